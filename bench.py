#!/usr/bin/env python
"""Benchmark of the B200 anisotropic-PQ hot path (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], "config2"): n = 1,183,514 unit
vectors, d = 100, M = 50 subspaces x 16 codewords (4-bit codes), T = 0.2.
One step = one batch of 10,000 queries through the query path: float64 LUT
build, 4-bit ADC scoring of every (query, point) pair with exact top-100
selection, exact-dot rerank to top-10 (ids and scores bit-identical to the
reference). `value` = ADC scores/s (query x point) with index and queries
resident in HBM; `e2e` = the same through the host-buffer C-ABI call
(queries H2D, results D2H inside the timed region). The secondary object
`encode` reports anisotropic-encode points/s (configs[2] shape: n = 1e7,
d = 128, 3 coordinate-descent sweeps).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N   (weak scaling: one shard per rank)

Data are seeded synthetic stand-ins (GloVe-1.2M is not available offline):
paper_1908_10396_b200/workload.py.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADC scores/sec (query\u00d7point) + anisotropic-encode points/sec, % HBM roofline"  # BASELINE.json
UNIT = "scores/s"


# ---------------------------------------------------------------------------------------
def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=1_183_514, help="database rows per shard")
    p.add_argument("--nq", type=int, default=10_000, help="queries per step")
    p.add_argument("--encode-n", type=int, default=10_000_000)
    p.add_argument("--no-encode", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-c4", action="store_true", help="skip the config-4 search object")
    p.add_argument("--no-c5", action="store_true", help="skip the config-5 training object")
    p.add_argument("--no-dropin", action="store_true", help="skip the single-query drop-in call")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def sharded_mode(ws):
    """The multi-GPU code path (shared sharded index, NCCL collectives);
    BENCH_SHARDED=1 runs it as a one-rank world, to exercise it on one GPU."""
    return ws > 1 or os.environ.get("BENCH_SHARDED") == "1"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def traffic_record():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return {}


BENCH_INDEX = os.path.join(ROOT, "bench_data", "config2_codebook.npz")


def search_config(w, n):
    """The `config` both arms print (identical dicts: same workload, index and
    query set; the per-step query count is a separate top-level key)."""
    return {"workload": "config2", "n_per_gpu": n, "d": w.d, "M": w.M, "k": 16,
            "threshold": w.threshold, "adc_topn": 100, "rerank_to": 10,
            "index": "codebook of train_apq (warm start + 10 iterations, T = 0.2, seed 0; "
                     "bench_data/config2_codebook.npz is the reference's), codes of "
                     "pq_quantize (3 passes)",
            "queries": "config2 query set (workload.config2, 10,000 unit vectors)"}


def reference_codebook():
    """The config-2 codebook trained by the reference (tools/make_bench_index.py)."""
    try:
        return np.load(BENCH_INDEX)["dictionaries"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list[str] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
def build_index(aq, wl, n, nq, seed_shard, session):
    """Config-2 shard (setup, untimed): data, queries and the trained index —
    train_apq on the device exactly as configs[1] states (warm start, 10
    alternating iterations, T = 0.2), bit-identical to the reference's trainer."""
    import ctypes as C

    w = wl.config2(n=n, nq=nq, seed=0, shard=seed_shard)
    cfg = aq.TrainConfig(max_iterations=w.iterations, relative_tolerance=0.0, seed=0)
    L = aq._L
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if sharded_mode(ws):
        return build_index_sharded(aq, w, n, ws, seed_shard, session, cfg)
    ds = session.upload_dataset(w.base)
    # the first run builds the index and warms every kernel (module loading,
    # clocks); the second, identical (deterministic) run is the one timed
    hist0 = []
    dcb, dc = aq.dev_train_apq(ds, w.M, w.k, aq.ThresholdWeights(w.threshold), cfg, True, hist0)
    # best of two timed runs (host wall clock around the synchronous trainer;
    # the phases are device events of the same run)
    train_s, phases = None, None
    for _ in range(2):
        del dcb, dc
        L.aq_session_timing(session.h, 1)
        for slot in range(8):
            L.aq_session_timer_read(session.h, slot, None, None, 1)
        session.sync()
        t0 = time.perf_counter()
        hist = []
        dcb, dc = aq.dev_train_apq(ds, w.M, w.k, aq.ThresholdWeights(w.threshold), cfg, True,
                                   hist)
        session.sync()
        ts = time.perf_counter() - t0
        assert hist == hist0, "train_apq is deterministic"
        ph = {}
        for slot, name in [(0, "encode"), (5, "assemble"), (6, "llt_solve"),
                           (7, "kmeans_warm_start")]:
            ms, cnt = C.c_double(0), C.c_uint64(0)
            L.aq_session_timer_read(session.h, slot, C.byref(ms), C.byref(cnt), 1)
            ph[name] = {"ms": round(ms.value, 2), "launches": int(cnt.value)}
        L.aq_session_timing(session.h, 0)
        if train_s is None or ts < train_s:
            train_s, phases = ts, ph
    cb = dcb.download()
    return w, cb, ds, dcb, dc, {"train_apq_s": round(train_s, 2), "loss_first": hist[0],
                                "loss_last": hist[-1], "iterations": len(hist) - 1,
                                "phases": phases, "trainer": "train_apq on device, warm start"}


def build_index_sharded(aq, w, n, ws, rank, session, cfg):
    """N > 1: one index over all shards — the codebook trained jointly by the
    row-sharded trainer (per-shard partial sums, NCCL all-gather, rank-ordered
    combination; paper_1908_10396_b200/distributed.py), every rank holding
    the same codebook and its shard's codes."""
    import ctypes as C
    import torch
    from paper_1908_10396_b200.distributed import DeviceShard, ShardedTrainer

    L = aq._L
    rows = torch.from_numpy(w.base).cuda(session.device)
    sh = DeviceShard(session, rows, aq.ThresholdWeights(w.threshold))
    trainer = ShardedTrainer(sh, n * ws, rank * n)
    trainer.train_apq(w.M, w.k, cfg, True)  # warms every kernel and collective
    L.aq_session_timing(session.h, 1)
    for slot in range(8):
        L.aq_session_timer_read(session.h, slot, None, None, 1)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    t0 = time.perf_counter()
    hist = []
    trainer.train_apq(w.M, w.k, cfg, True, hist)
    torch.cuda.synchronize()
    t = torch.tensor([time.perf_counter() - t0], device=f"cuda:{session.device}")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ph = {}
    for slot, name in [(0, "encode"), (5, "assemble"), (6, "llt_solve"),
                       (7, "kmeans_warm_start")]:
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(session.h, slot, C.byref(ms), C.byref(cnt), 1)
        ph[name] = {"ms": round(ms.value, 2), "launches": int(cnt.value)}
    L.aq_session_timing(session.h, 0)
    cb = sh.cb.download()
    return w, cb, sh.ds, sh.cb, sh.codes, {
        "train_apq_s": round(float(t.item()), 2), "loss_first": hist[0], "loss_last": hist[-1],
        "iterations": len(hist) - 1, "phases": ph,
        "trainer": f"row-sharded train_apq over {ws} GPUs (NCCL), one shared codebook"}


def train_record(w, n, info, codes_h, cpu):
    """train_apq on configs[1] (setup of the search bench, timed on the host
    around the synchronous trainer; phases from device events)."""
    its = info["iterations"]
    ph = info["phases"]
    km = ph["kmeans_warm_start"]["ms"] / 1e3
    per_it = (info["train_apq_s"] - km) / max(its, 1)
    asm_s = ph["assemble"]["ms"] / 1e3 / max(its, 1)
    M = w.M
    # lower-triangle coupling MACs per iteration: every point meets each pair
    # (m2 <= m) of its codes with sd^2 = 4 products
    macs = n * (M * (M + 1) // 2) * 4
    # shared-memory read-modify-write ceiling: 4 MACs per (point, m2) touch
    # 4 doubles read + written = 64 B -> 8 MACs per 128-B wavefront per SM
    ceil = 148 * 8 * 1.965e9
    return {"metric": "train_apq iterations/sec", "workload": "config2",
            "value": round(1.0 / per_it, 3), "unit": "iterations/s",
            "ms_per_iteration": round(per_it * 1e3, 2), "iterations": its,
            "warm_start_s": round(km, 3), "total_s": info["train_apq_s"],
            "phases_ms": {k: v["ms"] for k, v in ph.items()},
            "assembly_roofline": {"bound": "smem read-modify-write", "macs_per_iteration": macs,
                                  "achieved_gmacs": round(macs / asm_s / 1e9, 1),
                                  "ceiling_gmacs": round(ceil / 1e9, 1),
                                  "frac": round(macs / asm_s / ceil, 4),
                                  "note": "float64 entries, each a point-ordered chain "
                                          "(bit-exact with pq.hpp:320-339); ceiling = 16 B of "
                                          "shared-memory read-modify-write per MAC at 128 B/clk/SM",
                                  "ncu": "k_assemble_sd2 at config 2: L1/shared pipe 62.5% busy, "
                                         "~22 wavefronts per point and warp (16 the accumulator "
                                         "read-modify-write); the update takes about as long as "
                                         "the longest strip's chain (35k-104k points per strip) "
                                         "(profiles/r01_ncu_assemble_full.csv, DESIGN.md 4.4)"},
            "exact": "codebooks, codes and loss history bit-identical to the reference",
            "cpu_baseline": cpu}


def train_cpu_baseline(args, w, dc_h, n):
    """Reference pq_codebook_update (oracle/_ref, serial assembly + LLT) on a
    bounded prefix of the config-2 shard with the trained codes, extrapolated
    to the full shard: assembly is linear in n, the LLT is timed once."""
    try:
        from oracle import Reference
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}
    if not Reference.available():
        return None
    R = Reference()
    x = w.base
    norms = np.sqrt(np.einsum("ij,ij->i", x.astype(np.float64), x.astype(np.float64)))
    d = x.shape[1]
    times = []
    for m in (4000, 16000):
        xs = x[:m].astype(np.float64)
        nr = norms[:m]
        rho = (w.threshold / nr) ** 2
        hp = (d - 1) * rho / (1 - rho)
        ho = np.ones(m)
        t0 = time.perf_counter()
        R.pq_codebook_update(xs, dc_h[:m], hp, ho, w.M, w.k)
        times.append((m, time.perf_counter() - t0))
    (m1, t1), (m2, t2) = times
    per_pt = (t2 - t1) / (m2 - m1)
    fixed = max(t1 - per_pt * m1, 0.0)
    est = fixed + per_pt * n
    return {"value": round(1.0 / est, 5), "unit": "iterations/s (codebook update only)",
            "cores": 1, "kind": "reference",
            "sample": f"pq_codebook_update on the first {m1} and {m2} rows ({t1:.1f} s, "
                      f"{t2:.1f} s), linear in n -> {est:.1f} s at n = {n} (serial in the "
                      f"reference: pq.hpp:303-343)"}


def run_ours(args):
    import torch
    import ctypes as C

    ws, rank, local = dist_env()
    sharded = sharded_mode(ws)
    if sharded:
        import torch.distributed as dist
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_1908_10396_b200 import anisoq as aq
    from paper_1908_10396_b200 import workload as wl

    L = aq._L
    sess = aq.Session(local)
    stream = torch.cuda.ExternalStream(sess.stream, device=torch.device("cuda", local))
    w, cb, ds, dcb, dc, train_info = build_index(aq, wl, args.n, args.nq, rank, sess)
    n, nq, M, d = args.n, args.nq, w.M, w.d
    ref_cb = reference_codebook()
    if ws == 1 and n == 1_183_514 and ref_cb is not None:
        # the device trainer reproduces the reference's codebook bit for bit
        train_info["codebook_equals_reference"] = bool(np.array_equal(cb.dictionaries, ref_cb))
    # the searched index: the trained codebook + pq_quantize codes (the
    # reference pipeline's train -> encode), the same in both arms
    trained_codes = dc
    dc = sess.alloc_codes(n, M, 16)
    aq.dev_pq_quantize(ds, dcb, aq.ThresholdWeights(w.threshold), 3, dc)
    sess.sync()
    topn, keep = 100, 10
    Qh = np.ascontiguousarray(w.queries, np.float64)
    Qd = torch.from_numpy(Qh).cuda(local)
    te, ke = min(topn, n), min(keep, topn)
    aid = torch.empty((nq, te), dtype=torch.int32, device=f"cuda:{local}")
    asc = torch.empty((nq, te), dtype=torch.float64, device=f"cuda:{local}")
    rid = torch.empty((nq, ke), dtype=torch.int32, device=f"cuda:{local}")
    rsc = torch.empty((nq, ke), dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    # events on the session stream (single GPU); on torch's stream bracketing
    # the host-synchronous calls + collectives when sharded
    tstream = stream if not sharded else torch.cuda.current_stream(local)

    def step_dev():
        aq._check(L.aq_dev_search_rerank_d(ds.h, dc.h, dcb.h, Qd.data_ptr(), nq, topn, keep,
                                           aid.data_ptr(), asc.data_ptr(), rid.data_ptr(),
                                           rsc.data_ptr()))

    hid = np.zeros((nq, ke), np.uint32)
    hsc = np.zeros((nq, ke), np.float64)
    Qpin = torch.from_numpy(Qh).pin_memory()
    hid_t = torch.from_numpy(hid)
    hsc_t = torch.from_numpy(hsc)

    def step_e2e():
        aq._check(L.aq_dev_search_rerank(ds.h, dc.h, dcb.h, Qpin.data_ptr(), nq, topn, keep,
                                         None, None, hid_t.data_ptr(), hsc_t.data_ptr()))

    if sharded:
        # row shards: this rank owns global ids [rank*n, (rank+1)*n); one NCCL
        # all-gather of per-shard candidates + exact merge per step
        from paper_1908_10396_b200 import distributed as D

        def step_dev():  # noqa: F811
            D.sharded_search_rerank(ds, dc, dcb, Qd, rank * n, topn, keep, n_total=n * ws)

        def step_e2e():  # noqa: F811
            q = Qpin.to(f"cuda:{local}", non_blocking=True)
            _, _, r_ids, r_sc = D.sharded_search_rerank(ds, dc, dcb, q, rank * n, topn, keep,
                                                        n_total=n * ws)
            hid_t.copy_(r_ids.to(torch.int32).cpu())
            hsc_t.copy_(r_sc.cpu())

    def timed(fn, steps, warmup, with_clocks=False):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if sharded:
            torch.distributed.barrier()
        L.aq_session_timing(sess.h, 1)
        for slot in range(5):
            L.aq_session_timer_read(sess.h, slot, None, None, 1)
        launches0 = sess.launches
        total = 0.0
        sampler = ClockSampler(local) if with_clocks else None
        if sampler:
            sampler.__enter__()
        for _ in range(steps):
            flush.zero_()  # > L2 (126 MB): every step starts cold
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(tstream)
            fn()
            if sharded:
                torch.cuda.synchronize()
            e1.record(tstream)
            e1.synchronize()
            total += e0.elapsed_time(e1)
        if sampler:
            sampler.__exit__()
        torch.cuda.synchronize()
        launches = sess.launches - launches0
        kt = {}
        for slot, name in enumerate(["encode", "adc_score", "adc_merge", "rerank", "lut"]):
            ms, cnt = C.c_double(0), C.c_uint64(0)
            L.aq_session_timer_read(sess.h, slot, C.byref(ms), C.byref(cnt), 1)
            if cnt.value:
                kt[name] = (ms.value, cnt.value)
        L.aq_session_timing(sess.h, 0)
        ms = total / steps
        if sharded:
            t = torch.tensor([ms], device=f"cuda:{local}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = t.item()
        return ms, launches, kt, (sampler.summary() if sampler else None)

    ms, launches, kt, clocks = timed(step_dev, args.steps, args.warmup, with_clocks=True)
    value = nq * n * ws / (ms / 1e3)
    ms_e2e, _, _, _ = timed(step_e2e, args.steps, max(1, args.warmup // 2))
    e2e = nq * n * ws / (ms_e2e / 1e3)

    # quality of the timed pipeline (untimed): recall@10 of ADC top-100 + exact
    # rerank against exact float64 ground truth (k_exact_score), this shard
    gt, _ = aq.dev_exact_search(ds, Qh, keep)
    step_e2e()
    recall = float(np.mean([len(set(hid[q].tolist()) & set(gt[q].tolist())) / keep
                            for q in range(nq)])) if ws == 1 else None

    # roofline of the dominant kernel: ADC scoring (algorithmic bytes: M/2
    # code bytes per (query, point) score)
    pk = peaks()
    ms_k, cnt_k = kt.get("adc_score", (float("nan"), 1))
    per_launch_s = ms_k / cnt_k / 1e3
    alg_bytes = nq * n * (M / 2)  # one scoring launch per step covers every score
    achieved = alg_bytes / per_launch_s / 1e9
    tr = traffic_record().get("adc_score")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                "traffic": tr, "kernel": "k_adc_score",
                "kernel_ms_per_step": round(ms_k / args.steps, 3),
                "share_of_step": round((ms_k / args.steps) / ms, 3),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in pk
                else "fallback 6650 GB/s",
                "note": "algorithmic bytes = M/2 code bytes per score (single-pass HBM figure); "
                        "queries are batched so the kernel is shared-memory-LUT bound"}
    # on-chip ceiling: one 128-byte shared-memory wavefront per SM per clock
    # = 32 LUT words = 64 (query, subspace) lookups of 16 bits; M per score
    sm_hz = (clocks or {}).get("sm_mhz") or 1965.0
    n_sms = torch.cuda.get_device_properties(local).multi_processor_count
    ceil = n_sms * 64 * sm_hz * 1e6 / M
    roofline["onchip"] = {"ceiling_scores_per_s": round(ceil, -8),
                          "kernel_scores_per_s": round(nq * n / per_launch_s, -8),
                          "frac": round(nq * n / per_launch_s / ceil, 4),
                          "basis": f"{n_sms} SMs x 64 lookups/clk x {sm_hz:.0f} MHz / M={M}"}

    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded stand-in for GloVe-1.2M shape, config2)",
           "config": dict(search_config(w, n), parallelism=f"dp{ws} (row shards)"),
           "queries_per_step": nq,
           "index_build": {k: v for k, v in train_info.items() if k != "phases"},
           "recall10_at_10": recall,
           "notes": {"filter": "13-bit integer LUT (bounded error), results f64 bit-exact",
                     "l2": "flushed (256 MiB write) before every timed step"},
           "e2e": {"value": round(e2e, 1), "unit": UNIT,
                   "h2d_bytes_per_step": int(nq * d * 8),
                   "d2h_bytes_per_step": int(nq * ke * (4 + 8))},
           "gpu_launches": int(launches), "roofline": roofline, "clocks": clocks,
           "kernel_ms": {k: round(v[0] / args.steps, 3) for k, v in kt.items()}}

    if rank == 0:
        tcpu = None
        if ws == 1 and not args.no_cpu_baseline:
            tcpu = train_cpu_baseline(args, w, trained_codes.download().codes, n)
        out["train"] = train_record(w, n * ws, train_info, None, tcpu)
    if not args.no_encode:
        out["encode"] = bench_encode(args, aq, wl, sess, stream, flush, local, ws, pk)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, w, cb, dc, n)
    if ws == 1 and not args.no_dropin:
        out["dropin_adc_search"] = bench_dropin_search(aq, sess, w, cb, dc, n)
    del trained_codes, dc, dcb, ds, aid, asc, rid, rsc, Qd
    torch.cuda.empty_cache()
    if ws == 1 and not args.no_c4:
        out["search_c4"] = bench_search_c4(args, aq, wl, sess, local, pk, stream)
    if ws == 1 and not args.no_c5:
        out["train_c5"] = bench_train_c5(args, aq, sess, local)
    if rank == 0:
        emit(json.dumps(out))
    if sharded:
        torch.distributed.destroy_process_group()


def bench_encode(args, aq, wl, sess, stream, flush, local, ws, pk):
    """configs[2]: n = 1e7, d = 128, M = 64, 3 sweeps, lognormal norms."""
    import torch
    import ctypes as C

    L = aq._L
    w = wl.config3(n=args.encode_n)
    n = args.encode_n
    ds = sess.upload_dataset(w.base)
    cb = sess.upload_codebook(aq.ProductCodebook(64, 16, 2, w.codebook))
    out = sess.alloc_codes(n, 64, 16)
    wt = aq.ThresholdWeights(w.threshold, "parallel_only")
    for _ in range(args.warmup):
        aq.dev_pq_quantize(ds, cb, wt, 3, out)
    multi = torch.distributed.is_available() and torch.distributed.is_initialized()

    def max_over_ranks(v):  # every number below is the slowest rank's
        if not multi:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return t.item()

    torch.cuda.synchronize()
    if multi:
        torch.distributed.barrier()
    L.aq_session_timing(sess.h, 1)
    L.aq_session_timer_read(sess.h, 0, None, None, 1)
    tot = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        aq.dev_pq_quantize(ds, cb, wt, 3, out)
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ms_k, cnt = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(sess.h, 0, C.byref(ms_k), C.byref(cnt), 1)
    L.aq_session_timing(sess.h, 0)
    ms = max_over_ranks(tot / args.steps)
    value = n * ws / (ms / 1e3)
    # e2e: host rows in -> host codes out through the C ABI (pq_quantize), from
    # page-locked host buffers (the contract's pinned inputs: the library DMAs
    # straight from / into them) and, for comparison, from pageable numpy
    # arrays (the library stages those through its own page-locked ring)
    keep = []
    cw = aq._weights(wt, n, keep)
    x_pin = torch.from_numpy(w.base).pin_memory()
    codes_pin = torch.zeros((n, 64), dtype=torch.int32).pin_memory()
    xs = np.ascontiguousarray(w.base)
    codes_h = np.zeros((n, 64), np.uint32)

    def e2e_call(xp, op):
        aq._check(L.aq_pq_quantize(sess.h, xp, n, 128, w.codebook.ctypes.data, 64,
                                   16, 2, C.byref(cw), 3, op))

    def e2e_time(xp, op):
        e2e_call(xp, op)  # warm-up: first-touch of the host buffers, device scratch
        steps = max(2, min(args.steps, 3))
        if multi:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            e2e_call(xp, op)
        return max_over_ranks((time.perf_counter() - t0) / steps), steps

    e2e_s, e2e_steps = e2e_time(x_pin.data_ptr(), codes_pin.data_ptr())
    e2e_pg_s, _ = e2e_time(xs.ctypes.data, codes_h.ctypes.data)
    same_codes = bool(np.array_equal(codes_pin.numpy().view(np.uint32), codes_h))
    del x_pin, codes_pin
    cpu = None
    if not args.no_cpu_baseline and int(os.environ.get("RANK", "0")) == 0 and ws == 1:
        cpu = encode_cpu_baseline(args, w)
    per_launch = ms_k.value / max(cnt.value, 1) / 1e3
    ops_per_pt = 64 * 16 * (3 + 3 * 8)   # M k [(sd+1) + S (sd+6)]
    fp32_peak = 148 * 128 * 1.965e9      # FP32 pipe ops/s (FFMA = 1 op)
    achieved_ops = n * ops_per_pt / per_launch
    del ds, cb, out
    return {"metric": "anisotropic-encode points/sec", "value": round(value, 1),
            "unit": "points/s", "ms_per_step": round(ms, 3), "workload": "config3",
            "n_per_gpu": n, "d": 128, "M": 64, "passes": 3,
            "roofline": {"bound": "fp32", "achieved": round(achieved_ops / 1e12, 2),
                         "peak": round(fp32_peak / 1e12, 2), "unit": "Tops/s",
                         "frac": round(achieved_ops / fp32_peak, 4),
                         "note": "27,648 algorithmic f32 ops/point (SURVEY.md §8(d)); HBM side "
                                 "544 B/point is << HBM peak; the kernel is issue/latency "
                                 "bound (ncu: ~71% issue active, no pipe above 46%; the "
                                 "per-point float64 coordinate-descent chain, DESIGN.md §4.1)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(n / e2e_s, 1), "unit": "points/s",
                    "h2d_bytes_per_step": int(n * 128 * 4), "d2h_bytes_per_step": int(n * 64 * 4),
                    "pageable_value": round(n / e2e_pg_s, 1),
                    "codes_equal_pageable": same_codes,
                    "note": f"host wall clock of the synchronous aq_pq_quantize call (host "
                            f"rows in, host uint32 codes out, both page-locked: H2D / D2H "
                            f"straight from / into them), mean of {e2e_steps} calls after "
                            f"one warm-up; pageable_value = the same call on pageable numpy "
                            f"arrays (staged through the library's page-locked ring)"}}


def bench_dropin_search(aq, sess, w, cb, dc, n):
    """The reference-signature single-query call anisoq::adc_search(q, codes,
    cb, topn) (index.hpp:118): host uint32 codes in, host hits out, so every
    call uploads and packs the whole index (n x M x 4 B). The resident
    batched path above is the one to use for query batches."""
    L = aq._L
    import ctypes as C
    codes = np.ascontiguousarray(dc.download().codes, np.uint32)
    Q = np.ascontiguousarray(w.queries[:4], np.float64)
    ids = np.zeros(100, np.uint32)
    sc = np.zeros(100, np.float64)
    cnt = C.c_size_t(0)

    def call(q):
        aq._check(L.aq_adc_search(sess.h, q.ctypes.data, q.size, codes.ctypes.data, n, w.M, 16,
                                  cb.dictionaries.ctypes.data, w.M, 16, 2, 100, ids.ctypes.data,
                                  sc.ctypes.data, C.byref(cnt)))

    call(Q[0])
    t0 = time.perf_counter()
    for q in Q[1:]:
        call(q)
    ms = (time.perf_counter() - t0) / (len(Q) - 1) * 1e3
    return {"call": "aq_adc_search (C++ anisoq::adc_search), one query, host codes",
            "ms_per_query": round(ms, 2), "scores_per_s": round(n / (ms / 1e3), 1),
            "h2d_bytes_per_call": int(n * ((((w.M + 1) // 2) + 7) // 8 * 8) + 8 * w.d),
            "note": "dominated by the per-call index upload (the reference signature passes "
                    "the codes by value, 4 bytes per code: packed to 4 bits by every host "
                    "core into page-locked memory, then copied); batched queries on the "
                    "resident index: `value`"}


def bench_search_c4(args, aq, wl, sess, local, pk, stream):
    """configs[3]: ADC top-100 of 4,096 queries over 1e8 uniform 4-bit codes
    (M = 48), resident; the largest single-GPU search configuration."""
    import ctypes as C
    import torch

    L = aq._L
    w = wl.config4()
    n, M, nq = w.n, w.M, len(w.queries)
    dc = sess.upload_packed_codes(w.packed_codes, n, M, 16)
    del w.packed_codes
    dcb = sess.upload_codebook(aq.ProductCodebook(M, 16, 2, w.codebook))
    Qd = torch.from_numpy(np.ascontiguousarray(w.queries, np.float64)).cuda(local)
    ids = torch.empty((nq, 100), dtype=torch.int32, device=f"cuda:{local}")
    sc = torch.empty((nq, 100), dtype=torch.float64, device=f"cuda:{local}")

    def step():
        aq._check(L.aq_dev_adc_search_d(dc.h, dcb.h, Qd.data_ptr(), nq, 100, ids.data_ptr(),
                                        sc.data_ptr()))

    step()
    torch.cuda.synchronize()
    L.aq_session_timing(sess.h, 1)
    L.aq_session_timer_read(sess.h, 1, None, None, 1)
    steps = 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    msk, cnt = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(sess.h, 1, C.byref(msk), C.byref(cnt), 1)
    L.aq_session_timing(sess.h, 0)
    per_launch = msk.value / max(cnt.value, 1) / 1e3
    hbm = nq * n * (M / 2) / per_launch / 1e9
    del dc, dcb
    # the search takes the tensor-core filter (csrc/adc_tc.cu) for long
    # per-SM slices (search.cu: >= 1.5e6 points of a 128-query block per SM)
    tc = M <= 50 and ((nq + 127) // 128) * n / 148 >= 1.5e6 and os.environ.get("AQ_ADC_TC") != "0"
    if tc:
        # the filter as executed: a u8 x u8 GEMM, K = 32 M bytes per (query,
        # point) (hi and lo one-hot images of each 4-bit code), 2 ops per MAC;
        # int8 peak taken as twice the measured bf16 burst (sm_100 issues int8
        # at twice the bf16 rate; tools/mb/umma_i8_test.cu measured 8,176
        # MAC/clk/SM for M = 128, N = 256, i.e. 4.75 POPS at 1,965 MHz)
        i8_peak = 2 * pk["bf16_tflops"]
        ach = nq * n * 32 * M * 2 / per_launch / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 1), "peak": round(i8_peak, 1),
                "unit": "TOPS (int8)", "frac": round(ach / i8_peak, 4), "kernel": "k_adc_tc",
                "hbm_single_pass": {"achieved_gbs": round(hbm, 1), "frac": round(hbm / pk["hbm_gbs"], 4)},
                "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (int8 not measured by the driver)",
                "note": "tcgen05.mma.kind::i8, M = 128 queries, N = 64 points, K = 32 per subspace; "
                        "per-instruction floor ~72 cycles for N <= 128 (microbenchmark), so N = 64 "
                        "tiles cap the tensor pipe near 45% of peak"}
    else:
        ceil = 148 * 64 * 1.965e9 / M
        roof = {"bound": "hbm", "achieved": round(hbm, 1), "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": round(hbm / pk["hbm_gbs"], 4),
                "kernel": "k_adc_score",
                "onchip_frac": round(nq * n / per_launch / ceil, 4),
                "note": "M/2 code bytes per score; 16 queries per code pass, so the "
                        "bound is the shared-memory LUT (onchip_frac: 64 lookups/clk/SM)"}
    return {"metric": "ADC scores/sec", "workload": "config4", "value": round(nq * n / (ms / 1e3), 1),
            "unit": "scores/s", "ms_per_step": round(ms, 2), "n": n, "M": M,
            "queries_per_step": nq, "topn": 100, "roofline": roof,
            "exact": "ids and scores equal the reference's over all 1e8 codes "
                     "(tests/test_config_pins_gpu.py::test_c4_all_codes_top100)"}


def bench_train_c5(args, aq, sess, local):
    """configs[4]: train_apq at n = 1e7, d = 256, M = 128, k = 16, T = 0.2,
    warm start + 20 iterations (the dim-4096 normal equations); rows drawn on
    the device (torch, seeded) with config 5's distribution."""
    import ctypes as C
    import torch

    L = aq._L
    n, d, M, comps = 10_000_000, 256, 128, 4096
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    means = torch.randn((comps, d), generator=g, device=dev, dtype=torch.float32)
    x = torch.empty((n, d), dtype=torch.float32, device=dev)
    for b in range(0, n, 1 << 20):
        e = min(n, b + (1 << 20))
        comp = torch.randint(0, comps, (e - b,), generator=g, device=dev)
        v = means[comp] + 0.4 * torch.randn((e - b, d), generator=g, device=dev)
        x[b:e] = v / torch.linalg.vector_norm(v, dim=1, keepdim=True)
    torch.cuda.synchronize()
    ds = sess.wrap_device_rows(x.data_ptr(), n, d)
    cfg = aq.TrainConfig(max_iterations=20, relative_tolerance=0.0, seed=0)
    L.aq_session_timing(sess.h, 1)
    for slot in range(9):
        L.aq_session_timer_read(sess.h, slot, None, None, 1)
    hist = []
    t0 = time.perf_counter()
    dcb, dc = aq.dev_train_apq(ds, M, 16, aq.ThresholdWeights(0.2), cfg, True, hist)
    sess.sync()
    tt = time.perf_counter() - t0
    ph = {}
    for slot, name in [(0, "encode"), (5, "assemble"), (6, "llt_solve"), (7, "kmeans_warm_start")]:
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(sess.h, slot, C.byref(ms), C.byref(cnt), 1)
        ph[name] = round(ms.value, 1)
    L.aq_session_timing(sess.h, 0)
    its = len(hist) - 1
    per_it = (tt - ph["kmeans_warm_start"] / 1e3) / max(its, 1)
    macs = n * (M * (M + 1) // 2) * 4
    asm_s = ph["assemble"] / 1e3 / max(its, 1)
    del ds, dcb, dc, x, means
    torch.cuda.empty_cache()
    return {"metric": "train_apq iterations/sec", "workload": "config5", "n": n, "d": d, "M": M,
            "value": round(1.0 / per_it, 3), "unit": "iterations/s",
            "ms_per_iteration": round(per_it * 1e3, 1), "total_s": round(tt, 2),
            "iterations": its, "phases_ms": ph, "loss_first": hist[0], "loss_last": hist[-1],
            "assembly_roofline": {"bound": "smem read-modify-write",
                                  "achieved_gmacs": round(macs / asm_s / 1e9, 1),
                                  "ceiling_gmacs": 2326.6,
                                  "frac": round(macs / asm_s / 2.3266e12, 4),
                                  "ncu": "k_assemble_sd2r at config 5: L1/shared pipe 73.9% "
                                         "busy (LSU wavefronts 70.6% of peak), ~20 wavefronts "
                                         "per point and warp of which 16 the accumulator "
                                         "read-modify-write (profiles/r01_ncu_assemble_ring_full.csv)"},
            "data": "synthetic on the device (torch, seeded): 4,096-component mixture, "
                    "sigma 0.4, unit norm",
            "exact": "bit-identical to the reference at the config-5 shape "
                     "(tests/test_config_pins_gpu.py::test_c5_shape_train, n = 2e5)"}


def encode_cpu_baseline(args, w):
    """Reference pq_quantize (oracle/_ref, all host cores) on a bounded prefix
    of the config-3 rows."""
    try:
        from oracle import Port, Reference
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}
    if Reference.available():
        R, kind, cores = Reference(), "reference", os.cpu_count() or 1
    else:
        R, kind, cores = Port(), "port", 1
    x = w.base
    norms = np.sqrt(np.einsum("ij,ij->i", x.astype(np.float64), x.astype(np.float64)))
    m = int(min(len(x), 20000))
    while True:
        xs = x[:m].astype(np.float64)
        nr = norms[:m]
        rho = np.where(nr > w.threshold, (w.threshold / nr) ** 2, 0.0)
        hp = np.where(nr > w.threshold, (127 * rho) / (1 - np.where(rho < 1, rho, 0)), 1.0)
        ho = np.where(nr > w.threshold, 1.0, 0.0)
        t0 = time.perf_counter()
        if kind == "reference":
            R.pq_quantize(xs, w.codebook, 64, 16, 2, hp, ho, 3, threads=cores)
        else:
            R.pq_quantize(xs, w.codebook, 64, 16, 2, hp, ho, 3)
        dt = time.perf_counter() - t0
        if dt > args.cpu_seconds / 3 or m >= len(x):
            break
        m = min(len(x), int(m * max(2.0, args.cpu_seconds / 2 / max(dt, 1e-3))))
    return {"value": round(m / dt, 1), "unit": "points/s", "cores": cores, "kind": kind,
            "sample": f"first {m} config-3 rows, pq_quantize passes=3, {dt:.1f} s"}


def cpu_baseline(args, w, cb, dc, n):
    """The reference itself (oracle/_ref, compiled in place) on this host's
    cores, on a bounded sample of the same step (queries subset x full shard)."""
    try:
        from oracle import Port, Reference
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}
    codes = dc.download().codes
    if Reference.available():
        R, kind = Reference(), "reference"
        cores = os.cpu_count() or 1
    else:
        R, kind = Port(), "port"
        cores = 1
    Q = np.ascontiguousarray(w.queries, np.float64)
    x64 = w.base.astype(np.float64)
    nq_s = 4
    while True:
        t0 = time.perf_counter()
        ids, _ = (R.adc_search_batch(Q[:nq_s], codes, 16, cb.dictionaries, w.M, 16, 2, 100,
                                     threads=cores) if kind == "reference" else
                  R.adc_search_batch(Q[:nq_s], codes, 16, cb.dictionaries, w.M, 16, 2, 100))
        R.rerank(Q[:nq_s], x64, ids, 10)
        dt = time.perf_counter() - t0
        if dt > args.cpu_seconds / 3 or nq_s >= len(Q):
            break
        nq_s = min(len(Q), int(nq_s * max(2.0, args.cpu_seconds / 2 / max(dt, 1e-3))))
    return {"value": round(nq_s * n / dt, 1), "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{nq_s} queries x {n} points (adc_search top-100 + rerank to 10), "
                      f"{dt:.1f} s"}


def run_reference(args):
    """--impl reference: the reference CPU implementation (oracle/_ref) on the
    host cores, same metric/config, each step a bounded query sample."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import Port, Reference
    from paper_1908_10396_b200 import workload as wl

    n = args.n
    w = wl.config2(n=n, nq=args.nq, seed=0)
    M = w.M
    # the index of the GPU arm: the config-2 codebook as trained by the
    # reference itself (bench_data/, tools/make_bench_index.py; the device
    # trainer reproduces it bit for bit) and pq_quantize codes below
    dic = reference_codebook() if n == 1_183_514 else None
    same_index = dic is not None
    if dic is None:  # other shard sizes: a codebook sampled from the rows
        g = np.random.Generator(np.random.PCG64([0, 7]))
        dic = np.empty((M, 16, 2))
        for m in range(M):
            idx = g.choice(n, size=16, replace=False)
            dic[m] = w.base[idx, m * 2:(m + 1) * 2]
        dic = dic.ravel()
    if Reference.available():
        R, kind, cores = Reference(), "reference", os.cpu_count() or 1
    else:
        R, kind, cores = Port(), "port", 1
    x64 = w.base.astype(np.float64)
    hp = np.empty(n)
    norms = np.sqrt(np.einsum("ij,ij->i", x64, x64))
    rho = (w.threshold / norms) ** 2
    hp[:] = (w.d - 1) * rho / (1 - rho)
    ho = np.ones(n)
    # index build with the reference's own encoder (setup, untimed)
    codes = (R.pq_quantize(x64, dic, M, 16, 2, hp, ho, 3, threads=cores) if kind == "reference"
             else R.pq_quantize(x64, dic, M, 16, 2, hp, ho, 3))
    Q = np.ascontiguousarray(w.queries, np.float64)
    # one parallel_for chunk of 16 queries (index.hpp evaluate's chunking, as
    # adc_search_batch uses) per host thread, so every core works each step
    per_step = max(1, min(len(Q), int(os.environ.get("REF_QUERIES_PER_STEP", str(16 * cores)))))

    def step(i):
        q = Q[(i * per_step) % len(Q):][:per_step]
        ids, _ = (R.adc_search_batch(q, codes, 16, dic, M, 16, 2, 100, threads=cores)
                  if kind == "reference" else R.adc_search_batch(q, codes, 16, dic, M, 16, 2, 100))
        R.rerank(q, x64, ids, 10)
        return len(q)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    done = 0
    for i in range(args.steps):
        done += step(i)
    dt = time.perf_counter() - t0
    value = done * n / dt
    emit(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded stand-in for GloVe-1.2M shape, config2)",
        "config": (dict(search_config(w, n), parallelism=f"dp{ws} (row shards)") if same_index
                   else {"workload": "config2", "n_per_gpu": n, "d": w.d, "M": M, "k": 16,
                         "index": "sampled codebook + pq_quantize codes"}),
        "queries_per_step": per_step,
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{per_step} queries x {n} points per step"},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


_STDOUT_FD = None


def emit(line: str) -> None:
    """The one JSON line on the real stdout (everything else — NCCL banners,
    library prints — was sent to stderr)."""
    sys.stderr.flush()
    if _STDOUT_FD is not None:
        os.write(_STDOUT_FD, (line + "\n").encode())
    else:
        print(line, flush=True)


def launch_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: start N ranks (one process
    per GPU) under torch.distributed.run on this node and relay rank 0's line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is None and a.gpus > 1:
        sys.exit(launch_ranks(a))
    if world is not None and int(world) != a.gpus:
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if a.impl == "ours" and a.gpus > 1:
        import torch
        if torch.cuda.device_count() < a.gpus and int(os.environ.get("LOCAL_RANK", "0")) == 0:
            sys.exit(f"bench.py: --gpus {a.gpus} but only {torch.cuda.device_count()} visible")
    sys.stdout.flush()
    _STDOUT_FD = os.dup(1)
    os.dup2(2, 1)  # C-level and Python prints during the run go to stderr
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
