"""anisoq_b200 verbs on the B200 against the oracle: train (pq and vq),
encode, search and eval write the files the reference tool writes
(anisoq_main.cpp:358-579) with the oracle's codebooks, codes, loss history,
hits and exact ground truth."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.test_cli import EXE, run

pytestmark = pytest.mark.gpu
P = Port()


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    t = tmp_path_factory.mktemp("cli")
    base, q = t / "base.fvecs", t / "q.fvecs"
    assert run("gen", "--out", str(base), "--kind", "gaussian_mixture", "--n", "3000", "--d",
               "16", "--seed", "2", "--centers", "12", "--spread", "0.3",
               "--normalize").returncode == 0
    assert run("gen", "--out", str(q), "--kind", "gaussian_mixture", "--n", "20", "--d", "16",
               "--seed", "3", "--centers", "12", "--spread", "0.3",
               "--normalize").returncode == 0
    x = aq.read_fvecs(str(base)).values.astype(np.float64)
    Q = aq.read_fvecs(str(q)).values.astype(np.float64)
    hp, ho = P.threshold_weights(P.row_norms(x), 16, 0.2, 0)
    return t, base, q, x, Q, hp, ho


def _history(path):
    rows = [ln for ln in open(path).read().splitlines() if ln and not ln.startswith("#")]
    assert rows[0] == "iteration,total_loss"
    return np.array([float(r.split(",")[1]) for r in rows[1:]])


def test_train_pq_encode_search_eval(files):
    t, base, qf, x, Q, hp, ho = files
    out = t / "pq"
    r = run("train", "--data", str(base), "--out", str(out), "--M", "8", "--k", "16",
            "--iters", "5", "--tol", "0", "--seed", "1")
    assert r.returncode == 0, r.stderr
    cb, codes, hist = P.train_apq(x, 8, 16, hp, ho, max_it=5, tol=0.0, seed=1)
    got_cb = aq.load_codebook(str(out / "codebook.bin"))
    assert np.array_equal(got_cb.dictionaries, cb.astype(np.float32).astype(np.float64))
    assert np.array_equal(aq.load_codes(str(out / "codes.bin")).codes, codes)
    assert np.array_equal(_history(out / "train_log.csv"), hist)
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "train" and man["iterations_run"] == len(hist) - 1
    assert man["final_loss"] == hist[-1] and man["loss"]["loss"] == "score_aware"
    assert r.stdout.startswith("trained pq codebook: k=16 M=8 final_loss=")

    # encode with the saved (float32) codebook, 2 sweeps
    enc = t / "enc.bin"
    r = run("encode", "--data", str(base), "--codebook", str(out / "codebook.bin"), "--out",
            str(enc), "--passes", "2")
    assert r.returncode == 0, r.stderr
    assert r.stdout == "encoded 3000 datapoints\n"
    want = P.pq_quantize(x, got_cb.dictionaries, 8, 16, 2, hp, ho, 2)
    assert np.array_equal(aq.load_codes(str(enc)).codes, want)
    assert json.loads(open(str(enc) + ".meta.json").read())["options"]["passes"] == 2

    # search: one line per hit, "%zu %zu %u %.9g"
    r = run("search", "--codebook", str(out / "codebook.bin"), "--codes", str(enc),
            "--queries", str(qf), "--topn", "7")
    assert r.returncode == 0, r.stderr
    ids, sc = P.adc_search_batch(Q, want, 16, got_cb.dictionaries, 8, 16, 2, 7)
    lines = ["# query rank index score"] + [
        "%d %d %d %.9g" % (qi, rk, ids[qi, rk], sc[qi, rk]) for qi in range(20)
        for rk in range(7)]
    assert r.stdout.splitlines() == lines
    r = run("search", "--codebook", str(out / "codebook.bin"), "--codes", str(enc),
            "--queries", str(qf), "--topn", "3", "--query-index", "4")
    assert r.returncode == 0 and len(r.stdout.splitlines()) == 4
    assert r.stdout.splitlines()[1].startswith(f"4 0 {ids[4, 0]} ")
    r = run("search", "--codebook", str(out / "codebook.bin"), "--codes", str(enc),
            "--queries", str(qf), "--query-index", "20")
    assert r.returncode == 2 and "query index out of range" in r.stderr

    # eval: exact ground truth cached as ivecs, report files
    ev = t / "eval"
    r = run("eval", "--data", str(base), "--queries", str(qf), "--codebook",
            str(out / "codebook.bin"), "--codes", str(enc), "--out", str(ev), "--Ns", "1,10")
    assert r.returncode == 0, r.stderr
    man = json.loads((ev / "manifest.json").read_text())
    assert man["ground_truth"]["source"] == "computed"
    gt = aq.read_ivecs(man["ground_truth"]["path"])
    want_gt, _ = P.exact_search_batch(Q, x, 10)
    assert np.array_equal(np.array(gt), want_gt.astype(np.int32))
    rep = json.loads((ev / "eval_report.json").read_text())
    assert rep["num_queries"] == 20 and rep["num_datapoints"] == 3000 and rep["kk"] == 10
    adc10, _ = P.adc_search_batch(Q, want, 16, got_cb.dictionaries, 8, 16, 2, 10)
    recall = np.mean([len(set(adc10[i]) & set(want_gt[i])) / 10 for i in range(20)])
    assert abs(rep["recall_kk"] - recall) < 1e-12
    assert (ev / "eval_report.txt").read_text().startswith("num_queries 20\n")
    r = run("eval", "--data", str(base), "--queries", str(qf), "--codebook",
            str(out / "codebook.bin"), "--codes", str(enc), "--out", str(ev), "--Ns", "1,10")
    assert json.loads((ev / "manifest.json").read_text())["ground_truth"]["source"] == "cache"
    # a supplied ground truth file is used as is; a missing one is computed there
    ev2 = t / "eval2"
    r = run("eval", "--data", str(base), "--queries", str(qf), "--codebook",
            str(out / "codebook.bin"), "--codes", str(enc), "--out", str(ev2), "--Ns", "1,10",
            "--ground-truth", man["ground_truth"]["path"])
    assert r.returncode == 0, r.stderr
    assert json.loads((ev2 / "manifest.json").read_text())["ground_truth"]["source"] == "supplied"
    rep2 = json.loads((ev2 / "eval_report.json").read_text())
    rep2.pop("latency_us")
    assert rep2 == {k: v for k, v in rep.items() if k != "latency_us"}
    gt_new = t / "gt_new.ivecs"
    r = run("eval", "--data", str(base), "--queries", str(qf), "--codebook",
            str(out / "codebook.bin"), "--codes", str(enc), "--out", str(ev2), "--Ns", "1,10",
            "--ground-truth", str(gt_new))
    assert r.returncode == 0 and np.array_equal(np.array(aq.read_ivecs(str(gt_new))),
                                                want_gt.astype(np.int32))


def test_train_from_config_document(files):
    t, base, _, x, _, hp, ho = files
    cfg = t / "train.json"
    cfg.write_text(json.dumps({"seed": 3, "train": {"M": 4, "k": 8, "iters": 2, "tol": 0.0,
                                                    "warm-start": False}}))
    out = t / "cfg"
    r = run("train", "--data", str(base), "--out", str(out), "--config", str(cfg))
    assert r.returncode == 0, r.stderr
    cb, codes, hist = P.train_apq(x, 4, 8, hp, ho, max_it=2, tol=0.0, seed=3, warm_start=False)
    assert np.array_equal(aq.load_codes(str(out / "codes.bin")).codes, codes)
    man = json.loads((out / "manifest.json").read_text())
    assert man["options"]["seed"] == 3 and man["options"]["warm_start"] is False


def test_train_vq_and_reconstruction_loss(files):
    t, base, _, x, _, hp, ho = files
    out = t / "vq"
    r = run("train", "--data", str(base), "--out", str(out), "--quantizer", "vq", "--k", "24",
            "--iters", "4", "--tol", "0", "--seed", "5")
    assert r.returncode == 0, r.stderr
    cw, a, hist = P.train_avq(x, 24, hp, ho, max_it=4, tol=0.0, seed=5)
    cb = aq.load_codebook(str(out / "codebook.bin"))
    assert (cb.M, cb.k, cb.sub_dimension) == (1, 24, 16)
    assert np.array_equal(cb.dictionaries, cw.ravel().astype(np.float32).astype(np.float64))
    assert np.array_equal(aq.load_codes(str(out / "codes.bin")).codes.ravel(), a)
    assert np.array_equal(_history(out / "train_log.csv"), hist)
    # reconstruction loss = isotropic weights; explicit eta overrides the threshold
    out2 = t / "l2"
    r = run("train", "--data", str(base), "--out", str(out2), "--M", "4", "--k", "8",
            "--iters", "3", "--tol", "0", "--loss", "reconstruction", "--no-warm-start")
    assert r.returncode == 0, r.stderr
    ones = np.ones(len(x))
    cbw, codes, h2 = P.train_apq(x, 4, 8, ones, ones, max_it=3, tol=0.0, seed=0,
                                 warm_start=False)
    assert np.array_equal(aq.load_codes(str(out2 / "codes.bin")).codes, codes)
    assert np.array_equal(_history(out2 / "train_log.csv"), h2)
    r = run("train", "--data", str(base), "--out", str(t / "bad"), "--M", "5")
    assert r.returncode == 2 and "divisible" in r.stderr
