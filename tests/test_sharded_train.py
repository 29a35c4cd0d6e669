"""Row-sharded trainer (distributed.ShardedTrainer): host orchestration on CPU.

* world of one: the sharded trainer with the oracle as its per-shard backend
  equals the oracle's single-process train_apq / train_l2_pq bit for bit
  (every partial is then the full sequential sum);
* world of two (gloo): both ranks hold identical dictionaries, the result is
  deterministic, and it matches the single-process trainer up to float64
  re-association at the shard boundary;
* a failure on one rank raises the same error on every rank.
The device backend (DeviceShard) is covered in test_sharded_train_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_10396_b200.distributed import HostRng, ShardedTrainer, shard_bounds
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho
from tests.shard_cpu import OracleShard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_host_rng_sample_distinct_matches_oracle():
    from oracle import Port

    P = Port()
    for seed, n, k in [(0, 10, 10), (7, 1000, 16), (123, 5, 3), (2**63 + 5, 100000, 256)]:
        assert HostRng(seed).sample_distinct(n, k) == P.sample_distinct(seed, n, k).tolist()


def _data(n=600, d=8, seed=5):
    x = mixture_rows(n, d, seed).astype(np.float64)
    hp, ho = threshold_hp_ho(x, 0.2)
    return x, hp, ho


@pytest.mark.parametrize("warm", [True, False])
def test_world_one_equals_oracle_train_apq(warm):
    from oracle import Port

    x, hp, ho = _data()
    M, k = 4, 16
    cfg = aq.TrainConfig(max_iterations=6, relative_tolerance=0.0, seed=3)
    sh = OracleShard(x, hp, ho)
    hist = []
    dict_ = ShardedTrainer(sh, len(x), 0).train_apq(M, k, cfg, warm, hist)
    cb, codes, h = Port().train_apq(x, M, k, hp, ho, max_it=6, tol=0.0, seed=3,
                                    warm_start=warm)
    assert np.array_equal(dict_.numpy(), cb)
    assert np.array_equal(sh.codes, codes)
    assert hist == h.tolist()


def test_world_one_isotropic_and_reseed_paths():
    """Isotropic weights (mean path) and a dataset with duplicated rows, so
    partitions empty out and get reseeded from the loss ranking."""
    from oracle import Port

    base = mixture_rows(40, 8, 9).astype(np.float64)
    x = np.repeat(base, 8, axis=0)  # 320 rows, only 40 distinct
    one = np.ones(len(x))
    M, k = 2, 64
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=1)
    for (hp, ho), warm in [((one, one), False), (threshold_hp_ho(x, 0.2), False),
                           (threshold_hp_ho(x, 0.2), True)]:
        sh = OracleShard(x, hp, ho)
        hist = []
        dict_ = ShardedTrainer(sh, len(x), 0).train_apq(M, k, cfg, warm, hist)
        cb, codes, h = Port().train_apq(x, M, k, hp, ho, max_it=4, tol=0.0, seed=1,
                                        warm_start=warm)
        assert np.array_equal(dict_.numpy(), cb)
        assert np.array_equal(sh.codes, codes)
        assert hist == h.tolist()


def _worker(rank, world, port, x, hp, ho, M, k, warm, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(len(x), rank, world)
    sh = OracleShard(x[lo:hi], hp[lo:hi], ho[lo:hi])
    cfg = aq.TrainConfig(max_iterations=5, relative_tolerance=0.0, seed=4)
    hist = []
    dict_ = ShardedTrainer(sh, len(x), lo).train_apq(M, k, cfg, warm, hist)
    out[rank] = (dict_.numpy().copy(), sh.codes.copy(), list(hist))
    dist.destroy_process_group()


def _run_world(world, x, hp, ho, M, k, warm):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), x, hp, ho, M, k, warm, out), nprocs=world,
             join=True)
    return dict(out)


@pytest.mark.parametrize("warm,world", [(True, 2), (False, 2), (True, 3)])
def test_ranks_match_single_process(warm, world):
    """W ranks re-associate each float64 sum at W - 1 shard boundaries
    (rank-ordered chain). The north_star bar: codebooks within a stated
    relative tolerance (1e-12 here), loss history within 1e-12, and codes
    equal except near-ties — a differing code must be within
    eps_c = 2^-20 x max loss of the single-process code under the trained
    codebook (SURVEY.md §8(c) rule 1)."""
    from oracle import Port

    P = Port()
    x, hp, ho = _data(n=500)
    M, k = 4, 16
    res = _run_world(world, x, hp, ho, M, k, warm)
    d0, _, h0 = res[0]
    for r in range(1, world):
        assert np.array_equal(res[r][0], d0) and res[r][2] == h0  # replicated state
    codes = np.concatenate([res[r][1] for r in range(world)])
    cb, ref_codes, h = Port().train_apq(x, M, k, hp, ho, max_it=5, tol=0.0, seed=4,
                                        warm_start=warm)
    assert np.allclose(d0, cb, rtol=0, atol=1e-12 * np.abs(cb).max())
    assert np.allclose(h0, h, rtol=1e-12)
    loss = P.pq_point_losses(x, d0, M, k, 2, hp, ho, codes)
    eps = 2.0 ** -20 * loss.max()
    for i in np.nonzero((codes != ref_codes).any(axis=1))[0]:
        alt = P.pq_point_losses(x[i:i + 1], d0, M, k, 2, hp[i:i + 1], ho[i:i + 1],
                                ref_codes[i:i + 1])
        assert abs(alt[0] - loss[i]) <= eps, (i, codes[i], ref_codes[i])
    again = _run_world(world, x, hp, ho, M, k, warm)  # deterministic for a given world size
    assert np.array_equal(again[0][0], d0)


def _zero_worker(rank, world, port, x, hp, ho, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(len(x), rank, world)
    sh = OracleShard(x[lo:hi], hp[lo:hi], ho[lo:hi])
    cfg = aq.TrainConfig(max_iterations=2, seed=0)
    try:
        ShardedTrainer(sh, len(x), lo).train_apq(2, 4, cfg, False)
        out[rank] = "no error"
    except aq.ZeroNormDatapoint as e:
        out[rank] = str(e)
    dist.destroy_process_group()


def test_failure_on_one_rank_raises_on_all():
    """A zero-norm anisotropic point in rank 1's shard fails its assignment
    pass (pq.hpp:137-146); both ranks raise the same error instead of rank 0
    waiting in a collective."""
    x, _, _ = _data(n=100)
    x[70] = 0.0
    hp = np.full(len(x), 4.0)
    ho = np.ones(len(x))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_zero_worker, args=(2, _free_port(), x, hp, ho, out), nprocs=2, join=True)
    assert out[0] == out[1]
    assert out[0].startswith("ZeroNormDatapoint")


def test_validation_errors():
    x, hp, ho = _data(n=20)
    t = ShardedTrainer(OracleShard(x, hp, ho), len(x), 0)
    with pytest.raises(aq.DimensionNotDivisible):
        t.train_apq(3, 4, aq.TrainConfig())
    with pytest.raises(aq.InvalidArgument):
        t.train_apq(2, 21, aq.TrainConfig())
    with pytest.raises(aq.EmptyDataset):
        ShardedTrainer(OracleShard(x[:0], hp[:0], ho[:0]), 0, 0).train_apq(2, 4, aq.TrainConfig())
