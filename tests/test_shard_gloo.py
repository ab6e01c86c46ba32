"""Row-sharded multi-process Lloyd plumbing (shard.ShardComm) on CPU with the
gloo backend, world_size 2: the per-iteration packed all-reduce of the
float64 partials and the cross-rank farthest-point reseed must reproduce the
single-process reference results (kmeans.py:167-171, 197-206)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((103, 5)).astype(np.float32)
    labels = rng.integers(0, 6, 103).astype(np.int64)
    labels[labels == 4] = 5  # cluster 4 stays empty
    sq = rng.random(103)
    sq[[17, 80]] = 9.0       # tie across shards: lowest global row wins
    return x, labels, sq


def _reference(x, labels, sq, k):
    sums = np.zeros((k, x.shape[1]))
    for f in range(x.shape[1]):
        sums[:, f] = np.bincount(labels, weights=x[:, f].astype(np.float64), minlength=k)
    counts = np.bincount(labels, minlength=k)
    inertia = float(np.sum(sq))
    far = int(np.argmax(sq))  # first maximum
    return sums, counts, inertia, far


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2408_01391_b200.shard import ShardComm

        x, labels, sq = _data()
        k = 6
        lo, hi = ShardComm.shard_bounds(len(x), WORLD, rank)
        comm = ShardComm(lo)
        xs, ls = x[lo:hi], labels[lo:hi]
        sums = torch.zeros((k, x.shape[1]), dtype=torch.float64)
        for f in range(x.shape[1]):
            sums[:, f] = torch.from_numpy(
                np.bincount(ls, weights=xs[:, f].astype(np.float64), minlength=k))
        counts = torch.from_numpy(np.bincount(ls, minlength=k).astype(np.int64))
        ctl_f64 = torch.tensor([float(np.sum(sq[lo:hi])), 0.0], dtype=torch.float64)
        ctl_i32 = torch.tensor([1 if rank == 0 else 0], dtype=torch.int32)  # rank 1 changed
        comm.reduce_partials(sums, counts, ctl_f64, ctl_i32)
        cent = torch.zeros((k, x.shape[1]), dtype=torch.float32)
        sq_t = torch.from_numpy(sq[lo:hi].copy())
        comm.reseed(torch.from_numpy(xs), counts, sq_t, cent)
        out[rank] = (sums.numpy().copy(), counts.numpy().copy(), float(ctl_f64[0]),
                     int(ctl_i32[0]), cent.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_sharded_partials_and_reseed_match_single_process():
    x, labels, sq = _data()
    ref_sums, ref_counts, ref_inertia, far = _reference(x, labels, sq, 6)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
        res = dict(out)
    for rank in range(WORLD):
        sums, counts, inertia, unchanged, cent = res[rank]
        # f64 partials summed per shard then across ranks: equal to ~1 ulp
        np.testing.assert_allclose(sums, ref_sums, rtol=1e-15, atol=1e-12)
        assert np.array_equal(counts, ref_counts)
        assert abs(inertia - ref_inertia) <= 1e-12 * abs(ref_inertia)
        assert unchanged == 0  # one rank changed labels -> not unchanged
        # empty cluster 4 takes the global farthest point, lowest global row on ties
        assert far == 17
        assert np.array_equal(cent[4], x[far])
    # every rank holds the same result (the all-reduce is the only exchange)
    assert all(np.array_equal(res[0][0], res[r][0]) for r in range(WORLD))
    assert all(np.array_equal(res[0][4], res[r][4]) for r in range(WORLD))
