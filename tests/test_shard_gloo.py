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
        lo, hi = ShardComm.shard_bounds(len(x), WORLD, rank, align=1)
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


def test_shard_bounds_aligned_and_covering():
    from paper_2408_01391_b200.shard import ALIGN, ShardComm

    for n, w in [(1_000_000, 8), (100_000_000, 8), (1000, 3), (300, 2), (5, 4)]:
        b = [ShardComm.shard_bounds(n, w, r) for r in range(w)]
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[r][1] == b[r + 1][0] for r in range(w - 1))
        assert all(lo % ALIGN == 0 or lo == n for lo, _ in b)


# ---- the sharded ENGINE (GPU): two ranks on one GPU over gloo (eager
# steps), and one rank over NCCL with the all-reduce captured in the graphs


def _engine_run(x, c0, k, steps, dist=None, graph=False):
    dt = x.dtype.type
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200.kmeans import LloydEngine
    from paper_2408_01391_b200.tiles import default_config
    from paper_2408_01391_b200.abft import Threshold

    eng = LloydEngine(E.to_dev(x), c0, k, dt, default_config(dt), "abft",
                      Threshold.default_for(dt), 8, dist=dist, graph=graph)
    hist = []
    for it in range(steps):
        inertia, _, moved = eng.step(it, more=(lambda it=it: it + 1 < steps))
        hist.append((inertia, moved))
    labels, inertia = eng.final(steps)
    cent = E.to_host(eng.cent)
    eng.close()
    return labels, cent, hist, inertia


def _engine_data(dtype=np.float32):
    rng = np.random.default_rng(11)
    centers = rng.random((40, 24)) * 10
    lab = rng.integers(0, 40, 60_000)
    x = (centers[lab] + 0.3 * rng.standard_normal((60_000, 24))).astype(dtype)
    c0 = np.ascontiguousarray(x[rng.choice(len(x), 40, replace=False)])
    return x, c0


def _engine_worker(rank, port, backend, world, out, dtype_name="float32"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        from paper_2408_01391_b200.shard import ShardComm

        x, c0 = _engine_data(np.dtype(dtype_name).type)
        lo, hi = ShardComm.shard_bounds(len(x), world, rank)
        comm = ShardComm(lo)
        labels, cent, hist, inertia = _engine_run(x[lo:hi], c0, 40, 10, dist=comm,
                                                  graph=backend == "nccl")
        out[rank] = (lo, labels, cent, hist, inertia)
    finally:
        dist.destroy_process_group()


def _cuda_ok():
    return torch.cuda.is_available()


@pytest.mark.gpu
@pytest.mark.parametrize("backend,world,dtype_name", [("gloo", 2, "float32"), ("nccl", 1, "float32"),
                                                      ("gloo", 2, "float64")])
def test_sharded_engine_matches_single_process(backend, world, dtype_name):
    """LloydEngine(dist=ShardComm): gloo world 2 (eager steps, both ranks on
    cuda:0) and NCCL world 1 (the packed all-reduce captured in the step
    graphs) reproduce the single-process engine: labels identical,
    centroids / inertia equal to float64 re-association (world 2) or bitwise
    (world 1)."""
    if not _cuda_ok():
        pytest.skip("needs a CUDA device")
    x, c0 = _engine_data(np.dtype(dtype_name).type)
    ref_lab, ref_c, ref_hist, ref_inertia = _engine_run(x, c0, 40, 10, graph=True)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_engine_worker, args=(_free_port(), backend, world, out, dtype_name), nprocs=world,
                 join=True)
        res = dict(out)
    labels = np.concatenate([res[r][1] for r in range(world)])
    assert np.array_equal(labels, ref_lab)
    for r in range(world):
        _, _, cent, hist, inertia = res[r]
        if world == 1:
            assert cent.tobytes() == ref_c.tobytes()
            assert hist == ref_hist and inertia == ref_inertia
        else:
            np.testing.assert_allclose(cent, ref_c, rtol=1e-6, atol=0)
            assert abs(inertia - ref_inertia) <= 1e-12 * ref_inertia
            assert all(abs(a[0] - b[0]) <= 1e-12 * b[0] for a, b in zip(hist, ref_hist))
    assert all(np.array_equal(res[0][2], res[r][2]) for r in range(world))
