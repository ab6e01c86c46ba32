"""CPU oracle for the FT K-means Lloyd hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker or as the timed CPU baseline.  The product package
(``paper_2408_01391_b200``) never imports it.

It restates the reference package ``ftkmeans`` 0.1.0 (numba, CPU) on top of
the C restatement in ``ftk_oracle.c``:

* ``assign``          -> gemm.fused_assign / _kernels._assign_range
                          (gemm.py:88-141, _kernels.py:432-475)
* ``row_sq_norms``    -> matrix.row_sq_norms / _kernels._row_sq_norms
                          (matrix.py:113-120, _kernels.py:106-114)
* ``update_step``     -> kmeans.update_step (kmeans.py:135-207, DMR omitted:
                          a fault-free duplicate is bitwise equal by construction)
* ``init_centroids``  -> kmeans.init_centroids (kmeans.py:69-103)
* ``lloyd``           -> kmeans.lloyd, fault-free (kmeans.py:210-319)
* ``pairwise_sum``    -> numpy float64 add.reduce (used for inertia)

Pinning: tests/test_oracle.py checks every function against the golden
vectors in tests/golden/, which tests/golden/make_golden.py produced by
running the reference itself in the build container.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _cpu_has_avx2():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    return " avx2 " in line + " "
    except OSError:
        pass
    return False


def build():
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    name = "libftk_oracle_v3.so" if _cpu_has_avx2() else "libftk_oracle_v2.so"
    path = os.path.join(_HERE, "_build", name)
    if not os.path.exists(path):
        build()
    L = ctypes.CDLL(path)
    i64, p, dbl, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double, ctypes.c_int
    for nm in ("ftko_row_sq_norms_f32", "ftko_row_sq_norms_f64"):
        getattr(L, nm).argtypes = [p, i64, i64, p]
    for nm in ("ftko_assign_f32", "ftko_assign_f64"):
        getattr(L, nm).argtypes = [p, p, p, i64, i64, i64, p, p, ci]
    L.ftko_dot_f32.argtypes = [p, p, i64]
    L.ftko_dot_f32.restype = ctypes.c_float
    L.ftko_dot_f64.argtypes = [p, p, i64]
    L.ftko_dot_f64.restype = dbl
    L.ftko_update_sums.argtypes = [ci, p, p, i64, i64, i64, p, p, ci]
    L.ftko_pairwise_sum.argtypes = [p, i64]
    L.ftko_pairwise_sum.restype = dbl
    L.ftko_row_norms_pairwise.argtypes = [p, i64, i64, p]
    L.ftko_checked_assign.argtypes = [ci, p, p, p, i64, i64, i64, i64, i64, i64, dbl, dbl, p, p, ci]
    L.ftko_checked_assign.restype = i64
    _LIB = L
    return L


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _threads(threads):
    return int(threads) if threads else (os.cpu_count() or 1)


def row_sq_norms(x):
    x = np.ascontiguousarray(x)
    out = np.empty(x.shape[0], dtype=x.dtype)
    fn = lib().ftko_row_sq_norms_f32 if x.dtype == np.float32 else lib().ftko_row_sq_norms_f64
    fn(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
    return out


def assign(x, y, y_norms=None, threads=None):
    """Returns (labels int64, min_dists dtype) exactly as fused_assign."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    if y_norms is None:
        y_norms = row_sq_norms(y)
    yn = np.ascontiguousarray(y_norms, dtype=x.dtype)
    m = x.shape[0]
    idx = np.empty(m, dtype=np.int64)
    val = np.empty(m, dtype=x.dtype)
    fn = lib().ftko_assign_f32 if x.dtype == np.float32 else lib().ftko_assign_f64
    fn(_ptr(x), _ptr(y), _ptr(yn), m, y.shape[0], x.shape[1], _ptr(idx), _ptr(val),
       _threads(threads))
    return idx, val


def checked_assign(x, y, y_norms=None, block=None, delta_rel=None, abs_tol=0.0, threads=None):
    """abft.checked_assign's fault-free path (abft.py:247-365, _kernels.py:479-612):
    the same labels/min_dists as ``assign`` plus the reference's per-tile,
    per-k-interval e1 column-checksum verification.  Detection only: returns
    (labels, min_dists, violations); a violation cannot be diagnosed here."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    if y_norms is None:
        y_norms = row_sq_norms(y)
    yn = np.ascontiguousarray(y_norms, dtype=x.dtype)
    f64 = x.dtype == np.float64
    if block is None:  # the reference's default tiles (tiles.py:70-74)
        block = (64, 64, 16) if f64 else (32, 256, 16)
    if delta_rel is None:  # Threshold.default_for (abft.py:41-68)
        delta_rel = 1e-10 if f64 else 1e-4
    m = x.shape[0]
    idx = np.empty(m, dtype=np.int64)
    val = np.empty(m, dtype=x.dtype)
    nv = lib().ftko_checked_assign(1 if f64 else 0, _ptr(x), _ptr(y), _ptr(yn), m, y.shape[0],
                                   x.shape[1], int(block[0]), int(block[1]), int(block[2]),
                                   float(delta_rel), float(abs_tol), _ptr(idx), _ptr(val),
                                   _threads(threads))
    return idx, val, int(nv)


def exact_dot(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    if a.dtype == np.float32:
        return np.float32(lib().ftko_dot_f32(_ptr(a), _ptr(b), a.shape[0]))
    return np.float64(lib().ftko_dot_f64(_ptr(a), _ptr(b), a.shape[0]))


def update_sums(x, labels, k, threads=None):
    x = np.ascontiguousarray(x)
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    sums = np.empty((k, x.shape[1]), dtype=np.float64)
    counts = np.empty(k, dtype=np.int64)
    lib().ftko_update_sums(1 if x.dtype == np.float64 else 0, _ptr(x), _ptr(lab), x.shape[0],
                           x.shape[1], k, _ptr(sums), _ptr(counts), _threads(threads))
    return sums, counts


def pairwise_sum(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().ftko_pairwise_sum(_ptr(a), a.shape[0]))


def row_norms(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty(a.shape[0], dtype=np.float64)
    lib().ftko_row_norms_pairwise(_ptr(a), a.shape[0], a.shape[1], _ptr(out))
    return out


def update_step(x, labels, k, sq_dists=None, threads=None):
    """kmeans.update_step (kmeans.py:135-207), fault-free."""
    x = np.ascontiguousarray(x)
    sums, counts = update_sums(x, labels, k, threads)
    cent = np.zeros((k, x.shape[1]), dtype=np.float64)
    ne = counts > 0
    cent[ne] = sums[ne] / counts[ne, None]
    empty = np.flatnonzero(~ne)
    if empty.size:
        if sq_dists is None:
            own = cent[labels]
            sq_dists = ((x.astype(np.float64) - own) ** 2).sum(axis=1)
        sq = np.array(sq_dists, dtype=np.float64)
        for j in empty:
            far = int(np.argmax(sq))
            cent[j] = x[far].astype(np.float64)
            sq[far] = -np.inf
    return np.ascontiguousarray(cent, dtype=x.dtype), counts


def init_centroids(x, k, seed=0, method="kmeanspp"):
    """kmeans.init_centroids (kmeans.py:69-103): numpy Generator draws."""
    m = x.shape[0]
    rng = np.random.default_rng(seed)
    if method == "random-sample":
        return np.ascontiguousarray(x[rng.choice(m, size=k, replace=False)])
    x64 = x.astype(np.float64)
    cs = np.empty((k, x.shape[1]), dtype=np.float64)
    cs[0] = x64[int(rng.integers(0, m))]
    d2 = ((x64 - cs[0]) ** 2).sum(axis=1)
    for c in range(1, k):
        tot = d2.sum()
        if tot <= 0:
            pick = int(rng.integers(0, m))
        else:
            pick = min(int(np.searchsorted(np.cumsum(d2), rng.random() * tot, side="right")), m - 1)
        cs[c] = x64[pick]
        d2 = np.minimum(d2, ((x64 - cs[c]) ** 2).sum(axis=1))
    return np.ascontiguousarray(cs, dtype=x.dtype)


def _assign_ft(x, c, ft_mode, threads):
    if ft_mode == "off":
        return assign(x, c, threads=threads)
    lab, md, nv = checked_assign(x, c, threads=threads)
    if nv:
        raise RuntimeError(f"oracle checked_assign: {nv} checksum violations (not diagnosed here)")
    return lab, md


def lloyd(x, k, max_iters=300, tol=1e-4, seed=0, init="kmeanspp", threads=None,
          centroids=None, ft_mode="off"):
    """kmeans.lloyd (kmeans.py:210-319), fault-free.  ft_mode "abft" runs the
    checksum-verified assignment (same results: a fault-free protected run is
    bit-identical to the unprotected one, test_abft.py:141-149), so its cost
    is the reference's; a checksum violation raises."""
    x = np.ascontiguousarray(x)
    t_tot = time.perf_counter_ns()
    t0 = time.perf_counter_ns()
    c = init_centroids(x, k, seed, init) if centroids is None else np.array(centroids, dtype=x.dtype)
    timings = {"init_ns": time.perf_counter_ns() - t0, "assign_ns": 0, "update_ns": 0}
    x_sq = row_sq_norms(x).astype(np.float64)
    eps = float(np.finfo(x.dtype).eps)
    labels = None
    hist = []
    iters = 0
    converged = False
    for it in range(max_iters):
        t0 = time.perf_counter_ns()
        new, md = _assign_ft(x, c, ft_mode, threads)
        timings["assign_ns"] += time.perf_counter_ns() - t0
        sq = md.astype(np.float64) + x_sq
        hist.append(max(0.0, pairwise_sum(sq)))
        unchanged = labels is not None and np.array_equal(labels, new)
        labels = new
        t0 = time.perf_counter_ns()
        nc, _ = update_step(x, labels, k, sq_dists=sq, threads=threads)
        timings["update_ns"] += time.perf_counter_ns() - t0
        iters = it + 1
        num = row_norms(nc.astype(np.float64) - c.astype(np.float64))
        den = row_norms(c.astype(np.float64)) + eps
        moved = float((num / den).max()) if k else 0.0
        c = nc
        if unchanged or moved < tol:
            converged = True
            break
    labels, md = _assign_ft(x, c, ft_mode, threads)
    inertia = max(0.0, pairwise_sum(md.astype(np.float64) + x_sq))
    timings["total_ns"] = time.perf_counter_ns() - t_tot
    return {
        "centroids": c, "assignments": labels, "inertia": inertia, "iters": iters,
        "converged": converged, "inertia_history": hist, "timings": timings,
    }
