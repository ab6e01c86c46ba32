"""k-means++ seeding time on the c2 shape (N=1e6, D=128, K=1024 fp32):
device D^2 updates + device pairwise total + device searchsorted, one
host read per pick.  Also checks the first 64 picks against a host replay of
the reference's own numpy recurrence (float64)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import _kmeanspp_dev  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
x, _, _ = P.gaussian_mixture(n, 128, 1024, 0.25, precision="single", seed=0)
x_t = E.to_dev(x)
_kmeanspp_dev(x_t, 8, np.random.default_rng(1))  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
picks = _kmeanspp_dev(x_t, 1024, np.random.default_rng(0))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
# reference recurrence (kmeans.py:86-103) for the first 64 picks
rng = np.random.default_rng(0)
x64 = x.astype(np.float64)
ref = [int(rng.integers(0, n))]
d2 = ((x64 - x64[ref[0]]) ** 2).sum(axis=1)
for c in range(1, 64):
    tot = d2.sum()
    p = int(rng.integers(0, n)) if tot <= 0 else min(int(np.searchsorted(np.cumsum(d2), rng.random() * tot, side="right")), n - 1)
    ref.append(p)
    d2 = np.minimum(d2, ((x64 - x64[p]) ** 2).sum(axis=1))
print(f"kmeanspp N={n} K=1024: {dt:.3f} s ({dt / 1024 * 1e3:.3f} ms/pick); first 64 picks equal the "
      f"reference recurrence: {list(picks[:64]) == ref}")
