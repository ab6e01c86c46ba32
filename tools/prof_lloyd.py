"""Per-phase timing of Lloyd iterations on c2 (N=1e6, D=128, K=1024)."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--ft", default="off")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--k", type=int, default=1024)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402

x, _, _ = P.gaussian_mixture(a.n, a.d, a.k, 0.25, precision="single", seed=0)
x_t = E.to_dev(x)
c0 = P.init_centroids(x, a.k, seed=0, method="random-sample")
eng = LloydEngine(x_t, c0, a.k, np.float32, P.default_config(np.float32), a.ft,
                  P.Threshold.default_for(np.float32), 64)
for it in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inertia, unch, moved = eng.step(it)
    wall = (time.perf_counter() - t0) * 1e3
    fb = E.tc_fallback_rows()
    print(f"it {it}: wall {wall:.3f} ms  assign {eng.assign_ms:.3f} ms  update {eng.update_ms:.3f} ms  "
          f"inertia {inertia:.1f} fallback {fb}")
