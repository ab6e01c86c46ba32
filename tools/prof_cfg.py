"""Time Lloyd steps of any BASELINE config on one GPU (device-resident data).

  python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--ft", default="off")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--variant", default="auto")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import gemm  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402

gemm.set_variant(a.variant)
dt = np.float32 if a.dtype == "f32" else np.float64
x, _, _ = P.gaussian_mixture(a.n, a.d, a.k, 0.25, precision="single" if dt == np.float32 else "double",
                             seed=0)
x_t = E.to_dev(x)
c0 = P.init_centroids(x, a.k, seed=0, method="random-sample")
eng = LloydEngine(x_t, c0, a.k, dt, P.default_config(dt), a.ft, P.Threshold.default_for(dt), 64)
flops = 2.0 * a.n * a.d * a.k
for it in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inertia, unch, moved = eng.step(it)
    wall = (time.perf_counter() - t0) * 1e3
    print(f"it {it}: wall {wall:.3f} ms  assign {eng.assign_ms:.3f} ms "
          f"({flops / eng.assign_ms / 1e9:.1f} TFLOP/s)  update {eng.update_ms:.3f} ms")
eng.close()
