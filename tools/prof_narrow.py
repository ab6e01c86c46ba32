"""c3 wide-row shapes through the narrow screen: per Lloyd step, the screen
kernel (CUDA events), the whole assignment, the winner-pass / exact-row counts.

  python tools/prof_narrow.py [--n 1000000] [--ft off|abft] [--steps 6]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--ft", default="off")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--shapes", default="16x512,32x2048,8x512,8x2048,16x2048,32x512")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import _native as N  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402

peak = 6464.0
lib = N.load()
for sh in a.shapes.split(","):
    k, d = (int(v) for v in sh.split("x"))
    x, _, _ = P.gaussian_mixture(a.n, d, k, 0.25, precision="single", seed=0)
    x_t = E.to_dev(x)
    c0 = P.init_centroids(x, k, seed=0, method="random-sample")
    eng = LloydEngine(x_t, c0, k, np.float32, P.default_config(np.float32), a.ft,
                      P.Threshold.default_for(np.float32), 64)
    floor_ms = a.n * d * 4 / peak / 1e6
    for it in range(a.steps):
        eng.step(it)
        torch.cuda.synchronize()
        ms = ctypes.c_float(0)
        lib.ftk_tc_last_kernel_ms(E.ctx(), ctypes.byref(ms))
        st = (ctypes.c_int64 * 3)()
        lib.ftk_tc_fallback_rows(E.ctx(), st, E.stream())
        print(f"K{k} D{d} {a.ft} it {it}: screen {ms.value:.3f} ms ({a.n * d * 4 / ms.value / 1e6:.0f} GB/s, "
              f"floor {floor_ms:.3f}) assign {eng.assign_ms:.3f} update {eng.update_ms:.3f} "
              f"winner_rows {st[0]} exact_rows {st[1]} flags {st[2]}", flush=True)
    eng.close()
    del x_t
    torch.cuda.empty_cache()
