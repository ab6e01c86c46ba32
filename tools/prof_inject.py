"""Cost of an injected Lloyd step at c2 (graph steps, ABFT): per-step CUDA
event times with one scheduled flip every 4th iteration, and (under ncu) the
launch list of those steps.

  python tools/prof_inject.py [--steps 24]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=24)
ap.add_argument("--n", type=int, default=1_000_000)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402
from paper_2408_01391_b200.tiles import default_config  # noqa: E402

K, D = 1024, 128
x, _, _ = P.gaussian_mixture(a.n, D, K, 0.25, precision="single", seed=0)
x_t = E.to_dev(x)
c0 = P.init_centroids(x, K, seed=0, method="random-sample")
rng = np.random.default_rng(0)
ents = [FaultEntry(it, (int(rng.integers(0, a.n // 32)), int(rng.integers(0, 4))),
                   (int(rng.integers(0, 32)), int(rng.integers(0, 256))), 27)
        for it in range(4, a.steps + 8, 4)]
hook = ScheduledFaultHook(FaultSchedule(ents))
eng = LloydEngine(x_t, c0, K, np.float32, default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64, gemm_hook=hook, graph=True)
times = []
for it in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.step(it)
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t0) * 1e3)
for it, t in enumerate(times):
    print(f"it {it:3d} {'INJ' if it % 4 == 0 and it >= 4 else '   '} wall {t:.3f} ms")
clean = [t for i, t in enumerate(times) if i >= 2 and not (i % 4 == 0 and i >= 4)]
inj = [t for i, t in enumerate(times) if i >= 4 and i % 4 == 0]
print(f"median clean {np.median(clean):.3f} ms, injected {np.median(inj):.3f} ms; "
      f"report: {eng.report.detections} detections, {eng.report.corrections} corrections")
eng.close()
