"""Per-step device times of the c2 ABFT Lloyd loop under a fault schedule
(which steps are injected, which replay a graph)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.faults import ScheduledFaultHook  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402
from paper_2408_01391_b200.tiles import default_config  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
x = bench.make_data()
x_t = E.to_dev(x)
K = bench.K
c0 = P.init_centroids(x, K, seed=0, method="random-sample")
sched = bench._campaign_schedule(2e-6, steps + 1, x.shape[0], K, seed=2)
hook = ScheduledFaultHook(sched)
eng = LloydEngine(x_t, c0, K, np.float32, default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64, gemm_hook=hook, graph=True)
inj_its = sorted({e.iteration for e in sched.entries}) if hasattr(sched, "entries") else []
for it in range(steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record()
    eng.step(it)
    b.record()
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) * 1e3
    g = "graph" if eng._graph_ok(it) else "eager"
    print(f"it {it:3d} {g} inj={bool(sched.for_iteration(it))} dev {a.elapsed_time(b):7.3f} ms wall {w:7.3f} ms "
          f"det {eng.report.n_detections if hasattr(eng.report, 'n_detections') else len(eng.report.events)}")
eng.close()
