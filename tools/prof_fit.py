"""Phase timeline of one fit from pinned host X (the e2e leg), max_iters=10:
H2D, engine setup (row norms, row bounds), each step (graph capture shows
up in the first graph step)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402
from paper_2408_01391_b200.tiles import default_config  # noqa: E402

x = bench.make_data()
xp = torch.from_numpy(x).pin_memory()
P.lloyd(xp[:4096], P.KMeansConfig(k=16, max_iters=2, init="random-sample"))
graph = os.environ.get("GRAPH", "1") == "1"
import gc
gc.disable()
for rep in range(3):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    lab = []
    x_t = E.to_dev(xp)
    torch.cuda.synchronize(); T.append(time.perf_counter()); lab.append("h2d")
    c0 = P.init_centroids(x, bench.K, seed=0, method="random-sample")
    T.append(time.perf_counter()); lab.append("init")
    eng = LloydEngine(x_t, c0, bench.K, np.float32, default_config(np.float32), "abft",
                      P.Threshold.default_for(np.float32), 64, graph=graph)
    torch.cuda.synchronize(); T.append(time.perf_counter()); lab.append("engine")
    for it in range(10):
        eng.step(it)
        T.append(time.perf_counter()); lab.append(f"s{it}")
    eng.final(10)
    torch.cuda.synchronize(); T.append(time.perf_counter()); lab.append("final")
    eng.close()
    print(f"rep {rep} total {1e3*(T[-1]-T[0]):.1f} ms: " +
          " ".join(f"{l}={1e3*(b-a):.2f}" for l, a, b in zip(lab, T, T[1:])))
