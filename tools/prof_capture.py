"""Cost of capturing the Lloyd step graph: torch.cuda.graph vs manual capture."""
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
x_t = E.to_dev(x)
c0 = P.init_centroids(x, bench.K, seed=0, method="random-sample")
eng = LloydEngine(x_t, c0, bench.K, np.float32, default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64, graph=True)
eng.step(0)
torch.cuda.synchronize()
pool = torch.cuda.graph_pool_handle()
s = torch.cuda.Stream()
for rep in range(3):
    g = torch.cuda.CUDAGraph()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        g.capture_begin()
        t1 = time.perf_counter()
        eng._device_part(1)
        t2 = time.perf_counter()
        g.capture_end()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    g.replay()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    g.replay()
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"manual: begin {1e3*(t1-t0):.2f} ms record {1e3*(t2-t1):.2f} end+inst {1e3*(t3-t2):.2f} "
          f"first replay {1e3*(t5-t4):.2f} second {1e3*(t6-t5):.2f}")
for rep in range(2):
    g = torch.cuda.CUDAGraph()
    t0 = time.perf_counter()
    with torch.cuda.graph(g, pool=pool):
        eng._device_part(1)
    print(f"torch.cuda.graph: {1e3*(time.perf_counter()-t0):.2f} ms")
