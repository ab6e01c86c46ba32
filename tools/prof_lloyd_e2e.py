"""Repeated public-API fits from pinned host X (bench.py's e2e leg) with the
fit's own phase timings, to see where slow fits lose time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402

x = bench.make_data()
xp = torch.from_numpy(x).pin_memory()
conf = P.KMeansConfig(k=bench.K, max_iters=10, tol=0.0, seed=0, init="random-sample", ft_mode="abft")
for r in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.lloyd(xp, conf)
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) * 1e3
    tm = {k: round(v / 1e6, 2) for k, v in res.timings.items()}
    print(f"fit {r}: {w:.1f} ms {tm}")
