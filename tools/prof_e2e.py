"""Wall time of the public-API fit from pinned host X (bench.py's e2e leg),
repeated, with a cProfile of one call."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402

x = bench.make_data()
xp = torch.from_numpy(x).pin_memory()
conf = P.KMeansConfig(k=bench.K, max_iters=50, tol=0.0, seed=0, init="random-sample", ft_mode="abft")
P.lloyd(xp[:4096], P.KMeansConfig(k=16, max_iters=2, init="random-sample"))
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if r == 2:
        pr = cProfile.Profile()
        pr.enable()
    res = P.lloyd(xp, conf)
    torch.cuda.synchronize()
    if r == 2:
        pr.disable()
    print(f"fit {r}: {time.perf_counter() - t0:.4f} s, iters {res.iters}")
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
