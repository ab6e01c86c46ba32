"""bench.py's e2e leg alone: a 10-iteration ABFT fit through the public lloyd
from a numpy array (pageable host memory), median wall time of 5 fits after
one warm fit.  FTK_H2D_THREADS sets the staged uploader's copy threads."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402

x = bench.make_data(bench.CONFIGS["c2"])
conf = P.KMeansConfig(k=1024, max_iters=10, tol=0.0, seed=0, init="random-sample", ft_mode="abft")
P.lloyd(x, conf)
walls = []
for r in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.lloyd(x, conf)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
w = statistics.median(walls)
print(f"threads={os.environ.get('FTK_H2D_THREADS', 'default')}: fit {w * 1e3:.1f} ms, {res.iters / w:.1f} iter/s "
      f"({[round(v * 1e3, 1) for v in walls]})")
