"""Pass-1 pair-kernel time (CUDA events) under the FTK_TC_DEBUG switches:
1 = no screen math, 2 = no refine math, 4 = TMEM drain only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.matrix import gaussian_mixture  # noqa: E402

x, _, _ = gaussian_mixture(1_000_000, 128, 1024, 0.25, precision="single", seed=0)
rng = np.random.default_rng(0)
y = np.ascontiguousarray(x[rng.choice(len(x), 1024, replace=False)])
x_t, y_t = E.to_dev(x), E.to_dev(y)
yn = E.row_sq_norms_dev(y_t)
chk = os.environ.get("CHK", "1") == "1"
for r in range(4):
    ev = E.DevEvents(64 * 64)
    E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant="tc", checked=chk, delta_rel=1e-4,
                 abs_tol=0.0, events=ev)
    torch.cuda.synchronize()
print(f"dbg={os.environ.get('FTK_TC_DEBUG', '0')} chk={chk} pass-1 kernel {E.tc_last_kernel_ms():.4f} ms")
