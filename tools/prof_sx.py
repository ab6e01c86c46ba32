"""Pass-1 pair-kernel time at c3 shapes (streamed X), with FTK_TC_DEBUG honoured."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.matrix import gaussian_mixture  # noqa: E402

n, d, k = (int(v) for v in sys.argv[1:4])
x, _, _ = gaussian_mixture(n, d, k, 0.25, precision="single", seed=0)
rng = np.random.default_rng(0)
y = np.ascontiguousarray(x[rng.choice(len(x), k, replace=False)])
x_t, y_t = E.to_dev(x), E.to_dev(y)
yn = E.row_sq_norms_dev(y_t)
for r in range(3):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant="tc")
    en.record()
    torch.cuda.synchronize()
print(f"n={n} d={d} k={k} dbg={os.environ.get('FTK_TC_DEBUG', '0')}: assign {st.elapsed_time(en):.3f} ms, "
      f"pass-1 kernel {E.tc_last_kernel_ms():.3f} ms, fallback {E.tc_fallback_rows()}")
