"""Short driver for ncu captures / timing: fused assignment of the c2 shape
(N=1e6, D=128, K=1024 f32) per variant, after a warm-up call."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="tc")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--iters", type=int, default=0, help="Lloyd iterations to converge centroids first")
ap.add_argument("--checked", action="store_true", help="ABFT (checksum-protected) assignment")
a = ap.parse_args()

import torch  # noqa: E402

from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.matrix import gaussian_mixture  # noqa: E402

x, _, _ = gaussian_mixture(a.n, a.d, a.k, 0.25, precision="single", seed=0)
rng = np.random.default_rng(0)
y = np.ascontiguousarray(x[rng.choice(a.n, a.k, replace=False)])
x_t, y_t = E.to_dev(x), E.to_dev(y)
if a.iters:
    import paper_2408_01391_b200 as P
    from paper_2408_01391_b200.kmeans import LloydEngine
    eng = LloydEngine(x_t, y, a.k, np.float32, P.default_config(np.float32), "off", None, 1)
    for it in range(a.iters):
        eng.step(it)
    y_t = eng.cent
yn = E.row_sq_norms_dev(y_t)
for r in range(a.reps):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    if a.checked:
        ev = E.DevEvents(64)
        E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant=a.variant, checked=True, delta_rel=1e-4,
                     abs_tol=0.0, events=ev)
    else:
        E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant=a.variant)
    en.record()
    torch.cuda.synchronize()
    fb = E.tc_fallback_rows() if a.variant == "tc" else (-1, -1)
    print(f"rep {r}: {st.elapsed_time(en):.3f} ms  uncertified(pass1, pass2)={fb}  "
          f"TFLOP/s={2 * a.n * a.d * a.k / st.elapsed_time(en) / 1e9:.1f}")
