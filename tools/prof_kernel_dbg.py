"""Pass-1 CTA-pair kernel time at c2 with parts of its work switched off
(FTK_TC_DEBUG bits: 1 skip the screen math, 2 skip the refine, 4 TMEM drain
only) -- which role bounds the kernel.  Results are wrong under the bits (rows
go uncertified); only the pass-1 kernel time (CUDA events) is read."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402

x, _, _ = P.gaussian_mixture(1_000_000, 128, 1024, 0.25, precision="single", seed=0)
c0 = P.init_centroids(x, 1024, seed=0, method="random-sample")
eng = LloydEngine(E.to_dev(x), c0, 1024, np.float32, P.default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64)
for it in range(4):
    eng.step(it)
cent = eng.cent.clone()
yn = E.row_sq_norms_dev(cent)
for dbg in ([int(v) for v in sys.argv[1:]] or [0, 2, 1, 4, 3, 6, 0]):
    os.environ["FTK_TC_DEBUG"] = str(dbg)
    ms = []
    for r in range(3):
        ev = E.DevEvents(64)
        E.assign_dev(eng.x_t, cent, yn, (32, 256, 16), variant="pair", checked=True, delta_rel=1e-4,
                     abs_tol=0.0, events=ev)
        torch.cuda.synchronize()
        ms.append(E.tc_last_kernel_ms())
    print(f"dbg={dbg}: pass-1 kernel {np.median(ms):.4f} ms  ({ms})", flush=True)
