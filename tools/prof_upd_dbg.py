"""Replayed-chain and pass-2 counts of eager c2 Lloyd steps (FTK_UPD_DEBUG=1
prints the update's replayed chains; tc_fallback_rows the rows pass 1 left
uncertified).  python tools/prof_upd_dbg.py [steps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FTK_UPD_DEBUG"] = "1"
import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x, _, _ = P.gaussian_mixture(1_000_000, 128, 1024, 0.25, precision="single", seed=0)
x_t = E.to_dev(x)
c0 = P.init_centroids(x, 1024, seed=0, method="random-sample")
eng = LloydEngine(x_t, c0, 1024, np.float32, P.default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64, graph=False)
for it in range(steps):
    eng.step(it, eager=True)
    print(f"it {it}: assign {eng.assign_ms:.3f} ms update {eng.update_ms:.3f} ms "
          f"fallback rows {E.tc_fallback_rows()}", file=sys.stderr, flush=True)
eng.close()
