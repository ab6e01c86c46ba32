import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_01391_b200 import _engine as E
sys.path.insert(0, "oracle")
import oracle as O
for d in (256, 260, 288, 512):
    for k in (16, 200):
        rng = np.random.default_rng(1)
        x = np.ascontiguousarray(rng.standard_normal((2048, d)), dtype=np.float32)
        y = np.ascontiguousarray(x[rng.choice(2048, k, replace=False)] + 0.3 * rng.standard_normal((k, d)).astype(np.float32))
        x_t, y_t = E.to_dev(x), E.to_dev(y)
        idx, val = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), (32, 256, 16), variant="tc")
        fb = E.tc_fallback_rows()
        lab, v = O.assign(x, y)
        print(d, k, "fallback", fb, "labels ok", np.array_equal(E.to_host(idx), lab))
