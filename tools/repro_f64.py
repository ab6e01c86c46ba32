import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_01391_b200 as P
rng = np.random.default_rng(202)
for case in range(40):
    m, n, k = int(rng.integers(1, 192)), int(rng.integers(1, 64)), int(rng.integers(1, 80))
    x = np.ascontiguousarray(rng.standard_normal((m, n)), dtype=np.float64)
    y = np.ascontiguousarray(rng.standard_normal((k, n)), dtype=np.float64)
    which = sys.argv[1]
    if which == "plain":
        r = P.fused_assign(x, y)
    else:
        r, rep = P.checked_assign(x, y)
    import torch; torch.cuda.synchronize()
    print(case, m, n, k, "ok", flush=True)
