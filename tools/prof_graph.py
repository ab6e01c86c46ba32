"""Lloyd steps with and without CUDA-graph replay (c2 shape)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_01391_b200 as P
from paper_2408_01391_b200 import _engine as E
from paper_2408_01391_b200.kmeans import LloydEngine
ft = sys.argv[1] if len(sys.argv) > 1 else "abft"
x, _, _ = P.gaussian_mixture(1000000, 128, 1024, 0.25, precision="single", seed=0)
x_t = E.to_dev(x)
c0 = P.init_centroids(x, 1024, seed=0, method="random-sample")
res = {}
for graph in (False, True):
    eng = LloydEngine(x_t, c0, 1024, np.float32, P.default_config(np.float32), ft,
                      P.Threshold.default_for(np.float32), 64, graph=graph)
    outs = []
    for it in range(4):
        outs.append(eng.step(it))
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for it in range(4, 24):
        outs.append(eng.step(it))
    en.record(); torch.cuda.synchronize()
    res[graph] = (st.elapsed_time(en) / 20, outs, E.to_host(eng.cent).copy())
    eng.close()
print(f"{ft}: eager {res[False][0]:.3f} ms/step, graph {res[True][0]:.3f} ms/step")
assert res[False][1] == res[True][1], "step outputs differ"
assert res[False][2].tobytes() == res[True][2].tobytes(), "centroids differ"
print("graph == eager (bitwise)")
