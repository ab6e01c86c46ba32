"""Host turnaround per Lloyd step: graph replays back to back (no control
readback between them) vs the engine's step() (replay, sync, host decisions)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_01391_b200 as P  # noqa: E402
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.kmeans import LloydEngine  # noqa: E402
from paper_2408_01391_b200.tiles import default_config  # noqa: E402

x = bench.make_data()
x_t = E.to_dev(x)
c0 = P.init_centroids(x, bench.K, seed=0, method="random-sample")
eng = LloydEngine(x_t, c0, bench.K, np.float32, default_config(np.float32), "abft",
                  P.Threshold.default_for(np.float32), 64, graph=True)
for it in range(6):
    eng.step(it)
torch.cuda.synchronize()
n = 40
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for it in range(6, 6 + n):
    eng.step(it)
en.record()
torch.cuda.synchronize()
step_ms = st.elapsed_time(en) / n
g0, g1 = eng.graphs[0][0], eng.graphs[1][0]
torch.cuda.synchronize()
st.record()
for i in range(n):
    (g0 if i % 2 == 0 else g1).replay()
en.record()
torch.cuda.synchronize()
rep_ms = st.elapsed_time(en) / n
print(f"step() {step_ms:.4f} ms, back-to-back replay {rep_ms:.4f} ms, turnaround {step_ms - rep_ms:.4f} ms")
eng.close()
