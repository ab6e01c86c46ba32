# r2x: DADD latency; c4 cluster sizes
OUT=gpurun_out/r2x; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/dadd tools/probes/dadd_latency.cu && /tmp/dadd | tee $OUT/dadd.log
python - > $OUT/c4_sizes.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_01391_b200 as P
from paper_2408_01391_b200 import _engine as E
from paper_2408_01391_b200.kmeans import LloydEngine
x, _, _ = P.gaussian_mixture(10_000_000, 64, 256, 0.25, precision="double", seed=0)
c0 = P.init_centroids(x, 256, seed=0, method="random-sample")
eng = LloydEngine(E.to_dev(x), c0, 256, np.float64, P.default_config(np.float64), "off", None, 64)
for it in range(4):
    eng.step(it)
    lab = eng.A.labels[eng.slot].cpu().numpy()
    cnt = np.bincount(lab, minlength=256)
    print(it, "update", round(eng.update_ms, 3), "counts min/mean/max", cnt.min(), cnt.mean(), cnt.max(), "top5", sorted(cnt)[-5:])
PY
cat $OUT/c4_sizes.log
