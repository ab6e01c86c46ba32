# r2u: CTA-pair role timing in the engine (rowinfo registered); c4 ordered-chain kernel full capture + cluster sizes
OUT=gpurun_out/r2u; mkdir -p $OUT
P=paper_2408_01391_b200/_lib/var_probe/libftkb200.so
FTK_LIB_PATH=$P FTK_PAIR_CLK=1 python tools/prof_cfg.py --ft abft --steps 5 > $OUT/probe_c2.log 2>&1; tail -8 $OUT/probe_c2.log
python - > $OUT/c4_sizes.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_01391_b200 as P
from paper_2408_01391_b200 import _engine as E
from paper_2408_01391_b200.kmeans import LloydEngine
x, _, _ = P.gaussian_mixture(10_000_000, 64, 256, 0.25, precision="double", seed=0)
c0 = P.init_centroids(x, 256, seed=0, method="random-sample")
eng = LloydEngine(E.to_dev(x), c0, 256, np.float64, P.default_config(np.float64), "abft", P.Threshold.default_for(np.float64), 64)
for it in range(4):
    eng.step(it)
    cnt = eng.counts_buf.cpu().numpy()
    print(it, "assign", round(eng.assign_ms, 3), "update", round(eng.update_ms, 3), "counts min/mean/max", cnt.min(), cnt.mean(), cnt.max())
PY
cat $OUT/c4_sizes.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:chain_pipe -s 2 -c 1 \
  -o $OUT/chain python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/ncu_chain.log 2>&1; echo "ncu-chain rc=$?"
