# r2z: c4 tc64 per-kernel launch list + uncertified counts
OUT=gpurun_out/r2z; mkdir -p $OUT
python - > $OUT/c4_fb.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2408_01391_b200 as P
from paper_2408_01391_b200 import _engine as E, gemm
from paper_2408_01391_b200.kmeans import LloydEngine
gemm.set_variant("pair")
x, _, _ = P.gaussian_mixture(10_000_000, 64, 256, 0.25, precision="double", seed=0)
c0 = P.init_centroids(x, 256, seed=0, method="random-sample")
eng = LloydEngine(E.to_dev(x), c0, 256, np.float64, P.default_config(np.float64), "abft", P.Threshold.default_for(np.float64), 64)
for it in range(5):
    eng.step(it)
    lab = eng.A.labels[eng.slot].cpu().numpy()
    cnt = np.bincount(lab[lab >= 0], minlength=256)
    print(it, "assign", round(eng.assign_ms, 3), "update", round(eng.update_ms, 3), "fallback", E.tc_fallback_rows(), "counts max", cnt.max(), "mean", cnt.mean(), "top", sorted(cnt)[-4:])
PY
cat $OUT/c4_fb.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/c4_launches.csv \
  python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 --variant pair > $OUT/c4_ncu.log 2>&1
python tools/ncu_summary.py $OUT/c4_launches.csv 2>&1 | head -25
