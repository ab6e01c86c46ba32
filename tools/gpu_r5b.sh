# r5b: centroid norms staged once (k <= 2048) and early TMEM buffer release
OUT=gpurun_out/r5b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_tc64.py tests/test_gpu_configs.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
bash tools/ab.sh r5b/ab base noyall norel
for v in base noyall norel; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_kernel_dbg.py 0 1 4 0 > $OUT/dbg_$v.log 2>&1; echo dbg $v; grep "dbg=" $OUT/dbg_$v.log | head -4
done
