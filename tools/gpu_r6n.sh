# r6n: per-k-block X landing barriers (FTK_PAIR_XKB): a row tile's first MMAs start before its last X k-blocks land
OUT=gpurun_out/r6n; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_xkb/libftkb200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_tc64.py -q -x > $OUT/pytest_xkb.log 2>&1; tail -1 $OUT/pytest_xkb.log
bash tools/ab.sh r6n/ab base xkb
for v in base xkb; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_kernel_dbg.py 0 2 0 2 > $OUT/dbg_$v.log 2>&1; echo dbg $v; grep "dbg=" $OUT/dbg_$v.log
done
