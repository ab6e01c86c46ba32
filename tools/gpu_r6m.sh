# r6m: refine: k-blocks 2-3 of the hinted centroid prefetched into L1 (FTK_PAIR_PFL1) A/B + role breakdown
OUT=gpurun_out/r6m; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_pfl1/libftkb200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x > $OUT/pytest_pfl1.log 2>&1; tail -1 $OUT/pytest_pfl1.log
bash tools/ab.sh r6m/ab base pfl1
for v in base pfl1; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_kernel_dbg.py 0 2 0 2 > $OUT/dbg_$v.log 2>&1; echo dbg $v; grep "dbg=" $OUT/dbg_$v.log
done
