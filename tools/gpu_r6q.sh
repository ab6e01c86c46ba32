# r6q: speculative refine against the hinted centroid (FTK_PAIR_SPEC) -- parity + A/B + role breakdown
OUT=gpurun_out/r6q; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_spec/libftkb200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > $OUT/pytest_spec.log 2>&1; tail -1 $OUT/pytest_spec.log
bash tools/ab.sh r6q/ab base spec
for v in base spec; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_kernel_dbg.py 0 2 0 2 > $OUT/dbg_$v.log 2>&1; echo dbg $v; grep "dbg=" $OUT/dbg_$v.log
done
