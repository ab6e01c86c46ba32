# r3w: swg3r (setmaxnreg within the CTA budget): quick hang check, parity, A/B -- everything under short timeouts
OUT=gpurun_out/r3w; mkdir -p $OUT
L=paper_2408_01391_b200/_lib/var_swg3r/libftkb200.so
FTK_LIB_PATH=$L timeout 90 python tools/prof_assign.py --variant pair --reps 2 > $OUT/quick.log 2>&1; echo "quick rc=$?"; tail -2 $OUT/quick.log
if grep -q "rep 1" $OUT/quick.log; then
  FTK_LIB_PATH=$L timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_swg3r.log 2>&1; tail -2 $OUT/pytest_swg3r.log
  bash tools/ab.sh r3w base swg3r 2>&1
fi
