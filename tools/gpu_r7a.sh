# r7a: pass-2 COLLECT drain in chunk pairs on top of the branch-free compare (FTK_PAIR_CX2) A/B
OUT=gpurun_out/r7a; mkdir -p $OUT
L=paper_2408_01391_b200/_lib/var_cx2/libftkb200.so
FTK_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > $OUT/pytest_cx2.log 2>&1; tail -1 $OUT/pytest_cx2.log
for v in base cx2; do
  if [ $v = base ]; then lp=""; else lp=$L; fi
  FTK_LIB_PATH=$lp timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$v.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
  echo "== $v c2"; python tools/iter_breakdown.py $OUT/launches_$v.csv 30 | grep -E "kernel sum|<0, 1"
  FTK_LIB_PATH=$lp timeout 600 python tools/prof_c5.py 1e8 off > $OUT/c5_$v.log 2>&1; echo "== $v c5"; tail -3 $OUT/c5_$v.log
done
