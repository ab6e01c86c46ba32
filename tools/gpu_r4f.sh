# r4f: chain groups of 32 rows (barrier overhead per member halved)
OUT=gpurun_out/r4f; mkdir -p $OUT
for v in base gs32 gs32b; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4_$v.log 2>&1; echo $v; tail -2 $OUT/c4_$v.log
done
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_gs32/libftkb200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or update" > $OUT/pytest_gs32.log 2>&1; tail -1 $OUT/pytest_gs32.log
