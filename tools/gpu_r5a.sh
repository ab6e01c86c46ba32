# r5a: pass-2 (COLLECT) work items split per column tile
OUT=gpurun_out/r5a; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_tc64.py tests/test_gpu_configs.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for v in base nosplit; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_$v.log 2>&1; echo c4 $v; tail -2 $OUT/c4_$v.log
done
bash tools/ab.sh r5a/ab base nosplit
