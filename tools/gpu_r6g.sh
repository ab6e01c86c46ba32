# r6g: X2 drain as the default; full GPU suite; A/B base (x2) vs x64 (one 64-column LDTM per pair) vs nox2 (pipelined drain)
OUT=gpurun_out/r6g; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_x64/libftkb200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x > $OUT/pytest_x64.log 2>&1; tail -1 $OUT/pytest_x64.log
bash tools/ab.sh r6g/ab base x64 nox2
for cfg in "--n 1000000 --d 64 --k 256 --dtype f64 --variant pair" "--n 20000000 --d 128 --k 4096"; do
  for v in base nox2; do
    if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
    echo "$v $cfg"; FTK_LIB_PATH=$lp timeout 300 python tools/prof_cfg.py $cfg --ft abft --steps 4 2>&1 | tail -2
  done
done
