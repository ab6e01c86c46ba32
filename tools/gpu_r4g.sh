# r4g: narrow screen with the runner-up hint: parity (narrow + configs + tc64 extras) and c3 timings vs FTK_NARROW_NOH2
OUT=gpurun_out/r4g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_configs.py tests/test_gpu_tc64.py -q -x -rf > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for shp in "512 16" "512 8" "2048 32" "2048 8"; do set -- $shp
  for v in h2 noh2; do
    if [ $v = noh2 ]; then export FTK_NARROW_NOH2=1; else unset FTK_NARROW_NOH2; fi
    timeout 300 python tools/prof_cfg.py --n 1000000 --d $1 --k $2 --ft abft --steps 8 > $OUT/c3_$1_$2_$v.log 2>&1
    echo "d=$1 k=$2 $v: $(tail -2 $OUT/c3_$1_$2_$v.log | tr '\n' ' ')"
  done
done
unset FTK_NARROW_NOH2
