# r6w: branch-free COLLECT compare (bit mask + set-bit pass); tests, c5 steps, c2 launch breakdown
OUT=gpurun_out/r6w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tc64.py -q -x > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 600 python tools/prof_c5.py 1e8 off > $OUT/c5.log 2>&1; tail -4 $OUT/c5.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 6
