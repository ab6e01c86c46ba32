# r4c: refine with rowinfo/constants prefetched: c4 screen time, c2 A/B numbers, parity
OUT=gpurun_out/r4c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_tc64.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_screen_kernel -c 6 --csv --log-file $OUT/c4.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > /dev/null 2>&1
grep pair_screen $OUT/c4.csv | awk -F'","' '{print $5, $NF}' | head -6
timeout 300 python tools/prof_kernel_dbg.py 0 0 > $OUT/c2.log 2>&1; grep dbg $OUT/c2.log
