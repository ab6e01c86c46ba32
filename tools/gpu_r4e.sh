# r4e: F64+ABFT checksum reference formed before the partials: parity + c4 screen time
OUT=gpurun_out/r4e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc64.py tests/test_gpu_configs.py -q -x -rf -k "tc64 or c4" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_screen_kernel -c 6 --csv --log-file $OUT/c4.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > /dev/null 2>&1
grep pair_screen $OUT/c4.csv | awk -F'","' '{print $5, $NF}' | head -6
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4.log 2>&1; tail -2 $OUT/c4.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4_off.log 2>&1; tail -2 $OUT/c4_off.log
