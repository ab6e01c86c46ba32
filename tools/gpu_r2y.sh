# r2y: float64 through the tf32 pair screen: parity + c4 timing (pair vs dmma)
OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc64.py -q -x -rf > $OUT/pytest.log 2>&1; tail -15 $OUT/pytest.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_pair.log 2>&1; cat $OUT/c4_pair.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4_pair_off.log 2>&1; cat $OUT/c4_pair_off.log
