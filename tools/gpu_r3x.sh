# r3x: float64 pass 2 by COLLECT re-screen + float64 candidates: parity + c4 timing vs DMMA pass 2
OUT=gpurun_out/r3x; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tc64.py -q -x -rf > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
FTK_T64_NO_P2=1 timeout 600 python -m pytest tests/test_gpu_tc64.py -q -x -rf > $OUT/pytest_nop2.log 2>&1; tail -1 $OUT/pytest_nop2.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 6 --variant pair > $OUT/c4.log 2>&1; tail -3 $OUT/c4.log
FTK_T64_NO_P2=1 timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 6 --variant pair > $OUT/c4_nop2.log 2>&1; tail -3 $OUT/c4_nop2.log
