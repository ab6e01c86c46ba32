# r3a: full GPU suite after tc64 + X-buffer change; c1/c4/c2 timings
OUT=gpurun_out/r3a; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log; tail -4 $OUT/pytest_gpu.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_pair.log 2>&1; tail -3 $OUT/c4_pair.log
FTK_PAIR_NA2=1 timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_pair_na2.log 2>&1; tail -3 $OUT/c4_pair_na2.log
timeout 300 python tools/prof_cfg.py --n 100000 --d 32 --k 64 --steps 6 > $OUT/c1.log 2>&1; tail -3 $OUT/c1.log
FTK_PAIR_NA2=1 timeout 300 python tools/prof_cfg.py --n 100000 --d 32 --k 64 --steps 6 > $OUT/c1_na2.log 2>&1; tail -3 $OUT/c1_na2.log
timeout 300 python tools/prof_cfg.py --ft abft --steps 5 > $OUT/c2.log 2>&1; tail -3 $OUT/c2.log
