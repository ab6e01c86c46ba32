# r2v: bulk-copy ordered chains: parity + c4 update timing
OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or update" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/c4.log 2>&1; cat $OUT/c4.log
FTK_UPD_CHAIN=0 timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/c4_old.log 2>&1; cat $OUT/c4_old.log
