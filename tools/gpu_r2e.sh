# r2e: narrow screen parity + c3 timings
OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_narrow.py -q -x -rf > $OUT/pytest_narrow.log 2>&1; echo "rc=$?" >> $OUT/pytest_narrow.log
tail -30 $OUT/pytest_narrow.log
timeout 600 python -m pytest tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_cfg.log 2>&1; echo "rc=$?" >> $OUT/pytest_cfg.log
tail -5 $OUT/pytest_cfg.log
timeout 600 python tools/prof_narrow.py --steps 5 > $OUT/narrow_off.log 2>&1; cat $OUT/narrow_off.log
timeout 600 python tools/prof_narrow.py --steps 4 --ft abft --shapes 16x512,32x2048 > $OUT/narrow_abft.log 2>&1; cat $OUT/narrow_abft.log
