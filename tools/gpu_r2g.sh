# r2g: narrow screen after hoisting the chain loads (A/B: transposed operand)
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_narrow.py -q -x -rf > $OUT/pytest_narrow.log 2>&1; echo "rc=$?" >> $OUT/pytest_narrow.log
tail -3 $OUT/pytest_narrow.log
timeout 600 python tools/prof_narrow.py --steps 4 > $OUT/narrow_off.log 2>&1; cat $OUT/narrow_off.log
FTK_NARROW_CT=1 timeout 600 python tools/prof_narrow.py --steps 3 --shapes 16x512,32x2048 > $OUT/narrow_ct.log 2>&1; cat $OUT/narrow_ct.log
timeout 600 python tools/prof_narrow.py --steps 4 --ft abft --shapes 16x512,32x2048 > $OUT/narrow_abft.log 2>&1; cat $OUT/narrow_abft.log
