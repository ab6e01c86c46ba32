# r2i: full GPU suite + c2 bench + narrow timings
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json
timeout 600 python tools/prof_narrow.py --steps 4 --shapes 16x512,32x2048 > $OUT/narrow_off.log 2>&1; cat $OUT/narrow_off.log
