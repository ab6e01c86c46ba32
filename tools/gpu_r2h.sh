# r2h: pair-kernel ABFT location/correction + full GPU suite + c2 bench
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_abft_tc.py -q -x -rf > $OUT/pytest_abft.log 2>&1; echo "rc=$?" >> $OUT/pytest_abft.log
tail -30 $OUT/pytest_abft.log
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json
