# r2s (session 3 re-entry): full GPU suite + smoke + bench (both arms) at the current commit
OUT=gpurun_out/r2s; mkdir -p $OUT
nproc > $OUT/host.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/host.txt; free -g >> $OUT/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
tail -3 $OUT/smoke.log; tail -25 $OUT/pytest_gpu.log; cat $OUT/bench.json $OUT/ref.json
