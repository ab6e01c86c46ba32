OUT=gpurun_out/r2a; mkdir -p $OUT
nproc > $OUT/host.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/host.txt; free -g >> $OUT/host.txt
timeout 60 python tools/probe_graph_events.py > $OUT/probe_events.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x > $OUT/pytest_cfg.log 2>&1; echo "rc=$?" >> $OUT/pytest_cfg.log
timeout 600 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
tail -3 $OUT/pytest_cfg.log $OUT/pytest_gpu.log; cat $OUT/probe_events.log
