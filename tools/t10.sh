mkdir -p gpurun_out/t10
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/t10/bench.json 2> gpurun_out/t10/bench.err; tail -c 2500 gpurun_out/t10/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t10/launches.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/t10/launches.csv | head -30
