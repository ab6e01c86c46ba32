timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 bash tools/t34.sh 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/t37.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
