timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k streamed 2>&1 | tail -15
timeout 120 python tools/prof_assign.py --n 1000000 --d 512 --k 16 --reps 2 --iters 2 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t47.csv python tools/prof_assign.py --n 1000000 --d 512 --k 16 --reps 2 --iters 2 > /dev/null 2>&1
