set -x
timeout 120 python tools/prof_assign.py --variant tc --reps 3 --n 4096 --k 256
timeout 120 python tools/prof_assign.py --variant tc --reps 3
FTK_TC_PAIR=0 timeout 120 python tools/prof_assign.py --variant tc --reps 3
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15
