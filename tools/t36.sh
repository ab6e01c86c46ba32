timeout 120 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_probe/libftkb200.so FTK_PAIR_CLK=1 timeout 120 python tools/prof_assign.py --checked --iters 3 --reps 3 2>&1 | tail -3
timeout 300 bash tools/t34.sh 2>&1 | tail -2
