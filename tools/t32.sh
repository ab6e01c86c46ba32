export FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_probe/libftkb200.so FTK_PAIR_CLK=1
python tools/prof_assign.py --iters 3 --reps 3 2>&1 | tail -6
python tools/prof_assign.py --checked --iters 3 --reps 3 2>&1 | tail -6
