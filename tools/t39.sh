for s in 5 4 3; do
echo "== S=$s"
FTK_PAIR_STAGES=$s FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_pnoinj/libftkb200.so FTK_PAIR_CLK=1 timeout 120 python tools/prof_assign.py --checked --iters 3 --reps 3 2>&1 | tail -3
done
