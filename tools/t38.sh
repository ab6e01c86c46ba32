for v in probe pnoinj pnosum pnoboth; do
echo "== $v"
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_$v/libftkb200.so FTK_PAIR_CLK=1 timeout 120 python tools/prof_assign.py --checked --iters 3 --reps 3 2>&1 | tail -3
done
