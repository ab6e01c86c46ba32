for dbg in 0 2 6 3; do echo "dbg=$dbg"; FTK_PAIR_CLK=1 FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_assign.py --variant tc --reps 3 2>&1 | grep -E "pair clk" | tail -1; done
