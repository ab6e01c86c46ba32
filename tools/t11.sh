mkdir -p gpurun_out/t11
for c in "" "--checked"; do FTK_PAIR_CLK=1 timeout 120 python tools/prof_assign.py --variant tc --reps 3 $c 2>&1 | grep -E "pair clk|rep 2" | tail -2; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 -o gpurun_out/t11/chk python tools/prof_assign.py --variant tc --reps 3 --checked > gpurun_out/t11/ncu.log 2>&1; tail -1 gpurun_out/t11/ncu.log
