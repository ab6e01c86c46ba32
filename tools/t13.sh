mkdir -p gpurun_out/t13
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 -o gpurun_out/t13/pair python tools/prof_assign.py --variant tc --reps 3 --iters 3 > gpurun_out/t13/ncu.log 2>&1; tail -1 gpurun_out/t13/ncu.log
