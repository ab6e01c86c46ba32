timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for dbg in 0 2 3; do echo "dbg=$dbg"; FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_assign.py --variant tc --reps 3 | tail -1; done
mkdir -p gpurun_out/t5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t5/l.csv python tools/prof_assign.py --variant tc --reps 3 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/t5/l.csv | head -5
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 -o gpurun_out/t5/pair python tools/prof_assign.py --variant tc --reps 3 > gpurun_out/t5/ncu.log 2>&1; tail -1 gpurun_out/t5/ncu.log
