timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out/t6
for dbg in 0 1 2 3; do FTK_TC_DEBUG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair --csv --log-file gpurun_out/t6/l$dbg.csv python tools/prof_assign.py --variant tc --reps 3 > /dev/null 2>&1; echo "dbg=$dbg"; python tools/ncu_summary.py gpurun_out/t6/l$dbg.csv | grep pair; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 -o gpurun_out/t6/pair python tools/prof_assign.py --variant tc --reps 3 > gpurun_out/t6/ncu.log 2>&1; tail -1 gpurun_out/t6/ncu.log
