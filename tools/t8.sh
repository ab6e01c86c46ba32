timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for dbg in 0 2; do echo "dbg=$dbg"; FTK_PAIR_CLK=1 FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_assign.py --variant tc --reps 3 2>&1 | grep -E "pair clk|rep 2" | tail -2; done
mkdir -p gpurun_out/t8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair --csv --log-file gpurun_out/t8/l.csv python tools/prof_assign.py --variant tc --reps 3 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/t8/l.csv | grep pair
