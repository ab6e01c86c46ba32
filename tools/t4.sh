timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for dbg in 0 1 2 3; do echo "dbg=$dbg"; FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_assign.py --variant tc --reps 3 | tail -1; done
mkdir -p gpurun_out/t4
for dbg in 0 3; do FTK_TC_DEBUG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t4/l$dbg.csv python tools/prof_assign.py --variant tc --reps 3 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/t4/l$dbg.csv | grep pair; done
for st in 2 3 4; do echo "stages=$st"; FTK_PAIR_STAGES=$st FTK_TC_DEBUG=3 timeout 120 python tools/prof_assign.py --variant tc --reps 3 | tail -1; done
