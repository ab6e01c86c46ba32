#!/bin/bash
# One GPU-box session: parity tests, bench line, ncu launch list + full capture of the top kernel.
# usage: bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo BUILD_FAIL
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 > $OUT/bench_ncu.log 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_screen -s 2 -c 1 \
  -o $OUT/tc_screen python tools/prof_assign.py --variant tc --reps 3 > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:update -s 4 -c 2 \
  -o $OUT/update python tools/prof_lloyd.py --steps 3 > $OUT/ncu_upd.log 2>&1; echo "ncu-upd rc=$?"
fi
