#!/bin/bash
# One GPU-box session: parity tests, smoke, bench line, ncu launch list + full
# captures of the top kernels.  usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo BUILD_FAIL
timeout 400 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3500 $OUT/bench.json
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 > $OUT/bench_ncu.log 2>&1; echo "ncu-list rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 8 -c 1 \
  -o $OUT/pair_chk python tools/prof_assign.py --variant tc --reps 3 --iters 3 --checked > $OUT/ncu_pair.log 2>&1; echo "ncu-pair rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_partials -s 2 -c 1 \
  -o $OUT/seg python tools/prof_lloyd.py --steps 4 > $OUT/ncu_seg.log 2>&1; echo "ncu-seg rc=$?"
fi
if [ -z "$NO_NCU" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dmma_screen -s 1 -c 1 \
  -o $OUT/dmma python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 2 > $OUT/ncu_dmma.log 2>&1; echo "ncu-dmma rc=$?"
fi
