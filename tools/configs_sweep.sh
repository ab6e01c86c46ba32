#!/bin/bash
# Per-iteration timings of every BASELINE config on one GPU (device-resident data),
# the numbers DESIGN.md section 8 quotes.  usage: bash tools/configs_sweep.sh > out.txt
run() { echo "== $*"; timeout 900 python tools/prof_cfg.py "$@" --steps 4 2>&1 | tail -2; }
run --n 100000 --d 32 --k 64 --ft off
run --n 100000 --d 32 --k 64 --ft abft
run --n 1000000 --d 128 --k 1024 --ft abft
run --n 1000000 --d 512 --k 16 --ft abft
run --n 1000000 --d 512 --k 16 --ft off
run --n 1000000 --d 2048 --k 32 --ft off
run --n 1000000 --d 8 --k 4096 --ft abft
run --n 1000000 --d 4 --k 4096 --ft abft
run --n 10000000 --d 64 --k 256 --dtype f64 --ft abft
echo "== c5 1 GPU"; timeout 900 python tools/prof_c5.py 2>&1 | tail -3
