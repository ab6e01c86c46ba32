# r2b: GPU tests, peaks, kmeanspp timing, bench, ncu launch list + screen capture
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo BUILD_FAIL
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 200 python tools/peaks_tf32_f64.py > $OUT/peaks.json 2>&1; cat $OUT/peaks.json
timeout 300 python tools/prof_kpp.py > $OUT/kpp.log 2>&1; cat $OUT/kpp.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --campaign-s 0 --c5 0 > $OUT/bench_ncu.log 2>&1; echo "ncu-list rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 8 -c 1 \
  -o $OUT/pair_chk python tools/prof_assign.py --variant tc --reps 3 --iters 3 --checked > $OUT/ncu_pair.log 2>&1; echo "ncu-pair rc=$?"
