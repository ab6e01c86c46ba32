# r6v: c5 launch breakdown after the pass-2 changes
OUT=gpurun_out/r6v; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_c5.py 1e8 off > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 12
grep "pair_screen_kernel<0, 1" $OUT/launches.csv | grep tensor | tail -2 | cut -d, -f5,13-15
