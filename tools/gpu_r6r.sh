# r6r: c5 (N=1e8, D=128, K=4096) per-step breakdown: eager steps with the fallback counts, then an ncu launch list
OUT=gpurun_out/r6r; mkdir -p $OUT
timeout 600 python tools/prof_c5.py 1e8 off > $OUT/c5.log 2>&1; tail -5 $OUT/c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_c5.py 1e8 off > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 20
