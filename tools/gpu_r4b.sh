# r4b: c4 F64 CHK screen: which part costs (dbg 2 = skip refine)
OUT=gpurun_out/r4b; mkdir -p $OUT
for dbg in 0 2; do
  FTK_TC_DEBUG=$dbg timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_screen_kernel -c 8 --csv --log-file $OUT/c4_$dbg.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > /dev/null 2>&1
  echo "== dbg $dbg"; grep pair_screen $OUT/c4_$dbg.csv | cut -d, -f5,15 | head -8
done
