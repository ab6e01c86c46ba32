# r4a: c4 kernel list FT off vs ABFT (where the 11 % goes)
OUT=gpurun_out/r4a; mkdir -p $OUT
for ft in off abft; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/c4_$ft.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft $ft --steps 4 --variant pair > /dev/null 2>&1
  echo "== $ft"; python tools/ncu_summary.py $OUT/c4_$ft.csv 2>&1 | head -16
done
