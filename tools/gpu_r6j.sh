# r6j: c4 float64 refine with the centroid table in shared memory (FTK_T64_CTAB A/B)
OUT=gpurun_out/r6j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc64.py tests/test_gpu_configs.py -q -x -k "tc64 or c4" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for r in 1 2; do for v in 1 0; do
  echo "ctab=$v"; FTK_T64_CTAB=$v timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair 2>&1 | tail -2
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:tc64_refine -c 2 --csv --log-file $OUT/t64.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 2 --variant pair > /dev/null 2>&1
grep -v "^==" $OUT/t64.csv | cut -d, -f5,13-15 | tail -6
timeout 900 python bench.py --steps 10 --warmup 3 --campaign-s 0.3 --reps 3 --c5 0 > $OUT/bench.json 2> $OUT/bench.err; python -c "
import json; j=json.load(open('$OUT/bench.json')); print('c2', j['value'], 'c4', j['c4_1gpu'])"
