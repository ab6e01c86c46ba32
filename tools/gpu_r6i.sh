# r6i: pass-2 COLLECT drain in chunk pairs (tests + launch breakdown); ncu --set full of the c4 float64 refine
OUT=gpurun_out/r6i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tc64.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc64_refine_tma -s 2 -c 1 -o $OUT/t64_refine python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > $OUT/ncu_t64.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/t64_refine.ncu-rep --page details --csv > $OUT/t64_details.csv 2>/dev/null; python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r6i/t64_details.csv')))
h=rows[0]
want=('Duration','DRAM Throughput','Memory Throughput','Achieved Occupancy','Registers Per Thread','Issue Slots Busy','No Eligible','Active Warps Per Scheduler','Eligible Warps Per Scheduler','L2 Hit Rate','Dynamic Shared Memory Per Block','Waves Per SM','Block Limit Shared Mem','Theoretical Occupancy')
for r in rows[1:]:
    d=dict(zip(h,r))
    if any(w in d.get('Metric Name','') for w in want): print(d['Section Name'][:28], '|', d['Metric Name'], '|', d['Metric Value'], d.get('Metric Unit',''))
PY
