# r7z: session-final checkpoint: full GPU suite, smoke, bench (both arms), launch list, tensor-pipe + traffic, role breakdown, ncu full of the c2 CHK screen
# the pass-1 kernel role breakdown (FTK_TC_DEBUG bits) and one ncu --set full capture of the c2 CHK screen
OUT=gpurun_out/r7z; mkdir -p $OUT
bash tools/gpu_r6a.sh > /dev/null 2>&1
mv gpurun_out/r6a/* $OUT/ 2>/dev/null; rmdir gpurun_out/r6a 2>/dev/null
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log
python - <<'PY'
import json
j=json.load(open('gpurun_out/r7z/bench.json'))
print('value', j['value'], 'frac', j['roofline']['frac'], 'kernel', j['roofline']['kernel_ms'], 'ft%', j['ft_overhead_pct'], 'launches', j['gpu_launches'])
print('campaign', {k: j['ft_campaign'][k] for k in ('overhead_pct_median','label_divergence','detections','corrections','false_alarms','injected_per_s','tc_checksum_flags')})
print('e2e', j['e2e']['value'], 'c4', j['c4_1gpu']['iter_per_s'], 'c5', j['c5_1gpu']['iter_per_s'], j['c5_1gpu']['frac'], 'clocks', j['clocks'])
PY
timeout 300 python tools/prof_kernel_dbg.py 0 2 1 4 0 > $OUT/kernel_dbg.log 2>&1; grep "dbg=" $OUT/kernel_dbg.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 8 -c 1 -o $OUT/pair_chk python tools/prof_assign.py --variant tc --reps 3 --iters 3 --checked > $OUT/ncu_pair.log 2>&1; echo "ncu-full rc=$?"
ncu -i $OUT/pair_chk.ncu-rep --page details --csv > $OUT/pair_details.csv 2>/dev/null; python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r7z/pair_details.csv')))
h=rows[0]
want=('Duration','DRAM Throughput','Issue Slots Busy','No Eligible','Eligible Warps','Registers Per Thread','L1/TEX Cache Throughput','Compute (SM) Throughput')
for r in rows[1:]:
    d=dict(zip(h,r))
    if any(w == d.get('Metric Name','') for w in want): print(d['Kernel Name'][:40], '|', d['Metric Name'], '|', d['Metric Value'], d.get('Metric Unit',''))
PY
