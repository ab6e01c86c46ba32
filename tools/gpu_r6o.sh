# r6o: ncu --set full of the pass-2 kernels at c2 steady state (candidate evaluation and the COLLECT screen)
OUT=gpurun_out/r6o; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none -k regex:"cand_exact|cand_finalize|pass2_gather" -s 12 -c 3 -o $OUT/pass2 python tools/prof_lloyd.py --steps 8 --ft abft > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/pass2.ncu-rep --page details --csv > $OUT/pass2_details.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r6o/pass2_details.csv')))
h=rows[0]
want=('Duration','Grid Size','Achieved Occupancy','Issue Slots Busy','Elapsed Cycles','SM Active Cycles','Executed Instructions','Memory Throughput','DRAM Throughput','Warp Cycles Per Issued Instruction','Threads')
for r in rows[1:]:
    d=dict(zip(h,r))
    if d.get('Metric Name','') in want: print(d['Kernel Name'][:22], '|', d['Metric Name'], '|', d['Metric Value'], d.get('Metric Unit',''))
PY
