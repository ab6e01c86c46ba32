# r3r: c2 pass-2 statistics per step (rows, candidates, rows to the exact kernel) + per-step launch timeline
OUT=gpurun_out/r3r; mkdir -p $OUT
FTK_TC_P2_DEBUG=1 timeout 300 python tools/prof_cfg.py --ft abft --steps 12 > $OUT/p2.log 2>&1; grep -E "pass 2|it " $OUT/p2.log | tail -16
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/steps.csv python tools/prof_cfg.py --ft abft --steps 12 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r3r/steps.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[hi]
ki,vi=h.index('Kernel Name'),h.index('Metric Value')
seq=[(r[ki].split('(')[0][-40:], float(r[vi].replace(',',''))/1e3) for r in rows[hi+1:] if len(r)>vi]
# print the last ~40 launches (the last two steps)
tot=0
for n,ms in seq[-45:]:
    print(f"{ms:8.4f}  {n}")
PY
