#!/bin/bash
# Short GPU check: c2 bench line (0.3 s campaign) + ncu launch list of a few
# Lloyd iterations; summarise with tools/iter_breakdown.py gpurun_out/qb_launches.csv
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/qb_launches.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python bench.py --campaign-s 0.3 > gpurun_out/qb.json 2> gpurun_out/qb.err
python -c "
import json;j=json.load(open('gpurun_out/qb.json'));c=j['ft_campaign']
print('%.1f'%j['value'],'ovh %.1f'%j['ft_overhead_pct'],j['step_ms'],'e2e',round(j['e2e']['value'],1))
print('campaign',round(c['ms_per_step'],4),c['injected'],round(c['overhead_vs_ft_off_pct'],2))"
python tools/iter_breakdown.py gpurun_out/qb_launches.csv 8
