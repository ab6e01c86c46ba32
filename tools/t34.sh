python -m pytest tests/test_gpu_parity.py -x -q -k "update or lloyd or graph" 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t34.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python bench.py --campaign-s 0.3 > gpurun_out/t34.json 2>gpurun_out/t34.err; python -c "
import json;j=json.load(open('gpurun_out/t34.json'));c=j['ft_campaign']
print('%.1f'%j['value'],'ovh %.1f'%j['ft_overhead_pct'],j['step_ms'],'e2e',j['e2e']['value'])
print('campaign',c['ms_per_step'],c['injected'],c['overhead_vs_ft_off_pct'])"
