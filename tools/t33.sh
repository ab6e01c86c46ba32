python tools/prof_steps.py 8 2>&1 | tail -8
python tools/prof_e2e.py 2>&1 | head -4
python -m pytest tests/test_gpu_parity.py -x -q -k "graph" 2>&1 | tail -2
python bench.py > gpurun_out/t33.json 2>gpurun_out/t33.err; python -c "
import json;j=json.load(open('gpurun_out/t33.json'));c=j['ft_campaign']
print('%.1f'%j['value'],'ovh %.1f'%j['ft_overhead_pct'],j['step_ms']['abft'],'e2e',j['e2e'])
print('campaign',c['ms_per_step'],c['injected'],c['injected_per_s'],c['detections'],c['overhead_vs_ft_off_pct'])"
