for r in 1 2; do
python bench.py --steps 50 --warmup 5 > gpurun_out/t30_$r.json 2>gpurun_out/t30_$r.err
python -c "
import json;j=json.load(open('gpurun_out/t30_$r.json'));c=j['ft_campaign']
print('%.1f'%j['value'],'ovh %.1f'%j['ft_overhead_pct'],j['step_ms']['abft'],j['faults'],'e2e %.1f'%j['e2e']['value'])
print('campaign',c['ms_per_step'],c['injected'],c['injected_per_s'],c['detections'],c['overhead_vs_ft_off_pct'])"
done
