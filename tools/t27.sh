for r in 1 2 3 4; do
python bench.py --steps 50 --warmup 5 --campaign-s 0.3 > gpurun_out/t27_$r.json 2>gpurun_out/t27_$r.err
python -c "import json;j=json.load(open('gpurun_out/t27_$r.json'));print('%.1f'%j['value'],j['step_ms'],j['faults']['injected'],'e2e %.1f'%j['e2e']['value'],'%.4f'%j['e2e']['wall_s'])"
done
