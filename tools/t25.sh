mkdir -p gpurun_out/t25
python tools/prof_assign.py --checked --iters 3 --reps 5 2>&1 | tail -3
python tools/prof_assign.py --iters 3 --reps 5 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 > gpurun_out/t25/bench.json 2> gpurun_out/t25/bench.err
python -c "import json;j=json.load(open('gpurun_out/t25/bench.json'));print(j['value'],j['ms_per_step'],j['roofline']['kernel_ms'],j['ft_off_kernel_ms'],j['ft_overhead_pct'],j['e2e']['value'])"
