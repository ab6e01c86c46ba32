# r6h: checkpoint after the X2 drain: full GPU suite, smoke, bench (both arms), launch list, tensor-pipe + traffic
OUT=gpurun_out/r6h; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log; tail -4 $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
python - <<'PY'
import json
j=json.load(open('gpurun_out/r6h/bench.json'))
print('value', j['value'], 'frac', j['roofline']['frac'], 'kernel', j['roofline']['kernel_ms'], 'ft%', j['ft_overhead_pct'], 'launches', j['gpu_launches'])
print('campaign', {k: j['ft_campaign'][k] for k in ('overhead_pct_median','label_divergence','detections','corrections','false_alarms','injected_per_s','tc_checksum_flags')})
print('dmr', j['dmr']); print('e2e', j['e2e']['value'], j['e2e']['pinned']['value']); print('c4', j['c4_1gpu']); print('c5', j['c5_1gpu']); print('clocks', j['clocks'])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --c4 0 --c5 0 --campaign-s 0 > $OUT/bench_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active --clock-control none -k regex:pair_screen_kernel -c 12 --csv --log-file $OUT/pair_metrics.csv python tools/prof_cfg.py --ft abft --steps 6 > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pair_screen|tc64_refine|chain_spec|dmma" -c 16 --csv --log-file $OUT/c4_metrics.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 --variant pair > /dev/null 2>&1; echo "ncu3 rc=$?"
