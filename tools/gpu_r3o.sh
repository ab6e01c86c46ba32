# r3o: checkpoint: full GPU suite, smoke, bench (both arms), launch list
OUT=gpurun_out/r3o; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log; tail -14 $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
python - <<'PY'
import json
j=json.load(open('gpurun_out/r3o/bench.json'))
print('value', j['value'], 'frac', j['roofline']['frac'], 'kernel', j['roofline']['kernel_ms'], 'ft%', j['ft_overhead_pct'])
print('campaign', {k: j['ft_campaign'][k] for k in ('overhead_pct_median','label_divergence','detections','corrections','false_alarms','injected_per_s')})
print('dmr', j['dmr']); print('e2e', j['e2e']['value'], j['e2e']['pinned']['value']); print('c4', j['c4_1gpu']); print('c5', j['c5_1gpu'])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --c4 0 --c5 0 --campaign-s 0 > $OUT/bench_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1; head -25 $OUT/launches_summary.txt
