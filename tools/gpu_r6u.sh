# r6u: pass-2 candidates flushed once per work item (not per tile); tests, c5 steps, bench
OUT=gpurun_out/r6u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_tc64.py -q -x > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 600 python tools/prof_c5.py 1e8 off > $OUT/c5.log 2>&1; tail -5 $OUT/c5.log
timeout 900 python bench.py --steps 10 --warmup 3 --campaign-s 0.3 --reps 3 > $OUT/bench.json 2> $OUT/bench.err; python -c "
import json; j=json.load(open('$OUT/bench.json')); print('c2', j['value'], j['roofline']['kernel_ms'], 'c4', j['c4_1gpu']['iter_per_s'], 'c5', j['c5_1gpu']['iter_per_s'], j['c5_1gpu']['assign_ms'], j['c5_1gpu']['screen_ms'])"
