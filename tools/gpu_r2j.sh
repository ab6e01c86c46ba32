# r2j: pair ABFT group location (no per-chunk work) + bench
OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abft_tc.py tests/test_gpu_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; j=json.load(open("gpurun_out/r2j/bench.json"))
print("value", j["value"], "kernel", j["roofline"]["kernel_ms"], "frac", j["roofline"]["frac"], "off_kernel", j["ft_off_kernel_ms"], "ft%", j["ft_overhead_pct"], "campaign%", j["ft_campaign"]["overhead_pct_median"], "div", j["ft_campaign"]["label_divergence"])
PY
timeout 300 python tools/prof_inject.py > $OUT/inject.log 2>&1; tail -8 $OUT/inject.log
