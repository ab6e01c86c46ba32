# r2o: full suite with the shipped variant table; bench; c4 DMMA ncu; injected-step launch list
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -6 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; j=json.load(open("gpurun_out/r2o/bench.json"))
print("value", j["value"], "kernel", j["roofline"]["kernel_ms"], "frac", j["roofline"]["frac"], "off_kernel", j["ft_off_kernel_ms"], "ft%", j["ft_overhead_pct"], "campaign%", j["ft_campaign"]["overhead_pct_median"], "div", j["ft_campaign"]["label_divergence"], "e2e", j["e2e"]["value"])
PY
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/c4.log 2>&1; cat $OUT/c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmma_screen -s 2 -c 1 -o $OUT/dmma python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/ncu_dmma.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/inject_launches.csv python tools/prof_inject.py --steps 14 > $OUT/inject.log 2>&1; echo "ncu2 rc=$?"; tail -3 $OUT/inject.log
