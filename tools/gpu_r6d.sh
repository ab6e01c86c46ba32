# r6d: replay sub-segment chains from LDS.128 registers; full GPU suite
OUT=gpurun_out/r6d; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python tools/prof_upd_dbg.py 10 > $OUT/upd_dbg.log 2>&1; tail -8 $OUT/upd_dbg.log
bash tools/ab.sh r6d/ab old base
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 30
