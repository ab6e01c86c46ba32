mkdir -p gpurun_out/t31
for ft in off abft; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t31/$ft.csv python tools/prof_lloyd.py --steps 8 --ft $ft > /dev/null 2>&1
done
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
