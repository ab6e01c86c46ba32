timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 bash tools/t34.sh 2>&1 | tail -2
python tools/iter_breakdown.py gpurun_out/t34.csv 5
for cfg in "--n 1000000 --d 512 --k 16" "--n 100000 --d 32 --k 64"; do
echo "== $cfg abft"; timeout 300 python tools/prof_cfg.py $cfg --steps 4 --ft abft 2>&1 | tail -1
done
