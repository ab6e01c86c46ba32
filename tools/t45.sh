timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "update or lloyd or dmr" 2>&1 | tail -2
for cfg in "--n 1000000 --d 512 --k 16" "--n 1000000 --d 2048 --k 8" "--n 100000 --d 32 --k 64"; do
echo "== $cfg"; timeout 300 python tools/prof_cfg.py $cfg --steps 4 2>&1 | tail -1
done
timeout 300 bash tools/t34.sh 2>&1 | tail -2
python tools/iter_breakdown.py gpurun_out/t34.csv 7
