timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -4
for cfg in "--n 1000000 --d 512 --k 16" "--n 1000000 --d 2048 --k 8" "--n 1000000 --d 512 --k 32"; do
echo "== $cfg"; timeout 300 python tools/prof_cfg.py $cfg --steps 4 2>&1 | tail -1
echo "== $cfg abft"; timeout 300 python tools/prof_cfg.py $cfg --steps 4 --ft abft 2>&1 | tail -1
done
