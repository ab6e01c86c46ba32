timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
python tools/dbg_sx.py 2>&1 | tail -8
for cfg in "--n 1000000 --d 512 --k 16" "--n 1000000 --d 2048 --k 8" "--n 1000000 --d 512 --k 32" "--n 100000 --d 32 --k 64" "--n 1000000 --d 8 --k 4096"; do
echo "== $cfg abft"; timeout 300 python tools/prof_cfg.py $cfg --steps 4 --ft abft 2>&1 | tail -1
done
