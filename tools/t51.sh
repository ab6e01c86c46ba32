echo "== c4 N=1e7 D=64 K=256 f64 abft"; timeout 600 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 2>&1 | tail -1
echo "== c3 D=8 K=4096"; timeout 300 python tools/prof_cfg.py --n 1000000 --d 8 --k 4096 --steps 3 2>&1 | tail -1
echo "== c3 D=4 K=4096"; timeout 300 python tools/prof_cfg.py --n 1000000 --d 4 --k 4096 --steps 3 2>&1 | tail -1
echo "== c3 D=2048 K=32"; timeout 300 python tools/prof_cfg.py --n 1000000 --d 2048 --k 32 --steps 3 2>&1 | tail -1
echo "== c5 1 GPU"; timeout 900 python tools/prof_c5.py 2>&1 | tail -4
