timeout 240 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3
timeout 120 python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft off --steps 3
