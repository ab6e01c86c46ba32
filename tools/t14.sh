timeout 300 python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3
timeout 300 python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft off --steps 3
timeout 300 python tools/prof_cfg.py --n 1000000 --d 512 --k 16 --steps 3
timeout 300 python tools/prof_cfg.py --n 1000000 --d 4 --k 4096 --steps 3
timeout 300 python tools/prof_cfg.py --n 100000 --d 32 --k 64 --steps 3
