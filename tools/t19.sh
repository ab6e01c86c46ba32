timeout 240 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 120 python tools/prof_cfg.py --n 2000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3
timeout 120 python tools/prof_cfg.py --n 1000000 --d 512 --k 16 --steps 3
