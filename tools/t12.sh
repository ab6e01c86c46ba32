timeout 180 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FTK_PAIR_CLK=1 timeout 60 python tools/prof_lloyd.py --steps 6 --ft abft 2>&1 | tail -4
FTK_PAIR_CLK=1 timeout 60 python tools/prof_lloyd.py --steps 6 --ft off 2>&1 | tail -4
