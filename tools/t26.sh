python tools/prof_steps.py 12 2>&1 | tail -12
python -m pytest tests/test_gpu_parity.py -x -q -k "graph or inject or campaign" 2>&1 | tail -3
bash tools/ab.sh ab2 base nohint
