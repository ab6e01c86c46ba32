python -m pytest tests/test_gpu_parity.py -x -q -k "graph or inject or campaign or checked" 2>&1 | tail -5
python tools/prof_steps.py 16 2>&1 | tail -16
