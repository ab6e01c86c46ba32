timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 bash tools/t34.sh 2>&1 | tail -2
python tools/iter_breakdown.py gpurun_out/t34.csv 8
