python -m pytest tests/test_gpu_parity.py -x -q -k "update or lloyd or dmr" 2>&1 | tail -2
bash tools/t34.sh 2>&1 | tail -2
