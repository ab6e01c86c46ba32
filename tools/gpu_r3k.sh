# r3k: N=128 accumulator tiles (4 TMEM buffers) vs N=256: parity on the variant lib + A/B
OUT=gpurun_out/r3k; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_bn128/libftkb200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_bn128.log 2>&1; tail -2 $OUT/pytest_bn128.log
bash tools/ab.sh r3k base bn128 2>&1
