# r6l: A/B of the X2 drain's wait without a memory clobber (norm loads may move above it)
OUT=gpurun_out/r6l; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_nomem/libftkb200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x > $OUT/pytest_nomem.log 2>&1; tail -1 $OUT/pytest_nomem.log
bash tools/ab.sh r6l/ab base nomem
