# r3m: warp-id priority A/B: refine warps 0..3 (reflow) vs 8..11 (base)
OUT=gpurun_out/r3m; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_reflow/libftkb200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x -rf > $OUT/pytest_reflow.log 2>&1; tail -2 $OUT/pytest_reflow.log
bash tools/ab.sh r3m base reflow 2>&1
