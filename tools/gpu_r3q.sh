# r3q: three screen warpgroups (swg3, 96-register cap with spills) vs two (base): parity + A/B
OUT=gpurun_out/r3q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_base.log 2>&1; tail -2 $OUT/pytest_base.log
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_swg3/libftkb200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_swg3.log 2>&1; tail -2 $OUT/pytest_swg3.log
bash tools/ab.sh r3q base swg3 2>&1
