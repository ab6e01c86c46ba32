# r3v: three screen warpgroups with setmaxnreg rebalancing (swg3r) vs base: parity + A/B
OUT=gpurun_out/r3v; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_swg3r/libftkb200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest_swg3r.log 2>&1; tail -2 $OUT/pytest_swg3r.log
bash tools/ab.sh r3v base swg3r 2>&1
