# r6k: centroid-table refine sized against the shared-memory limit; float64 + config tests
OUT=gpurun_out/r6k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc64.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
