# r2q: staged diagnose panels; injected-step timing; kmeans++ timing
OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_cli.py -q -x -rf > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -4 $OUT/pytest.log
timeout 300 python tools/prof_inject.py --steps 40 > $OUT/inject.log 2>&1; tail -1 $OUT/inject.log; grep INJ $OUT/inject.log | head -12
timeout 300 python tools/prof_kpp.py > $OUT/kpp.log 2>&1; tail -5 $OUT/kpp.log
