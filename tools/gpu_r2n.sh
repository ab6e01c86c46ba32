# r2n: pair screen with streamed X over several column tiles; parity + re-tune
OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_variants.py tests/test_gpu_abft_tc.py tests/test_gpu_narrow.py -q -x -rf > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
FTK_VARIANT_TABLE=0 timeout 1200 python tools/tune_variants.py --out $OUT/variants_b200.csv > $OUT/tune.log 2>&1; echo "tune rc=$?"; tail -2 $OUT/tune.log
