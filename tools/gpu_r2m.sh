# r2m: variant families + selector; full GPU suite; variant table measurement
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_variants.py -q -x -rf > $OUT/pytest_var.log 2>&1; echo "rc=$?" >> $OUT/pytest_var.log
tail -15 $OUT/pytest_var.log
FTK_VARIANT_TABLE=0 timeout 1200 python tools/tune_variants.py --out $OUT/variants_b200.csv > $OUT/tune.log 2>&1; echo "tune rc=$?"; tail -3 $OUT/tune.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -6 $OUT/pytest_gpu.log
