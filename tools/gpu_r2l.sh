# r2l: ABFT flag records + post-pass events; A/B vs the narrow-commit build; tests
OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abft_tc.py tests/test_gpu_tc.py tests/test_gpu_narrow.py -q -x -rf > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
bash tools/ab.sh r2l base head
