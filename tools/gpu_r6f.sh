# r6f: screen drain A/B: x2 = both chunks of a pair loaded with one wait, two tournaments in one block;
#      x2r = x2 + the TMEM buffer released as soon as the tile's last values are in registers
OUT=gpurun_out/r6f; mkdir -p $OUT
for v in x2 x2r; do
  FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_$v/libftkb200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x > $OUT/pytest_$v.log 2>&1; echo $v; tail -1 $OUT/pytest_$v.log
done
bash tools/ab.sh r6f/ab base x2 x2r
