# r3h: refine timing probes (bits 8: no centroid loads, 16: no exact chain) + tc parity
OUT=gpurun_out/r3h; mkdir -p $OUT
P=paper_2408_01391_b200/_lib/var_probe/libftkb200.so
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py -q -x -rf > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for dbg in 0 8 16 24; do
  FTK_LIB_PATH=$P FTK_PAIR_CLK=1 FTK_TC_DEBUG=$dbg timeout 300 python tools/prof_cfg.py --ft abft --steps 5 > $OUT/probe_$dbg.log 2>&1
  echo "dbg=$dbg"; grep "pair clk" $OUT/probe_$dbg.log | sed -n 7,8p
done
