# r3l: refine loop probes: 8 no c loads, 16 no chain, 32 no X smem reads, 64 no csum smem reads
OUT=gpurun_out/r3l; mkdir -p $OUT
P=paper_2408_01391_b200/_lib/var_probe/libftkb200.so
for dbg in 0 24 56 120; do
  FTK_LIB_PATH=$P FTK_PAIR_CLK=1 FTK_TC_DEBUG=$dbg timeout 300 python tools/prof_cfg.py --ft abft --steps 4 > $OUT/probe_$dbg.log 2>&1
  echo "dbg=$dbg"; grep "pair clk" $OUT/probe_$dbg.log | sed -n 5,6p
done
FTK_LIB_PATH=$P FTK_PAIR_CLK=1 timeout 300 python tools/prof_cfg.py --ft off --steps 4 > $OUT/probe_off.log 2>&1
echo "ft off"; grep "pair clk" $OUT/probe_off.log | sed -n 5,6p
