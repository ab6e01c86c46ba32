# r2w: chain_spec loader/ring sweep at c4
OUT=gpurun_out/r2w; mkdir -p $OUT
for v in base l5 l11 l13; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 4 > $OUT/c4_$v.log 2>&1; echo $v; tail -2 $OUT/c4_$v.log
done
