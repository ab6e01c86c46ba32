# r3t: chain ring depth at c4 (7 loaders; 8 / 12 / 16 slots of 16 rows; 3 loaders 8 slots)
OUT=gpurun_out/r3t; mkdir -p $OUT
for v in base ng12 ng16 l3ng8; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4_$v.log 2>&1; echo $v; tail -2 $OUT/c4_$v.log
done
