# r4d: same-box A/B: rowinfo/constant prefetch in the refine (base) vs previous (prev)
OUT=gpurun_out/r4d; mkdir -p $OUT
bash tools/ab.sh r4d base prev 2>&1
for v in base prev; do
  if [ $v = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python tools/prof_kernel_dbg.py 0 0 2>&1 | grep dbg | sed "s/^/$v /"
done
