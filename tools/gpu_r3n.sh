# r3n: is the X-buffer hand-back the MMA's wait?  dbg 128 releases X before the refine loop
OUT=gpurun_out/r3n; mkdir -p $OUT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_probe/libftkb200.so timeout 600 python tools/prof_kernel_dbg.py 0 128 2 0 128 > $OUT/dbg.log 2>&1; grep dbg $OUT/dbg.log
