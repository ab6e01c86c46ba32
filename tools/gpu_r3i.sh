# r3i: pass-1 pair kernel time with roles switched off (which role bounds it)
OUT=gpurun_out/r3i; mkdir -p $OUT
timeout 600 python tools/prof_kernel_dbg.py > $OUT/dbg.log 2>&1; cat $OUT/dbg.log | grep dbg
