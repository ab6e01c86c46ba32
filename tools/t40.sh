for lib in "" paper_2408_01391_b200/_lib/var_noinj/libftkb200.so; do
echo "== lib=$lib"
for dbg in 0 1 2 3 4; do FTK_LIB_PATH=$lib FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_dbg.py 2>&1 | tail -1; done
FTK_LIB_PATH=$lib CHK=0 timeout 120 python tools/prof_dbg.py 2>&1 | tail -1
done
