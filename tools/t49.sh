for dbg in 0 1 2; do FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_sx.py 1000000 512 16 2>&1 | tail -1; done
for dbg in 0 2; do FTK_TC_DEBUG=$dbg timeout 120 python tools/prof_sx.py 1000000 2048 8 2>&1 | tail -1; done
timeout 120 python tools/prof_sx.py 1000000 256 16 2>&1 | tail -1
