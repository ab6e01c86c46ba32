# r2t: CTA-pair screen role timing (probe build) + debug pipeline splits at c2; c4 launch list
OUT=gpurun_out/r2t; mkdir -p $OUT
P=paper_2408_01391_b200/_lib/var_probe/libftkb200.so
python tools/prof_assign.py --checked --iters 3 --reps 5 > $OUT/base.log 2>&1; tail -2 $OUT/base.log
FTK_TC_DEBUG=1 python tools/prof_assign.py --checked --iters 3 --reps 5 > $OUT/dbg1.log 2>&1; tail -2 $OUT/dbg1.log
FTK_TC_DEBUG=4 python tools/prof_assign.py --checked --iters 3 --reps 5 > $OUT/dbg4.log 2>&1; tail -2 $OUT/dbg4.log
FTK_LIB_PATH=$P FTK_PAIR_CLK=1 python tools/prof_assign.py --checked --iters 3 --reps 4 > $OUT/probe.log 2>&1; tail -6 $OUT/probe.log
FTK_LIB_PATH=$P FTK_PAIR_CLK=1 FTK_TC_DEBUG=4 python tools/prof_assign.py --checked --iters 3 --reps 3 > $OUT/probe4.log 2>&1; tail -4 $OUT/probe4.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/c4_launches.csv \
  python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 > $OUT/c4_ncu.log 2>&1
python tools/ncu_summary.py $OUT/c4_launches.csv 2>&1 | head -30
