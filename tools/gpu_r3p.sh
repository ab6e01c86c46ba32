# r3p: TMA-fed float64 refine: parity + c4 timing vs the LDG version
OUT=gpurun_out/r3p; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc64.py -q -x -rf > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_tma.log 2>&1; tail -3 $OUT/c4_tma.log
FTK_T64_REFINE_LDG=1 timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 5 --variant pair > $OUT/c4_ldg.log 2>&1; tail -3 $OUT/c4_ldg.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tc64_refine -c 4 --csv --log-file $OUT/refine.csv python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > /dev/null 2>&1
grep tc64_refine $OUT/refine.csv | cut -d, -f5,13- | head
