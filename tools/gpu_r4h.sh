# r4h: ncu full captures of the F64 pair screen at c4, CHK vs non-CHK
OUT=gpurun_out/r4h; mkdir -p $OUT
timeout 500 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 \
  -o $OUT/f64chk python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 3 --variant pair > $OUT/ncu1.log 2>&1; echo "rc=$?"
timeout 500 ncu --set full --clock-control none --import-source on -k regex:pair_screen -s 2 -c 1 \
  -o $OUT/f64off python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 3 --variant pair > $OUT/ncu2.log 2>&1; echo "rc=$?"
