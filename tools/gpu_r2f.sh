# r2f: ncu of the narrow screen (hinted iteration) at c3 K16 D512
OUT=gpurun_out/r2f; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:narrow_screen -s 1 -c 1 \
  -o $OUT/narrow_k16 python tools/prof_narrow.py --steps 2 --shapes 16x512 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 $OUT/ncu.log
