# r3s: ncu full capture of the warp-specialised float64 chain kernel at c4
OUT=gpurun_out/r3s; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_spec -s 2 -c 1 \
  -o $OUT/chain_spec python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 4 --variant pair > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
