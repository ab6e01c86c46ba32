# r3c: DMR graph test; full ncu capture (source) of the c2 ABFT pair screen in the engine
OUT=gpurun_out/r3c; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dmr" > $OUT/pytest_dmr.log 2>&1; tail -3 $OUT/pytest_dmr.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_screen_kernel -s 6 -c 1 \
  -o $OUT/pair_c2 python tools/prof_cfg.py --ft abft --steps 5 > $OUT/ncu_pair.log 2>&1; echo "ncu rc=$?"
