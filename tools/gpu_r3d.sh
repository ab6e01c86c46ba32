# r3d: chain slab widths: parity + c4 update timing
OUT=gpurun_out/r3d; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or update" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for sl in auto 512 256 128; do
  if [ $sl = auto ]; then unset FTK_CS_SLAB; else export FTK_CS_SLAB=$sl; fi
  timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4_$sl.log 2>&1; echo $sl; tail -2 $OUT/c4_$sl.log
done
