# r3u: chain consumer loads batched per group: parity + c4 update
OUT=gpurun_out/r3u; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or update or dmr" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 5 --variant pair > $OUT/c4.log 2>&1; tail -3 $OUT/c4.log
