# r6e: coalesced segment fold (32 chains per block, warps stride the segments) + replay grid 148*8
OUT=gpurun_out/r6e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_shard_gloo.py -q -x -m gpu > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
bash tools/ab.sh r6e/ab old base
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python tools/iter_breakdown.py $OUT/launches.csv 30
for cfg in "--n 1000000 --d 512 --k 16" "--n 1000000 --d 2048 --k 32"; do
  timeout 300 python tools/prof_cfg.py $cfg --ft abft --steps 5 2>&1 | tail -2
  FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_old/libftkb200.so timeout 300 python tools/prof_cfg.py $cfg --ft abft --steps 5 2>&1 | tail -2
done
