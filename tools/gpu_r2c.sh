# r2c: sharded-engine tests, kpp timing, tensor-pipe calibration
OUT=gpurun_out/r2c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo BUILD_FAIL
timeout 600 python -m pytest tests/test_shard_gloo.py tests/test_gpu_parity.py -m gpu -q -x -k "sharded or kmeanspp or upload or phase" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 300 python tools/prof_kpp.py > $OUT/kpp.log 2>&1; cat $OUT/kpp.log
M=sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg,sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"gemm|Kernel|sm100|nvjet|cutlass" -c 10 python tools/ncu_tensor_calib.py > $OUT/calib.csv 2>&1; echo "calib rc=$?"
timeout 300 ncu --metrics $M --clock-control none --csv -k regex:pair_screen -s 8 -c 2 python tools/prof_assign.py --variant tc --reps 3 --iters 3 --checked > $OUT/calib_pair.csv 2>&1; echo "calib pair rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:kpp -c 40 python tools/prof_kpp.py 200000 > $OUT/kpp_ncu.csv 2>&1; echo "kpp ncu rc=$?"
