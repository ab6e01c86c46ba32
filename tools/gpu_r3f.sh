# r3f: per-warp yn staging (no named barrier) + hint prefetch: parity, A/B, role timing
OUT=gpurun_out/r3f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_abft_tc.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for r in 1 2; do for v in hint nohint; do
  if [ $v = nohint ]; then export FTK_PAIR_NOHINT=1; else unset FTK_PAIR_NOHINT; fi
  python bench.py --steps 50 --warmup 5 --campaign-s 0.3 --reps 3 --c5 0 --c4 0 > $OUT/$v.$r.json 2> $OUT/$v.$r.err
  python -c "import json;j=json.load(open('$OUT/$v.$r.json'));print('$v', '%.1f'%j['value'],'ms %.4f'%j['ms_per_step'],'k %.4f'%j['roofline']['kernel_ms'],'off %.4f'%j['ft_off_kernel_ms'],'frac %.3f'%j['roofline']['frac'])"
done; done
unset FTK_PAIR_NOHINT
FTK_LIB_PATH=paper_2408_01391_b200/_lib/var_probe/libftkb200.so FTK_PAIR_CLK=1 python tools/prof_cfg.py --ft abft --steps 5 > $OUT/probe.log 2>&1; tail -4 $OUT/probe.log
