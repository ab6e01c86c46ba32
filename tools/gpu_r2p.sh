# r2p: DMMA 2-CTA tiles (A/B vs 128-row), f64 parity, block_absmax, injected-step python profile
OUT=gpurun_out/r2p; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -rf > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/c4_mt2.log 2>&1; cat $OUT/c4_mt2.log
FTK_DMMA_MT=4 timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft abft --steps 4 > $OUT/c4_mt4.log 2>&1; cat $OUT/c4_mt4.log
timeout 300 python tools/prof_cfg.py --n 10000000 --d 64 --k 256 --dtype f64 --ft off --steps 4 > $OUT/c4_off.log 2>&1; cat $OUT/c4_off.log
timeout 300 python -c "
import cProfile, pstats, sys, runpy
sys.argv=['tools/prof_inject.py','--steps','40']
cProfile.run(\"runpy.run_path('tools/prof_inject.py', run_name='__main__')\", '$OUT/inject.prof')
p=pstats.Stats('$OUT/inject.prof'); p.sort_stats('cumulative').print_stats(35)
" > $OUT/inject_prof.log 2>&1; grep -A60 "median clean" $OUT/inject_prof.log | head -70
