timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "update or lloyd or dmr" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t44.csv python tools/prof_cfg.py --n 1000000 --d 512 --k 16 --steps 5 > /dev/null 2>&1
FTK_UPD_DEBUG=1 timeout 120 python tools/prof_cfg.py --n 1000000 --d 512 --k 16 --steps 4 2>&1 | tail -3
