mkdir -p gpurun_out/t9
timeout 300 ncu --set full --clock-control none --import-source on -k regex:seg_ -s 4 -c 2 -o gpurun_out/t9/seg python tools/prof_lloyd.py --steps 4 > gpurun_out/t9/ncu.log 2>&1; tail -2 gpurun_out/t9/ncu.log
