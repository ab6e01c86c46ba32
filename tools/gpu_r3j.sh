# r3j: gated screen experiment (data order vs rows grouped by cluster), c2 and c5-shape
OUT=gpurun_out/r3j; mkdir -p $OUT
timeout 600 python tools/prof_gate.py > $OUT/gate_c2.log 2>&1; cat $OUT/gate_c2.log | grep -v Warn
timeout 600 python tools/prof_gate.py 1000000 128 4096 > $OUT/gate_k4096.log 2>&1; cat $OUT/gate_k4096.log | grep -v Warn
