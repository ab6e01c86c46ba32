# r4i: the multi-rank bench path end to end on one GPU (2 ranks over gloo, both on cuda:0), c2 and reference arm
OUT=gpurun_out/r4i; mkdir -p $OUT
FTK_BENCH_DEVICE=0 FTK_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --campaign-s 0 > $OUT/bench2.json 2> $OUT/bench2.err; echo "rc=$?"
tail -c 1500 $OUT/bench2.json; tail -5 $OUT/bench2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/ref2.json 2> $OUT/ref2.err; echo "ref rc=$?"; tail -c 600 $OUT/ref2.json
