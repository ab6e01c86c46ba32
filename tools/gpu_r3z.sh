# r3z: e2e (numpy input, 10-iteration ABFT fit) vs staged-uploader copy threads
OUT=gpurun_out/r3z; mkdir -p $OUT
for t in 6 10 14 4; do FTK_H2D_THREADS=$t timeout 300 python tools/prof_e2e_np.py 2>&1 | tail -1; done | tee $OUT/e2e_threads.log
