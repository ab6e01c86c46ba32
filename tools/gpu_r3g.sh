# r3g: same-box A/B: per-warp yn staging (base) vs shared + named barrier (ynshared)
OUT=gpurun_out/r3g; mkdir -p $OUT
bash tools/ab.sh r3g base ynshared 2>&1
