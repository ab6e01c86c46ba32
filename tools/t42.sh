for cfg in "--n 1000000 --d 512 --k 16" "--n 1000000 --d 2048 --k 8" "--n 100000 --d 32 --k 64" "--n 1000000 --d 512 --k 32" "--n 1000000 --d 8 --k 4096" "--n 1000000 --d 4 --k 4096"; do
for path in pipe seg; do
echo "== $cfg $path"; FTK_UPD_PATH=$path timeout 300 python tools/prof_cfg.py $cfg --steps 4 2>&1 | tail -1
done; done
