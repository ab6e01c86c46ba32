# A/B bench: bash tools/ab.sh OUT var1 var2 ...  ("base" = default build); 2 rounds each, alternating
out=gpurun_out/$1; shift; mkdir -p $out
for r in 1 2; do for v in "$@"; do
  if [ "$v" = base ]; then lp=""; else lp=paper_2408_01391_b200/_lib/var_$v/libftkb200.so; fi
  FTK_LIB_PATH=$lp timeout 300 python bench.py --steps 50 --warmup 5 --campaign-s 0.3 --reps 3 --c5 0 --c4 0 > $out/$v.$r.json 2> $out/$v.$r.err
  FTK_LIB_PATH=$lp python -c "import json;j=json.load(open('$out/$v.$r.json'));print('$v', '%.1f'%j['value'],'ms %.4f'%j['ms_per_step'],'k %.4f'%j['roofline']['kernel_ms'],'off %.4f'%j['ft_off_kernel_ms'],'offstep %.4f'%j['ft_off_ms_per_step'],'e2e %.1f'%j['e2e']['value'])"
done; done
