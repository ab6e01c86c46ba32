mkdir -p gpurun_out/t22
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t22/l.csv python tools/prof_lloyd.py --steps 8 --ft abft > /dev/null 2>&1
python - <<'PY'
import sys
sys.path.insert(0,'tools')
import ncu_summary as S
seq=S.launches('gpurun_out/t22/l.csv')
# last 3 iterations: find indices of pair_screen_kernel<1, 0> launches
idx=[i for i,(n,ms) in enumerate(seq) if 'pair_screen_kernel<1, 0>' in n]
a,b=idx[-3],idx[-1]
tot=0
for n,ms in seq[a:b]:
    pass
import collections
agg=collections.OrderedDict()
for n,ms in seq[idx[-2]:idx[-1]]:
    agg.setdefault(n,[0,0.0]); agg[n][0]+=1; agg[n][1]+=ms
t=sum(v[1] for v in agg.values())
print("one ABFT iteration, kernel sum %.3f ms"%t)
for n,(c,ms) in sorted(agg.items(),key=lambda x:-x[1][1]): print(f"{n[:70]:70s} {c:3d} {ms:8.4f}")
PY
