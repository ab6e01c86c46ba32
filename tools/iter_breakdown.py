"""Kernel breakdown of one steady-state Lloyd iteration from an ncu launch list
of tools/prof_lloyd.py: python tools/iter_breakdown.py launches.csv [n]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as S  # noqa: E402

seq = S.launches(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
idx = [i for i, (name, ms) in enumerate(seq)
       if 'pair_screen_kernel<1, 0' in name or 'pair_screen_kernel<0, 0' in name]
agg = collections.OrderedDict()
for name, ms in seq[idx[-2]:idx[-1]]:
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += ms
print("one iteration, kernel sum %.3f ms" % sum(v[1] for v in agg.values()))
for name, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"  {name[:66]:66s} {c:3d} {ms:8.4f}")
