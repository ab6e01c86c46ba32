"""Top stall lines of an ncu report's SASS source page + barrier waits."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
agg = {h[i]: sum(float(r[i] or 0) for r in data) for i in sc}
print("samples", tot, {k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
for i, r in enumerate(sorted(range(len(data)), key=lambda j: -float(data[j][si] or 0))[:n]):
    row = data[r]
    st = sorted(((h[c], float(row[c] or 0)) for c in sc), key=lambda x: -x[1])[:2]
    prev = data[r - 1][1][:40] if r else ""
    print(row[0][-5:], row[1][:58].ljust(58), row[si].rjust(6), row[ie].rjust(9), st[0][0], "| prev:", prev)
