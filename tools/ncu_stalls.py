"""Top stall locations (SASS) of an .ncu-rep: python tools/ncu_stalls.py rep [n]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ci, si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
data = [r for r in rows[2:] if len(r) > ci]
tot = sum(float(r[ci] or 0) for r in data) or 1
agg = {}
for r in data:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print("stall totals:", {k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
for r in sorted(data, key=lambda r: -float(r[ci] or 0))[:n]:
    reasons = sorted(((h[i], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
    print(f"{100 * float(r[ci]) / tot:5.1f}%  {r[ai][-5:]}  {r[si].strip()[:70]:70s} {reasons}")
