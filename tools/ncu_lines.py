"""Top source lines of one kernel in an ncu report by instructions executed
(and by stall samples): python tools/ncu_lines.py REPORT KERNEL [N]"""
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", kernel],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
ie = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


data = [r for r in rows[hdr + 1:] if len(r) > ie and r[0].strip() and num(r[ie]) > 0]
tot = sum(num(r[ie]) for r in data) or 1
sst = sum(num(r[si]) for r in data) or 1
print(f"total instructions executed: {tot:.3e}")
for r in sorted(data, key=lambda r: -num(r[ie]))[:top]:
    print(f"{100 * num(r[ie]) / tot:5.1f}% inst {100 * num(r[si]) / sst:5.1f}% stall  {r[0]:>5}  {r[1].strip()[:100]}")
