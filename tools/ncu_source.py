"""Summarise an ncu source page (CUDA-source view): top lines by stall samples."""
import csv
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", kernel],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
src = 1
data = [r for r in rows[hdr + 1:] if len(r) > si and r[0].strip() and r[si].strip().isdigit()]
tot = sum(int(r[si]) for r in data) or 1
extra = [c for c in ("L2 Theoretical Sectors Global Excessive", "L2 Theoretical Sectors Global", "Instructions Executed") if c in h]
for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
    print(f"{100*int(r[si])/tot:5.1f}%  {r[0]:>5}  {r[src].strip()[:90]:90s} " + " ".join(f"{c.split()[-1]}={r[h.index(c)]}" for c in extra))
