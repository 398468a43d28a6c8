"""Per source line (all files) instruction-executed and stall-sample shares of one kernel in an ncu report.
usage: python tools/ncu_lines_exec.py REPORT KERNEL_REGEX [TOP]"""
import csv, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None; h = None; data = []
for r in rows:
    if r and r[0] == "File Name": f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": h = r; continue
    if h and len(r) == len(h) and r[0].isdigit():
        d = dict(zip(h, r))
        ex = d.get("Instructions Executed", "0") or "0"
        st = d.get("Warp Stall Sampling (All Samples)", "0") or "0"
        data.append((f, int(r[0]), r[1].strip(), int(ex) if ex.isdigit() else 0, int(st) if st.isdigit() else 0))
te = sum(x[3] for x in data) or 1; ts = sum(x[4] for x in data) or 1
print("total inst executed", te)
for x in sorted(data, key=lambda x: -x[3])[:top]:
    print(f"{100*x[3]/te:5.1f}% exec {100*x[4]/ts:5.1f}% stall  {str(x[0])[:18]:18s}:{x[1]:<5d} {x[2][:90]}")
