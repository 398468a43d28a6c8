"""Summarise an ncu --set full report for profiles/: per-kernel key metrics
(markdown) and DRAM traffic per launch (JSON read by bench.py).

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX
   -> OUT_PREFIX.md, and profiles/ncu_traffic.json (merged)
"""
import csv
import json
import os
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("launch__registers_per_thread", "registers"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "ld_sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "ld_requests"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}


def main(rep, prefix):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m, k in WANT:
            if m in h and r[h.index(m)] not in ("", "n/a"):
                v = float(r[h.index(m)].replace(",", ""))
                d[k] = v * UNIT.get(units[h.index(m)], 1) if k in ("duration", "dram_read", "dram_write") else v
        res.append(d)
    lines = [f"# ncu --set full summary ({os.path.basename(rep)})", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | DRAM % | L2 hit % | SM % | issue % | occupancy % | thr/inst | regs | ld sectors/req |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in res:
        spr = d.get("ld_sectors", 0) / d["ld_requests"] if d.get("ld_requests") else 0
        lines.append(f"| {d['kernel']} | {d.get('duration', 0) * 1e3:.3f} | {d.get('dram_read', 0) / 1e9:.2f} | "
                     f"{d.get('dram_write', 0) / 1e9:.2f} | {d.get('dram_pct', 0):.1f} | {d.get('l2_hit_pct', 0):.1f} | "
                     f"{d.get('sm_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get('threads_per_inst', 0):.1f} | "
                     f"{d.get('registers', 0):.0f} | {spr:.2f} |")
        if "dram_read" in d:
            name = d["kernel"].replace("mc::", "").replace("void ", "").split("<")[0].strip()
            traffic[name] = {
                "dram_bytes_per_launch": int(d["dram_read"] + d.get("dram_write", 0)),
                "source": os.path.basename(rep)}
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    # keep only kernels that still exist in libmc.so (renamed / removed ones are stale)
    live = {"k_sketch_partition", "k_sub_count", "k_sub_scatter", "k_sub_finalize", "k_heavy_select",
            "k_query_plan", "k_query_sketch_probe", "k_query_small", "k_query_medium", "k_query_large",
            "k_merge_classify"}
    old = {k: v for k, v in old.items() if k in live}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
