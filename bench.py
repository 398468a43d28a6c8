#!/usr/bin/env python3
"""bench.py -- MetaCache-GPU hot path on B200 (arXiv 2106.08150).

One step = the whole hot path over one batch of synthetic input:
  build   : clear the static table, insert every reference target (B1-B5),
            finalize (B6: sort + cap + condensed layout)
  query   : classify the read batch (Q1-Q9)
Workload (N=1): BASELINE.json configs[1] "bacterial subset": ~1,000 synthetic
genomes (~4.4 Gbp) + 1M paired-end 2x150 bp reads.  For N>1 every rank
builds its own ~4.4 Gbp partition (weak scaling) and the read batch is
all-gathered; candidates are merged with one all-to-all (see
paper_2106_08150_b200/dist.py).

Prints ONE JSON line on rank 0.  `value` = DB build Gbp/s (device-resident
inputs); `query` holds classified reads/s (each mate counts as a read,
SURVEY S22); `e2e` repeats both through the C-ABI with pinned HOST buffers
(host<->device copies inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOADS = {
    "subset": dict(n_targets=1000, n_pairs=1_000_000, read_len=150, ref_kw={},
                   desc="bacterial subset: ~1,000 synthetic genomes (~4 Gbp) DB build + 1M paired-end 150 bp reads"),
    # configs[2] / configs[4] query shapes against the subset DB (same build)
    "afs20": dict(n_targets=1000, n_pairs=10_000_000, read_len=101, ref_kw={}, reads="afs",
                  desc="AFS20-shaped query: 20-species mock community, 10M paired-end 2x101 bp reads against the "
                       "bacterial-subset DB (~1,000 synthetic genomes, ~4 Gbp; build included in the step)"),
    "kal": dict(n_targets=1000, n_pairs=4_000_000, read_len=101, ref_kw={}, reads="kal",
                desc="KAL_D-shaped query: 4M paired-end 2x101 bp reads, 95% from genomes absent from the DB, against "
                     "the bacterial-subset DB (build included in the step)"),
    # variable-length single-end query shapes (Table 2)
    "hiseq": dict(n_targets=1000, n_pairs=10_000_000, read_len=101, ref_kw={}, reads="hiseq",
                  desc="HiSeq-shaped query: 10M single-end reads of 19-101 bp (mean 92.3) against the "
                       "bacterial-subset DB (build included in the step)"),
    "miseq": dict(n_targets=1000, n_pairs=10_000_000, read_len=251, ref_kw={}, reads="miseq",
                  desc="MiSeq-shaped query: 10M single-end reads of 19-251 bp (mean 156.8, 1-3 windows) against the "
                       "bacterial-subset DB (build included in the step)"),
    # configs[3]: one per-GPU target shard (genus mod 8) of the RefSeq-202-shaped DB; at N=8
    # the 8 ranks build the whole ~70 Gbp / ~50k-sequence database; queried with KAL_D-shaped pairs
    "refseq8": dict(n_targets=0, n_pairs=4_000_000, read_len=101, ref_kw={}, reads="kal", refs="refseq8",
                    desc="RefSeq-202-shaped DB, one 1/8 target shard per GPU (~8-9 Gbp, ~6k sequences: viral, "
                         "strain-structured bacterial + plasmids, fungal chromosomes) + 4M KAL_D-shaped pairs 2x101 bp"),
    # one per-GPU shard (species mod 8) of the AFS31-shaped eukaryotic DB
    # (Table 1): chromosome-level and scaffold-level genomes, ~10^5 targets
    "afs31x8": dict(n_targets=0, n_pairs=4_000_000, read_len=101, ref_kw={}, reads="kal", refs="afs31x8",
                    desc="AFS31-shaped eukaryotic DB, one 1/8 species shard per GPU (~9.5 Gbp: long chromosomes + "
                         "~10^5 scaffold targets) + 4M KAL_D-shaped pairs 2x101 bp"),
    "small": dict(n_targets=100, n_pairs=100_000, read_len=150,
                  ref_kw=dict(median_len=4e5, min_len=1e5, max_len=1e6),
                  desc="small: 100 synthetic genomes (~40 Mbp) + 100k paired-end 150 bp reads"),
}
FALLBACK_HBM_GBS = 6650.0


BENCH_M = 4
# reads per internal query batch: host reads of batch b+1 are copied while
# batch b computes (libmc.so query pipeline)
READ_BATCH = 1 << 18


def make_db(mc, refs, world, rank, local, n_pairs, read_batch=READ_BATCH):
    """The database in the launch configuration bench.py times (also used by
    tests/test_gpu_fullsize.py for full-size parity)."""
    return mc.Database(refs.parent, refs.rank, n_partitions=world, partition_begin=rank, n_local_partitions=1,
                       capacity_bp=int(refs.total_bp * 1.01) + (1 << 20), max_targets=refs.n + 64,
                       read_batch=min(read_batch, n_pairs), device=local, max_candidates=BENCH_M)


def all_reduce_host(t, op):
    import torch.distributed as dist
    c = t.cpu()
    dist.all_reduce(c, op=op)
    return c.to(t.device)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=list(WORKLOADS), default="subset")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile", action="store_true", help="short run for ncu: no e2e, no CPU baseline")
    p.add_argument("--read-batch", type=int, default=READ_BATCH, help="reads per internal query batch")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path))["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# CPU oracle on a bounded sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_sample(refs, read_len, target_bp=12_000_000, n_pairs=10_000, seed=synth.READ_SEED):
    """First targets of the shard up to ~target_bp, plus pairs drawn from them."""
    lens = np.diff(refs.offsets).astype(np.int64)
    order = np.argsort(lens)  # smallest first so several targets (and species) are sampled
    sel, bp = [], 0
    for i in order:
        if bp >= target_bp:
            break
        sel.append(int(i))
        bp += int(lens[i])
    sel.sort()
    seqs = [refs.seq(i) for i in sel]
    sub = synth.references_from_list(seqs, refs.taxa[sel], refs.parent, ids=refs.target_ids[sel])
    rd = synth.paired_reads(sub, n_pairs, length=read_len, seed=seed)
    return sub, rd


def host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def run_oracle_step(sub, rd, threads=0):
    """Oracle build (1 thread) + query (1 thread); with threads > 0 also the
    query phase on `threads` host threads.  Returns (build s, query s[, query
    s on threads, threads])."""
    import oracle
    t0 = time.perf_counter()
    db = oracle.OracleDB(sub.parent)
    db.insert(sub.buf, sub.offsets, sub.target_ids, sub.taxa)
    db.finalize()
    t1 = time.perf_counter()
    db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
    t2 = time.perf_counter()
    if threads:
        db.classify_threads(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets, threads=threads)
        t3 = time.perf_counter()
        db.close()
        return t1 - t0, t2 - t1, t3 - t2, threads
    db.close()
    return t1 - t0, t2 - t1


def sample_desc(sub, rd):
    return (f"oracle (1 thread, std::map) on {sub.n} targets / {sub.total_bp / 1e6:.1f} Mbp of the workload's "
            f"references (build) + {rd.n} read pairs drawn from them (query)")


# ---------------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl, world, rank)
    import torch
    import torch.distributed as dist
    # MC_BENCH_REHEARSE=1: a multi-rank rehearsal on fewer GPUs than ranks (ranks share
    # devices, gloo process group staged through the host) -- exercises the N>1 code
    # path on the one-GPU box; never a reported number
    rehearse = os.environ.get("MC_BENCH_REHEARSE") == "1"
    if rehearse:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if rehearse:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import paper_2106_08150_b200 as mc
    from paper_2106_08150_b200 import dist as mcd

    # ---- synthetic workload (host), then device copies ----------------------
    t0 = time.time()
    if wl.get("refs") == "refseq8":
        if world > 8:
            raise SystemExit("refseq8: at most 8 ranks (one 1/8 shard each)")
        refs = synth.refseq_shard(rank, 8)
    elif wl.get("refs") == "afs31x8":
        if world > 8:
            raise SystemExit("afs31x8: at most 8 ranks (one 1/8 shard each)")
        refs = synth.afs31_shard(rank, 8)
    else:
        refs = synth.subset_shard(rank, world, n_targets=wl["n_targets"], **wl["ref_kw"])
    n_pairs, L = wl["n_pairs"], wl["read_len"]  # read records (pairs, or single reads), max read length
    lo, hi = mcd.slice_bounds(n_pairs, world, rank)
    gen = {"afs": synth.afs_reads, "kal": synth.kal_reads}.get(wl.get("reads"))
    if wl.get("reads") in ("hiseq", "miseq"):
        rd = getattr(synth, wl["reads"] + "_reads")(refs, hi - lo, seed=synth.READ_SEED + 40 + rank)
    elif gen:
        rd = gen(refs, hi - lo, length=L, seed=synth.READ_SEED + 20 + rank)
    else:
        rd = synth.paired_reads(refs, hi - lo, length=L, seed=synth.READ_SEED + rank)
    paired = rd.mates_buf is not None
    log(f"[rank {rank}] workload: {refs.n} targets, {refs.total_bp / 1e9:.3f} Gbp, {rd.n} local "
        f"{'pairs' if paired else 'reads'} ({time.time() - t0:.1f}s)")
    dev = torch.device(f"cuda:{local}")
    pin = lambda a: torch.from_numpy(a).pin_memory()
    h_buf = pin(refs.buf)
    h_offs = refs.offsets
    d_buf = h_buf.to(dev)
    d_offs = torch.from_numpy(refs.offsets.astype(np.int64)).to(dev)
    # reads as flat byte buffers + record offsets (fixed or variable length; mates optional)
    h_r1, o1 = pin(rd.buf), rd.offsets.astype(np.uint64)
    h_r2, o2 = (pin(rd.mates_buf), rd.mate_offsets.astype(np.uint64)) if paired else (None, None)
    h_o1 = pin(o1.astype(np.int64))
    h_o2 = pin(o2.astype(np.int64)) if paired else None
    pids = np.full(refs.n, rank, np.uint32)
    m = BENCH_M
    db = make_db(mc, refs, world, rank, local, n_pairs, args.read_batch)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    db.set_stream(stream)
    n_mine = hi - lo
    d_tax = torch.zeros(n_mine if world > 1 else n_pairs, dtype=torch.int32, device=dev)
    d_cand = torch.zeros((n_mine if world > 1 else n_pairs) * m * 4, dtype=torch.int32, device=dev)
    d_hits = torch.zeros(n_pairs * m * 6, dtype=torch.int32, device=dev)
    h_tax = torch.zeros(n_mine, dtype=torch.int32).pin_memory()
    h_cand = torch.zeros(n_mine * m * 4, dtype=torch.int32).pin_memory()

    def gather_reads(r1, a1, r2, a2):
        if world == 1:
            return r1, a1, r2, a2
        r1, a1 = mcd.allgather_flat(r1, a1)
        if r2 is not None:
            r2, a2 = mcd.allgather_flat(r2, a2)
        return r1, a1, r2, a2

    def query_device(r1, a1, r2, a2, out_tax, out_cand):
        r1, a1, r2, a2 = gather_reads(r1, a1, r2, a2)
        if world == 1:
            db.classify(r1, a1, r2, a2, out_taxon=out_tax, out_candidates=out_cand)
        else:
            db.query_partials(r1, a1, r2, a2, out_hits=d_hits)
            mine = mcd.exchange_hits(d_hits.view(n_pairs, m * 6), n_pairs)
            db.merge_classify(mine, world, n=n_mine, out_taxon=out_tax, out_candidates=out_cand)

    d_r1, d_o1 = h_r1.to(dev), h_o1.to(dev)
    d_r2, d_o2 = (h_r2.to(dev), h_o2.to(dev)) if paired else (None, None)

    def step_device():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        db.clear()
        db.insert_targets(d_buf, d_offs, refs.target_ids, refs.taxa, pids)
        db.finalize()
        e[1].record(stream)
        query_device(d_r1, d_o1, d_r2, d_o2, d_tax, d_cand)
        e[2].record(stream)
        return e

    def step_e2e():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        db.clear()
        db.insert_targets(h_buf, h_offs, refs.target_ids, refs.taxa, pids)
        db.finalize()
        e[1].record(stream)
        if world == 1:
            db.classify(h_r1, h_o1, h_r2, h_o2, out_taxon=h_tax, out_candidates=h_cand)
        else:
            cp = lambda t: t.to(dev, non_blocking=True) if t is not None else None
            query_device(cp(h_r1), cp(h_o1), cp(h_r2), cp(h_o2), d_tax, d_cand)
            h_tax.copy_(d_tax, non_blocking=True)
            h_cand.copy_(d_cand, non_blocking=True)
        e[2].record(stream)
        return e

    def timed(step, K, W, sample_clocks):
        for _ in range(W):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        db.reset_stats()
        evs = []
        with ClockSampler(local) if sample_clocks else _Null() as cs:
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            for _ in range(K):
                evs.append(step())
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
        tb = sum(e[0].elapsed_time(e[1]) for e in evs)
        tq = sum(e[1].elapsed_time(e[2]) for e in evs)
        t = torch.tensor([tb, tq], dtype=torch.float64, device=dev)
        if world > 1:
            t = all_reduce_host(t, dist.ReduceOp.MAX) if rehearse else t
            if not rehearse:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0]), float(t[1]), db.stats(), (cs.summary() if sample_clocks else None)

    K, W = args.steps, args.warmup
    if args.profile:
        args.no_e2e = args.no_cpu_baseline = True
    tb, tq, st, clocks = timed(step_device, K, W, not args.profile)
    total_bp = refs.total_bp * world  # every rank builds a partition of the same size class
    tot_bp = torch.tensor([float(refs.total_bp)], dtype=torch.float64, device=dev)
    if world > 1:
        if rehearse:
            tot_bp = all_reduce_host(tot_bp, dist.ReduceOp.SUM)
        else:
            dist.all_reduce(tot_bp)
    total_bp = float(tot_bp)
    reads = (2 if paired else 1) * n_pairs  # each mate counts as a read (S22)
    build_gbps = total_bp * K / (tb / 1e3) / 1e9
    reads_per_s = reads * K / (tq / 1e3)
    launches = sum(st["launches"].values())

    e2e = None
    if not args.no_e2e:
        eb, eq, _, _ = timed(step_e2e, K, max(1, min(W, 2)), False)
        h2d = refs.buf.nbytes + refs.offsets.nbytes + h_r1.numel() + o1.nbytes + \
            ((h_r2.numel() + o2.nbytes) if paired else 0)
        d2h = h_tax.numel() * 4 + h_cand.numel() * 4
        e2e = {"value": round(total_bp * K / (eb / 1e3) / 1e9, 3), "unit": "Gbp/s", "ms_per_step": round((eb + eq) / K, 3),
               "build_ms_per_step": round(eb / K, 3), "query_ms_per_step": round(eq / K, 3),
               "query_reads_per_s": round(reads * K / (eq / 1e3), 1),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- roofline of the dominant kernel (CUDA events inside libmc.so) -------
    peak, peak_src = peaks()
    roof = kernel_rooflines(st, K, refs, db, n_pairs, L, m, world)
    dom = max(roof.values(), key=lambda r: r["ms_per_step"]) if roof else None
    # (the committed ncu capture is of the default subset workload)
    traffic = ncu_traffic(dom["kernel"]) if dom and args.workload == "subset" else None
    roofline = None
    if dom and "alu_ops_per_s" in dom:
        # integer-ALU peak from the unit counts: 148 SMs x 128 INT32 lanes/clk x max SM clock
        smhz = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
        alu_peak = st["sms"] * 128 * smhz * 1e6
        roofline = {"bound": "alu", "kernel": dom["kernel"], "achieved": round(dom["alu_ops_per_s"] / 1e12, 3),
                    "peak": round(alu_peak / 1e12, 3), "unit": "Tintop/s",
                    "frac": round(dom["alu_ops_per_s"] / alu_peak, 4), "traffic": traffic,
                    "algorithmic_ops": "16 int ops per k-mer (DESIGN.md section 7)",
                    "peak_source": f"{st['sms']} SMs x 128 INT32 lanes x {smhz:.0f} MHz (B200_PROFILING.md / MEASURED_PEAKS sm_max_mhz)",
                    "hbm": {"achieved_gbs": dom["gbs"], "peak_gbs": peak, "frac": round(dom["gbs"] / peak, 4)},
                    "share_of_step": round(dom["ms_per_step"] / ((tb + tq) / K), 4)}
    elif dom:
        achieved = dom["gbs"]
        roofline = {"bound": "hbm", "kernel": dom["kernel"], "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                    "algorithmic_bytes_per_launch": dom["bytes_per_launch"], "peak_source": peak_src,
                    "share_of_step": round(dom["ms_per_step"] / ((tb + tq) / K), 4)}
        if "random_ops_frac_of_measured_ceiling" in dom:
            roofline["random_ops_frac_of_measured_ceiling"] = dom["random_ops_frac_of_measured_ceiling"]
            roofline["random_ceiling_ops_per_s"] = random_ceiling("read")

    path = path_roofline(st, K, tb, tq, refs, n_pairs, paired, peak, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sub, srd = oracle_sample(refs, L)
        bt, qt, qtn, nthr = run_oracle_step(sub, srd, threads=host_threads())
        cpu = {"value": round(sub.total_bp / bt / 1e9, 6), "unit": "Gbp/s", "cores": 1, "kind": "oracle",
               "sample": sample_desc(sub, srd), "query_reads_per_s": round(2 * srd.n / qt, 1),
               "build_s": round(bt, 3), "query_s": round(qt, 3),
               # the read-only query phase on every host core (SURVEY §8(d) oracle timing)
               "query_threads": {"cores": nthr, "reads_per_s": round(2 * srd.n / qtn, 1), "query_s": round(qtn, 3)},
               "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": "DB build Gbp/s and classified reads/s at 1/2/4/8 B200 vs HBM roofline",
            "value": round(build_gbps, 3), "unit": "Gbp/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": round((tb + tq) / K, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/u32 (integer path)", "data": "synthetic (seeded; synth/)",
            "config": {"workload": wl["desc"], "targets_per_gpu": refs.n, "bp_per_gpu": refs.total_bp,
                       "read_pairs" if paired else "reads": n_pairs, "paired": paired, "read_batch": min(args.read_batch, n_pairs), "read_len": L, "k": 16, "s": 16, "w": 127, "cap": 254, "m": m,
                       "partitions": world, "parallelism": f"target-partitioned x{world}",
                       "l2": "inputs and tables >> 126 MB L2 (no flush needed)"},
            "build": {"ms_per_step": round(tb / K, 3), "gbp_per_s": round(build_gbps, 3)},
            "query": {"value": round(reads_per_s, 1), "unit": "reads/s",
                      ("pairs_per_s" if paired else "records_per_s"): round(n_pairs * K / (tq / 1e3), 1),
                      "ms_per_step": round(tq / K, 3)},
            "e2e": e2e,
            "roofline": roofline,
            "path_roofline": path,
            "kernels": roof,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
            "stage_ms_per_step": {k: round(v / K, 4) for k, v in st["stage_ms"].items()},
            "db_stats": {k: v for k, v in st.items() if k not in ("stage_ms", "launches")},
        }
        print(json.dumps(line), flush=True)
    db.close()
    if world > 1:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


CEILINGS_FILE = os.path.join(ROOT, "profiles", "r02a_random_access_ceilings.jsonl")
_CEIL = {}


def random_ceiling(kind="read"):
    """Measured random-access rate of this part at the kernels' working-set
    size (tools/randbw.cu over a 4 GiB table, profiles/r02a_random_access_ceilings.jsonl):
    kind "read" = random 8-byte loads (the probe / gather shape; 125 B of DRAM
    per access by ncu, so this is the DRAM-line rate), "atomic" = random
    64-bit atomicAdd (sector read-modify-write).  None if the file is absent."""
    if kind not in _CEIL:
        want = {"read": "random_read_8B_ldg", "atomic": "random_atomicAdd_64_noret"}[kind]
        rate = None
        if os.path.exists(CEILINGS_FILE):
            for l in open(CEILINGS_FILE):
                d = json.loads(l)
                if d.get("op") == want and d.get("table_mib") == 4096 and "gops" in d:
                    rate = d["gops"] * 1e9
        _CEIL[kind] = rate
    return _CEIL[kind]


def dram_bytes_per_random_read():
    if os.path.exists(CEILINGS_FILE):
        for l in open(CEILINGS_FILE):
            d = json.loads(l)
            if d.get("op") == "random_read_8B_ldg" and "dram_read_bytes_per_op" in d:
                return d["dram_read_bytes_per_op"]
    return None


def kernel_rooflines(st, K, refs, db, n_pairs, L, m, world):
    """Algorithmic bytes per kernel over the K timed
    steps, divided by the event-timed kernel durations.  Random-access kernels
    also report random sector ops against the measured random-op ceiling."""
    ms, la = st["stage_ms"], st["launches"]
    p = st["partitions"][0]
    nslots, keys, nvals = p["table_slots"], p["keys"], p["values"]
    bp, locs = st["bp"], st["locations_inserted"]
    qfeat, qloc, read_bp, nrec = st["query_features"], st["query_locations"], st["read_bp"], st["reads"]
    # records and locations per query bin (small / medium / large); records of the
    # small bin also include those deferred out of it (their work is redone)
    nrec_all = nrec * db.n_local
    lbin = st.get("query_locations_by_bin", [qloc, 0, 0])
    rec_bin = [nrec_all - st["query_large_bin"], st["query_medium_bin"], st["query_large_bin"]]
    fpr = qfeat / max(nrec_all, 1)
    # stage: (launch key(s), algorithmic bytes, random sector ops)
    B = {
        # ASCII read once + (key, value) pair written per location
        "sketch_partition": ("k_sketch_partition", bp + 8 * locs, 0),
        # pairs read (8 B) per location
        "sub_count": ("k_sub_count", 8 * locs, 0),
        # pairs read (8 B) + regrouped pairs written (8 B) per location
        "sub_scatter": ("k_sub_scatter", 16 * locs, 0),
        # regrouped pairs read (8 B) per location + table written (8 B per slot) + values written (4 B each);
        # locs is summed over the K steps, nslots / nvals are per step
        "sub_finalize": ("k_sub_finalize", 8 * locs + K * 8 * nslots + K * 4 * nvals, 0),
        # reads + one 32 B key-table sector per probed feature + the 8 B probe word written per feature
        "query_sketch_probe": ("k_query_sketch_probe", read_bp + 32 * qfeat + 8 * qfeat, qfeat),
        # per record of the bin: its probe words (8 B per feature) + 4 B per gathered location + m hit records
        # (random ops: one list gather per probed feature of the bin's records)
        "query_small": ("k_query_small", 8 * fpr * rec_bin[0] + 4 * lbin[0] + 24 * m * rec_bin[0], fpr * rec_bin[0]),
        "query_medium": ("k_query_medium", 8 * fpr * rec_bin[1] + 4 * lbin[1] + 24 * m * rec_bin[1], 0),
        "query_large": ("k_query_large", 8 * fpr * rec_bin[2] + 4 * lbin[2] + 24 * m * rec_bin[2], 0),
        "merge_classify": ("k_merge_classify", nrec // max(world, 1) * (24 * m * world + 4 + 16 * m), 0),
    }
    rc = random_ceiling("read")  # every random-access kernel of the path reads (probes, gathers)
    # ALU-bound sketch: algorithmic integer ops per k-mer:
    # 2-bit code extract 2, ambiguity test 2, reverse complement 2, canonical min 1,
    # h1 8, bottom-s selection 1 -> 16 ops per k-mer (k-mers ~= reference bp)
    alu_ops = 16 * bp
    out = {}
    for stage, (kern, nbytes, rops) in B.items():
        t = ms.get(stage, 0.0)
        kerns = kern if isinstance(kern, tuple) else (kern,)
        n_l = sum(la.get(k, 0) for k in kerns)
        if t <= 0 or n_l == 0:
            continue
        d = {"kernel": "+".join(kerns), "ms_per_step": round(t / K, 4), "launches": n_l,
             "bytes_per_launch": int(nbytes / n_l), "gbs": round(nbytes / (t / 1e3) / 1e9, 2)}
        if rops and rc:
            d["random_ops_per_s"] = round(rops / (t / 1e3), 1)
            d["random_ops_frac_of_measured_ceiling"] = round(rops / (t / 1e3) / rc, 4)
            d["ceiling"] = "random 8-B reads over 4 GiB (tools/randbw.cu, r02a)"
        if stage in ("sketch_partition", "sketch_insert"):
            d["alu_ops_per_s"] = alu_ops / (t / 1e3)
        out[stage] = d
    return out


def path_roofline(st, K, tb, tq, refs, n_pairs, paired, peak, world):
    """Whole-path efficiency: the build's Gbp/s against the HBM
    time of its algorithmic bytes per reference bp, and the query's records/s
    against the random DRAM lines a record must touch, at the measured
    random-read rate.  Per GPU (every rank runs the same work)."""
    p = st["partitions"][0]
    bp = st["bp"] / K                       # per step, this GPU
    lpb = st["locations_inserted"] / K / max(bp, 1)  # locations per reference bp (~ s / stride)
    kpb = p["keys"] / max(bp, 1)            # distinct (feature, partition) keys per bp
    # 1 B ASCII read + per location a random sector read-modify-write
    # (32 B + 32 B) for the insert + finalize's slot read (16 B) + the 8 B value
    # written, + a 16 B key-table slot per key
    bytes_per_bp = 1.0 + lpb * (64 + 16 + 8) + kpb * 16
    build_gbps = bp / (tb / K / 1e3) / 1e9
    b_ceiling = peak / bytes_per_bp
    rrate = random_ceiling("read")
    arate = random_ceiling("atomic")
    out = {"build": {"gbp_per_s": round(build_gbps, 2), "algorithmic_bytes_per_bp": round(bytes_per_bp, 3),
                     "ceiling_gbp_per_s": round(b_ceiling, 1), "frac": round(build_gbps / b_ceiling, 4),
                     "peak_gbs": peak,
                     "random_insert_ceiling_gbp_per_s": round(arate / lpb / 1e9, 1) if arate else None,
                     "note": "bytes per bp per SURVEY 8(d); random_insert_ceiling = measured random atomic rate / "
                             "locations per bp (a per-location random-RMW insert design's bound)"}}
    nrec = st["reads"] / K                  # records per step (this GPU queries them all)
    if nrec:
        F = st["query_features"] / K / nrec
        Fh = st.get("query_features_found", 0) / K / nrec
        Lr = st["query_locations"] / K / nrec
        lines = F + Fh + 4.0 * Lr / 128.0   # probe line + first line of each list + the lists' extra lines
        rec_s = nrec / (tq / K / 1e3)
        q_ceiling = rrate / lines if rrate else None
        mult = 2 if paired else 1
        out["query"] = {"records_per_s": round(rec_s, 1), "reads_per_s": round(mult * rec_s, 1),
                        "features_per_record": round(F, 2), "lists_found_per_record": round(Fh, 2),
                        "locations_per_record": round(Lr, 1), "random_lines_per_record": round(lines, 1),
                        "random_read_rate_per_s": rrate, "dram_bytes_per_random_read": dram_bytes_per_random_read(),
                        "ceiling_records_per_s": round(q_ceiling, 1) if q_ceiling else None,
                        "frac": round(rec_s / q_ceiling, 4) if q_ceiling else None,
                        "note": "ceiling = measured random 8-B read rate (4 GiB table; each costs a 128-B DRAM line) "
                                "/ (probes + lists found + 4 B x locations / 128 B) per record"}
    return out


def ncu_traffic(kernel):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    v = d.get(kernel)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else v


def run_reference(args, wl, world, rank):
    """The reference arm: the CPU oracle (there is no reference code) on a
    bounded sample of the same workload, rank 0 only."""
    if rank != 0:
        return
    if wl.get("refs") == "refseq8":  # (the sample only needs a few small targets of the same recipe)
        refs = synth.refseq_shard(0, 8, scale=0.05)
    elif wl.get("refs") == "afs31x8":
        refs = synth.afs31_shard(0, 8, scale=0.01)
    else:
        refs = synth.subset_shard(0, 1, n_targets=wl["n_targets"], **wl["ref_kw"])
    sub, rd = oracle_sample(refs, wl["read_len"], target_bp=6_000_000, n_pairs=5_000)
    for _ in range(args.warmup):
        run_oracle_step(sub, rd)
    tb = tq = 0.0
    for _ in range(args.steps):
        b, q = run_oracle_step(sub, rd)
        tb += b
        tq += q
    K = args.steps
    val = sub.total_bp * K / tb / 1e9
    line = {
        "impl": "reference", "metric": "DB build Gbp/s and classified reads/s at 1/2/4/8 B200 vs HBM roofline",
        "value": round(val, 6), "unit": "Gbp/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": round((tb + tq) / K * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/u32 (integer path)", "data": "synthetic (seeded; synth/)",
        "config": {"workload": wl["desc"], "sample": sample_desc(sub, rd)},
        "query": {"value": round(2 * rd.n * K / tq, 1), "unit": "reads/s"},
        "cpu_baseline": {"value": round(val, 6), "unit": "Gbp/s", "cores": 1, "kind": "oracle",
                         "sample": sample_desc(sub, rd)},
        "e2e": {"value": round(val, 6), "unit": "Gbp/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
