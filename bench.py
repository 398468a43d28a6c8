#!/usr/bin/env python3
"""bench.py -- MetaCache-GPU hot path on B200 (arXiv 2106.08150).

One step = the whole hot path over one batch of synthetic input:
  build   : clear the static table, insert every reference target (B1-B5),
            finalize (B6: sort + cap + condensed layout)
  query   : classify the read batch (Q1-Q9)
Workload (N=1): BASELINE.json configs[1] "bacterial subset": ~1,000 synthetic
genomes (~4.1 Gbp) + 1M paired-end 2x150 bp reads.  N > 1 (weak scaling): ONE
multi-GPU handle (mc_config.n_gpus = N) -- partition g = its own ~4 Gbp shard
on GPU g, built concurrently; the 1M read pairs (slice g drawn from shard g)
are all-gathered per batch over NVLink peer memory, every GPU scores every
record, and GPU h merges + classifies slice h reading the other GPUs' hit
lists in place.  Under torchrun only rank 0 runs (it drives all N GPUs).

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
    # configs[4] at its stated size (~100M+ reads streamed in batches against the RefSeq-shaped DB): 50M
    # KAL_D-shaped pairs (Table 2: KAL_D has 26.1M pairs) streamed through mc_classify in 4M-pair
    # batches against one GPU's full 1/8 RefSeq-202-shaped shard
    "kal50m": dict(n_targets=0, n_pairs=50_000_000, read_len=101, ref_kw={}, reads="kal_stream", refs="refseq8",
                   read_batch=1 << 22,
                   desc="KAL_D-shaped stream: 50M paired-end 2x101 bp reads (100M reads, 95% from absent genomes) "
                        "classified in 4M-pair batches against a 1/8 RefSeq-202-shaped shard (~10 Gbp; build "
                        "included in the step)"),
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
    """The single-GPU database in the launch configuration bench.py times (also
    used by tests/test_gpu_fullsize.py for full-size parity)."""
    return mc.Database(refs.parent, refs.rank, n_partitions=world, partition_begin=rank, n_local_partitions=1,
                       capacity_bp=int(refs.total_bp * 1.01) + (1 << 20), max_targets=refs.n + 64,
                       read_batch=min(read_batch, n_pairs), device=local, max_candidates=BENCH_M)


class Workload:
    """The synthetic inputs of one bench run on G GPUs (weak scaling): shard g
    = one per-GPU reference set of the workload (its own ~4 Gbp of the subset,
    or its 1/8 of the RefSeq- / AFS31-shaped DB), built into partition g; the
    read records are n_pairs in total, slice g drawn from shard g."""

    def __init__(self, name: str, G: int = 1):
        wl = WORKLOADS[name]
        self.name, self.G, self.wl = name, G, wl
        self.n_pairs, self.L = wl["n_pairs"], wl["read_len"]
        self.shards = [self._refs(g) for g in range(G)]
        slices = []
        for g in range(G):
            q, r = divmod(self.n_pairs, G)
            n_g = q + (1 if g < r else 0)
            slices.append(self._reads(self.shards[g], n_g, g))
        self.reads = slices[0] if G == 1 else concat_reads(slices)
        self.paired = self.reads.mates_buf is not None
        self.parent, self.rank = self.shards[0].parent, self.shards[0].rank
        self.total_bp = sum(r.total_bp for r in self.shards)

    def _refs(self, g):
        wl, G = self.wl, self.G
        if wl.get("refs") in ("refseq8", "afs31x8"):
            if G > 8:
                raise SystemExit(f"{self.name}: at most 8 GPUs (one 1/8 shard each)")
            return (synth.refseq_shard if wl["refs"] == "refseq8" else synth.afs31_shard)(g, 8)
        return synth.subset_shard(g, G, n_targets=wl["n_targets"], **wl["ref_kw"])

    def _reads(self, refs, n, g):
        wl = self.wl
        if wl.get("reads") in ("hiseq", "miseq"):
            return getattr(synth, wl["reads"] + "_reads")(refs, n, seed=synth.READ_SEED + 40 + g)
        if wl.get("reads") == "kal_stream":
            return synth.kal_stream(refs, n, length=self.L, seed=synth.READ_SEED + 60 + g)
        gen = {"afs": synth.afs_reads, "kal": synth.kal_reads}.get(wl.get("reads"))
        if gen:
            return gen(refs, n, length=self.L, seed=synth.READ_SEED + 20 + g)
        return synth.paired_reads(refs, n, length=self.L, seed=synth.READ_SEED + g)


def concat_reads(parts):
    def cat(bufs, offs):
        base = np.cumsum([0] + [int(o[-1]) for o in offs[:-1]]).astype(np.uint64)
        o = np.concatenate([offs[0][:1].astype(np.uint64)] + [o[1:].astype(np.uint64) + b for o, b in zip(offs, base)])
        return np.concatenate(bufs), o
    buf, off = cat([r.buf for r in parts], [r.offsets for r in parts])
    mb = mo = None
    if parts[0].mates_buf is not None:
        mb, mo = cat([r.mates_buf for r in parts], [r.mate_offsets for r in parts])
    return synth.Reads(buf, off, mb, mo)


def make_group_db(mc, W: Workload, devices, read_batch=READ_BATCH):
    """The G-GPU database bench.py times at N > 1: ONE handle, n_gpus = G,
    partition g (shard g's references) on devices[g]."""
    return mc.Database(W.parent, W.rank, n_partitions=W.G, n_gpus=W.G, devices=list(devices),
                       capacity_bp=int(max(r.total_bp for r in W.shards) * W.G * 1.01) + (1 << 20),
                       max_targets=sum(r.n for r in W.shards) + 64 * W.G,
                       read_batch=min(read_batch, W.n_pairs), max_candidates=BENCH_M)


class Inputs:
    """Device-resident copies (shard g's references on devices[g], the reads on
    devices[0]) and pinned host copies of a Workload, plus result buffers."""

    def __init__(self, torch, W: Workload, devices):
        pin = lambda a: torch.from_numpy(a).pin_memory()
        d0 = torch.device(f"cuda:{devices[0]}")
        self.W, self.devices = W, devices
        self.h_bufs = [pin(r.buf) for r in W.shards]
        self.d_bufs = [h.to(torch.device(f"cuda:{d}")) for h, d in zip(self.h_bufs, devices)]
        self.d_offs = [torch.from_numpy(r.offsets.astype(np.int64)).to(torch.device(f"cuda:{d}"))
                       for r, d in zip(W.shards, devices)]
        self.pids = [np.full(r.n, g, np.uint32) for g, r in enumerate(W.shards)]
        rd = W.reads
        self.h_r1, self.h_o1 = pin(rd.buf), pin(rd.offsets.astype(np.int64))
        self.h_r2 = pin(rd.mates_buf) if W.paired else None
        self.h_o2 = pin(rd.mate_offsets.astype(np.int64)) if W.paired else None
        cp = lambda t: t.to(d0) if t is not None else None
        self.d_r1, self.d_o1, self.d_r2, self.d_o2 = cp(self.h_r1), cp(self.h_o1), cp(self.h_r2), cp(self.h_o2)
        n, m = W.n_pairs, BENCH_M
        self.d_tax = torch.zeros(n, dtype=torch.int32, device=d0)
        self.d_cand = torch.zeros(n * m * 4, dtype=torch.int32, device=d0)
        self.h_tax = torch.zeros(n, dtype=torch.int32).pin_memory()
        self.h_cand = torch.zeros(n * m * 4, dtype=torch.int32).pin_memory()

    def build(self, db, device_resident: bool):
        """Clear + insert every shard (B1-B5) + finalize (B6)."""
        W = self.W
        db.clear()
        if W.G == 1:
            r = W.shards[0]
            if device_resident:
                db.insert_targets(self.d_bufs[0], self.d_offs[0], r.target_ids, r.taxa, self.pids[0])
            else:
                db.insert_targets(self.h_bufs[0], r.offsets, r.target_ids, r.taxa, self.pids[0])
        else:
            db.insert_target_batches([((self.d_bufs[g], self.d_offs[g]) if device_resident else
                                       (self.h_bufs[g], r.offsets)) + (r.target_ids, r.taxa, self.pids[g])
                                      for g, r in enumerate(W.shards)])
        db.finalize()

    def query(self, db, device_resident: bool):
        """Classify every read record (Q1-Q9); results on device 0 or in pinned host memory."""
        if device_resident:
            db.classify(self.d_r1, self.d_o1, self.d_r2, self.d_o2, out_taxon=self.d_tax, out_candidates=self.d_cand)
        else:
            db.classify(self.h_r1, self.h_o1, self.h_r2, self.h_o2, out_taxon=self.h_tax, out_candidates=self.h_cand)


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
    p.add_argument("--read-batch", type=int, default=None,
                   help=f"read records per internal query batch (default: the workload's, else {READ_BATCH})")
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
    wl = WORKLOADS[args.workload]
    if args.read_batch is None:
        args.read_batch = wl.get("read_batch", READ_BATCH)
    if args.impl == "reference":
        return run_reference(args, wl, world, rank)
    if world > 1 and rank != 0:
        # ONE host process drives every GPU of the node through one multi-GPU
        # handle (mc_config.n_gpus; the paper's MetaCache-GPU is one process with
        # per-GPU batch arenas): the launcher's other ranks idle
        return
    import torch
    G = max(1, args.gpus if world == 1 else max(args.gpus, world))
    ndev = torch.cuda.device_count()
    # MC_BENCH_REHEARSE=1: N shards on fewer GPUs (ordinals repeat) -- exercises the
    # N > 1 code path on the one-GPU box; never a reported number
    rehearse = os.environ.get("MC_BENCH_REHEARSE") == "1"
    if G > ndev and not rehearse:
        raise SystemExit(f"--gpus {G}: only {ndev} GPUs visible")
    devices = [g % ndev for g in range(G)]
    torch.cuda.set_device(devices[0])
    import paper_2106_08150_b200 as mc

    t0 = time.time()
    Wl = Workload(args.workload, G)
    n_pairs, L, paired, m = Wl.n_pairs, Wl.L, Wl.paired, BENCH_M
    log(f"workload: {G} x {Wl.shards[0].n} targets, {Wl.total_bp / 1e9:.3f} Gbp, {n_pairs} "
        f"{'pairs' if paired else 'reads'} ({time.time() - t0:.1f}s)")
    inp = Inputs(torch, Wl, devices)
    if G == 1:
        db = make_db(mc, Wl.shards[0], 1, 0, devices[0], n_pairs, args.read_batch)
        stream = torch.cuda.Stream(device=devices[0])
        torch.cuda.set_stream(stream)
        db.set_stream(stream)  # the library's work runs on the timed stream
        streams = [stream]
    else:
        db = make_group_db(mc, Wl, devices, args.read_batch)
        # calls are synchronous: events on each device's stream around a call
        # bound that device's part of it (max over devices = the step)
        streams = [torch.cuda.current_stream(torch.device(f"cuda:{d}")) for d in devices]

    def step(device_resident):
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in streams]
        for e, s in zip(ev, streams):
            e[0].record(s)
        inp.build(db, device_resident)
        for e, s in zip(ev, streams):
            e[1].record(s)
        inp.query(db, device_resident)
        for e, s in zip(ev, streams):
            e[2].record(s)
        return ev

    def timed(device_resident, K, W, sample_clocks):
        for _ in range(W):
            step(device_resident)
        torch.cuda.synchronize()
        db.reset_stats()
        evs = []
        with ClockSampler(devices[0]) if sample_clocks else _Null() as cs:
            for d in set(devices):
                torch.cuda.synchronize(d)
            for _ in range(K):
                evs.append(step(device_resident))
            for d in set(devices):
                torch.cuda.synchronize(d)
        # per device, then the max over devices
        tb = max(sum(e[g][0].elapsed_time(e[g][1]) for e in evs) for g in range(len(streams)))
        tq = max(sum(e[g][1].elapsed_time(e[g][2]) for e in evs) for g in range(len(streams)))
        return tb, tq, db.stats(), (cs.summary() if sample_clocks else None)

    K, W = args.steps, args.warmup
    if args.profile:
        args.no_e2e = args.no_cpu_baseline = True
    tb, tq, st, clocks = timed(True, K, W, not args.profile)
    total_bp = Wl.total_bp
    reads = (2 if paired else 1) * n_pairs  # each mate counts as a read (S22)
    build_gbps = total_bp * K / (tb / 1e3) / 1e9
    reads_per_s = reads * K / (tq / 1e3)
    launches = sum(st["launches"].values())

    e2e = None
    if not args.no_e2e:
        eb, eq, _, _ = timed(False, K, max(1, min(W, 2)), False)
        rd = Wl.reads
        h2d = sum(r.buf.nbytes + r.offsets.nbytes for r in Wl.shards) + rd.buf.nbytes + rd.offsets.nbytes + \
            ((rd.mates_buf.nbytes + rd.mate_offsets.nbytes) if paired else 0)
        d2h = inp.h_tax.numel() * 4 + inp.h_cand.numel() * 4
        e2e = {"value": round(total_bp * K / (eb / 1e3) / 1e9, 3), "unit": "Gbp/s", "ms_per_step": round((eb + eq) / K, 3),
               "build_ms_per_step": round(eb / K, 3), "query_ms_per_step": round(eq / K, 3),
               "query_reads_per_s": round(reads * K / (eq / 1e3), 1),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- roofline of the dominant kernel (CUDA events inside libmc.so) -------
    peak, peak_src = peaks()
    refs = Wl.shards[0]
    roof = kernel_rooflines(st, K, refs, db, n_pairs, L, m, G)
    clean = [r for r in roof.values() if not r.get("overlapped_streams")]
    dom = max(clean or roof.values(), key=lambda r: r["ms_per_step"]) if roof else None
    # (the committed ncu capture is of the default subset workload)
    traffic = ncu_traffic(dom["kernel"]) if dom and args.workload == "subset" and G == 1 else None
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

    path = path_roofline(st, K, tb, tq, refs, n_pairs, paired, peak, G)

    cpu = None
    if G == 1 and not args.no_cpu_baseline:
        sub, srd = oracle_sample(refs, L)
        bt, qt, qtn, nthr = run_oracle_step(sub, srd, threads=host_threads())
        cpu = {"value": round(sub.total_bp / bt / 1e9, 6), "unit": "Gbp/s", "cores": 1, "kind": "oracle",
               "sample": sample_desc(sub, srd), "query_reads_per_s": round(2 * srd.n / qt, 1),
               "build_s": round(bt, 3), "query_s": round(qt, 3),
               # the read-only query phase on every host core (SURVEY §8(d) oracle timing)
               "query_threads": {"cores": nthr, "reads_per_s": round(2 * srd.n / qtn, 1), "query_s": round(qtn, 3)},
               "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}

    line = {
        "metric": "DB build Gbp/s and classified reads/s at 1/2/4/8 B200 vs HBM roofline",
        "value": round(build_gbps, 3), "unit": "Gbp/s", "n_gpus": G, "steps": K, "warmup": W,
        "ms_per_step": round((tb + tq) / K, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/u32 (integer path)", "data": "synthetic (seeded; synth/)",
        "config": {"workload": wl["desc"], "targets_per_gpu": refs.n, "bp_per_gpu": refs.total_bp,
                   "read_pairs" if paired else "reads": n_pairs, "paired": paired,
                   "read_batch": min(args.read_batch, n_pairs), "read_len": L, "k": 16, "s": 16, "w": 127,
                   "cap": 254, "m": m, "partitions": G,
                   "parallelism": "single GPU" if G == 1 else
                   f"target-partitioned x{G}: one multi-GPU handle (NVLink peer all-gather + fused merge)",
                   "devices": devices, "rehearsal": rehearse and G > ndev,
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
    # per GPU: a multi-GPU handle's stats sum the build counters and launches over
    # its `world` devices, take stage times as the max over them, and count the
    # query (every device scores every record) once
    ms, la = st["stage_ms"], {k: v / world for k, v in st["launches"].items()}
    p = st["partitions"][0]
    nslots, keys, nvals = p["table_slots"], p["keys"], p["values"]
    bp, locs = st["bp"] / world, st["locations_inserted"] / world
    qfeat, qloc, read_bp, nrec = st["query_features"], st["query_locations"], st["read_bp"], st["reads"]
    # records and locations per query bin (small / medium / large); records of the
    # small bin also include those deferred out of it (their work is redone)
    nrec_all = nrec * max(1, db.n_local // world)
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
    # query batches on two compute streams: a query kernel's event time then
    # includes sharing the GPU with the other stream's kernels (not its own
    # duration); such kernels are flagged and never picked as the dominant one
    overlapped = st.get("query_overlapped_calls", 0) > 0
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
        d = {"kernel": "+".join(kerns), "ms_per_step": round(t / K, 4), "launches": round(n_l),
             "bytes_per_launch": int(nbytes / n_l), "gbs": round(nbytes / (t / 1e3) / 1e9, 2)}
        if rops and rc:
            d["random_ops_per_s"] = round(rops / (t / 1e3), 1)
            d["random_ops_frac_of_measured_ceiling"] = round(rops / (t / 1e3) / rc, 4)
            d["ceiling"] = "random 8-B reads over 4 GiB (tools/randbw.cu, r02a)"
        if stage in ("sketch_partition", "sketch_insert"):
            d["alu_ops_per_s"] = alu_ops / (t / 1e3)
        if overlapped and stage.startswith(("query_", "merge_")):
            d["overlapped_streams"] = True
        out[stage] = d
    return out


def path_roofline(st, K, tb, tq, refs, n_pairs, paired, peak, world):
    """Whole-path efficiency: the build's Gbp/s against the HBM
    time of its algorithmic bytes per reference bp, and the query's records/s
    against the random DRAM lines a record must touch, at the measured
    random-read rate.  Per GPU (every rank runs the same work)."""
    p = st["partitions"][0]
    bp = st["bp"] / K / world               # per step, per GPU (weak scaling: equal shards)
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
