"""Where the e2e (pinned host input) classification time goes: per-stage
device times (library CUDA events) vs the event-timed call, subset workload."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, synth, paper_2106_08150_b200 as mc
wl = bench.WORKLOADS["subset"]
refs = synth.subset_shard(0, 1, n_targets=wl["n_targets"])
rd = synth.paired_reads(refs, wl["n_pairs"], length=150)
torch.cuda.set_device(0)
db = bench.make_db(mc, refs, 1, 0, 0, wl["n_pairs"], read_batch=int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18)
db.insert_targets(torch.from_numpy(refs.buf).cuda(), torch.from_numpy(refs.offsets.astype(np.int64)).cuda(),
                  refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
db.finalize()
pin = lambda a: torch.from_numpy(a).pin_memory()
r1, r2 = pin(rd.buf), pin(rd.mates_buf)
o1, o2 = pin(rd.offsets.astype(np.int64)), pin(rd.mate_offsets.astype(np.int64))
tax = torch.zeros(rd.n, dtype=torch.int32).pin_memory()
cand = torch.zeros(rd.n * 16, dtype=torch.int32).pin_memory()
for _ in range(2):
    db.classify(r1, o1, r2, o2, out_taxon=tax, out_candidates=cand)
torch.cuda.synchronize()
db.reset_stats()
t0 = time.perf_counter()
K = 5
for _ in range(K):
    db.classify(r1, o1, r2, o2, out_taxon=tax, out_candidates=cand)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
st = db.stats()
print(json.dumps({"wall_ms_per_call": round(wall, 3),
                  "stage_ms_per_call": {k: round(v / K, 3) for k, v in sorted(st["stage_ms"].items(), key=lambda t: -t[1])},
                  "launches_per_call": {k: v // K for k, v in st["launches"].items()}}))
