"""Timeline of one e2e (pinned host input) classification on the subset
workload: MC_TRACE=1 makes libmc.so print per-batch event times (stderr)."""
import os, sys, time
os.environ["MC_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, synth, paper_2106_08150_b200 as mc
wl = bench.WORKLOADS["subset"]
refs = synth.subset_shard(0, 1, n_targets=wl["n_targets"])
rd = synth.paired_reads(refs, wl["n_pairs"], length=150)
torch.cuda.set_device(0)
for rb in [int(x) for x in (sys.argv[1:] or [str(1 << 18)])]:
    db = bench.make_db(mc, refs, 1, 0, 0, wl["n_pairs"], read_batch=rb)
    db.insert_targets(torch.from_numpy(refs.buf).cuda(), torch.from_numpy(refs.offsets.astype(np.int64)).cuda(),
                      refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
    db.finalize()
    pin = lambda a: torch.from_numpy(a).pin_memory()
    r1, r2 = pin(rd.buf), pin(rd.mates_buf)
    o1, o2 = pin(rd.offsets.astype(np.int64)), pin(rd.mate_offsets.astype(np.int64))
    tax = torch.zeros(rd.n, dtype=torch.int32).pin_memory()
    cand = torch.zeros(rd.n * 16, dtype=torch.int32).pin_memory()
    for _ in range(3):
        db.classify(r1, o1, r2, o2, out_taxon=tax, out_candidates=cand)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    db.classify(r1, o1, r2, o2, out_taxon=tax, out_candidates=cand)
    print(f"read_batch {rb}: wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
    db.close()
