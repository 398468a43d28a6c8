"""Host phases of one build (insert + finalize) in the bench's launch
configuration: MC_TRACE=1 makes libmc.so print each phase's host wall time.
usage: python tools/host_trace.py [workload (afs31x8)] [host]  (host: pinned host input, as bench's e2e)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2106_08150_b200 as mc
name = sys.argv[1] if len(sys.argv) > 1 else "afs31x8"
dev_res = not (len(sys.argv) > 2 and sys.argv[2] == "host")
W = bench.Workload(name, 1)
torch.cuda.set_device(0)
inp = bench.Inputs(torch, W, [0])
db = bench.make_db(mc, W.shards[0], 1, 0, 0, W.n_pairs)
for _ in range(2):
    inp.build(db, dev_res)
torch.cuda.synchronize()
os.environ["MC_TRACE"] = "1"   # (read per call by the library)
t0 = time.perf_counter()
inp.build(db, dev_res)
torch.cuda.synchronize()
print(f"{name} ({'device' if dev_res else 'pinned host'} input): build wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
st = db.stats()
print({k: round(v / 3, 3) for k, v in st["stage_ms"].items()}, file=sys.stderr)
