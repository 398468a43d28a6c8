"""A/B timing of the insert (sketch + partition) kernel alone on the bench
subset: python tools/exp_insert.py [LIB.so ...] -> ms per insert per library."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2:  # one process per library (the binding loads one .so per process)
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib], env=dict(os.environ, MC_LIB_PATH=lib))
    sys.exit(0)
if len(sys.argv) == 2:
    os.environ["MC_LIB_PATH"] = sys.argv[1]
import numpy as np
import torch
import synth
import paper_2106_08150_b200 as mc

refs = synth.subset_shard(0, 1, n_targets=1000)
d = torch.from_numpy(refs.buf).cuda()
o = torch.from_numpy(refs.offsets.astype(np.int64)).cuda()
db = mc.Database(refs.parent, refs.rank, capacity_bp=int(refs.total_bp * 1.01) + (1 << 20), max_targets=refs.n + 64)
pids = np.zeros(refs.n, np.uint32)
for it in range(4):
    db.clear()
    if it == 1:
        db.reset_stats()
    db.insert_targets(d, o, refs.target_ids, refs.taxa, pids)
    torch.cuda.synchronize()
st = db.stats()
print(os.environ.get("MC_LIB_PATH", "default"), "sketch_partition ms/insert:",
      round(st["stage_ms"]["sketch_partition"] / 3, 3))
