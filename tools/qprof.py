"""Small-bin work counters (diagnostic build ab/qprof.so, -DMC_QPROF=1):
per-record locations, distinct blocks, gather iterations, claim-loop
iterations, Q7 blocks.  Usage (GPU): MC_LIB_PATH=$PWD/ab/qprof.so python tools/qprof.py [workload]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2106_08150_b200 as mc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "subset"
W = bench.Workload(name, 1)
refs, rd = W.shards[0], W.reads
db = bench.make_db(mc, refs, 1, 0, 0, W.n_pairs, read_batch=W.wl.get("read_batch", bench.READ_BATCH))
db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
db.finalize()
lib = ctypes.CDLL(os.environ["MC_LIB_PATH"])
buf = (ctypes.c_ulonglong * 16)()
lib.mc_debug_qprof(buf, 1)
db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
lib.mc_debug_qprof(buf, 0)
c = list(buf)
n = max(c[0], 1)
names = ["records (small bin, all attempts)", "L locations", "uniq blocks", "HS slots", "gather iters (warp max)",
         "gather iters (lane sum)", "misses (lane sum)", "claim-loop iters (warp)", "binsert bucket steps (lane sum)",
         "CAS lost (lane sum)", "F lists", "deferred", "Q7 occupied blocks", "block_best evaluated",
         "toplist inserts", "Q7 iters (warp max)"]
print(f"workload {name}: {rd.n} records")
for i, nm in enumerate(names):
    print(f"{nm:36s} total {c[i]:>14d}  per record {c[i] / n:10.2f}")
print(f"miss rate {c[6] / max(c[1], 1):.3f}; claim-loop iters per gather iter {c[7] / max(c[4], 1):.2f}; "
      f"bucket steps per miss {c[8] / max(c[6], 1):.2f}")
db.close()
