"""Time-to-query (the paper's Table 5 / Fig. 4:
on-the-fly build vs database write + load): build the bench workload's
database on one GPU from pinned host memory (the OTF path), save it with
mc_db_save, load it into a fresh handle with mc_db_load, and check the loaded
handle classifies the read batch identically.  Prints one JSON line.
usage: python tools/time_to_query.py [WORKLOAD] [PATH]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2106_08150_b200 as mc  # noqa: E402
import synth  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "subset"
path = sys.argv[2] if len(sys.argv) > 2 else "/tmp/mc_time_to_query.mcdb"
wl = bench.WORKLOADS[wl_name]
refs = synth.subset_shard(0, 1, n_targets=wl["n_targets"], **wl["ref_kw"])
rd = synth.paired_reads(refs, wl["n_pairs"], length=wl["read_len"])
torch.cuda.set_device(0)
h_buf = torch.from_numpy(refs.buf).pin_memory()
db = bench.make_db(mc, refs, 1, 0, 0, wl["n_pairs"])
pids = np.zeros(refs.n, np.uint32)


def sync_time(f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    f()
    torch.cuda.synchronize()
    return time.perf_counter() - t


def build():
    db.clear()
    db.insert_targets(h_buf, refs.offsets, refs.target_ids, refs.taxa, pids)
    db.finalize()


build()  # warm-up
t_build = min(sync_time(build) for _ in range(3))
t_save = sync_time(lambda: db.save(path))
size = os.path.getsize(path)
db2 = [None]
t_load = sync_time(lambda: db2.__setitem__(0, mc.Database.load(path)))
t1, c1 = db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
t2, c2 = db2[0].classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
same = bool(np.array_equal(t1, t2) and np.array_equal(c1.view(np.uint32), c2.view(np.uint32)))
os.remove(path)
print(json.dumps({"what": "time to query: OTF build from pinned host memory vs mc_db_save + mc_db_load",
                  "workload": wl["desc"], "bp": refs.total_bp, "build_s": round(t_build, 4),
                  "save_s": round(t_save, 3), "load_s": round(t_load, 3), "file_bytes": size,
                  "file_gbs_write": round(size / t_save / 1e9, 2), "file_gbs_read": round(size / t_load / 1e9, 2),
                  "loaded_handle_identical": same}))
assert same
