import os, sys
os.environ["MC_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, paper_2106_08150_b200 as mc
refs = synth.tiny_references(n_genomes=2, length=30000)
rd = synth.single_end_reads(refs, 3000, length=100)
db = mc.Database(refs.parent, capacity_bp=1 << 20, read_batch=1000)
db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
db.finalize()
t, c = db.classify(rd.buf, rd.offsets)
print("ok", (t != 0).mean())
