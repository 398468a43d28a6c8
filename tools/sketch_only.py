import sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch, synth
import paper_2106_08150_b200 as mc
refs = synth.subset_shard(0, 1, n_targets=1000)
d = torch.from_numpy(refs.buf).cuda()
o = torch.from_numpy(refs.offsets.astype(np.int64)).cuda()
for _ in range(2):
    mc.debug_sketch(d, o)
print("done", refs.total_bp)
