"""GPU parity on the AFS31-shaped recipe (-m gpu; SURVEY.md §8(f) NEXT rank 4,
Table 1): a species shard of synth.afs31_shard -- long
chromosomes plus a scaffold-level genome of thousands of short targets, all
sequences of a genome under one taxon, N runs -- built in the bench's launch
configuration and queried with genome-derived pairs and KAL_D-shaped pairs.
Checked against the feature-restricted oracle on
sampled pairs and sampled feature lists.  The shard is the one `bench.py
--workload afs31x8` builds and times (scale 1.0: 9.55 Gbp, 239 k targets, an
845 Mbp chromosome); the restricted oracle sketches all of it on the host's threads."""
import time

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _sample(rd, n, seed):
    idx = np.sort(np.random.default_rng(seed).choice(rd.n, min(n, rd.n), replace=False))
    cut = lambda buf, o: [buf[int(o[i]):int(o[i + 1])].tobytes() for i in idx]
    return idx, cut(rd.buf, rd.offsets), cut(rd.mates_buf, rd.mate_offsets)


@pytest.fixture(scope="module")
def afs31_run(oracle_mod):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    import paper_2106_08150_b200 as mc
    refs = synth.afs31_shard(0, 8)  # exactly the bench's shard 0
    assert refs.n > 1000  # scaffold-level genome present
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    sets = {"genomes": synth.paired_reads(refs, 200_000, length=150, seed=synth.READ_SEED + 9),
            "kal": synth.kal_reads(refs, 200_000)}
    db = bench.make_db(mc, refs, 1, 0, 0, 200_000)
    db.insert_targets(torch.from_numpy(refs.buf).to(dev), torch.from_numpy(refs.offsets.astype(np.int64)).to(dev),
                      refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
    db.finalize()
    out = {}
    for name, rd in sets.items():
        t, c = db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
        out[name] = (t, c.view(np.uint32).reshape(rd.n, -1))
    samples = {name: _sample(rd, 800, 41 + i) for i, (name, rd) in enumerate(sets.items())}
    feats = set()
    for _, r1, r2 in samples.values():
        for a in r1 + r2:
            for sk in oracle_mod.sketch(a):
                feats.update(int(x) for x in sk)
    o = oracle_mod.OracleDB(refs.parent, m=4)
    o.set_feature_filter(np.array(sorted(feats), np.uint32))
    t0 = time.time()
    o.insert_restricted(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    o.finalize()
    print(f"afs31 shard: {refs.n} targets, {refs.total_bp / 1e9:.2f} Gbp; restricted oracle {time.time() - t0:.1f}s")
    res = {}
    for name, (idx, r1, r2) in samples.items():
        s = synth.reads_from_list(r1, r2)
        ot, oc = o.classify(s.buf, s.offsets, s.mates_buf, s.mate_offsets)
        res[name] = (idx, ot, oc.view(np.uint32).reshape(len(idx), -1))
    yield dict(db=db, o=o, refs=refs, out=out, res=res, feats=np.array(sorted(feats), np.uint32))
    o.close()
    db.close()


@pytest.mark.parametrize("name,frac", [("genomes", (0.6, 1.0)), ("kal", (0.0, 0.2))])
def test_afs31_shard_sampled_candidates_and_taxa(afs31_run, name, frac):
    t, c = afs31_run["out"][name]
    idx, ot, oc = afs31_run["res"][name]
    bad = np.nonzero((c[idx] != oc).any(1))[0]
    assert bad.size == 0, f"{bad.size}/{len(idx)} sampled pairs differ; first {idx[bad[:5]]}"
    assert np.array_equal(t[idx], ot)
    assert frac[0] <= (ot != 0).mean() <= frac[1]


def test_afs31_shard_sampled_feature_lists(afs31_run):
    db, o = afs31_run["db"], afs31_run["o"]
    fs = np.random.default_rng(13).choice(afs31_run["feats"], min(3000, afs31_run["feats"].size), replace=False)
    for f in fs:
        assert np.array_equal(db.feature_locations(0, int(f)), o.feature_locations(0, int(f))), hex(int(f))


def test_afs31_shard_invariants(afs31_run):
    st = afs31_run["db"].stats()["partitions"][0]
    refs = afs31_run["refs"]
    n = np.maximum(np.diff(refs.offsets).astype(np.int64) - 15, 0)
    assert st["windows"] == int(((n + 111) // 112).sum())
    assert st["values"] == st["locations"] - st["truncated"]
