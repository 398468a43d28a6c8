"""GPU parity on the configs[3] recipe (-m gpu): a RefSeq-202-shaped target
shard (synth.refseq_shard: viral genomes, strain-structured bacteria with
plasmids, multi-chromosome fungi; target ids NOT in insertion order, so the
gapped -> ranked window conversion is exercised) built in the bench's launch
configuration, queried with strain-derived pairs and KAL_D-shaped pairs.
Checked against the feature-restricted oracle on
sampled pairs and sampled feature lists.  The shard is the one `bench.py
--workload refseq8` builds and times (scale 1.0: ~10 Gbp, ~6.3 k targets);
the restricted oracle sketches all of it on the host's threads."""
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
def refseq_run(oracle_mod):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    import paper_2106_08150_b200 as mc
    refs = synth.refseq_shard(0, 8)  # exactly the bench's shard 0
    assert not np.all(np.diff(refs.target_ids.astype(np.int64)) > 0)  # ids out of insertion order
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    sets = {"strains": synth.paired_reads(refs, 200_000, length=150, seed=synth.READ_SEED + 7),
            "kal": synth.kal_reads(refs, 200_000)}
    d_buf, d_offs = torch.from_numpy(refs.buf).to(dev), torch.from_numpy(refs.offsets.astype(np.int64)).to(dev)
    db = bench.make_db(mc, refs, 1, 0, 0, 200_000)
    db.insert_targets(d_buf, d_offs, refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
    db.finalize()
    out = {}
    for name, rd in sets.items():
        t, c = db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
        out[name] = (t, c.view(np.uint32).reshape(rd.n, -1))
    # configs[4] at its stated size, as `bench.py --workload kal50m` runs it: 50M KAL_D-shaped pairs
    # (100M reads) from pinned host memory through mc_classify in 4M-pair batches
    stream = synth.kal_stream(refs, 50_000_000, seed=synth.READ_SEED + 60)
    sdb = bench.make_db(mc, refs, 1, 0, 0, stream.n, read_batch=1 << 22)
    sdb.insert_targets(d_buf, d_offs, refs.target_ids, refs.taxa, np.zeros(refs.n, np.uint32))
    sdb.finalize()
    pin = lambda a: torch.from_numpy(a).pin_memory()
    h_in = [pin(stream.buf), pin(stream.offsets.astype(np.int64)), pin(stream.mates_buf),
            pin(stream.mate_offsets.astype(np.int64))]
    s_t = torch.zeros(stream.n, dtype=torch.int32).pin_memory()
    s_c = torch.zeros(stream.n * 16, dtype=torch.int32).pin_memory()
    t0 = time.time()
    sdb.classify(*h_in, out_taxon=s_t, out_candidates=s_c)
    print(f"kal50m stream: {stream.n} pairs classified in {time.time() - t0:.2f}s (host wall, pinned in/out)")
    out["stream"] = (s_t.numpy().view(np.uint32), s_c.numpy().view(np.uint32).reshape(stream.n, -1))
    sets["stream"] = stream
    sdb.close()
    del h_in
    # feature-restricted oracle over the whole shard, for the sampled pairs' features
    samples = {name: _sample(rd, 1000 if name == "stream" else 800, 31 + i) for i, (name, rd) in enumerate(sets.items())}
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
    print(f"refseq shard: {refs.n} targets, {refs.total_bp / 1e9:.2f} Gbp; restricted oracle {time.time() - t0:.1f}s")
    res = {}
    for name, (idx, r1, r2) in samples.items():
        s = synth.reads_from_list(r1, r2)
        ot, oc = o.classify(s.buf, s.offsets, s.mates_buf, s.mate_offsets)
        res[name] = (idx, ot, oc.view(np.uint32).reshape(len(idx), -1))
    yield dict(db=db, o=o, refs=refs, out=out, res=res, feats=np.array(sorted(feats), np.uint32))
    o.close()
    db.close()


@pytest.mark.parametrize("name,frac", [("strains", (0.6, 1.0)), ("kal", (0.0, 0.2)), ("stream", (0.0, 0.2))])
def test_refseq_shard_sampled_candidates_and_taxa(refseq_run, name, frac):
    t, c = refseq_run["out"][name]
    idx, ot, oc = refseq_run["res"][name]
    bad = np.nonzero((c[idx] != oc).any(1))[0]
    assert bad.size == 0, f"{bad.size}/{len(idx)} sampled pairs differ; first {idx[bad[:5]]}"
    assert np.array_equal(t[idx], ot)
    assert frac[0] <= (ot != 0).mean() <= frac[1]


def test_refseq_shard_sampled_feature_lists(refseq_run):
    db, o = refseq_run["db"], refseq_run["o"]
    fs = np.random.default_rng(11).choice(refseq_run["feats"], min(3000, refseq_run["feats"].size), replace=False)
    for f in fs:
        assert np.array_equal(db.feature_locations(0, int(f)), o.feature_locations(0, int(f))), hex(int(f))


def test_refseq_shard_invariants(refseq_run):
    st = refseq_run["db"].stats()["partitions"][0]
    refs = refseq_run["refs"]
    n = np.maximum(np.diff(refs.offsets).astype(np.int64) - 15, 0)
    assert st["windows"] == int(((n + 111) // 112).sum())
    assert st["values"] == st["locations"] - st["truncated"]
