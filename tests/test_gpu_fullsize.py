"""Full-size GPU parity (-m gpu): BASELINE.json configs[1] "bacterial subset"
(1,000 synthetic genomes, ~4.13 Gbp, 1M read pairs 2 x 150 bp) built and
classified in exactly the launch configuration bench.py times
(bench.make_db, device-resident inputs, clear + rebuild on one handle);
against the same database, configs[2] "AFS20-shaped" (10M pairs 2 x 101 bp
from 20 species, log-normal abundances) and a KAL_D-shaped stream (configs[4]
read mix: 95 % from absent genomes, 2 x 101 bp; 4M pairs in 1M-pair batches,
scaled down from 100M+ reads against the 8-GPU RefSeq-shaped database).

The full std::map oracle does not fit at this size, so parity is checked on
sampled outputs with the feature-restricted oracle:
the oracle sketches a seeded sample of read pairs, keeps only the locations
of their features while sketching every reference window (host threads over
independent targets), applies the cap and classifies the sampled pairs.  A
pair's result depends only on its own features' lists, so the sampled
candidates and taxa must match bit-exactly; so must the location lists of
sampled features.  Whole-database properties that hold at any size are
checked on the GPU statistics.
"""
import os
import time

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

N_SAMPLE = int(os.environ.get("MC_FULLSIZE_SAMPLE", "1500"))
N_AFS = int(os.environ.get("MC_FULLSIZE_AFS_PAIRS", "10000000"))
N_KAL = int(os.environ.get("MC_FULLSIZE_KAL_PAIRS", "4000000"))
# HiSeq / MiSeq-shaped single-end variable-length reads (Table 2)
N_SE = int(os.environ.get("MC_FULLSIZE_SE_READS", "2000000"))


@pytest.fixture(scope="module")
def fullsize():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    import paper_2106_08150_b200 as mc
    wl = bench.WORKLOADS["subset"]
    refs = synth.subset_shard(0, 1, n_targets=wl["n_targets"], **wl["ref_kw"])
    n_pairs, L = wl["n_pairs"], wl["read_len"]
    rd = synth.paired_reads(refs, n_pairs, length=L, seed=synth.READ_SEED)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    db = bench.make_db(mc, refs, 1, 0, 0, n_pairs)
    stream = torch.cuda.Stream(device=dev)
    db.set_stream(stream)
    d_buf = torch.from_numpy(refs.buf).to(dev)
    d_offs = torch.from_numpy(refs.offsets.astype(np.int64)).to(dev)
    d_r1 = torch.from_numpy(rd.buf.reshape(-1, L)).to(dev)
    d_r2 = torch.from_numpy(rd.mates_buf.reshape(-1, L)).to(dev)
    d_ro = torch.from_numpy((np.arange(n_pairs + 1, dtype=np.int64) * L)).to(dev)
    pids = np.zeros(refs.n, np.uint32)
    outs = []
    for _ in range(2):  # build, classify; then clear + rebuild + classify (the bench step)
        d_tax = torch.zeros(n_pairs, dtype=torch.int32, device=dev)
        d_cand = torch.zeros(n_pairs * bench.BENCH_M * 4, dtype=torch.int32, device=dev)
        db.clear()
        db.insert_targets(d_buf, d_offs, refs.target_ids, refs.taxa, pids)
        db.finalize()
        db.classify(d_r1, d_ro, d_r2, d_ro, out_taxon=d_tax, out_candidates=d_cand)
        torch.cuda.synchronize()
        outs.append((d_tax.cpu().numpy().view(np.uint32), d_cand.cpu().numpy().view(np.uint32).reshape(n_pairs, -1)))
    stats = db.stats()
    extra = {}
    for name, gen, n in (("afs", synth.afs_reads, N_AFS), ("kal", synth.kal_reads, N_KAL)):
        r = gen(refs, n)
        Lr = int(r.offsets[1] - r.offsets[0])
        d1 = torch.from_numpy(r.buf).to(dev)
        d2 = torch.from_numpy(r.mates_buf).to(dev)
        do = torch.from_numpy(r.offsets.astype(np.int64)).to(dev)
        t = torch.zeros(n, dtype=torch.int32, device=dev)
        c = torch.zeros(n * bench.BENCH_M * 4, dtype=torch.int32, device=dev)
        db.classify(d1, do, d2, do, out_taxon=t, out_candidates=c)
        torch.cuda.synchronize()
        extra[name] = dict(rd=r, L=Lr, taxon=t.cpu().numpy().view(np.uint32),
                           cand=c.cpu().numpy().view(np.uint32).reshape(n, -1))
        del d1, d2, do, t, c
    for name, gen in (("hiseq", synth.hiseq_reads), ("miseq", synth.miseq_reads)):
        r = gen(refs, N_SE)
        d1 = torch.from_numpy(r.buf).to(dev)
        do = torch.from_numpy(r.offsets.astype(np.int64)).to(dev)
        t = torch.zeros(N_SE, dtype=torch.int32, device=dev)
        c = torch.zeros(N_SE * bench.BENCH_M * 4, dtype=torch.int32, device=dev)
        db.classify(d1, do, None, None, out_taxon=t, out_candidates=c)
        torch.cuda.synchronize()
        extra[name] = dict(rd=r, L=None, taxon=t.cpu().numpy().view(np.uint32),
                           cand=c.cpu().numpy().view(np.uint32).reshape(N_SE, -1))
        del d1, do, t, c
    yield dict(mc=mc, db=db, refs=refs, rd=rd, L=L, outs=outs, stats=stats, extra=extra)
    db.close()


def _sample_pairs(rd, L, n, seed):
    """Sampled records as byte strings (mates None for single-end; any lengths)."""
    idx = np.sort(np.random.default_rng(seed).choice(rd.n, min(n, rd.n), replace=False))
    cut = lambda buf, o: [buf[int(o[i]):int(o[i + 1])].tobytes() for i in idx]
    r2 = cut(rd.mates_buf, rd.mate_offsets) if rd.mates_buf is not None else None
    return idx, cut(rd.buf, rd.offsets), r2


@pytest.fixture(scope="module")
def restricted(fullsize, oracle_mod):
    refs = fullsize["refs"]
    sets = {"subset": (fullsize["rd"], fullsize["L"], N_SAMPLE, 20210615)}
    for name, e in fullsize["extra"].items():
        sets[name] = (e["rd"], e["L"], 1000, 20210616 + len(sets))
    samples = {name: _sample_pairs(r, L, n, seed) for name, (r, L, n, seed) in sets.items()}
    feats = set()
    for _, r1, r2 in samples.values():
        for a in list(r1) + list(r2 or []):
            for sk in oracle_mod.sketch(bytes(a)):
                feats.update(int(x) for x in sk)
    o = oracle_mod.OracleDB(refs.parent, m=4)
    o.set_feature_filter(np.array(sorted(feats), np.uint32))
    t0 = time.time()
    o.insert_restricted(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    o.finalize()
    print(f"restricted oracle build: {len(feats)} features, {time.time() - t0:.1f}s")
    res = {}
    for name, (idx, r1, r2) in samples.items():
        sample = synth.reads_from_list(r1, r2)
        ot, oc = o.classify(sample.buf, sample.offsets, sample.mates_buf, sample.mate_offsets)
        res[name] = dict(idx=idx, taxon=ot, cand=oc)
    yield dict(o=o, feats=np.array(sorted(feats), np.uint32), res=res)
    o.close()


def _check_sample(t, c, r, min_classified):
    idx = r["idx"]
    oc = r["cand"].view(np.uint32).reshape(len(idx), -1)
    bad = np.nonzero((c[idx] != oc).any(1))[0]
    assert bad.size == 0, f"{bad.size}/{len(idx)} sampled pairs differ; first {idx[bad[:5]]}"
    assert np.array_equal(t[idx], r["taxon"])
    frac = (r["taxon"] != 0).mean()
    assert frac >= min_classified[0] and frac <= min_classified[1], frac


def test_fullsize_rebuild_is_deterministic(fullsize):
    (t0, c0), (t1, c1) = fullsize["outs"]
    assert np.array_equal(t0, t1)
    assert np.array_equal(c0, c1)


def test_fullsize_sampled_candidates_and_taxa(fullsize, restricted):
    t, c = fullsize["outs"][1]
    _check_sample(t, c, restricted["res"]["subset"], (0.5, 1.0))  # the sample exercises classification


def test_afs20_shaped_sampled_candidates_and_taxa(fullsize, restricted):
    e = fullsize["extra"]["afs"]
    _check_sample(e["taxon"], e["cand"], restricted["res"]["afs"], (0.5, 1.0))


def test_kal_shaped_stream_sampled_candidates_and_taxa(fullsize, restricted):
    """95 % of the pairs come from absent genomes: most stay unclassified."""
    e = fullsize["extra"]["kal"]
    _check_sample(e["taxon"], e["cand"], restricted["res"]["kal"], (0.0, 0.2))


@pytest.mark.parametrize("name", ["hiseq", "miseq"])
def test_variable_length_single_end_sampled_candidates_and_taxa(fullsize, restricted, name):
    """HiSeq-shaped (19-101 bp) and MiSeq-shaped (19-251 bp: 1-3 windows per
    read, sws 2-4) single-end reads cut from the database genomes."""
    e = fullsize["extra"][name]
    _check_sample(e["taxon"], e["cand"], restricted["res"][name], (0.5, 1.0))


def test_fullsize_sampled_feature_lists(fullsize, restricted):
    db, o = fullsize["db"], restricted["o"]
    rng = np.random.default_rng(7)
    fs = rng.choice(restricted["feats"], min(5000, restricted["feats"].size), replace=False)
    n_long = 0
    for f in fs:
        g = db.feature_locations(0, int(f))
        e = o.feature_locations(0, int(f))
        assert np.array_equal(g, e), f"feature {int(f):#x}: {g.size} vs {e.size} locations"
        n_long += e.size == 254
    print(f"{fs.size} sampled feature lists equal ({n_long} at the cap)")


def test_fullsize_database_invariants(fullsize):
    st = fullsize["stats"]
    part = st["partitions"][0]
    refs = fullsize["refs"]
    assert part["targets"] == refs.n
    assert part["bp"] == refs.total_bp
    # every window of every target (closed form, S5) is inserted once
    lens = np.diff(refs.offsets).astype(np.int64)
    n = np.maximum(lens - 15, 0)
    assert part["windows"] == int(((n + 111) // 112).sum())
    # stored values = inserted locations minus those cut by the cap (S7)
    assert part["values"] == part["locations"] - part["truncated"]
    assert part["keys"] <= part["locations"] <= 16 * part["windows"]
    assert part["table_slots"] >= part["keys"]
