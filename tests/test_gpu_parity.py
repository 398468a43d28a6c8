"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element, bit-exact (the path is integer throughout; north_star).

Run on the B200 box: python -m pytest tests -m gpu
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2106_08150_b200 import _build
    _build.build()
    import paper_2106_08150_b200 as m
    return m


def build_pair(mc, oracle_mod, refs, P=1, cap=254, m=4, partition_ids=None, **cfg):
    cap_bp = max(1 << 16, 2 * refs.total_bp)
    db = mc.Database(refs.parent, n_partitions=P, max_locations_per_feature=cap, max_candidates=m,
                     capacity_bp=cap_bp, **cfg)
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa, partition_ids)
    db.finalize()
    o = oracle_mod.OracleDB(refs.parent, k=cfg.get("k", 16), s=cfg.get("sketch_size", 16),
                            w=cfg.get("window_len", 127), cap=cap, m=m, n_partitions=P,
                            insert_size_max=cfg.get("insert_size_max", 0))
    o.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa, partition_ids)
    o.finalize()
    return db, o


def assert_db_equal(db, o, P):
    for p in range(P):
        gk, gc, gv = db.dump_partition(p)
        ok, oc, ov = o.dump_partition(p)
        assert np.array_equal(gk, ok), f"partition {p}: keys differ"
        assert np.array_equal(gc, oc), f"partition {p}: counts differ"
        assert np.array_equal(gv, ov), f"partition {p}: locations differ"


def assert_classify_equal(db, o, reads):
    t, c = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    ot, oc = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    bad = np.nonzero((c.view(np.uint32).reshape(len(t), -1) != oc.view(np.uint32).reshape(len(t), -1)).any(1))[0]
    assert bad.size == 0, f"{bad.size} records differ, first {bad[:5]}: gpu {c[bad[0]]} oracle {oc[bad[0]]}"
    assert np.array_equal(t, ot), "taxa differ"
    return t, c


# ---------------------------------------------------------------------------
# B1-B4: sketches (encode, windows, canonical k-mers, h1, s smallest unique)
# ---------------------------------------------------------------------------
def adversarial_seqs(rng):
    seqs = [b"", b"A", b"ACGT" * 3, b"A" * 15, b"A" * 16, b"C" * 127, b"AC" * 64, b"ACGTACGT" * 40,
            b"N" * 300, b"acgtNNNNacgt" * 30]
    for L in (16, 17, 126, 127, 128, 129, 239, 240, 241, 251, 1000, 5003):
        s = bytearray(synth.random_bases(rng, L).tobytes())
        seqs.append(bytes(s))
        t = bytearray(s)
        for p in rng.integers(0, L, size=max(1, L // 50)):
            t[p] = int(rng.choice(list(b"NRYKMnx-")))
        seqs.append(bytes(t))
        seqs.append(bytes(s).lower())
    pal = synth.random_bases(rng, 64)
    seqs.append((pal.tobytes() + synth.revcomp(pal).tobytes()) * 3)  # reverse-complement palindromes
    seqs.append((b"N" * 111 + synth.random_bases(rng, 40).tobytes()) * 3)  # N runs at window edges
    return seqs


@pytest.mark.parametrize("k,w,s", [(16, 127, 16), (12, 60, 8), (5, 8, 4), (16, 16, 16), (3, 130, 16), (1, 100, 3)])
def test_sketch_parity(mc, oracle_mod, k, w, s):
    rng = np.random.default_rng(k * 1000 + w)
    seqs = adversarial_seqs(rng)
    buf, offs = oracle_mod.pack_seqs(seqs)
    feats, counts, wo = mc.debug_sketch(buf, offs, k=k, window_len=w, sketch_size=s)
    for i, q in enumerate(seqs):
        exp = oracle_mod.sketch(q, k=k, s=s, w=w)
        got = [feats[j, :counts[j]].tolist() for j in range(int(wo[i]), int(wo[i + 1]))]
        assert got == exp, f"seq {i} (len {len(q)})"


def test_sketch_parity_device_input_and_alignment(mc, oracle_mod):
    rng = np.random.default_rng(3)
    seqs = [synth.random_bases(rng, int(L)).tobytes() for L in rng.integers(16, 3000, 60)]
    buf, offs = oracle_mod.pack_seqs(seqs)
    for shift in range(4):  # device buffers at every byte alignment
        dbuf = torch.zeros(len(buf) + 8, dtype=torch.uint8, device="cuda")
        dbuf[shift:shift + len(buf)] = torch.from_numpy(buf).cuda()
        view = dbuf[shift:shift + len(buf)]
        feats, counts, wo = mc.debug_sketch(view, torch.from_numpy(offs.astype(np.int64)).cuda())
        for i, q in enumerate(seqs):
            exp = oracle_mod.sketch(q)
            got = [feats[j, :counts[j]].tolist() for j in range(int(wo[i]), int(wo[i + 1]))]
            assert got == exp


# ---------------------------------------------------------------------------
# B5-B6: table + cap + condensed layout
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P", [1, 2, 4])
def test_db_parity_tiny(mc, oracle_mod, P):
    refs = synth.tiny_references()
    db, o = build_pair(mc, oracle_mod, refs, P=P)
    assert_db_equal(db, o, P)
    for t in refs.target_ids[:8]:
        assert db.partition_of(int(t)) == int(oracle_mod.plan_partitions(P, np.diff(refs.offsets))[t])
    st = db.stats()
    assert st["windows"] == refs.n * 1786
    db.close()


@pytest.mark.parametrize("cap", [1, 3, 254])
def test_db_parity_strains_and_cap(mc, oracle_mod, cap):
    refs = synth.strain_references(seed=11, n_targets=40, median_len=30_000, min_len=5_000, max_len=80_000,
                                   max_strains=20, id_stride=3, id_offset=7)
    db, o = build_pair(mc, oracle_mod, refs, P=2, cap=cap)
    assert_db_equal(db, o, 2)
    db.close()


def test_heavy_keys_cap_254(mc, oracle_mod):
    """300 near-identical strains: features with > 254 locations (heavy
    finalize path) keep the 254 smallest (target, window)."""
    rng = np.random.default_rng(5)
    base = synth.random_bases(rng, 3000)
    seqs = [synth.mutate(rng, base, 0.002).tobytes() for _ in range(300)]
    ids = rng.permutation(300).astype(np.uint32) * 5 + 1
    refs = synth.references_from_list(seqs, [2] * 300, [0, 1, 1], ids=ids)
    db, o = build_pair(mc, oracle_mod, refs)
    assert_db_equal(db, o, 1)
    st = db.stats()["partitions"][0]
    assert st["truncated"] > 0
    db.close()


def test_feature_zero_first_in_table(mc, oracle_mod):
    """Poly-A: canonical k-mer 0, feature h1(0) = 0 -- key 0, home slot 0, bucket
    offset 0 (an all-zero shared-memory entry must still read as occupied)."""
    refs = synth.references_from_list([b"A" * 600, b"T" * 300], [2, 2], [0, 1, 1])
    db, o = build_pair(mc, oracle_mod, refs)
    assert 0 in o.dump_partition(0)[0].tolist()
    assert_db_equal(db, o, 1)


def test_low_complexity_repeats_aggregated_insert(mc, oracle_mod):
    """Homopolymers / dinucleotide repeats: every window of a target holds the
    same few features, so one warp inserts equal keys (warp-aggregated path)."""
    seqs = [b"A" * 5000, b"AC" * 3000, b"ACG" * 2000, b"AAAAC" * 1000, b"ACGTTGCA" * 800]
    refs = synth.references_from_list(seqs, [2] * 5, [0, 1, 1])
    db, o = build_pair(mc, oracle_mod, refs, cap=1023)
    assert_db_equal(db, o, 1)
    db.close()


# ---------------------------------------------------------------------------
# Q1-Q9: classification
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P", [1, 2])
def test_classify_parity_tiny_config(mc, oracle_mod, P):
    """configs[0]: 8 x 200 kbp, 10k single-end 100 bp reads."""
    refs = synth.tiny_references()
    reads = synth.single_end_reads(refs, 10_000, length=100)
    db, o = build_pair(mc, oracle_mod, refs, P=P)
    t, c = assert_classify_equal(db, o, reads)
    src = reads.source_target
    ok = (src >= 0) & (t != 0)
    assert (t[ok] == refs.taxa[src[ok]]).mean() > 0.99
    db.close()


@pytest.mark.parametrize("P,m", [(1, 4), (3, 2), (4, 4), (2, 8), (1, 1), (1, 6), (8, 4), (8, 8)])
def test_classify_parity_paired_strains(mc, oracle_mod, P, m):
    refs = synth.strain_references(seed=21, n_targets=30, median_len=60_000, min_len=10_000, max_len=150_000,
                                   max_strains=12, id_stride=11)
    reads = synth.paired_reads(refs, 3000, length=150, random_frac=0.05, n_rate=0.001)
    db, o = build_pair(mc, oracle_mod, refs, P=P, m=m)
    assert_classify_equal(db, o, reads)
    db.close()


@pytest.mark.parametrize("k,w,s", [(12, 63, 8), (14, 113, 12), (16, 31, 4), (10, 41, 16), (15, 101, 10), (16, 143, 16)])
def test_classify_parity_non_default_sketch_params(mc, oracle_mod, k, w, s):
    """Whole path (build, cap, query bins, range scan, classification) with
    k / window / sketch sizes other than the paper's defaults (strides 52, 100, 87, 128,
    16, 32: up to 10 windows per 150 bp mate, sws up to 20)."""
    refs = synth.strain_references(seed=31, n_targets=16, median_len=40_000, min_len=10_000, max_len=80_000,
                                   max_strains=6, id_stride=5)
    reads = synth.paired_reads(refs, 1500, length=150, random_frac=0.05, n_rate=0.001)
    db, o = build_pair(mc, oracle_mod, refs, P=2, k=k, window_len=w, sketch_size=s)
    assert_db_equal(db, o, 2)
    assert_classify_equal(db, o, reads)
    db.close()


@pytest.mark.parametrize("ism", [400, 560, 900, 5000])
def test_classify_parity_insert_size_max(mc, oracle_mod, ism):
    """Reading S25: pairs widen their window range to
    insert_size_max (sws 5, 7, 10, 46 for 2 x 150); single-end records are
    unaffected.  Inserts N(600, 150) put the mates 2-6 windows apart."""
    refs = synth.strain_references(seed=23, n_targets=24, median_len=60_000, min_len=10_000, max_len=150_000,
                                   max_strains=8, id_stride=7)
    reads = synth.paired_reads(refs, 3000, length=150, insert_mean=600, insert_sd=150, random_frac=0.05)
    db, o = build_pair(mc, oracle_mod, refs, P=2, insert_size_max=ism)
    assert_classify_equal(db, o, reads)
    assert_classify_equal(db, o, synth.reads_from_list(
        [reads.buf[int(reads.offsets[i]):int(reads.offsets[i + 1])].tobytes() for i in range(500)]))
    db.close()


def test_classify_variable_lengths_and_edges(mc, oracle_mod):
    refs = synth.strain_references(seed=5, n_targets=12, median_len=40_000, min_len=10_000, max_len=60_000,
                                   max_strains=4)
    rd = synth.single_end_reads(refs, 2000, length_range=(0, 600), seed=9)
    edge = [b"", b"A", b"ACGT" * 3 + b"A" * 3, b"N" * 200, refs.seq(0)[:16], refs.seq(0)[:127],
            refs.seq(0)[:128], refs.seq(1)[5:244], refs.seq(1)[:240], refs.seq(2)[:251], refs.seq(2)[7:1400]]
    r1 = [rd.buf[int(rd.offsets[i]):int(rd.offsets[i + 1])].tobytes() for i in range(rd.n)] + edge
    r2 = [synth.revcomp(np.frombuffer(x, np.uint8)).tobytes() if i % 3 else b"" for i, x in enumerate(r1)]
    db, o = build_pair(mc, oracle_mod, refs, P=2)
    assert_classify_equal(db, o, synth.reads_from_list(r1))
    assert_classify_equal(db, o, synth.reads_from_list(r1, r2))
    db.close()


@pytest.mark.parametrize("m", [4, 8])
def test_query_bins_medium_and_large(mc, oracle_mod, m):
    """Records whose gathered location count exceeds the warp bin (512) and
    the medium bin (4096): 300 near-identical strains put up to 254
    locations behind every feature (up to 64*254 = 16256 per 2x150 pair).
    m = 8 runs every bin's 8-entry candidate-list instantiation (S14: m <= 8)."""
    rng = np.random.default_rng(8)
    base = synth.random_bases(rng, 4000)
    seqs = [synth.mutate(rng, base, 0.003).tobytes() for _ in range(300)]
    base2 = synth.random_bases(rng, 4000)
    seqs += [synth.mutate(rng, base2, 0.003).tobytes() for _ in range(20)]
    refs = synth.references_from_list(seqs, list(range(2, 322)), [0, 1] + [1] * 320)
    reads = synth.paired_reads(refs, 400, length=150, insert_mean=300, insert_sd=20)
    db, o = build_pair(mc, oracle_mod, refs, m=m)
    _, _, _, nl = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets, per_partition=True)
    assert nl.max() > 4096 and ((nl > 512) & (nl <= 4096)).any()
    assert_classify_equal(db, o, reads)
    db.close()


def test_query_large_bin_many_unique_windows(mc, oracle_mod):
    """3000 short targets, each sharing a random ~30% of one 300-bp region's
    k-mers: every feature keeps a different set of 254 targets, so a read of
    that region hits thousands of distinct windows (the 512-thread bin)."""
    rng = np.random.default_rng(17)
    R = synth.random_bases(rng, 300)
    seqs = [synth.mutate(rng, R, 0.073).tobytes() for _ in range(3000)]
    refs = synth.references_from_list(seqs, [2] * 3000, [0, 1, 1])
    rd = synth.reads_from_list([R[:150].tobytes()] * 3 + [R[:120].tobytes()],
                               [synth.revcomp(R[150:]).tobytes()] * 3 + [b""])
    db, o = build_pair(mc, oracle_mod, refs)
    assert_classify_equal(db, o, rd)
    db.close()


def test_partials_merge_equals_classify_and_multirank_split(mc, oracle_mod):
    refs = synth.strain_references(seed=31, n_targets=24, median_len=50_000, min_len=10_000, max_len=90_000,
                                   max_strains=6)
    reads = synth.paired_reads(refs, 1500, length=150)
    P = 2
    db, o = build_pair(mc, oracle_mod, refs, P=P)
    t, c = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    hits = db.query_partials(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    t2, c2 = db.merge_classify(hits, n_lists=P)
    assert np.array_equal(t, t2) and np.array_equal(c, c2)
    # two handles, one partition each (what each rank holds), explicit partition ids
    part = mc.plan_partitions(P, np.diff(refs.offsets))
    shards = []
    for p in range(P):
        sel = np.nonzero(part == p)[0]
        h = mc.Database(refs.parent, n_partitions=P, partition_begin=p, n_local_partitions=1,
                        capacity_bp=2 * refs.total_bp)
        bufs = [refs.seq(i) for i in sel]
        b, off = oracle_mod.pack_seqs(bufs)
        h.insert_targets(b, off, refs.target_ids[sel], refs.taxa[sel], np.full(sel.size, p, np.uint32))
        h.finalize()
        shards.append(h.query_partials(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets))
        if p == 1:
            merged = np.concatenate(shards, axis=1)
            t3, c3 = h.merge_classify(merged, n_lists=P)
        h.close()
    assert np.array_equal(t, t3) and np.array_equal(c, c3)
    db.close()


def test_device_resident_inputs_and_outputs(mc, oracle_mod):
    refs = synth.tiny_references(n_genomes=4, length=60_000)
    reads = synth.paired_reads(refs, 2000, length=150)
    db, o = build_pair(mc, oracle_mod, refs)
    t, c = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    d = lambda a: torch.from_numpy(a.view(np.uint8) if a.dtype == np.uint8 else a.astype(np.int64)).cuda()
    dt = torch.zeros(reads.n, dtype=torch.int32, device="cuda")
    dc = torch.zeros(reads.n * 4 * 4, dtype=torch.int32, device="cuda")
    db.classify(d(reads.buf), d(reads.offsets), d(reads.mates_buf), d(reads.mate_offsets), out_taxon=dt,
                out_candidates=dc)
    torch.cuda.synchronize()
    assert np.array_equal(dt.cpu().numpy().view(np.uint32), t)
    assert np.array_equal(dc.cpu().numpy().view(np.uint32), c.view(np.uint32).reshape(-1))
    # device-resident build gives the same database
    db2 = mc.Database(refs.parent, capacity_bp=1 << 20)
    db2.insert_targets(d(refs.buf), d(refs.offsets), refs.target_ids, refs.taxa)
    db2.finalize()
    assert_db_equal(db2, o, 1)
    db.close()
    db2.close()


def test_spill_and_staging_paths(mc, oracle_mod, monkeypatch):
    """Tiny region buckets force the spill area; tiny staging buffers force the
    double-buffered host->device streaming over many chunks; an undersized
    hash table (below the HyperLogLog sizing) forces the full-size retry."""
    import subprocess, sys, json, os
    code = r"""
import numpy as np, synth, oracle, json
import paper_2106_08150_b200 as mc
refs = synth.strain_references(seed=13, n_targets=30, median_len=40_000, min_len=10_000, max_len=80_000, max_strains=8)
db = mc.Database(refs.parent, capacity_bp=40 * refs.total_bp)
db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
db.finalize()
o = oracle.OracleDB(refs.parent)
o.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
o.finalize()
ok = all(np.array_equal(a, b) for a, b in zip(db.dump_partition(0), o.dump_partition(0)))
print(json.dumps({"ok": bool(ok), "keys": int(db.stats()["partitions"][0]["keys"])}))
"""
    env = dict(os.environ, MC_TEST_BUCKET_CAP="1000", MC_TEST_STAGE_BYTES="200000", MC_TEST_TABLE_SLOTS="3000")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["keys"] > 0


def test_batched_insert_and_clear(mc, oracle_mod):
    """Several insert calls (greedy partition state carried across calls),
    clear() and rebuild give the same database."""
    refs = synth.strain_references(seed=41, n_targets=16, median_len=30_000, min_len=5_000, max_len=50_000)
    P = 3
    o = oracle_mod.OracleDB(refs.parent, n_partitions=P)
    db = mc.Database(refs.parent, n_partitions=P, capacity_bp=2 * refs.total_bp)
    for rep in range(2):
        for lo, hi in ((0, 5), (5, 6), (6, 16)):
            b, off = oracle_mod.pack_seqs([refs.seq(i) for i in range(lo, hi)])
            db.insert_targets(b, off, refs.target_ids[lo:hi], refs.taxa[lo:hi])
            if rep == 0:
                o.insert(b, off, refs.target_ids[lo:hi], refs.taxa[lo:hi])
        db.finalize()
        if rep == 0:
            o.finalize()
        assert_db_equal(db, o, P)
        db.clear()
    db.close()


# ---------------------------------------------------------------------------
# lifecycle / errors
# ---------------------------------------------------------------------------
def test_state_machine_and_errors(mc):
    refs = synth.tiny_references(n_genomes=2, length=5000)
    db = mc.Database(refs.parent, capacity_bp=1 << 16)
    r = synth.reads_from_list([b"ACGT" * 30])
    with pytest.raises(mc.MCError) as e:
        db.classify(r.buf, r.offsets)
    assert e.value.code == mc.MC_ERR_STATE
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf, refs.offsets, [1, 1], refs.taxa)
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf, refs.offsets, [1, 2], [0, 5])
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf, refs.offsets, [1, 0xFFFFFFFF], refs.taxa)
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    big = synth.tiny_references(n_genomes=1, length=200_000)
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(big.buf, big.offsets, [9], [8])
    assert e.value.code == mc.MC_ERR_CAPACITY
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf, refs.offsets, [5, 6], refs.taxa)
    assert e.value.code == mc.MC_ERR_STATE
    with pytest.raises(mc.MCError) as e:
        db.finalize()
    assert e.value.code == mc.MC_ERR_STATE
    t, c = db.classify(np.zeros(0, np.uint8), np.zeros(1, np.uint64))
    assert t.size == 0
    with pytest.raises(mc.MCError):
        mc.Database([0, 2, 1])  # cycle without a root
    db.close()


# ---------------------------------------------------------------------------
# pipelined query batches (§8(f) NEXT rank 2): host reads of batch b+1 are
# copied while batch b computes; status checked one batch later
# ---------------------------------------------------------------------------
def test_pipelined_query_batches_host_and_device(mc, oracle_mod):
    refs = synth.strain_references(seed=33, n_targets=24, median_len=50_000, min_len=10_000, max_len=120_000,
                                   max_strains=6)
    reads = synth.paired_reads(refs, 5_000, length=150, random_frac=0.1)
    db, o = build_pair(mc, oracle_mod, refs, read_batch=777)  # 7 batches, ragged tail
    ot, oc = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    t, c = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)  # pageable host
    assert np.array_equal(t, ot) and np.array_equal(c.view(np.uint32), oc.view(np.uint32))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    ht = torch.zeros(reads.n, dtype=torch.int32).pin_memory()
    hc = torch.zeros(reads.n * 4 * 4, dtype=torch.int32).pin_memory()
    db.classify(pin(reads.buf), reads.offsets, pin(reads.mates_buf), reads.mate_offsets, out_taxon=ht,
                out_candidates=hc)  # pinned host in and out: fully asynchronous copies
    assert np.array_equal(ht.numpy().view(np.uint32), ot)
    assert np.array_equal(hc.numpy().view(np.uint32), oc.view(np.uint32).reshape(-1))
    dev = torch.device("cuda")
    dt = torch.zeros(reads.n, dtype=torch.int32, device=dev)
    db.classify(torch.from_numpy(reads.buf).to(dev), torch.from_numpy(reads.offsets.astype(np.int64)).to(dev),
                torch.from_numpy(reads.mates_buf).to(dev),
                torch.from_numpy(reads.mate_offsets.astype(np.int64)).to(dev), out_taxon=dt, want_candidates=False)
    assert np.array_equal(dt.cpu().numpy().view(np.uint32), ot)
    db.close()


def test_pipelined_query_error_names_the_record(mc, oracle_mod):
    """Device-resident offsets are checked on the device; a bad record in a
    later batch is reported with its index in the whole call."""
    refs = synth.tiny_references(n_genomes=2, length=20_000)
    reads = synth.single_end_reads(refs, 3000, length=100)
    db, _ = build_pair(mc, oracle_mod, refs, read_batch=1000)
    offs = reads.offsets.astype(np.int64).copy()
    offs[2501] = offs[2500] - 5  # record 2500 ends before it starts
    dev = torch.device("cuda")
    with pytest.raises(mc.MCError) as e:
        db.classify(torch.from_numpy(reads.buf).to(dev), torch.from_numpy(offs).to(dev))
    assert e.value.code == mc.MC_ERR_INVALID_ARG and "2500" in str(e.value)
    t, _ = db.classify(reads.buf, reads.offsets)  # the handle stays usable
    assert t.size == reads.n
    db.close()


# ---------------------------------------------------------------------------
# AFS31-shaped eukaryotic references (§8(f) NEXT rank 4): long chromosomes and
# thousands of scaffold targets, many shorter than one window, with N runs
# ---------------------------------------------------------------------------
def test_eukaryotic_scaffolds_many_targets(mc, oracle_mod):
    refs = synth.scaffold_references(chrom_len=800_000, scaffolds_per_species=1500, scaffold_median=1000)
    assert refs.n > 12_000
    P = 3
    db, o = build_pair(mc, oracle_mod, refs, P=P, max_targets=refs.n + 16)
    assert_db_equal(db, o, P)
    reads = synth.paired_reads(refs, 20_000, length=101, insert_mean=250, insert_sd=30, random_frac=0.05)
    t, c = assert_classify_equal(db, o, reads)
    assert (t != 0).mean() > 0.5
    db.close()


# ---------------------------------------------------------------------------
# condensed dump / load (§8(f) NEXT rank 3)

@pytest.mark.parametrize("P,ids_in_order", [(1, True), (3, False)])
def test_save_load_round_trip(mc, oracle_mod, tmp_path, P, ids_in_order):
    """A loaded handle answers exactly like the saved one: partition dumps,
    feature lists, candidates and taxa (heavy keys over the cap included)."""
    refs = synth.strain_references(seed=41, n_targets=40, median_len=50_000, min_len=10_000, max_len=90_000,
                                   max_strains=12, id_stride=1 if ids_in_order else 13)
    reads = synth.paired_reads(refs, 2000, length=150, random_frac=0.05)
    db, o = build_pair(mc, oracle_mod, refs, P=P, cap=5)
    path = str(tmp_path / "db.mcdb")
    db.save(path)
    db2 = mc.Database.load(path)
    assert_db_equal(db2, o, P)
    t1, c1 = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    t2, c2 = db2.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    assert np.array_equal(t1, t2) and np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    assert_classify_equal(db2, o, reads)
    for t in refs.target_ids[:5]:
        assert db2.partition_of(int(t)) == db.partition_of(int(t))
    with pytest.raises(mc.MCError) as e:  # a loaded handle is finalized
        db2.insert_targets(refs.buf, refs.offsets, np.arange(refs.n) + 10 ** 6, refs.taxa)
    assert e.value.code == mc.MC_ERR_STATE
    db.close()
    db2.close()


def test_save_load_errors(mc, tmp_path):
    refs = synth.tiny_references(n_genomes=2, length=5000)
    db = mc.Database(refs.parent, capacity_bp=1 << 16)
    with pytest.raises(mc.MCError) as e:
        db.save(str(tmp_path / "x"))  # not finalized
    assert e.value.code == mc.MC_ERR_STATE
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    p = tmp_path / "db.mcdb"
    db.save(str(p))
    data = p.read_bytes()
    (tmp_path / "trunc").write_bytes(data[: len(data) // 2])
    (tmp_path / "junk").write_bytes(b"not a database" * 10)
    for bad in ("trunc", "junk", "missing"):
        with pytest.raises(mc.MCError) as e:
            mc.Database.load(str(tmp_path / bad))
        assert e.value.code == mc.MC_ERR_INVALID_ARG, bad
    db.close()
