"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the
paper prints (tests/golden/*.json, cited), closed forms, invariants, or a
brute force written here from the textbook definitions (string reverse
complement, base-4 digits, explicit range enumeration).  None of these tests
re-calls the oracle's internals to produce its expected value.
"""
import itertools
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
COMP = {"A": "T", "C": "G", "G": "C", "T": "A"}


def rc_str(s):
    return "".join(COMP.get(c, "N") for c in reversed(s.upper()))


def base4(s):
    v = 0
    for c in s.upper():
        v = v * 4 + "ACGT".index(c)
    return v


def brute_sketch(seq, k, s, w, table, canonical=True):
    """Textbook windows + canonical k-mers + table hash + s smallest unique."""
    n = len(seq) - k + 1
    stride = w - k + 1
    out = []
    if n <= 0:
        return out
    for j in range((n + stride - 1) // stride):
        vals = set()
        for i in range(j * stride, min((j + 1) * stride, n)):
            km = seq[i:i + k]
            if any(c not in "ACGTacgt" for c in km):
                continue
            v = base4(km)
            if canonical:
                v = min(v, base4(rc_str(km)))
            vals.add(int(table[v]))
        out.append(sorted(vals)[:s])
    return out


# ---------------------------------------------------------------------------
# §2 toy example P:187-197
# ---------------------------------------------------------------------------
def test_minhash_toy_example(oracle_mod):
    g = json.load(open(os.path.join(GOLD, "minhash_toy.json")))
    k = g["k"]
    table = np.full(4 ** k, 1000, np.uint32)  # k-mers absent from the example
    for km, v in g["hash"].items():
        table[base4(km)] = v
    sk = oracle_mod.sketch(g["sequence"], k=k, s=g["s"], w=g["window_len"], canonical=g["canonical"], table=table)
    assert sk == [g["expected_sketch"]]


# ---------------------------------------------------------------------------
# Figure 1 worked example P:336-435
# ---------------------------------------------------------------------------
def _fig1_locs(part):
    locs = []
    for t, wins in part.items():
        for j, c in wins.items():
            locs += [(int(t) << 32) | int(j)] * c
    rng = np.random.default_rng(1)
    locs = np.array(locs, np.uint64)
    rng.shuffle(locs)  # the oracle must sort (step 6) itself
    return locs


def test_fig1_partition_lists_and_merge(oracle_mod):
    g = json.load(open(os.path.join(GOLD, "fig1_candidates.json")))
    lists = []
    for part, exp in zip(g["partitions"], g["expected_partition_lists"]):
        c = oracle_mod.top_hits(_fig1_locs(part), g["sws"], g["m"])
        assert [list(map(int, x)) for x in c] == exp
        lists.append(c)
    merged = oracle_mod.merge_candidates(lists, g["m"])
    assert [list(map(int, x)) for x in merged] == g["expected_merged"]


def test_fig1_range_sums(oracle_mod):
    """The 8 / 7 / 12 printed over g1 are the best ranges from w3 / w4 / w1 on."""
    g = json.load(open(os.path.join(GOLD, "fig1_candidates.json")))
    g1 = g["partitions"][0]["1"]
    for key, first in (("from_w1", 1), ("from_w3", 3), ("from_w4", 4)):
        part = {"1": {j: c for j, c in g1.items() if int(j) >= first}}
        c = oracle_mod.top_hits(_fig1_locs(part), g["sws"], 1)
        assert int(c[0]["hits"]) == g["g1_range_sums"][key]


# ---------------------------------------------------------------------------
# encoding / canonical k-mers (S3/S4)
# ---------------------------------------------------------------------------
def test_canonical_all_4mers(oracle_mod):
    for t in itertools.product("ACGT", repeat=4):
        km = "".join(t)
        c = oracle_mod.canonical_kmer(km)
        assert c == min(base4(km), base4(rc_str(km)))
        assert c == oracle_mod.canonical_kmer(rc_str(km))
        assert oracle_mod.canonical_kmer(km.lower()) == c


def test_canonical_random_16mers_and_ambiguous(oracle_mod):
    rng = np.random.default_rng(5)
    for _ in range(300):
        km = "".join(rng.choice(list("ACGT"), 16))
        assert oracle_mod.canonical_kmer(km) == min(base4(km), base4(rc_str(km)))
    assert oracle_mod.canonical_kmer("ACGTNACGTACGTACG") is None
    assert oracle_mod.canonical_kmer("ACGTRACGTACGTACG") is None


# ---------------------------------------------------------------------------
# windows
# ---------------------------------------------------------------------------
def test_window_count_closed_form(oracle_mod):
    assert oracle_mod.window_count(200_000) == 1786  # SURVEY §8a B2 / tiny config
    for L in list(range(0, 400)) + [1000, 10_000, 123_457]:
        exp = 0 if L < 16 else -(-(L - 15) // 112)
        assert oracle_mod.window_count(L) == exp
    # every k-mer start lies in exactly one window: window j covers [112j, 112j+112)
    for L in (16, 127, 128, 239, 240, 251, 1000):
        n = L - 15
        cover = np.zeros(n, int)
        for j in range(oracle_mod.window_count(L)):
            cover[j * 112:min(j * 112 + 112, n)] += 1
        assert (cover == 1).all()


# ---------------------------------------------------------------------------
# sketch
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("k,w,s", [(4, 10, 3), (5, 12, 4), (4, 7, 16), (6, 21, 5)])
def test_sketch_bruteforce_table_hash(oracle_mod, k, w, s):
    rng = np.random.default_rng(k * 100 + w)
    table = rng.integers(0, 2 ** 32, size=4 ** k, dtype=np.uint64).astype(np.uint32)
    for _ in range(60):
        L = int(rng.integers(0, 41))
        seq = "".join(rng.choice(list("ACGTacgtN"), L, p=[.22, .22, .22, .22, .02, .02, .02, .02, .04]))
        assert oracle_mod.sketch(seq, k=k, s=s, w=w, table=table) == brute_sketch(seq, k, s, w, table)


def test_sketch_repeats_and_short_sketches(oracle_mod):
    rng = np.random.default_rng(9)
    k = 4
    table = rng.integers(0, 2 ** 32, size=4 ** k, dtype=np.uint64).astype(np.uint32)
    for seq in ["A" * 40, "AC" * 20, "ACGTACGT" * 4, "NNNNACGTNNNN", "ACG", "ACGT"]:
        assert oracle_mod.sketch(seq, k=4, s=16, w=10, table=table) == brute_sketch(seq, 4, 16, 10, table)
    assert oracle_mod.sketch("A" * 40, k=4, s=16, w=10, table=table)[0] == [int(table[0])]


def test_sketch_strand_symmetry(oracle_mod):
    """canonical k-mers make a single-window sketch strand-independent."""
    rng = np.random.default_rng(11)
    for L in (16, 40, 100, 127):
        seq = "".join(rng.choice(list("ACGT"), L))
        a = oracle_mod.sketch(seq)
        b = oracle_mod.sketch(rc_str(seq))
        assert len(a) == 1 and a == b
        assert len(a[0]) == min(16, len(set(a[0])))
        assert a[0] == sorted(set(a[0]))


def test_sketch_default_params_shape(oracle_mod):
    rng = np.random.default_rng(12)
    seq = "".join(rng.choice(list("ACGT"), 1000))
    sk = oracle_mod.sketch(seq)
    assert len(sk) == oracle_mod.window_count(1000)
    assert all(len(x) == 16 for x in sk)
    assert all(x == sorted(set(x)) for x in sk)


def test_h1_bijective(oracle_mod):
    """S1: h1 is a bijection on 32-bit words (its inverse mixer recovers x),
    so distinct canonical k-mers give distinct features.  h1 VALUES are a
    choice the paper leaves open: parity unpinned."""
    def inv(x):
        x = ((x >> 16) ^ x) * 0x119DE1F3 & 0xFFFFFFFF
        x = ((x >> 16) ^ x) * 0x119DE1F3 & 0xFFFFFFFF
        return (x >> 16) ^ x
    rng = np.random.default_rng(13)
    for x in list(rng.integers(0, 2 ** 32, 2000)) + [0, 1, 2 ** 32 - 1]:
        assert inv(oracle_mod.h1(int(x))) == int(x)


# ---------------------------------------------------------------------------
# partition plan (S9)
# ---------------------------------------------------------------------------
def test_partition_plan_greedy(oracle_mod):
    rng = np.random.default_rng(3)
    lens = rng.integers(1, 1000, 200)
    for P in (1, 2, 3, 8):
        got = oracle_mod.plan_partitions(P, lens)
        load = [0] * P
        for i, L in enumerate(lens):
            b = min(range(P), key=lambda q: (load[q], q))
            assert got[i] == b
            load[b] += int(L)


# ---------------------------------------------------------------------------
# table + cap
# ---------------------------------------------------------------------------
def _expected_db(refs, P, cap, part, k=16, s=16, w=127):
    exp = [dict() for _ in range(P)]
    import oracle as O
    for i in range(refs.n):
        sk = O.sketch(refs.seq(i), k=k, s=s, w=w)
        for j, feats in enumerate(sk):
            for f in feats:
                exp[part[i]].setdefault(f, []).append((int(refs.target_ids[i]) << 32) | j)
    for d in exp:
        for f in d:
            d[f] = sorted(d[f])[:cap]
    return exp


@pytest.mark.parametrize("P", [1, 3])
def test_db_bruteforce(oracle_mod, P):
    refs = synth.strain_references(seed=7, n_targets=12, median_len=3000, min_len=500, max_len=8000,
                                   max_strains=5, n_rate=1e-3, id_stride=7, id_offset=100)
    db = oracle_mod.OracleDB(refs.parent, cap=3, n_partitions=P)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    part = oracle_mod.plan_partitions(P, np.diff(refs.offsets))
    exp = _expected_db(refs, P, 3, part)
    for p in range(P):
        keys, counts, vals = db.dump_partition(p)
        assert keys.tolist() == sorted(exp[p])
        assert counts.tolist() == [len(exp[p][f]) for f in sorted(exp[p])]
        assert vals.tolist() == [v for f in sorted(exp[p]) for v in exp[p][f]]


@pytest.mark.parametrize("threads", [1, 5])
def test_restricted_threaded_build_bruteforce(oracle_mod, threads):
    """Feature-restricted build (used for full-size parity):
    with a filter, the threaded insert stores exactly the brute-force lists of
    the filtered features, in the same order, for any thread count."""
    refs = synth.strain_references(seed=11, n_targets=14, median_len=3000, min_len=500, max_len=8000,
                                   max_strains=5, n_rate=1e-3, id_stride=3, id_offset=50)
    P = 2
    part = oracle_mod.plan_partitions(P, np.diff(refs.offsets))
    exp = _expected_db(refs, P, 3, part)
    allf = sorted({f for p in range(P) for f in exp[p]})
    keep = set(np.random.default_rng(2).choice(allf, len(allf) // 3, replace=False).tolist())
    db = oracle_mod.OracleDB(refs.parent, cap=3, n_partitions=P)
    db.set_feature_filter(np.array(sorted(keep), np.uint32))
    db.insert_restricted(refs.buf, refs.offsets, refs.target_ids, refs.taxa, threads=threads)
    db.finalize()
    for p in range(P):
        keys, counts, vals = db.dump_partition(p)
        fs = sorted(f for f in exp[p] if f in keep)
        assert keys.tolist() == fs
        assert vals.tolist() == [v for f in fs for v in exp[p][f]]


def test_cap_keeps_smallest(oracle_mod):
    """300 identical strains: every feature has 300 locations per partition and
    keeps the 254 smallest (t, j) -- the 254 lowest target ids."""
    rng = np.random.default_rng(4)
    base = "".join(rng.choice(list("ACGT"), 300))
    n = 300
    ids = rng.permutation(np.arange(1000, 1000 + n)).astype(np.uint32)
    refs = synth.references_from_list([base] * n, [2] * n, [0, 1, 1], ids=ids)
    db = oracle_mod.OracleDB(refs.parent)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    keys, counts, vals = db.dump_partition(0)
    sk = oracle_mod.sketch(base)
    assert sorted({f for x in sk for f in x}) == keys.tolist()
    for f in keys:
        locs = db.feature_locations(0, int(f))
        assert len(locs) == 254
        full = sorted((int(t) << 32) | j for t in ids for j, x in enumerate(sk) if f in x)
        assert locs.tolist() == full[:254]


# ---------------------------------------------------------------------------
# top hits: brute force over all ranges (P:593-598, S11-S13)
# ---------------------------------------------------------------------------
def brute_top(locs, sws, m):
    cnt = {}
    for l in locs:
        t, j = int(l) >> 32, int(l) & 0xFFFFFFFF
        cnt.setdefault(t, {}).setdefault(j, 0)
        cnt[t][j] += 1
    best = []
    for t, wins in cnt.items():
        lo, hi = min(wins), max(wins)
        sums = {b: sum(c for j, c in wins.items() if b <= j <= b + sws - 1) for b in range(lo - sws, hi + 1)}
        mx = max(sums.values())
        b = min(j for j in wins if sums[j] == mx)  # smallest hit window reaching the max
        e = max(j for j in wins if b <= j <= b + sws - 1)
        best.append((t, mx, b, e))
    best.sort(key=lambda c: (-c[1], c[0]))
    return best[:m]


def test_top_hits_bruteforce(oracle_mod):
    rng = np.random.default_rng(6)
    for trial in range(200):
        n = int(rng.integers(0, 60))
        t = rng.integers(0, 6, n).astype(np.uint64)
        j = rng.integers(0, 20, n).astype(np.uint64)
        locs = (t << np.uint64(32)) | j
        sws = int(rng.integers(1, 6))
        m = int(rng.integers(1, 5))
        got = [tuple(map(int, c)) for c in oracle_mod.top_hits(locs, sws, m)]
        assert got == brute_top(locs, sws, m)


def test_union_topm_equals_global_topm(oracle_mod):
    """Q8: merging per-partition top-m lists equals top-m over all targets,
    because each target lives in exactly one partition."""
    rng = np.random.default_rng(8)
    for _ in range(100):
        n = int(rng.integers(0, 80))
        t = rng.integers(0, 12, n).astype(np.uint64)
        j = rng.integers(0, 15, n).astype(np.uint64)
        locs = (t << np.uint64(32)) | j
        sws, m, P = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
        lists = [oracle_mod.top_hits(locs[(t % P) == p], sws, m) for p in range(P)]
        merged = oracle_mod.merge_candidates(lists, m)
        assert [tuple(map(int, c)) for c in merged] == brute_top(locs, sws, m)


# ---------------------------------------------------------------------------
# taxonomy / LCA / classification rule (S15/S16, S24)
# ---------------------------------------------------------------------------
#        1(root)
#       /      \
#      2        3
#     / \        \
#    4   5        6
#   / \            \
#  7   8            9
PARENT = [0, 1, 1, 1, 2, 2, 3, 4, 4, 6]


def test_lca_hand_tree(oracle_mod):
    db = oracle_mod.OracleDB(PARENT)
    cases = {(7, 8): 4, (7, 5): 2, (7, 9): 1, (8, 4): 4, (9, 6): 6, (5, 5): 5, (7, 1): 1, (2, 3): 1}
    for (a, b), c in cases.items():
        assert db.lca(a, b) == c and db.lca(b, a) == c


def test_classify_rule(oracle_mod):
    # targets 0..3 with taxa 7, 8, 5, 9
    refs = synth.references_from_list(["ACGT"] * 4, [7, 8, 5, 9], PARENT)
    db = oracle_mod.OracleDB(PARENT, hits_min=5, hits_diff=4)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    C = lambda *cs: np.array([tuple(c) for c in cs], oracle_mod.CAND_DTYPE)
    assert db.classify_candidates(C()) == 0                                  # no hits
    assert db.classify_candidates(C((0, 4, 0, 0))) == 0                       # below hits_min
    assert db.classify_candidates(C((0, 12, 0, 0), (1, 7, 0, 0))) == 7        # 12-7 = 5 > 4
    assert db.classify_candidates(C((0, 12, 0, 0), (1, 8, 0, 0))) == 4        # tie within 4 -> LCA(7,8)
    assert db.classify_candidates(C((0, 12, 0, 0), (1, 8, 0, 0), (3, 9, 0, 0))) == 1
    assert db.classify_candidates(C((0, 12, 0, 0), (2, 10, 0, 0), (3, 3, 0, 0))) == 2  # LCA(7,5)
    assert db.sws(100) == 2 and db.sws(150, 150) == 4 and db.sws(250, 250) == 6


# ---------------------------------------------------------------------------
# whole pipeline: exact self-classification (north_star "exact self-classification")
# ---------------------------------------------------------------------------
def test_window_aligned_reads_hit_their_window(oracle_mod):
    refs = synth.tiny_references(n_genomes=4, length=20_000)
    db = oracle_mod.OracleDB(refs.parent)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    rng = np.random.default_rng(2)
    reads, exp = [], []
    for _ in range(50):
        t = int(rng.integers(0, refs.n))
        j = int(rng.integers(0, (20_000 - 127) // 112))
        r = refs.seq(t)[112 * j:112 * j + 127]
        if rng.random() < 0.5:
            r = rc_str(r.decode()).encode()
        reads.append(r)
        nf = len(oracle_mod.sketch(r)[0])
        exp.append((t, nf, j, j))
    rd = synth.reads_from_list(reads)
    taxon, cand = db.classify(rd.buf, rd.offsets)
    for i, (t, nf, j, _) in enumerate(exp):
        assert tuple(map(int, cand[i][0])) == (t, nf, j, j)
        assert taxon[i] == refs.taxa[t]


@pytest.mark.parametrize("gap", [3, 4, 6])
def test_insert_size_max_window_aligned_pairs(oracle_mod, gap):
    """Reading S25 (insertSizeMax-style sws for pairs) pinned by a closed form:
    mate 1 = exactly window j, mate 2 = reverse complement of exactly window
    j + gap of a random genome; each mate alone gives 16 hits on its own
    window.  S10 (insert_size_max 0): 2 x 127 bp -> sws = 2 + 254 // 112 = 4,
    so a range holds both mates' windows iff gap <= 3 (32 hits on [j, j+gap]),
    else the best is one mate: 16 hits on [j, j].  With insert_size_max =
    112 * (gap + 1) - 1: sws = gap + 2 > gap, so 32 hits on [j, j + gap] for
    every gap; single-end records ignore insert_size_max."""
    refs = synth.tiny_references(n_genomes=3, length=40_000)
    t, j = 1, 40
    g = refs.seq(t)
    m1 = g[112 * j:112 * j + 127]
    m2 = rc_str(g[112 * (j + gap):112 * (j + gap) + 127].decode()).encode()
    assert len(oracle_mod.sketch(m1)[0]) == len(oracle_mod.sketch(m2)[0]) == 16
    pair = synth.reads_from_list([m1], [m2])
    single = synth.reads_from_list([m1 + b"N" + m2])  # 255 bp single-end: sws = 4 regardless
    single_out = []
    for ism in (0, 112 * (gap + 1) - 1):
        db = oracle_mod.OracleDB(refs.parent, insert_size_max=ism)
        # the sws itself, by the closed form: S10 gives 2 + 254 // 112 = 4 for the
        # pair and 2 + 255 // 112 = 4 for the single-end record; S25 raises only
        # the paired one to 2 + (112 (gap + 1) - 1) // 112 = gap + 2
        assert db.sws(127, 127, paired=True) == (gap + 2 if ism else 4)
        assert db.sws(255, 0, paired=False) == 4
        assert db.sws(127, 127, paired=False) == 4  # a record without a mate never takes S25
        db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
        db.finalize()
        _, cand = db.classify(pair.buf, pair.offsets, pair.mates_buf, pair.mate_offsets)
        both = ism > 0 or gap <= 3
        assert tuple(map(int, cand[0][0])) == ((t, 32, j, j + gap) if both else (t, 16, j, j))
        single_out.append(db.classify(single.buf, single.offsets)[1])
        db.close()
    assert np.array_equal(single_out[0], single_out[1])


def test_exact_reads_self_classify(oracle_mod):
    refs = synth.tiny_references(n_genomes=8, length=30_000)
    db = oracle_mod.OracleDB(refs.parent)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    rd = synth.single_end_reads(refs, 400, length=100, random_frac=0.0, sub_rate=0.0, n_rate=0.0, seed=3)
    taxon, cand = db.classify(rd.buf, rd.offsets)
    classified = taxon != 0
    assert classified.mean() > 0.9
    assert (taxon[classified] == refs.taxa[rd.source_target[classified]]).all()
    # identical strains -> LCA = their parent species node
    rp = synth.references_from_list([refs.seq(0), refs.seq(0)], [16, 17], list(refs.parent) + [8, 8])
    db2 = oracle_mod.OracleDB(rp.parent)
    db2.insert(rp.buf, rp.offsets, rp.target_ids, rp.taxa)
    db2.finalize()
    r2 = synth.reads_from_list([refs.seq(0)[1000:1127]])
    t2, c2 = db2.classify(r2.buf, r2.offsets)
    assert t2[0] == 8 and c2[0][0]["hits"] == c2[0][1]["hits"]


def test_classify_threads_equals_classify(oracle_mod):
    """The threaded query phase (cpu_baseline's N-thread timing) returns the
    single-threaded results: records are independent (read-only maps)."""
    refs = synth.tiny_references(n_genomes=4, length=30_000)
    db = oracle_mod.OracleDB(refs.parent, n_partitions=2)
    db.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    rd = synth.paired_reads(refs, 301, length=150, seed=5)
    t1, c1 = db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
    for threads in (1, 3, 8):
        t2, c2 = db.classify_threads(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets, threads=threads)
        assert np.array_equal(t1, t2) and np.array_equal(c1, c2)


def test_s9_counts_explicitly_placed_targets(oracle_mod):
    """Reading S9 ("the partition with the fewest bp so far"): targets placed
    with explicit partition ids count towards their partition's bp, so a later
    S9-assigned batch fills the lighter partitions first."""
    rng = np.random.default_rng(9)
    seqs = ["".join(rng.choice(list("ACGT"), L)) for L in (1000, 100, 100, 100)]
    refs = synth.references_from_list(seqs, [2, 2, 2, 2], PARENT)
    db = oracle_mod.OracleDB(PARENT, n_partitions=2)
    db.insert(refs.buf[:1000], refs.offsets[:2], refs.target_ids[:1], refs.taxa[:1], np.zeros(1, np.uint32))
    db.insert(refs.buf[1000:], refs.offsets[1:] - 1000, refs.target_ids[1:], refs.taxa[1:])
    db.finalize()
    # partition 0 already holds 1000 bp: the three 100 bp targets all go to partition 1
    tg = [set((db.dump_partition(p)[2] >> 32).tolist()) for p in range(2)]
    assert tg[0] == {int(refs.target_ids[0])}
    assert tg[1] == set(int(t) for t in refs.target_ids[1:])
