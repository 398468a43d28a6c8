"""The seeded input recipes stated in DESIGN.md §3 (-m "not gpu"): shapes,
length distributions and determinism of the synthetic workloads.  synth/ holds
no method arithmetic; these only pin that the generators produce what the
bench and the parity tests claim to run."""
import numpy as np

import synth


def test_variable_length_reads_match_table2():
    refs = synth.subset_shard(0, 1, n_targets=20, median_len=2e5, min_len=1e5, max_len=4e5)
    for gen, lo, hi, mean in ((synth.hiseq_reads, 19, 101, 92.3), (synth.miseq_reads, 19, 251, 156.8)):
        rd = gen(refs, 200_000)
        L = np.diff(rd.offsets).astype(np.int64)
        assert L.min() == lo and L.max() == hi
        assert abs(L.mean() - mean) < 1.0, (gen.__name__, L.mean())
        assert rd.mates_buf is None and rd.buf.size == int(rd.offsets[-1])
        again = gen(refs, 200_000)
        assert np.array_equal(again.buf, rd.buf)  # seeded


def test_variable_length_reads_are_cut_from_their_targets():
    refs = synth.subset_shard(0, 1, n_targets=10, median_len=2e5, min_len=1e5, max_len=4e5)
    rd = synth.hiseq_reads(refs, 2000, sub_rate=0.0)
    comp = bytes.maketrans(b"ACGT", b"TGCA")
    for i in range(0, 2000, 97):
        r = rd.buf[int(rd.offsets[i]):int(rd.offsets[i + 1])].tobytes()
        g = refs.seq(int(rd.source_target[i]))
        assert r in g or r.translate(comp)[::-1] in g


def test_refseq_shard_recipe():
    n_shards, scale = 4, 0.05
    shards = [synth.refseq_shard(s, n_shards, scale=scale) for s in range(n_shards)]
    # one global taxonomy on every shard; disjoint target ids
    for s in shards[1:]:
        assert np.array_equal(s.parent, shards[0].parent)
    ids = np.concatenate([s.target_ids for s in shards])
    assert np.unique(ids).size == ids.size
    # species counts of the three kinds (9000 / 6360 / 100 at scale 1)
    species = np.unique(np.concatenate([s.species_of_target for s in shards]))
    assert abs(species.size - round(scale * 15460)) <= 2
    # every target is a leaf under a species -> genus -> family -> root chain
    par, rank = shards[0].parent, shards[0].rank
    for s in shards:
        for t in s.taxa[:50]:
            chain = [int(t)]
            while par[chain[-1]] != chain[-1]:
                chain.append(int(par[chain[-1]]))
            assert [int(rank[x]) for x in chain] == [4, 3, 2, 1, 0]
    # deterministic per shard
    assert np.array_equal(synth.refseq_shard(1, n_shards, scale=scale).buf, shards[1].buf)
    # lengths: viral 10-200 kbp, chromosomes >= 2 Mbp, plasmids 5-200 kbp
    L = np.concatenate([np.diff(s.offsets) for s in shards]).astype(np.int64)
    assert L.min() >= 5_000 and L.max() <= 13_000_000


def test_afs31_shard_recipe():
    """AFS31-shaped shards (Table 1): 31 species over the
    shards, one global taxonomy, disjoint ids, scaffold-level genomes with
    many targets, every sequence of a genome under the genome's taxon."""
    n_shards, scale = 8, 0.004
    shards = [synth.afs31_shard(s, n_shards, scale=scale) for s in range(n_shards)]
    for s in shards[1:]:
        assert np.array_equal(s.parent, shards[0].parent)
    ids = np.concatenate([s.target_ids for s in shards])
    assert np.unique(ids).size == ids.size
    sp = [set(np.unique(s.species_of_target).tolist()) for s in shards]
    assert set().union(*sp) == set(range(31)) and sum(len(x) for x in sp) == 31
    for k, s in enumerate(shards):
        assert all(x % n_shards == k for x in sp[k])
    total = sum(s.total_bp for s in shards)
    assert abs(total - 77e9 * scale) < 31 * 20_000 + 1e6
    par, rank = shards[0].parent, shards[0].rank
    for s in shards:
        for x in np.unique(s.species_of_target):
            m = s.species_of_target == x
            assert np.unique(s.taxa[m]).size == 1           # one genome taxon
            t = int(s.taxa[m][0])
            chain = [t]
            while par[chain[-1]] != chain[-1]:
                chain.append(int(par[chain[-1]]))
            assert [int(rank[c]) for c in chain] == [4, 3, 2, 1, 0]
            L = np.diff(s.offsets)[m].astype(np.int64)
            if x % 3 == 0:                                  # scaffold level
                assert L.min() >= 1 and L.max() <= 2_000_000 and m.sum() > 20
                assert np.median(L) < 20_000
            else:                                           # chromosome level
                assert 8 <= m.sum() <= 40
    assert np.array_equal(synth.afs31_shard(3, n_shards, scale=scale).buf, shards[3].buf)
    # N runs (assembly gaps) present, only ACGTN bytes
    b = shards[0].buf
    assert set(np.unique(b).tolist()) <= set(b"ACGTN") and (b == ord("N")).any()
