"""Multi-GPU handle (mc_config.n_gpus = G > 1) vs the oracle with P partitions,
bit-exact: the partitioned build, the per-batch all-gather of
reads and the exchange fused into the merge, the double-buffered
batch pipeline.  On the one-GPU box the G shards share device 0
(repeated ordinals): the same code path runs, its peer copies degenerate to
same-device copies and the merge kernel's "peer" loads to local ones."""
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


@pytest.fixture(scope="module")
def refs():
    return synth.strain_references(seed=41, n_targets=40, median_len=60_000, min_len=10_000, max_len=150_000,
                                   max_strains=12, id_stride=13)


def group(mc, refs, G, P, read_batch=700, m=4, **cfg):
    return mc.Database(refs.parent, n_partitions=P, n_gpus=G, devices=[0] * G, max_candidates=m,
                       capacity_bp=max(1 << 16, 2 * refs.total_bp), read_batch=read_batch, **cfg)


def oracle_db(oracle_mod, refs, P, m=4):
    o = oracle_mod.OracleDB(refs.parent, n_partitions=P, m=m)
    o.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    o.finalize()
    return o


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.mark.parametrize("G,P", [(2, 2), (2, 4), (2, 8), (4, 4), (4, 8), (8, 8)])
def test_group_build_and_classify_equal_oracle(mc, oracle_mod, refs, G, P):
    reads = synth.paired_reads(refs, 2500, length=150, random_frac=0.05, n_rate=0.001, seed=77)
    db = group(mc, refs, G, P)
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    o = oracle_db(oracle_mod, refs, P)
    for p in range(P):  # every partition lives on its shard, identical to the oracle's
        gk, gc, gv = db.dump_partition(p)
        ok, oc, ov = o.dump_partition(p)
        assert np.array_equal(gk, ok) and np.array_equal(gc, oc) and np.array_equal(gv, ov), p
    plan = oracle_mod.plan_partitions(P, np.diff(refs.offsets))  # S9 over all P partitions
    for i in range(0, refs.n, 3):
        assert db.partition_of(int(refs.target_ids[i])) == plan[i]
    ot, oc = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    t, c = db.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)  # 4 batches of 700
    assert same(c, oc) and np.array_equal(t, ot)
    # per-partition lists (every shard's columns of out_hits) equal the oracle's
    _, _, opc, _ = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets, per_partition=True)
    hits = db.query_partials(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    assert hits.shape == (reads.n, P, 4)
    got = np.stack([hits["tgt"], hits["hits"], hits["win_beg"], hits["win_end"]], -1)
    exp = np.stack([opc["tgt"], opc["hits"], opc["win_beg"], opc["win_end"]], -1)
    assert np.array_equal(got, exp)
    db.close()


@pytest.mark.parametrize("inputs", ["pinned", "device"])
def test_group_query_input_kinds(mc, oracle_mod, refs, inputs):
    G, P = 2, 4
    reads = synth.paired_reads(refs, 1999, length=150, random_frac=0.05, seed=78)
    db = group(mc, refs, G, P, read_batch=512)
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    o = oracle_db(oracle_mod, refs, P)
    ot, oc = o.classify(reads.buf, reads.offsets, reads.mates_buf, reads.mate_offsets)
    if inputs == "pinned":
        args = [torch.from_numpy(reads.buf).pin_memory(), torch.from_numpy(reads.offsets.astype(np.int64)).pin_memory(),
                torch.from_numpy(reads.mates_buf).pin_memory(),
                torch.from_numpy(reads.mate_offsets.astype(np.int64)).pin_memory()]
        out_t = torch.zeros(reads.n, dtype=torch.int32).pin_memory()
        out_c = torch.zeros(reads.n * 16, dtype=torch.int32).pin_memory()
    else:
        dev = torch.device("cuda:0")
        args = [torch.from_numpy(reads.buf).to(dev), torch.from_numpy(reads.offsets.astype(np.int64)).to(dev),
                torch.from_numpy(reads.mates_buf).to(dev), torch.from_numpy(reads.mate_offsets.astype(np.int64)).to(dev)]
        out_t = torch.zeros(reads.n, dtype=torch.int32, device=dev)
        out_c = torch.zeros(reads.n * 16, dtype=torch.int32, device=dev)
    db.classify(*args, out_taxon=out_t, out_candidates=out_c)
    torch.cuda.synchronize()
    assert np.array_equal(out_t.cpu().numpy().view(np.uint32), ot)
    assert np.array_equal(out_c.cpu().numpy().view(np.uint32), oc.view(np.uint32).reshape(-1))
    db.close()


def test_group_batched_insert_device_resident(mc, oracle_mod, refs):
    """mc_db_insert_target_batches: two device-resident batches (explicit
    partitions for the first, S9 for the second), built by every shard
    concurrently; clear + rebuild gives the same database."""
    G, P = 2, 4
    half = refs.n // 2
    dev = torch.device("cuda:0")
    cut = int(refs.offsets[half])
    b1 = (torch.from_numpy(refs.buf[:cut]).to(dev), refs.offsets[:half + 1], refs.target_ids[:half], refs.taxa[:half],
          (np.arange(half) % P).astype(np.uint32))
    b2 = (torch.from_numpy(refs.buf[cut:]).to(dev), refs.offsets[half:] - cut, refs.target_ids[half:],
          refs.taxa[half:], None)
    db = group(mc, refs, G, P)
    o = oracle_mod.OracleDB(refs.parent, n_partitions=P)
    o.insert(refs.buf[:cut], refs.offsets[:half + 1], refs.target_ids[:half], refs.taxa[:half], b1[4])
    o.insert(refs.buf[cut:], refs.offsets[half:] - cut, refs.target_ids[half:], refs.taxa[half:])
    o.finalize()
    reads = synth.single_end_reads(refs, 1500, length=100, seed=79)
    ot, oc = o.classify(reads.buf, reads.offsets)
    for rep in range(2):
        db.insert_target_batches([b1, b2])
        db.finalize()
        for p in range(P):
            assert all(np.array_equal(x, y) for x, y in zip(db.dump_partition(p), o.dump_partition(p))), (rep, p)
        t, c = db.classify(reads.buf, reads.offsets)
        assert same(c, oc) and np.array_equal(t, ot)
        db.clear()
    db.close()


def test_group_config_errors(mc, refs):
    for bad in (dict(n_gpus=3, n_partitions=4), dict(n_gpus=2, n_partitions=1), dict(n_gpus=9, n_partitions=9),
                dict(n_gpus=2, n_partitions=2, n_local_partitions=1), dict(n_gpus=2, n_partitions=2, devices=[0, 99])):
        with pytest.raises(mc.MCError) as e:
            mc.Database(refs.parent, **bad)
        assert e.value.code == mc.MC_ERR_INVALID_ARG, bad
    db = group(mc, refs, 2, 2)
    with pytest.raises(mc.MCError) as e:
        db.set_stream(None)
    assert e.value.code == mc.MC_ERR_STATE
    db.close()


def test_group_variable_lengths_and_insert_size(mc, oracle_mod, refs):
    """Variable-length single-end records (MiSeq-shaped, 1-3 windows, the
    medium / large bins) and paired records with insert_size_max (reading S25)
    through a G = 2 handle: identical to the oracle with P = 4."""
    G, P = 2, 4
    miseq = synth.miseq_reads(refs, 1500, seed=81)
    for ism in (0, 560):
        db = group(mc, refs, G, P, read_batch=400, insert_size_max=ism)
        db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
        db.finalize()
        o = oracle_mod.OracleDB(refs.parent, n_partitions=P, insert_size_max=ism)
        o.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
        o.finalize()
        pairs = synth.paired_reads(refs, 1200, length=150, insert_mean=600, insert_sd=150, seed=82)
        for rd in (miseq, pairs):
            t, c = db.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
            ot, oc = o.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
            assert same(c, oc) and np.array_equal(t, ot), ism
        db.close()
