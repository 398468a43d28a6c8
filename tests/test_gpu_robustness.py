"""GPU checks of the ABI's input handling: converted input
buffers outlive the call, offsets that go backwards are INVALID_ARG with the
handle still usable, the reserved target id is never 'found'."""
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
def built(mc, oracle_mod):
    refs = synth.tiny_references(n_genomes=4, length=40_000)
    db = mc.Database(refs.parent, capacity_bp=1 << 20)
    db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    db.finalize()
    o = oracle_mod.OracleDB(refs.parent)
    o.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    o.finalize()
    return refs, db, o


def test_converted_read_buffers_outlive_the_call(mc, built):
    refs, db, o = built
    rd = synth.paired_reads(refs, 500, length=150, seed=11)
    ot, oc = o.classify(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
    # int8 buffers and python-list offsets are converted (copied) by the binding
    t, c = db.classify(rd.buf.view(np.int8), list(map(int, rd.offsets)), rd.mates_buf.view(np.int8),
                       list(map(int, rd.mate_offsets)))
    assert np.array_equal(t, ot) and np.array_equal(c.view(np.uint32), oc.view(np.uint32))
    # a strided (non-contiguous) buffer: every other byte of a doubled buffer
    wide = np.zeros(2 * rd.buf.size, np.uint8)
    wide[::2] = rd.buf
    t2, _ = db.classify(wide[::2], rd.offsets, rd.mates_buf, rd.mate_offsets)
    assert np.array_equal(t2, ot)


@pytest.mark.parametrize("where", ["host", "device"])
def test_backward_offsets_are_invalid_arg_and_handle_survives(mc, built, where):
    refs, db, o = built
    rd = synth.single_end_reads(refs, 300, length=100, seed=12)
    bad = rd.offsets.astype(np.uint64).copy()
    bad[1], bad[2] = 100, 50  # record 0 = [0, 100), record 1 = [100, 50): backwards; record 2 starts at 50
    bad[3] = 150
    buf, offs = rd.buf, bad
    if where == "device":
        buf = torch.from_numpy(rd.buf).cuda()
        offs = torch.from_numpy(bad.astype(np.int64)).cuda()
    with pytest.raises(mc.MCError) as e:
        db.classify(buf, offs)
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    # record 1 starts before the batch's first byte in a second shape: [100, 0, 200]
    bad2 = rd.offsets.astype(np.uint64).copy()
    bad2[0], bad2[1] = 100, 0
    with pytest.raises(mc.MCError) as e:
        db.classify(rd.buf, bad2)
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    t, c = db.classify(rd.buf, rd.offsets)  # the handle is still usable
    ot, oc = o.classify(rd.buf, rd.offsets)
    assert np.array_equal(t, ot) and np.array_equal(c.view(np.uint32), oc.view(np.uint32))


def test_reserved_target_id_is_unknown(mc, built):
    refs, db, _ = built
    with pytest.raises(mc.MCError) as e:
        db.partition_of(0xFFFFFFFF)
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    assert db.partition_of(int(refs.target_ids[0])) == 0


def test_duplicate_id_rolls_back_the_insert(mc, oracle_mod):
    """The duplicate-id check runs while the GPU sketches the call's targets;
    a duplicate rolls the call back (pair-store cursors + HyperLogLog
    restored): the handle stays usable and the database equals the oracle's
    built from the accepted calls only."""
    refs = synth.strain_references(seed=5, n_targets=12, median_len=30_000, min_len=10_000, max_len=60_000,
                                   max_strains=4)
    cut = 6
    c0 = int(refs.offsets[cut])
    a = (refs.buf[:c0], refs.offsets[:cut + 1], refs.target_ids[:cut], refs.taxa[:cut])
    b = (refs.buf[c0:], refs.offsets[cut:] - c0, refs.target_ids[cut:].copy(), refs.taxa[cut:])
    bad = (b[0], b[1], b[2].copy(), b[3])
    bad[2][3] = refs.target_ids[1]  # collides with the first call
    db = mc.Database(refs.parent, n_partitions=2, capacity_bp=4 * refs.total_bp)
    db.insert_targets(*a)
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(*bad)
    assert e.value.code == mc.MC_ERR_INVALID_ARG and "duplicate" in str(e.value)
    with pytest.raises(mc.MCError):  # a duplicate inside one call
        dup = (b[0], b[1], b[2].copy(), b[3])
        dup[2][1] = dup[2][0]
        db.insert_targets(*dup)
    db.insert_targets(*b)
    db.finalize()
    o = oracle_mod.OracleDB(refs.parent, n_partitions=2)
    o.insert(*a)
    o.insert(*b)
    o.finalize()
    for p in range(2):
        assert all(np.array_equal(x, y) for x, y in zip(db.dump_partition(p), o.dump_partition(p))), p
    rd = synth.single_end_reads(refs, 800, length=100, seed=13)
    t, c = db.classify(rd.buf, rd.offsets)
    ot, oc = o.classify(rd.buf, rd.offsets)
    assert np.array_equal(t, ot) and np.array_equal(c.view(np.uint32), oc.view(np.uint32))


def test_failure_in_a_later_chunk_rolls_back(mc, oracle_mod, monkeypatch):
    """Validation and capacity are checked chunk by chunk while earlier chunks
    already sketch on the GPU: a failure in a later chunk (here: the static
    window capacity, then decreasing offsets) rolls the whole call back."""
    refs = synth.tiny_references(n_genomes=8, length=20_000)
    monkeypatch.setenv("MC_TEST_STAGE_BYTES", "45000")  # ~2 targets per host chunk
    db = mc.Database(refs.parent, capacity_bp=90_000, max_targets=8)  # windows for ~4.5 of the 8 targets
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
    assert e.value.code == mc.MC_ERR_CAPACITY
    bad = refs.offsets.astype(np.uint64).copy()
    bad[4] = bad[3] - 1  # target 3 ends before it starts
    with pytest.raises(mc.MCError) as e:
        db.insert_targets(refs.buf[:int(refs.offsets[4])], bad[:5], refs.target_ids[:4], refs.taxa[:4])
    assert e.value.code == mc.MC_ERR_INVALID_ARG
    keep = 3
    c = int(refs.offsets[keep])
    db.insert_targets(refs.buf[:c], refs.offsets[:keep + 1], refs.target_ids[:keep], refs.taxa[:keep])
    db.finalize()
    o = oracle_mod.OracleDB(refs.parent)
    o.insert(refs.buf[:c], refs.offsets[:keep + 1], refs.target_ids[:keep], refs.taxa[:keep])
    o.finalize()
    assert all(np.array_equal(x, y) for x, y in zip(db.dump_partition(0), o.dump_partition(0)))
