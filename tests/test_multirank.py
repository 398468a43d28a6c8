"""N>1 host logic on CPU with gloo, world_size 2: target-partitioned shards,
read all-gather and the candidate all-to-all (paper_2106_08150_b200.dist),
checked against a single-process oracle over the whole database.  The
per-partition hits come from the oracle here (no GPU); on the B200s the same
exchange carries mc_query_partials output into mc_merge_classify."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2106_08150_b200 import dist as mcd
        oracle.build()
        kw = dict(n_targets=10, median_len=40_000, min_len=10_000, max_len=60_000, max_strains=4)
        refs = synth.subset_shard(rank, world, **kw)
        # this rank's partition (global partition id = rank)
        odb = oracle.OracleDB(refs.parent, n_partitions=1)
        odb.insert(refs.buf, refs.offsets, refs.target_ids, refs.taxa)
        odb.finalize()
        # each rank draws its share of pairs from its shard; all-gather -> full batch
        n_total = 301
        lo, hi = mcd.slice_bounds(n_total, world, rank)
        rd = synth.paired_reads(refs, hi - lo, length=150, seed=(synth.READ_SEED + rank))
        counts = [b - a for a, b in (mcd.slice_bounds(n_total, world, r) for r in range(world))]
        r1 = mcd.allgather_records(torch.from_numpy(rd.buf.reshape(-1, 150)), counts)
        r2 = mcd.allgather_records(torch.from_numpy(rd.mates_buf.reshape(-1, 150)), counts)
        offs = np.arange(n_total + 1, dtype=np.uint64) * 150
        _, _, pc, _ = odb.classify(r1.numpy().reshape(-1), offs, r2.numpy().reshape(-1), offs, per_partition=True)
        m = odb.m
        hits = np.zeros((n_total, m, 6), np.uint32)
        hits[:, :, :4] = pc[:, 0, :].view(np.uint32).reshape(n_total, m, 4)
        for i in range(n_total):
            for j in range(m):
                t = int(hits[i, j, 0])
                if t != 0xFFFFFFFF:
                    hits[i, j, 4] = refs.taxa[np.nonzero(refs.target_ids == t)[0][0]]
        mine = mcd.exchange_hits(torch.from_numpy(hits.view(np.int32).reshape(n_total, m * 6)), n_total)
        out_q.put((rank, lo, hi, mine.numpy().view(np.uint32), r1.numpy(), r2.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    import oracle
    kw = dict(n_targets=10, median_len=40_000, min_len=10_000, max_len=60_000, max_strains=4)
    shards = [synth.subset_shard(r, world, **kw) for r in range(world)]
    # single-process oracle over both partitions (explicit partition ids = shard)
    full = oracle.OracleDB(shards[0].parent, n_partitions=world)
    for r, s in enumerate(shards):
        full.insert(s.buf, s.offsets, s.target_ids, s.taxa, np.full(s.n, r, np.uint32))
    full.finalize()
    r1, r2 = res[0][4], res[0][5]
    assert np.array_equal(r1, res[1][4])  # every rank holds the same gathered batch
    n_total = r1.shape[0]
    offs = np.arange(n_total + 1, dtype=np.uint64) * 150
    taxon, cand, pc, _ = full.classify(r1.reshape(-1), offs, r2.reshape(-1), offs, per_partition=True)
    m = full.m
    for rank, lo, hi, mine, _, _ in res:
        mine = mine.reshape(hi - lo, world, m, 6)
        # rank's slice holds, per record, partition p's list from rank p
        assert np.array_equal(mine[:, :, :, :4].reshape(-1), pc[lo:hi].view(np.uint32).reshape(-1))
        # merging the exchanged lists reproduces the global top-m and taxon
        for i in range(hi - lo):
            lists = [np.array([tuple(x[:4]) for x in mine[i, p] if x[0] != 0xFFFFFFFF], oracle.CAND_DTYPE)
                     for p in range(world)]
            merged = oracle.merge_candidates(lists, m)
            exp = cand[lo + i][cand[lo + i]["tgt"] != 0xFFFFFFFF]
            assert np.array_equal(merged, exp)
            assert full.classify_candidates(merged) == taxon[lo + i]


def _flat_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_08150_b200 import dist as mcd
        kw = dict(n_targets=6, median_len=30_000, min_len=10_000, max_len=50_000, max_strains=3)
        refs = synth.subset_shard(rank, world, **kw)
        rd = synth.miseq_reads(refs, 97 + 50 * rank, seed=synth.READ_SEED + 40 + rank)  # ragged: 97 / 147 reads
        buf, offs = mcd.allgather_flat(torch.from_numpy(rd.buf), torch.from_numpy(rd.offsets.astype(np.int64)))
        # with the sizes known up front: no size exchange, same result
        o = offs.numpy()
        sizes = [(97, int(o[97])), (147, int(o[-1] - o[97]))]
        buf2, offs2 = mcd.allgather_flat(torch.from_numpy(rd.buf), torch.from_numpy(rd.offsets.astype(np.int64)),
                                         sizes=sizes)
        assert np.array_equal(buf2.numpy(), buf.numpy()) and np.array_equal(offs2.numpy(), o)
        out_q.put((rank, rd.buf, rd.offsets, buf.numpy(), offs.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_allgather_of_variable_length_reads():
    """The multi-node read exchange for variable-length single-end records
    (HiSeq / MiSeq-shaped): every rank ends with the rank-ordered concatenation,
    with or without the sizes known up front."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_flat_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp_buf = np.concatenate([r[1] for r in res])
    exp_offs = np.concatenate([[0], res[0][2][1:], res[1][2][1:] + res[0][2][-1]]).astype(np.int64)
    for _, _, _, buf, offs in res:
        assert np.array_equal(buf, exp_buf)
        assert np.array_equal(offs, exp_offs)
    assert exp_offs.size == 97 + 147 + 1
