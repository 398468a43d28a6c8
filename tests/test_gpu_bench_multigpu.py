"""bench.py's N = 2 launch configuration (one multi-GPU handle, partition g =
shard g's references, reads all-gathered per batch, exchange fused into the
merge), rehearsed with both shards on device 0, compared with the oracle
(P = 2) record by record: every candidate and every taxon, for the
device-resident (`value`) and the pinned-host (`e2e`) inputs."""
import numpy as np
import pytest

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


def test_bench_two_gpu_path_equals_oracle(mc, oracle_mod):
    import bench
    G = 2
    W = bench.Workload("small", G)
    devices = [0] * G
    inp = bench.Inputs(torch, W, devices)
    db = bench.make_group_db(mc, W, devices, read_batch=1 << 15)  # 4 batches of the 100k pairs
    o = oracle_mod.OracleDB(W.parent, n_partitions=G, m=bench.BENCH_M)
    for g, r in enumerate(W.shards):
        o.insert(r.buf, r.offsets, r.target_ids, r.taxa, np.full(r.n, g, np.uint32))
    o.finalize()
    rd = W.reads
    ot, oc = o.classify_threads(rd.buf, rd.offsets, rd.mates_buf, rd.mate_offsets)
    for device_resident in (True, False):
        inp.build(db, device_resident)
        inp.query(db, device_resident)
        torch.cuda.synchronize()
        t = (inp.d_tax if device_resident else inp.h_tax).cpu().numpy().view(np.uint32)
        c = (inp.d_cand if device_resident else inp.h_cand).cpu().numpy().view(np.uint32).reshape(rd.n, -1)
        bad = np.nonzero((c != oc.view(np.uint32).reshape(rd.n, -1)).any(1))[0]
        assert bad.size == 0, f"{bad.size} records differ (device_resident={device_resident}), first {bad[:5]}"
        assert np.array_equal(t, ot)
    st = db.stats()
    assert st["n_gpus"] == G and len(st["partitions"]) == G
    assert sum(p["bp"] for p in st["partitions"]) == W.total_bp
    db.close()
