"""C-ABI contract checks that need no GPU (-m "not gpu"): the library loads,
exports every symbol include/mc.h declares, host-only entry points behave,
and the package fails loudly without the extension."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mc():
    from paper_2106_08150_b200 import _build
    _build.build()
    import paper_2106_08150_b200 as m
    m.lib()
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mc_[a-z_]+)\s*\(", src)))


def test_header_declares_what_binding_lists(mc):
    assert declared_symbols() == sorted(mc.EXPORTS)


def test_library_exports_every_declared_symbol(mc):
    out = subprocess.check_output(["nm", "-D", "--defined-only", mc.LIB_PATH], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for s in declared_symbols():
        assert s in exported, s
        assert getattr(mc.lib(), s) is not None


def test_library_is_sm100a_cuda(mc):
    out = subprocess.check_output(["cuobjdump", "--list-elf", mc.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", mc.LIB_PATH], text=True)
    for k in ("k_sketch_partition", "k_sub_count", "k_sub_scatter", "k_sub_finalize", "k_heavy_select",
              "k_query_plan", "k_query_sketch_probe", "k_query_small", "k_query_medium", "k_query_large",
              "k_merge_classify"):
        assert k in sass, k


def test_config_defaults_are_the_papers(mc):
    c = mc.config()
    assert (c.k, c.sketch_size, c.window_len) == (16, 16, 127)
    assert c.max_locations_per_feature == 254
    assert c.max_candidates == 4                                        # P:596-598, Fig. 1
    assert (c.hits_min, c.hits_diff) == (5, 4)                          # S15 / S16
    assert c.insert_size_max == 0                                       # S10 unless set (S25)
    assert C.sizeof(mc.Config) == 128


def test_plan_partitions_matches_oracle(mc, oracle_mod):
    rng = np.random.default_rng(0)
    for P in (1, 2, 3, 8):
        lens = rng.integers(0, 10_000_000, 300).astype(np.uint64)
        run_a = np.zeros(P, np.uint64)
        run_b = np.zeros(P, np.uint64)
        a = np.concatenate([mc.plan_partitions(P, lens[:100], run_a), mc.plan_partitions(P, lens[100:], run_a)])
        b = np.concatenate([oracle_mod.plan_partitions(P, lens[:100], run_b),
                            oracle_mod.plan_partitions(P, lens[100:], run_b)])
        assert np.array_equal(a, b) and np.array_equal(run_a, run_b)


def test_bad_config_rejected_without_gpu_work(mc):
    for bad in (dict(k=0), dict(k=17), dict(sketch_size=0), dict(sketch_size=17), dict(window_len=10, k=16),
                dict(window_len=200)):
        with pytest.raises(mc.MCError) as e:
            mc.debug_sketch(np.zeros(1, np.uint8), np.zeros(1, np.uint64), **bad)
        assert e.value.code == mc.MC_ERR_INVALID_ARG
    with pytest.raises(mc.MCError):
        mc.Database([0, 1], k=0)
    for bad in (dict(insert_size_max=1022 * 112 + 1), dict(reserved2=1)):  # S25 bound, reserved field
        with pytest.raises(mc.MCError) as e:
            mc.Database([0, 1], **bad)
        assert e.value.code == mc.MC_ERR_INVALID_ARG, bad


def test_null_handle_calls_fail_cleanly(mc):
    L = mc.lib()
    assert L.mc_db_finalize(None) == mc.MC_ERR_INVALID_ARG
    assert L.mc_db_clear(None) == mc.MC_ERR_INVALID_ARG
    L.mc_db_destroy(None)  # no-op
    assert b"NULL" in L.mc_last_error()


def test_missing_extension_fails_loudly(tmp_path):
    """The product path has no CPU fallback: without libmc.so the package raises."""
    pkg = os.path.join(ROOT, "paper_2106_08150_b200", "__init__.py")
    d = tmp_path / "paper_2106_08150_b200"
    d.mkdir()
    (d / "__init__.py").write_text(open(pkg).read())
    code = "import paper_2106_08150_b200 as m\ntry:\n    m.lib()\nexcept ImportError as e:\n    print('RAISED', e)\n"
    out = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert "RAISED" in out.stdout and "no CPU fallback" in out.stdout


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2106_08150_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "oracle.cpp" not in txt and "or_" + "db" not in txt, f


def test_corrupt_database_file_rejected_without_gpu(mc, tmp_path):
    """mc_db_load reads the header and the taxonomy before touching a GPU: a
    corrupt array count (here 2^40 parents) or a truncated file must come back
    as INVALID_ARG, never as a huge allocation or an exception through the ABI."""
    cfg = mc.config()
    head = b"MCDB\0\0\0\x02" + np.uint64(C.sizeof(cfg)).tobytes() + bytes(cfg)
    cases = {
        "huge_count": head + np.uint64(1 << 40).tobytes() + b"\0" * 64,
        "truncated_taxonomy": head + np.uint64(1000).tobytes() + b"\0" * 40,
        "bad_magic": b"XXXX" + head[4:],
        "empty": b"",
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.mcdb"
        p.write_bytes(blob)
        with pytest.raises(mc.MCError) as e:
            mc.Database.load(str(p))
        assert e.value.code == mc.MC_ERR_INVALID_ARG, name
