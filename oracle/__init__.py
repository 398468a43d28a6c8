"""MetaCache oracle: ctypes wrapper around oracle/oracle.cpp.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_2106_08150_b200`` never imports it and
shares no code with it (see oracle/oracle.cpp header for the citations and
the pins that hold it to the paper).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++ -O2, single-threaded C++17)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-pthread", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class Candidate(C.Structure):
    _fields_ = [("tgt", C.c_uint32), ("hits", C.c_uint32), ("win_beg", C.c_uint32), ("win_end", C.c_uint32)]


class SketchParams(C.Structure):
    _fields_ = [("k", C.c_uint32), ("s", C.c_uint32), ("w", C.c_uint32), ("canonical", C.c_uint32),
                ("table", C.POINTER(C.c_uint32))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u32, u64, vp, cp = C.c_uint32, C.c_uint64, C.c_void_p, C.c_char_p
        P = C.POINTER
        L.or_h1.restype = u32; L.or_h1.argtypes = [u32]
        L.or_window_count.restype = u64; L.or_window_count.argtypes = [u64, u32, u32]
        L.or_canonical_kmer.restype = u32; L.or_canonical_kmer.argtypes = [cp, u32, P(C.c_int)]
        L.or_sketch_sequence.restype = u64
        L.or_sketch_sequence.argtypes = [P(SketchParams), cp, u64, vp, vp]
        L.or_plan_partitions.restype = None; L.or_plan_partitions.argtypes = [u32, u32, vp, vp, vp]
        L.or_top_hits.restype = u32; L.or_top_hits.argtypes = [u64, vp, u32, u32, vp]
        L.or_merge_candidates.restype = u32; L.or_merge_candidates.argtypes = [u32, u32, vp, vp, vp]
        L.or_db_create.restype = vp
        L.or_db_create.argtypes = [u32, u32, u32, u32, u32, u32, u32, u32, u32, vp]
        L.or_db_destroy.restype = None; L.or_db_destroy.argtypes = [vp]
        L.or_db_set_insert_size_max.restype = None; L.or_db_set_insert_size_max.argtypes = [vp, u64]
        L.or_db_set_feature_filter.restype = None; L.or_db_set_feature_filter.argtypes = [vp, u64, vp]
        L.or_db_insert.restype = C.c_int; L.or_db_insert.argtypes = [vp, u32, vp, vp, vp, vp, vp]
        L.or_db_insert_restricted.restype = C.c_int
        L.or_db_insert_restricted.argtypes = [vp, u32, vp, vp, vp, vp, vp, u32]
        L.or_db_finalize.restype = None; L.or_db_finalize.argtypes = [vp]
        L.or_db_feature_locations.restype = u32; L.or_db_feature_locations.argtypes = [vp, u32, u32, vp, u32]
        L.or_db_dump_partition.restype = None; L.or_db_dump_partition.argtypes = [vp, u32, vp, vp, vp, vp, vp]
        L.or_lca.restype = u32; L.or_lca.argtypes = [vp, u32, u32]
        L.or_classify_candidates.restype = u32; L.or_classify_candidates.argtypes = [vp, u32, vp]
        L.or_sws.restype = u32; L.or_sws.argtypes = [vp, u64, u64, C.c_int]
        L.or_classify.restype = C.c_int
        L.or_classify.argtypes = [vp, u64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.or_classify_threads.restype = C.c_int
        L.or_classify_threads.argtypes = [vp, u64, vp, vp, vp, vp, vp, vp, u32]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


CAND_DTYPE = np.dtype([("tgt", "<u4"), ("hits", "<u4"), ("win_beg", "<u4"), ("win_end", "<u4")])
EMPTY_TGT = 0xFFFFFFFF


def h1(x: int) -> int:
    return lib().or_h1(x)


def window_count(L: int, k: int = 16, w: int = 127) -> int:
    return lib().or_window_count(L, k, w)


def canonical_kmer(kmer: str) -> int | None:
    ok = C.c_int(0)
    v = lib().or_canonical_kmer(kmer.encode(), len(kmer), C.byref(ok))
    return v if ok.value else None


def sketch(seq: bytes | str, k=16, s=16, w=127, canonical=True, table=None):
    """List (one entry per window) of sorted unique features (S6: may be short)."""
    if isinstance(seq, str):
        seq = seq.encode()
    nwin = window_count(len(seq), k, w)
    feats = np.zeros(max(nwin, 1) * s, np.uint32)
    counts = np.zeros(max(nwin, 1), np.uint32)
    tab = None
    if table is not None:
        table = np.ascontiguousarray(table, dtype=np.uint32)
        assert table.size == 4 ** k
        tab = table.ctypes.data_as(C.POINTER(C.c_uint32))
    p = SketchParams(k, s, w, 1 if canonical else 0, tab)
    n = lib().or_sketch_sequence(C.byref(p), seq, len(seq), _ptr(feats), _ptr(counts))
    return [feats[j * s: j * s + counts[j]].tolist() for j in range(n)]


def plan_partitions(P: int, lengths, running_bp=None):
    lengths = np.ascontiguousarray(lengths, dtype=np.uint64)
    run = np.zeros(P, np.uint64) if running_bp is None else running_bp
    out = np.zeros(lengths.size, np.uint32)
    lib().or_plan_partitions(P, lengths.size, _ptr(lengths), _ptr(run), _ptr(out))
    return out


def top_hits(locs, sws: int, m: int):
    locs = np.ascontiguousarray(locs, dtype=np.uint64)
    out = np.zeros(m, CAND_DTYPE)
    n = lib().or_top_hits(locs.size, _ptr(locs), sws, m, _ptr(out))
    return out[:n]


def merge_candidates(lists, m: int):
    P = len(lists)
    buf = np.zeros(P * m, CAND_DTYPE)
    sizes = np.zeros(P, np.uint32)
    for i, l in enumerate(lists):
        buf[i * m: i * m + len(l)] = l
        sizes[i] = len(l)
    out = np.zeros(m, CAND_DTYPE)
    n = lib().or_merge_candidates(P, m, _ptr(buf), _ptr(sizes), _ptr(out))
    return out[:n]


def pack_seqs(seqs):
    """list of bytes -> (concatenated uint8 array, uint64 offsets[n+1])."""
    seqs = [s.encode() if isinstance(s, str) else bytes(s) for s in seqs]
    offs = np.zeros(len(seqs) + 1, np.uint64)
    offs[1:] = np.cumsum([len(s) for s in seqs], dtype=np.uint64)
    buf = np.frombuffer(b"".join(seqs) + b"\0", dtype=np.uint8).copy()
    return buf, offs


class OracleDB:
    """Ordered-map MetaCache database (one std::map per partition)."""

    def __init__(self, parent, k=16, s=16, w=127, cap=254, m=4, hits_min=5, hits_diff=4, n_partitions=1,
                 insert_size_max=0):
        self.parent = np.ascontiguousarray(parent, dtype=np.uint32)
        self.k, self.s, self.w, self.cap, self.m = k, s, w, cap, m
        self.P = n_partitions
        self.h = lib().or_db_create(k, s, w, cap, m, hits_min, hits_diff, n_partitions,
                                    self.parent.size, _ptr(self.parent))
        if insert_size_max:  # reading S25 (pairs: sws from max(|r1|+|r2|, insert_size_max))
            lib().or_db_set_insert_size_max(self.h, insert_size_max)

    def close(self):
        if self.h:
            lib().or_db_destroy(self.h)
            self.h = None

    __del__ = close

    def set_feature_filter(self, feats):
        f = np.ascontiguousarray(feats, dtype=np.uint32)
        lib().or_db_set_feature_filter(self.h, f.size, _ptr(f))

    def insert(self, buf, offsets, ids, taxa, partition_ids=None):
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        taxa = np.ascontiguousarray(taxa, dtype=np.uint32)
        pid = None if partition_ids is None else np.ascontiguousarray(partition_ids, dtype=np.uint32)
        rc = lib().or_db_insert(self.h, ids.size, _ptr(buf), _ptr(offsets), _ptr(ids), _ptr(taxa), _ptr(pid))
        if rc != 0:
            raise ValueError("oracle insert rejected input")

    def insert_restricted(self, buf, offsets, ids, taxa, partition_ids=None, threads=None):
        """Feature-restricted insert (needs set_feature_filter first): targets
        sketched on `threads` host threads, filtered locations appended in
        insertion order."""
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        taxa = np.ascontiguousarray(taxa, dtype=np.uint32)
        pid = None if partition_ids is None else np.ascontiguousarray(partition_ids, dtype=np.uint32)
        threads = threads or max(1, len(os.sched_getaffinity(0)))
        rc = lib().or_db_insert_restricted(self.h, ids.size, _ptr(buf), _ptr(offsets), _ptr(ids), _ptr(taxa),
                                           _ptr(pid), threads)
        if rc != 0:
            raise ValueError("oracle restricted insert rejected input (filter set?)")

    def finalize(self):
        lib().or_db_finalize(self.h)

    def feature_locations(self, p: int, f: int):
        out = np.zeros(1 << 16, np.uint64)
        n = lib().or_db_feature_locations(self.h, p, f, _ptr(out), out.size)
        return out[:n]

    def dump_partition(self, p: int):
        nk, nv = C.c_uint64(0), C.c_uint64(0)
        lib().or_db_dump_partition(self.h, p, None, None, None, C.byref(nk), C.byref(nv))
        keys = np.zeros(nk.value, np.uint32)
        counts = np.zeros(nk.value, np.uint32)
        vals = np.zeros(nv.value, np.uint64)
        lib().or_db_dump_partition(self.h, p, _ptr(keys), _ptr(counts), _ptr(vals), C.byref(nk), C.byref(nv))
        return keys, counts, vals

    def lca(self, a: int, b: int) -> int:
        return lib().or_lca(self.h, a, b)

    def sws(self, len1: int, len2: int = 0, paired: bool = False) -> int:
        """Window range of the contiguous-range top hits for a record of mate
        lengths len1 / len2; `paired` = the record has a mate (reading S25 then
        applies insert_size_max)."""
        return lib().or_sws(self.h, len1, len2, 1 if paired else 0)

    def classify_candidates(self, cands) -> int:
        c = np.ascontiguousarray(cands, dtype=CAND_DTYPE)
        return lib().or_classify_candidates(self.h, c.size, _ptr(c))

    def classify_threads(self, reads_buf, read_offsets, mates_buf=None, mate_offsets=None, threads=None):
        """classify() on `threads` host threads (contiguous record slices; same results)."""
        n = len(read_offsets) - 1
        threads = threads or max(1, len(os.sched_getaffinity(0)))
        reads_buf = np.ascontiguousarray(reads_buf, dtype=np.uint8)
        read_offsets = np.ascontiguousarray(read_offsets, dtype=np.uint64)
        if mates_buf is not None:
            mates_buf = np.ascontiguousarray(mates_buf, dtype=np.uint8)
            mate_offsets = np.ascontiguousarray(mate_offsets, dtype=np.uint64)
        taxon = np.zeros(n, np.uint32)
        cand = np.zeros(n * self.m, CAND_DTYPE)
        rc = lib().or_classify_threads(self.h, n, _ptr(reads_buf), _ptr(read_offsets), _ptr(mates_buf),
                                       _ptr(mate_offsets), _ptr(taxon), _ptr(cand), threads)
        if rc != 0:
            raise RuntimeError("oracle classify before finalize")
        return taxon, cand.reshape(n, self.m)

    def classify(self, reads_buf, read_offsets, mates_buf=None, mate_offsets=None, per_partition=False):
        n = len(read_offsets) - 1
        reads_buf = np.ascontiguousarray(reads_buf, dtype=np.uint8)
        read_offsets = np.ascontiguousarray(read_offsets, dtype=np.uint64)
        if mates_buf is not None:
            mates_buf = np.ascontiguousarray(mates_buf, dtype=np.uint8)
            mate_offsets = np.ascontiguousarray(mate_offsets, dtype=np.uint64)
        taxon = np.zeros(n, np.uint32)
        cand = np.zeros(n * self.m, CAND_DTYPE)
        pc = np.zeros(n * self.P * self.m, CAND_DTYPE) if per_partition else None
        nl = np.zeros(n * self.P, np.uint64) if per_partition else None
        rc = lib().or_classify(self.h, n, _ptr(reads_buf), _ptr(read_offsets), _ptr(mates_buf),
                               _ptr(mate_offsets), _ptr(taxon), _ptr(cand), _ptr(pc), _ptr(nl))
        if rc != 0:
            raise RuntimeError("oracle classify before finalize")
        cand = cand.reshape(n, self.m)
        if per_partition:
            return taxon, cand, pc.reshape(n, self.P, self.m), nl.reshape(n, self.P)
        return taxon, cand
