"""B200-native MetaCache-GPU hot path: thin ctypes binding over libmc.so.

Argument marshalling only -- every step of the method runs in the CUDA
kernels behind the C-ABI declared in include/mc.h (names are the same).
There is no CPU fallback: importing this package raises if libmc.so is
missing; build it with ``python -m paper_2106_08150_b200._build`` or
``__graft_entry__.build()``.

Array arguments may be numpy arrays (host), torch tensors (host, pinned, or
CUDA device memory) or raw integer addresses.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MC_LIB_PATH") or os.path.join(_HERE, "libmc.so")  # override: A/B builds

MC_OK = 0
MC_ERR_INVALID_ARG = -1
MC_ERR_STATE = -2
MC_ERR_CAPACITY = -3
MC_ERR_CUDA = -4
MC_ERR_OOM = -5
MC_ERR_PEER = -6  # multi-GPU transport (peer access over NVLink); SURVEY §8(b)'s MC_ERR_NCCL
MC_ERR_NCCL = MC_ERR_PEER
EMPTY_TGT = 0xFFFFFFFF

# every entry point include/mc.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "mc_config_init", "mc_db_create", "mc_db_insert_targets", "mc_db_insert_target_batches", "mc_db_finalize",
    "mc_classify",
    "mc_query_partials", "mc_merge_classify", "mc_db_destroy", "mc_db_clear", "mc_db_set_stream",
    "mc_last_error", "mc_plan_partitions", "mc_debug_sketch", "mc_db_partition_of",
    "mc_db_feature_locations", "mc_db_dump_partition", "mc_db_stats", "mc_db_reset_stats",
    "mc_db_save", "mc_db_load", "mc_db_get_config",
]


class MCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("k", C.c_uint32), ("sketch_size", C.c_uint32), ("window_len", C.c_uint32),
                ("max_locations_per_feature", C.c_uint32), ("max_candidates", C.c_uint32),
                ("hits_min", C.c_uint32), ("hits_diff", C.c_uint32), ("n_partitions", C.c_uint32),
                ("partition_begin", C.c_uint32), ("n_local_partitions", C.c_uint32), ("device", C.c_int32),
                ("flags", C.c_uint32), ("capacity_bp", C.c_uint64), ("max_targets", C.c_uint64),
                ("read_batch", C.c_uint64), ("table_slots_per_location", C.c_double),
                ("insert_size_max", C.c_uint32), ("reserved2", C.c_uint32),
                ("n_gpus", C.c_uint32), ("devices", C.c_int32 * 8)]


class TargetBatch(C.Structure):
    _fields_ = [("n", C.c_uint32), ("seqs", C.c_void_p), ("offsets", C.c_void_p), ("target_ids", C.c_void_p),
                ("taxa", C.c_void_p), ("partition_ids", C.c_void_p)]


class Taxonomy(C.Structure):
    _fields_ = [("n_taxa", C.c_uint32), ("parent", C.c_void_p), ("rank", C.c_void_p)]


CAND_DTYPE = np.dtype([("tgt", "<u4"), ("hits", "<u4"), ("win_beg", "<u4"), ("win_end", "<u4")])
HIT_DTYPE = np.dtype([("tgt", "<u4"), ("hits", "<u4"), ("win_beg", "<u4"), ("win_end", "<u4"),
                      ("taxon", "<u4"), ("reserved", "<u4")])

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, ip = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "mc_config_init": (None, [vp]),
            "mc_db_create": (ip, [vp, vp, vp]),
            "mc_db_insert_targets": (ip, [vp, u32, vp, vp, vp, vp, vp]),
            "mc_db_insert_target_batches": (ip, [vp, u32, vp]),
            "mc_db_finalize": (ip, [vp]),
            "mc_classify": (ip, [vp, u64, vp, vp, vp, vp, vp, vp]),
            "mc_query_partials": (ip, [vp, u64, vp, vp, vp, vp, vp]),
            "mc_merge_classify": (ip, [vp, u64, u32, vp, vp, vp]),
            "mc_db_destroy": (None, [vp]),
            "mc_db_clear": (ip, [vp]),
            "mc_db_set_stream": (ip, [vp, vp]),
            "mc_last_error": (C.c_char_p, []),
            "mc_plan_partitions": (ip, [u32, u32, vp, vp, vp]),
            "mc_debug_sketch": (ip, [vp, u32, vp, vp, vp, vp, vp]),
            "mc_db_partition_of": (ip, [vp, u32, vp]),
            "mc_db_feature_locations": (ip, [vp, u32, u32, vp, u32, vp]),
            "mc_db_dump_partition": (ip, [vp, u32, vp, vp, vp, vp, vp]),
            "mc_db_stats": (ip, [vp, vp, u64]),
            "mc_db_reset_stats": (ip, [vp]),
            "mc_db_save": (ip, [vp, C.c_char_p]),
            "mc_db_load": (ip, [C.c_char_p, C.c_int32, vp]),
            "mc_db_get_config": (ip, [vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != MC_OK:
        raise MCError(rc, lib().mc_last_error().decode(errors="replace"))


def _addr(x):
    """numpy array / torch tensor / int / None -> raw address (no copies)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


def _np(x, dtype):
    if isinstance(x, np.ndarray) or isinstance(x, (list, tuple)):
        return np.ascontiguousarray(x, dtype=dtype)
    return x


def config(**kw) -> Config:
    c = Config()
    lib().mc_config_init(C.byref(c))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise TypeError(f"unknown config field {k}")
        if k == "devices":  # list of device ordinals of the shards (multi-GPU handle)
            v = list(v) + [-1] * (8 - len(v))
            v = (C.c_int32 * 8)(*v)
        setattr(c, k, v)
    return c


def plan_partitions(P: int, lengths, running_bp=None) -> np.ndarray:
    lengths = np.ascontiguousarray(lengths, dtype=np.uint64)
    run = np.zeros(P, np.uint64) if running_bp is None else running_bp
    out = np.zeros(lengths.size, np.uint32)
    _check(lib().mc_plan_partitions(P, lengths.size, _addr(lengths), _addr(run), _addr(out)))
    return out


def debug_sketch(buf, offsets, **cfg):
    """GPU sketches of every window: returns (features[W, s], counts[W], window_offsets[n+1])."""
    c = config(**cfg)
    offsets = _np(offsets, np.uint64)
    n = (len(offsets) if isinstance(offsets, np.ndarray) else offsets.numel()) - 1
    wo = np.zeros(n + 1, np.uint64)
    buf = _np(buf, np.uint8)
    _check(lib().mc_debug_sketch(C.byref(c), n, _addr(buf), _addr(offsets), None, None, _addr(wo)))
    W = int(wo[-1])
    feats = np.zeros(max(W, 1) * c.sketch_size, np.uint32)
    counts = np.zeros(max(W, 1), np.uint32)
    _check(lib().mc_debug_sketch(C.byref(c), n, _addr(buf), _addr(offsets), _addr(feats), _addr(counts), _addr(wo)))
    return feats[:W * c.sketch_size].reshape(W, c.sketch_size), counts[:W], wo


class Database:
    """One mc_db handle: one GPU with one or more logical partitions, or (n_gpus
    = G > 1) G GPUs, shard g holding partitions [g P/G, (g+1) P/G) on devices[g]."""

    def __init__(self, parent, rank=None, **cfg):
        self.cfg = config(**cfg)
        self._parent = np.ascontiguousarray(parent, dtype=np.uint32)
        self._rank = None if rank is None else np.ascontiguousarray(rank, dtype=np.uint8)
        tax = Taxonomy(self._parent.size, _addr(self._parent), _addr(self._rank))
        h = C.c_void_p()
        _check(lib().mc_db_create(C.byref(self.cfg), C.byref(tax), C.byref(h)))
        self.h = h
        self.m = self.cfg.max_candidates
        P = self.cfg.n_partitions
        self.n_local = self.cfg.n_local_partitions or P

    @classmethod
    def load(cls, path: str, device: int = -1) -> "Database":
        """A finalized handle from an mc_db_save file (condensed dump/load)."""
        h = C.c_void_p()
        _check(lib().mc_db_load(os.fsencode(path), device, C.byref(h)))
        self = cls.__new__(cls)
        self.h = h
        self.cfg = Config()
        _check(lib().mc_db_get_config(self.h, C.byref(self.cfg)))
        self.m = self.cfg.max_candidates
        self.n_local = self.cfg.n_local_partitions or self.cfg.n_partitions
        return self

    def save(self, path: str):
        _check(lib().mc_db_save(self.h, os.fsencode(path)))

    def close(self):
        if getattr(self, "h", None):
            lib().mc_db_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- lifecycle ----------------------------------------------------------
    def insert_targets(self, buf, offsets, target_ids, taxa, partition_ids=None):
        offsets = _np(offsets, np.uint64)
        target_ids = _np(target_ids, np.uint32)
        taxa = _np(taxa, np.uint32)
        partition_ids = _np(partition_ids, np.uint32)
        buf = _np(buf, np.uint8)  # (bound to a local: a converted copy must outlive the C call)
        n = len(target_ids) if isinstance(target_ids, np.ndarray) else target_ids.numel()
        _check(lib().mc_db_insert_targets(self.h, n, _addr(buf), _addr(offsets), _addr(target_ids),
                                          _addr(taxa), _addr(partition_ids)))

    def insert_target_batches(self, batches):
        """batches: list of (buf, offsets, target_ids, taxa, partition_ids-or-None); on a
        multi-GPU handle every device builds its partitions' share concurrently."""
        keep, arr = [], (TargetBatch * max(len(batches), 1))()
        for i, (buf, offsets, target_ids, taxa, pids) in enumerate(batches):
            buf = _np(buf, np.uint8)
            offsets = _np(offsets, np.uint64)
            target_ids = _np(target_ids, np.uint32)
            taxa = _np(taxa, np.uint32)
            pids = _np(pids, np.uint32)
            keep += [buf, offsets, target_ids, taxa, pids]  # converted copies outlive the C call
            n = len(target_ids) if isinstance(target_ids, np.ndarray) else target_ids.numel()
            arr[i] = TargetBatch(n, _addr(buf), _addr(offsets), _addr(target_ids), _addr(taxa), _addr(pids))
        _check(lib().mc_db_insert_target_batches(self.h, len(batches), arr))

    def finalize(self):
        _check(lib().mc_db_finalize(self.h))

    def clear(self):
        _check(lib().mc_db_clear(self.h))

    def set_stream(self, stream):
        """stream: torch.cuda.Stream / raw cudaStream_t int / None."""
        s = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        _check(lib().mc_db_set_stream(self.h, s))

    # ---- query --------------------------------------------------------------
    def classify(self, reads, read_offsets, mates=None, mate_offsets=None, out_taxon=None, out_candidates=None,
                 want_candidates=True):
        read_offsets = _np(read_offsets, np.uint64)
        mate_offsets = _np(mate_offsets, np.uint64)
        reads, mates = _np(reads, np.uint8), _np(mates, np.uint8)  # locals: copies outlive the C call
        n = (len(read_offsets) if isinstance(read_offsets, np.ndarray) else read_offsets.numel()) - 1
        if out_taxon is None:
            out_taxon = np.zeros(n, np.uint32)
        if out_candidates is None and want_candidates:
            out_candidates = np.zeros(n * self.m, CAND_DTYPE)
        _check(lib().mc_classify(self.h, n, _addr(reads), _addr(read_offsets), _addr(mates), _addr(mate_offsets),
                                 _addr(out_taxon), _addr(out_candidates)))
        if isinstance(out_candidates, np.ndarray):
            out_candidates = out_candidates.reshape(n, self.m)
        return out_taxon, out_candidates

    def query_partials(self, reads, read_offsets, mates=None, mate_offsets=None, out_hits=None):
        read_offsets = _np(read_offsets, np.uint64)
        mate_offsets = _np(mate_offsets, np.uint64)
        reads, mates = _np(reads, np.uint8), _np(mates, np.uint8)  # locals: copies outlive the C call
        n = (len(read_offsets) if isinstance(read_offsets, np.ndarray) else read_offsets.numel()) - 1
        if out_hits is None:
            out_hits = np.zeros(n * self.n_local * self.m, HIT_DTYPE)
        _check(lib().mc_query_partials(self.h, n, _addr(reads), _addr(read_offsets), _addr(mates),
                                       _addr(mate_offsets), _addr(out_hits)))
        if isinstance(out_hits, np.ndarray):
            out_hits = out_hits.reshape(n, self.n_local, self.m)
        return out_hits

    def merge_classify(self, hits, n_lists: int, n: int | None = None, out_taxon=None, out_candidates=None):
        if isinstance(hits, np.ndarray):
            hits = np.ascontiguousarray(hits.reshape(-1), dtype=HIT_DTYPE)
            n = hits.size // (n_lists * self.m)
        if out_taxon is None:
            out_taxon = np.zeros(n, np.uint32)
        if out_candidates is None:
            out_candidates = np.zeros(n * self.m, CAND_DTYPE)
        _check(lib().mc_merge_classify(self.h, n, n_lists, _addr(hits), _addr(out_taxon), _addr(out_candidates)))
        if isinstance(out_candidates, np.ndarray):
            out_candidates = out_candidates.reshape(n, self.m)
        return out_taxon, out_candidates

    # ---- diagnostics --------------------------------------------------------
    def partition_of(self, target_id: int) -> int:
        p = C.c_uint32()
        _check(lib().mc_db_partition_of(self.h, target_id, C.byref(p)))
        return p.value

    def feature_locations(self, partition: int, feature: int) -> np.ndarray:
        out = np.zeros(4096, np.uint64)
        n = C.c_uint32()
        _check(lib().mc_db_feature_locations(self.h, partition, feature, _addr(out), out.size, C.byref(n)))
        return out[:n.value]

    def dump_partition(self, partition: int):
        nk, nv = C.c_uint64(), C.c_uint64()
        _check(lib().mc_db_dump_partition(self.h, partition, None, None, None, C.byref(nk), C.byref(nv)))
        keys = np.zeros(max(nk.value, 1), np.uint32)
        counts = np.zeros(max(nk.value, 1), np.uint32)
        vals = np.zeros(max(nv.value, 1), np.uint64)
        _check(lib().mc_db_dump_partition(self.h, partition, _addr(keys), _addr(counts), _addr(vals),
                                          C.byref(nk), C.byref(nv)))
        return keys[:nk.value], counts[:nk.value], vals[:nv.value]

    def stats(self) -> dict:
        buf = C.create_string_buffer(1 << 16)
        _check(lib().mc_db_stats(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def reset_stats(self):
        _check(lib().mc_db_reset_stats(self.h))
