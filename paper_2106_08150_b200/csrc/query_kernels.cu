// Query-side kernels (Q2-Q9): read sketch + key-table probe + location gather
// + per-record sort + window counts + contiguous-range top hits (per
// partition), then partition merge + classification.
//
// Paper: §4.2 P:584-618 (query), §5.2 steps (1)-(8) P:680-691, §5.3
// (minhash + query kernel), §5.4 P:743-752 (compaction), §5.5
// (segmented sort), §5.6 P:771-793 (top candidate generation).
//
// B200 design: instead of materialising all location lists and
// running a batch-wide segmented sort (the paper's dominant query cost, F5
// P:946-950), each record is processed end to end by one group -- a warp
// (small bin), a 128-thread CTA (medium) or a 512-thread CTA (large) --
// entirely in shared memory: every gathered location is counted straight
// into a per-record shared-memory hash keyed by ranked window id (the window
// count statistic, compaction and sort subsumed), each hit window's range sum
// over the next sws-1 windows is read back from the hash, and the top-m
// targets are reduced out.  Records with more unique windows than a bin's
// hash holds are deferred to the next bin (size-binned like Hou et al. [12],
// P:283-296).
#include <algorithm>

#include "mc_block.cuh"
#include "mc_kernels.cuh"

namespace mc {

constexpr uint32_t kEmptyTgt = 0xffffffffu;
constexpr uint32_t kSlotTile = 256;  // read windows per CTA tile in the sketch+probe kernel
#ifndef MC_SMALL_U
#define MC_SMALL_U 4
#endif
#ifndef MC_QPROF
#define MC_QPROF 0  // diagnostic build: small-bin work counters (mc_debug_qprof)
#endif
#if MC_QPROF
__device__ unsigned long long g_qprof[16];
#define QP(...) __VA_ARGS__
#else
#define QP(...)
#endif
#ifndef MC_PRECLAIM
#define MC_PRECLAIM 0
#endif
#ifndef MC_PRECLAIM_MINLEN
#define MC_PRECLAIM_MINLEN 8
#endif
#ifndef MC_FIND4
#define MC_FIND4 1
#endif

// Window counts of a block entry: four 16-bit lanes (uint2), or four 8-bit
// lanes (one word) where a record has <= 255 features, so no count overflows
template <int CB>
struct Cnt4;
template <>
struct Cnt4<16> {
  using T = uint2;
  static constexpr uint32_t bytes = 8;
  __device__ __forceinline__ static uint2 unpack(uint2 w) { return w; }
  __device__ __forceinline__ static void add(uint32_t* c32, uint32_t slot, uint32_t loc) {
    atomicAdd(&c32[2 * slot + ((loc >> 1) & 1u)], 1u << (16 * (loc & 1u)));
  }
};
template <>
struct Cnt4<8> {
  using T = uint32_t;
  static constexpr uint32_t bytes = 4;
  __device__ __forceinline__ static uint2 unpack(uint32_t w) {  // -> 16-bit lanes
    return make_uint2(__byte_perm(w, 0u, 0x4140u), __byte_perm(w, 0u, 0x4342u));
  }
  __device__ __forceinline__ static void add(uint32_t* c32, uint32_t slot, uint32_t loc) {
    atomicAdd(&c32[slot], __funnelshift_l(0u, 1u, loc << 3));  // 1 << 8 (loc & 3): the wrap shift takes it mod 32
  }
};

template <uint32_t H, uint32_t FCAP, int NT, int CB = 16>
struct RecLayout {
  // byte offsets inside the group's shared-memory slice
  static constexpr uint32_t foff = 0;                                    // uint64[FCAP] list offsets
  static constexpr uint32_t fcnt = foff + 8 * FCAP;                      // uint32[FCAP] list lengths
  static constexpr uint32_t fpos = fcnt + 4 * FCAP;                      // uint32[FCAP+1] scan of lengths
  static constexpr uint32_t bcnt = (fpos + 4 * (FCAP + 1) + 15) & ~15u;  // Cnt4[H] window counts
  static constexpr uint32_t bkey = bcnt + Cnt4<CB>::bytes * H;           // uint32[H] block id (window >> 2)
  static constexpr uint32_t scr = bkey + 4 * H;                          // uint32[NT/32+2]
  static constexpr uint32_t scr64 = (scr + 4 * (NT / 32 + 2) + 7) & ~7u;  // uint64[NT/32]
  static constexpr uint32_t meta = scr64 + 8 * (NT / 32);                // uint32[4]: overflow, winner target
  static constexpr uint32_t bytes = (meta + 16 + 15) & ~15u;
};

__device__ __forceinline__ uint32_t n_windows(uint64_t L, const SketchCfg& c) {
  return L < c.k ? 0u : (uint32_t)((L - c.k + c.stride) / c.stride);  // ceil((L-k+1)/stride)
}

__device__ __forceinline__ void write_hit(HitRec* o, uint32_t tgt, uint32_t hits, uint32_t b, uint32_t e,
                                          uint32_t taxon) {
  o->tgt = tgt;
  o->hits = hits;
  o->win_beg = b;
  o->win_end = e;
  o->taxon = taxon;
  o->reserved = 0;
}

enum : int { kDone = 0, kDefer = 1 };
constexpr uint32_t kEmptyLoc = 0xffffffffu;  // ranked window ids (and block ids) never reach this value

__device__ __forceinline__ uint32_t hslot(uint32_t x, uint32_t lg) { return (x * 2654435761u) >> (32 - lg); }

// The record's block hash is probed in BUCKETS of 4 slots (one LDS.128 reads
// a bucket's 4 keys): linear probing over buckets, slots claimed in order, so
// a key is absent once a bucket with an empty slot has been passed.  Probe
// chains -- and the lanes of a warp waiting on the longest one -- stay short.
// index of the first slot of bucket q holding x, 4 if none
__device__ __forceinline__ uint32_t find4(uint4 q, uint32_t x) {
#if MC_FIND4
  uint32_t i = q.w == x ? 3u : 4u;  // a select chain: no mask, no find-first-set
  i = q.z == x ? 2u : i;
  i = q.y == x ? 1u : i;
  return q.x == x ? 0u : i;
#else
  const uint32_t mm = (q.x == x ? 1u : 0u) | (q.y == x ? 2u : 0u) | (q.z == x ? 4u : 0u) | (q.w == x ? 8u : 0u);
  return mm ? __ffs(mm) - 1 : 4u;
#endif
}

// the 4 window counts of block `kb` in the record's hash (0 if absent); lg = log2 slots
template <typename CT>
__device__ __forceinline__ uint2 blookup(const uint32_t* bkey, const CT* bcnt, uint32_t lg, uint32_t kb) {
  using C4 = Cnt4<sizeof(CT) == 8 ? 16 : 8>;
  const uint32_t bmask = (1u << (lg - 2)) - 1u;
  for (uint32_t b = hslot(kb, lg - 2), i = 0; i <= bmask; ++i, b = (b + 1) & bmask) {
    const uint4 q = reinterpret_cast<const uint4*>(bkey)[b];
    const uint32_t mi = find4(q, kb);
    if (mi < 4) return C4::unpack(bcnt[4 * b + mi]);
    if (find4(q, kEmptyLoc) < 4) break;
  }
  return make_uint2(0, 0);
}

// slot of block `kb`, claimed if new (*claimed = 1); -1 if the table is full
__device__ __forceinline__ int binsert(uint32_t* bkey, uint32_t lg, uint32_t kb, uint32_t* claimed) {
  const uint32_t bmask = (1u << (lg - 2)) - 1u;
  uint32_t b = hslot(kb, lg - 2);
  for (uint32_t i = 0; i <= bmask;) {
    QP(++claimed[1]);
    const uint4 q = reinterpret_cast<const uint4*>(bkey)[b];
    const uint32_t mi = find4(q, kb);
    if (mi < 4) return (int)(4 * b + mi);
    const uint32_t ei = find4(q, kEmptyLoc);
    if (ei == 4) {
      b = (b + 1) & bmask;
      ++i;
      continue;
    }
    const uint32_t slot = 4 * b + ei;
    const uint32_t old = atomicCAS(&bkey[slot], kEmptyLoc, kb);
    if (old == kEmptyLoc) {
      *claimed = 1;
      return (int)slot;
    }
    if (old == kb) return (int)slot;
    QP(++claimed[2]);
    // lost the slot to another block: re-read this bucket
  }
  return -1;
}

__device__ __forceinline__ uint32_t cnt16(uint2 w, uint32_t q) { return ((q < 2 ? w.x : w.y) >> (16 * (q & 1))) & 0xffffu; }

// sum of the four 16-bit window counts of a block entry
__device__ __forceinline__ uint32_t hsum16(uint2 w) { return ((w.x + w.y) * 0x10001u) >> 16; }

// Best range start among the 4 windows of a block (S11: most hits, then the
// smallest start; only starts with hits), its range sum over SWS windows and
// its tight end offset.  w0 = the block, w1 / w2 = the next two blocks.
template <int SWS>
__device__ __forceinline__ void block_best(uint2 w0, uint2 w1, uint2 w2, uint32_t& bs, uint32_t& bi, uint32_t& be) {
  static_assert(SWS >= 2 && SWS <= 8, "3 blocks cover starts 0..3 plus SWS - 1 windows");
  uint32_t c[12];
  c[0] = w0.x & 0xffffu; c[1] = w0.x >> 16; c[2] = w0.y & 0xffffu; c[3] = w0.y >> 16;
  c[4] = w1.x & 0xffffu; c[5] = w1.x >> 16; c[6] = w1.y & 0xffffu; c[7] = w1.y >> 16;
  c[8] = w2.x & 0xffffu; c[9] = w2.x >> 16; c[10] = w2.y & 0xffffu; c[11] = w2.y >> 16;
  uint32_t s = 0, nz = 0;
#pragma unroll
  for (int d = 0; d < SWS; ++d) s += c[d];
#pragma unroll
  for (int q = 0; q < SWS + 3; ++q) nz |= (c[q] != 0 ? 1u : 0u) << q;
  bs = 0;
  bi = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i) s += c[i + SWS - 1] - c[i - 1];  // slide the range by one window
    if (c[i] != 0 && s > bs) { bs = s; bi = (uint32_t)i; }  // strict: smallest start wins ties
  }
  be = 31u - __clz(nz & ((2u << (bi + SWS - 1)) - 1u)) - bi;  // last hit window of the range
}

// Per-thread list of the best M candidates with distinct targets, ordered by
// key = hits << 32 | ~window (descending; 0 = empty).
template <int M>
struct TopList {
  uint64_t k[M];
  uint32_t t[M], e[M];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < M; ++i) k[i] = 0, t[i] = 0, e[i] = 0;
  }
  __device__ __forceinline__ void remove_target(uint32_t tt) {
    bool found = false;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      found |= k[i] != 0 && t[i] == tt;
      if (found) {
        k[i] = i + 1 < M ? k[i + 1] : 0ull;
        t[i] = i + 1 < M ? t[i + 1] : 0u;
        e[i] = i + 1 < M ? e[i + 1] : 0u;
      }
    }
  }
  // key > k[M-1] must hold
  __device__ __forceinline__ void insert(uint64_t key, uint32_t tt, uint32_t ee) {
#pragma unroll
    for (int i = 0; i < M; ++i)
      if (k[i] != 0 && t[i] == tt) {
        if (key <= k[i]) return;  // the target's better candidate is already listed
        remove_target(tt);
        break;
      }
#pragma unroll
    for (int i = M - 1; i > 0; --i) {
      if (k[i - 1] < key) { k[i] = k[i - 1]; t[i] = t[i - 1]; e[i] = e[i - 1]; }
      else if (k[i] < key) { k[i] = key; t[i] = tt; e[i] = ee; }
    }
    if (k[0] < key) { k[0] = key; t[0] = tt; e[0] = ee; }
  }
};

// ---------------------------------------------------------------------------
// One read record (mate 1 + optional mate 2) against one partition.
// Called by all NT threads of the group with the same r.  The window count
// statistic lives in a shared-memory hash of 4-window BLOCKS (block id =
// ranked window >> 2, four 16-bit counts per entry; a window's count is at
// most the record's feature count, <= 1024): consecutive windows of one
// target -- the reads' strain-shared hits -- share entries, and every range
// sum of one block reads its own entry plus (sws + 2) / 4 neighbours.
// H = capacity in blocks (distinct blocks <= 3H/4 except in the last bin).
// ---------------------------------------------------------------------------
template <int NT, uint32_t H, uint32_t FCAP, uint32_t LMAX, bool kLastBin, int kU, int M, int CB = 16>
__device__ int process_record(const QueryArgs& a, uint64_t r, uint8_t* sm, uint64_t& n_feat, uint64_t& n_loc) {
  using Lay = RecLayout<H, FCAP, NT, CB>;
  using C4 = Cnt4<CB>;
  static_assert(CB == 16 || FCAP <= 255, "8-bit window counts need <= 255 features per record");
  static_assert((H & (H - 1)) == 0, "hash capacity must be a power of two");
  uint64_t* foff = reinterpret_cast<uint64_t*>(sm + Lay::foff);
  uint32_t* fcnt = reinterpret_cast<uint32_t*>(sm + Lay::fcnt);
  uint32_t* fpos = reinterpret_cast<uint32_t*>(sm + Lay::fpos);
  typename C4::T* bcnt = reinterpret_cast<typename C4::T*>(sm + Lay::bcnt);
  uint32_t* bcnt32 = reinterpret_cast<uint32_t*>(sm + Lay::bcnt);
  uint32_t* bkey = reinterpret_cast<uint32_t*>(sm + Lay::bkey);
  uint32_t* scr = reinterpret_cast<uint32_t*>(sm + Lay::scr);
  uint64_t* scr64 = reinterpret_cast<uint64_t*>(sm + Lay::scr64);
  uint32_t* meta = reinterpret_cast<uint32_t*>(sm + Lay::meta);

  const SketchCfg& c = a.c;
  const uint32_t tid = group_rank<NT>();

  // ---- record geometry (S10, S17): each mate windowed separately ----------
  const uint64_t len1 = a.rb.o1[r + 1] - a.rb.o1[r];
  const uint64_t len2 = a.rb.r2 ? a.rb.o2[r + 1] - a.rb.o2[r] : 0;
  const uint32_t nwt = (uint32_t)(a.wbase[r + 1] - a.wbase[r]);
  HitRec* out = a.out + (r * a.n_lists + a.list) * a.m;
  if (nwt * c.s > FCAP) return kDefer;
  // S10: sws from the record's length; S25: pairs span at least insert_size_max
  const uint64_t span = a.rb.r2 && a.insert_size_max > len1 + len2 ? a.insert_size_max : len1 + len2;
  const uint32_t sws = 2u + (uint32_t)(span / c.stride);

  // ---- Q2 + Q3 ran in k_query_sketch_probe: the record's probe results.
  // Features with an empty list (absent keys, padding) are dropped here, so
  // every list the gather walks is non-empty (their order does not matter:
  // the window counts are sums) ----------------------------------------------
  uint32_t F;
  {
    const uint64_t fb = a.wbase[r] * c.s;
    const uint32_t F0 = nwt * c.s;
    if constexpr (NT == 32) {
      uint32_t nn = 0;
      for (uint32_t i0 = 0; i0 < F0; i0 += 32) {
        const uint64_t w = i0 + tid < F0 ? a.qfeat[fb + i0 + tid] : 0ull;
        const uint32_t cnt = (uint32_t)(w & 0xffffffu);
        const uint32_t bal = __ballot_sync(kFull, cnt != 0);
        if (cnt) {
          const uint32_t j = nn + __popc(bal & ((1u << tid) - 1u));
          fcnt[j] = cnt;
          foff[j] = w >> 24;
        }
        nn += __popc(bal);
      }
      F = nn;
    } else {
      if (tid == 0) meta[2] = 0;
      group_sync<NT>();
      for (uint32_t i = tid; i < F0; i += NT) {
        const uint64_t w = a.qfeat[fb + i];
        const uint32_t cnt = (uint32_t)(w & 0xffffffu);
        if (cnt) {
          const uint32_t j = atomicAdd(&meta[2], 1u);
          fcnt[j] = cnt;
          foff[j] = w >> 24;
        }
      }
      group_sync<NT>();
      F = meta[2];
    }
  }
  group_sync<NT>();

  // ---- Q4: exclusive scan of list lengths (replaces compaction) --
  const uint32_t per = (F + NT - 1) / NT;
  uint32_t mysum = 0;
  for (uint32_t i = tid * per; i < min(F, tid * per + per); ++i) mysum += fcnt[i];
  uint32_t L;
  uint32_t run = group_exclusive_scan<NT>(mysum, scr, &L);
  for (uint32_t i = tid * per; i < min(F, tid * per + per); ++i) {
    fpos[i] = run;
    run += fcnt[i];
  }
  if (tid == 0) fpos[F] = L;  // sentinel for the gather's forward walk
  if (L > LMAX) return kDefer;  // too many locations for this group size
  if (L == 0) {
    for (uint32_t i = tid; i < a.m; i += NT) write_hit(out + i, kEmptyTgt, 0, 0, 0, 0);
    return kDone;
  }
  // hash capacity for this record: >= 2 L blocks' worth, at most H
  const uint32_t lg = min(31u - __clz(H), max(5u, 32u - __clz(2 * L - 1)));
  const uint32_t HS = 1u << lg;
  for (uint32_t i = tid; i < HS; i += NT) {
    bkey[i] = kEmptyLoc;
    bcnt[i] = typename C4::T{};
  }
  if (tid == 0) meta[0] = 0;
  group_sync<NT>();
  uint32_t claims = 0;
#if MC_PRECLAIM
  // records with long lists (many strains share the read's features): the
  // blocks of MC_PRECLAIM lists spread over the record's windows are claimed
  // first, one list entry per lane (coalesced loads, distinct blocks), so the
  // gather below mostly finds its blocks in their home buckets instead of every
  // lane claiming kU new blocks one after another on an empty table
  if constexpr (NT == 32) {
    if (L >= MC_PRECLAIM_MINLEN * F) {
      uint32_t pk[MC_PRECLAIM];
#pragma unroll
      for (int q = 0; q < MC_PRECLAIM; ++q) {
        const uint32_t f = (F * (uint32_t)q) / MC_PRECLAIM;
        pk[q] = tid < fcnt[f] ? __ldg(a.pv.values + foff[f] + tid) >> 2 : kEmptyLoc;
      }
#pragma unroll
      for (int q = 0; q < MC_PRECLAIM; ++q) {
        if (pk[q] == kEmptyLoc || (q > 0 && pk[q] == pk[q - 1])) continue;
        uint32_t cl[3] = {0, 0, 0};  // (diagnostic builds count probe steps in cl[1..2])
        if (binsert(bkey, lg, pk[q], cl) < 0) meta[0] = 1;
        claims += cl[0];
      }
    }
  }
#endif

  // ---- Q5-Q6: gather every location and accumulate the window count ---------
  // statistic in the block hash instead of sorting.
  // each thread gathers a contiguous run of locations: its feature index is
  // found once and then only walks forward; kU value loads are kept in flight
  // each thread gathers a contiguous run of locations with a pointer into the
  // current feature's bucket (measured faster than positions strided over the
  // group: coalesced loads, but divergent feature walks and less L2 reuse)
  const uint32_t run_len = (L + NT - 1) / NT;
  const uint32_t i_beg = min(L, tid * run_len), i_end = min(L, i_beg + run_len);
  QP(uint32_t qp_iter = 0; uint32_t qp_witer = 0; uint32_t qp_miss = 0; uint32_t qp_cl[3] = {0, 0, 0};)
  if (i_beg < i_end) {
    uint32_t f = upper_index(fpos, F, i_beg);  // (lists are non-empty: fpos is strictly increasing)
    const uint32_t* src = a.pv.values + foff[f];
    uint32_t j = i_beg - fpos[f], cnt = fcnt[f];  // position in feature f's list, its length
    for (uint32_t i0 = i_beg; i0 < i_end; i0 += kU) {
      QP(++qp_iter);
      uint32_t loc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        // (one predicate per step, no reconvergence branch around it)
        const bool ok = i0 + u < i_end;
        if (ok && j == cnt) {  // next feature (never empty)
          ++f;
          src = a.pv.values + foff[f];
          j = 0;
          cnt = fcnt[f];
        }
        loc[u] = ok ? __ldg(src + j) : kEmptyLoc;
        j += ok ? 1u : 0u;
      }
      // the kU home buckets are read together (independent LDS.128 in flight);
      // a block already in its home bucket -- the common case -- is counted
      // straight away, anything else takes the claiming probe loop
      uint4 q0[kU];
      uint32_t hb[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        hb[u] = hslot(loc[u] >> 2, lg - 2);
        if (loc[u] != kEmptyLoc) q0[u] = reinterpret_cast<const uint4*>(bkey)[hb[u]];
      }
      uint32_t miss = 0;  // locations whose block is not in its home bucket (yet)
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (loc[u] == kEmptyLoc) continue;
        const uint32_t mi = find4(q0[u], loc[u] >> 2);
        if (mi < 4) C4::add(bcnt32, 4 * hb[u] + mi, loc[u]);
        else miss |= 1u << u;
      }
      // the misses of all kU locations share ONE claiming loop (the warp runs it
      // max-misses-per-lane times instead of once per location index)
      QP({
        const uint32_t am = __activemask();
        qp_miss += __popc(miss);
        const uint32_t mx = __reduce_max_sync(am, __popc(miss));
        if ((uint32_t)(__ffs(am) - 1) == (threadIdx.x & 31u)) qp_witer += mx;
      })
      while (miss) {
        const int u = __ffs(miss) - 1;
        miss &= miss - 1;
        uint32_t lu = loc[0];
#pragma unroll
        for (int q = 1; q < kU; ++q) lu = u == q ? loc[q] : lu;
#if MC_QPROF
        qp_cl[0] = 0;
        const int h = binsert(bkey, lg, lu >> 2, qp_cl);
        claims += qp_cl[0];
        const uint32_t cl = 0;
        (void)cl;
#else
        uint32_t cl = 0;
        const int h = binsert(bkey, lg, lu >> 2, &cl);
        claims += cl;
#endif
        if (h < 0) meta[0] = 1;  // table full
        else C4::add(bcnt32, (uint32_t)h, lu);
      }
    }
  }
  group_sync<NT>();
  uint32_t uniq;
  if constexpr (NT == 32) uniq = __reduce_add_sync(kFull, claims);  // (only the total is needed)
  else group_exclusive_scan<NT>(claims, scr, &uniq);
#if MC_QPROF
  if constexpr (NT == 32) {
    const uint32_t it_max = __reduce_max_sync(kFull, qp_iter), it_sum = __reduce_add_sync(kFull, qp_iter);
    const uint32_t ms = __reduce_add_sync(kFull, qp_miss), st = __reduce_add_sync(kFull, qp_cl[1]);
    const uint32_t cf = __reduce_add_sync(kFull, qp_cl[2]), wi = __reduce_add_sync(kFull, qp_witer);
    if (tid == 0) {
      atomicAdd(&g_qprof[0], 1ull);
      atomicAdd(&g_qprof[1], (unsigned long long)L);
      atomicAdd(&g_qprof[2], (unsigned long long)uniq);
      atomicAdd(&g_qprof[3], (unsigned long long)HS);
      atomicAdd(&g_qprof[4], (unsigned long long)it_max);
      atomicAdd(&g_qprof[5], (unsigned long long)it_sum);
      atomicAdd(&g_qprof[6], (unsigned long long)ms);
      atomicAdd(&g_qprof[7], (unsigned long long)wi);
      atomicAdd(&g_qprof[8], (unsigned long long)st);
      atomicAdd(&g_qprof[9], (unsigned long long)cf);
      atomicAdd(&g_qprof[10], (unsigned long long)F);
      if (meta[0] || (!kLastBin && uniq > (HS >> 2) * 3)) atomicAdd(&g_qprof[11], 1ull);
    }
  }
#endif
  if (meta[0] || (!kLastBin && uniq > (HS >> 2) * 3)) return kDefer;  // too many distinct blocks for this bin
  if (tid == 0) n_loc += L;

  // ---- Q7: best contiguous range per block and the --------
  // per-thread top-M with distinct targets (S13).  Ranked window ids of
  // different targets are >= kRankGap >= sws apart, so window b + d (d < sws)
  // always belongs to b's target.
  TopList<M> top;
  top.clear();
  const uint32_t nb = (sws + 2) >> 2;  // neighbour blocks a range starting in this block can reach
  // warp groups first compact the occupied slots (into the dead feature
  // arrays) so every lane works on a block; CTA groups walk the slots
  constexpr bool kCompact = NT == 32 && 2 * H <= 16 * FCAP;
  uint32_t nocc = HS;
  uint16_t* occ = reinterpret_cast<uint16_t*>(sm + Lay::foff);
  if constexpr (kCompact) {
    group_sync<NT>();  // (the feature arrays are no longer read)
    nocc = 0;
    for (uint32_t h0 = 0; h0 < HS; h0 += 32) {
      const bool o = bkey[h0 + tid] != kEmptyLoc;
      const uint32_t bal = __ballot_sync(kFull, o);
      if (o) occ[nocc + __popc(bal & ((1u << tid) - 1u))] = (uint16_t)(h0 + tid);
      nocc += __popc(bal);
    }
    __syncwarp();
  }
  QP(uint32_t qp_bb = 0, qp_ins = 0, qp_q7 = 0;)
  for (uint32_t j = tid; j < nocc; j += NT) {
    QP(++qp_q7);
    const uint32_t h = kCompact ? occ[j] : j;
    const uint32_t kb = bkey[h];
    if (!kCompact && kb == kEmptyLoc) continue;
    const uint2 own = C4::unpack(bcnt[h]);
    uint32_t bs = 0, bi = 0, be = 0;
    if (sws <= 8) {
      const uint2 w1 = blookup(bkey, bcnt, lg, kb + 1);
      const uint2 w2 = sws >= 6 ? blookup(bkey, bcnt, lg, kb + 2) : make_uint2(0, 0);
      // no range starting in this block can beat the list: skip it
      const uint32_t bound = hsum16(own) + hsum16(w1) + hsum16(w2);
      if ((((uint64_t)bound << 32) | 0xffffffffull) <= top.k[M - 1]) continue;
      QP(++qp_bb);
      switch (sws) {
        case 2: block_best<2>(own, w1, w2, bs, bi, be); break;
        case 3: block_best<3>(own, w1, w2, bs, bi, be); break;
        case 4: block_best<4>(own, w1, w2, bs, bi, be); break;
        case 5: block_best<5>(own, w1, w2, bs, bi, be); break;
        case 6: block_best<6>(own, w1, w2, bs, bi, be); break;
        case 7: block_best<7>(own, w1, w2, bs, bi, be); break;
        default: block_best<8>(own, w1, w2, bs, bi, be); break;
      }
    } else {  // long records: walk the (sws + 2) / 4 neighbour blocks
      uint32_t s4[4] = {0, 0, 0, 0}, e4[4] = {0, 0, 0, 0};
      for (uint32_t jb = 0; jb <= nb; ++jb) {
        const uint2 w = jb == 0 ? own : blookup(bkey, bcnt, lg, kb + jb);
        if ((w.x | w.y) == 0) continue;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          const uint32_t cq = cnt16(w, q);
          if (cq == 0) continue;
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            const int d = (int)(4 * jb + q) - (int)i;  // window offset from start 4 kb + i
            if (d >= 0 && d < (int)sws) { s4[i] += cq; e4[i] = (uint32_t)d; }
          }
        }
      }
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i)
        if (cnt16(own, i) != 0 && s4[i] > bs) { bs = s4[i]; bi = i; be = e4[i]; }
    }
    const uint32_t b = 4 * kb + bi;
    const uint64_t key = ((uint64_t)bs << 32) | (uint64_t)(~b);
    if (key <= top.k[M - 1]) continue;
    QP(++qp_ins);
    top.insert(key, target_of(a.pv, b), be);
  }
#if MC_QPROF
  if constexpr (NT == 32) {
    const uint32_t a0 = __reduce_add_sync(kFull, qp_bb), a1 = __reduce_add_sync(kFull, qp_ins);
    const uint32_t a2 = __reduce_max_sync(kFull, qp_q7);
    if (tid == 0) {
      atomicAdd(&g_qprof[12], (unsigned long long)nocc);
      atomicAdd(&g_qprof[13], (unsigned long long)a0);
      atomicAdd(&g_qprof[14], (unsigned long long)a1);
      atomicAdd(&g_qprof[15], (unsigned long long)a2);
    }
  }
#endif

  // ---- top-m over the group: m rounds of max over the list heads; the owner
  // writes the hit, every thread drops that target from its list ------------
  uint32_t round = 0;
  if constexpr (NT == 32) {
    // warp: the 64-bit max is two REDUX.MAX (hits, then ~window among the
    // lanes holding those hits); lane `round` keeps round's winner and the
    // hits are written after the rounds, so their target-table loads overlap
    uint32_t my_rk = 0, my_b = 0, my_e = 0, my_h = 0;
    for (; round < a.m; ++round) {
      const uint32_t hi = (uint32_t)(top.k[0] >> 32), lo = (uint32_t)top.k[0];
      const uint32_t mh = __reduce_max_sync(kFull, hi);
      if (mh == 0) break;  // every list is empty (a listed candidate has >= 1 hit)
      const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
      const uint32_t lane_of = __ffs(__ballot_sync(kFull, hi == mh && lo == ml)) - 1;
      const uint32_t wt = __shfl_sync(kFull, top.t[0], lane_of);
      const uint32_t we = __shfl_sync(kFull, top.e[0], lane_of);
      if (tid == round) my_rk = wt, my_b = ~ml, my_e = we, my_h = mh;
      top.remove_target(wt);
    }
    if (tid < round) {
      const uint32_t base = a.pv.rank_base[my_rk];
      write_hit(out + tid, a.pv.tgt_id[my_rk], my_h, my_b - base, my_b + my_e - base, a.pv.taxon[my_rk]);
    }
    for (uint32_t i = round + tid; i < a.m; i += NT) write_hit(out + i, kEmptyTgt, 0, 0, 0, 0);
    group_sync<NT>();
    return kDone;
  }
  for (; round < a.m; ++round) {
    const uint64_t best = group_max_u64<NT>(top.k[0], scr64);
    if (best == 0) break;
    uint32_t win_t;
    const bool owner = top.k[0] == best;
    if (owner) {
      const uint32_t rk = top.t[0], b = ~(uint32_t)best;
      const uint32_t base = a.pv.rank_base[rk];
      write_hit(out + round, a.pv.tgt_id[rk], (uint32_t)(best >> 32), b - base, b + top.e[0] - base, a.pv.taxon[rk]);
    }
    if constexpr (NT == 32) {
      const uint32_t lane_of = __ffs(__ballot_sync(kFull, owner)) - 1;
      win_t = __shfl_sync(kFull, top.t[0], lane_of);
    } else {
      if (owner) meta[1] = top.t[0];
      __syncthreads();
      win_t = meta[1];
    }
    top.remove_target(win_t);
  }
  for (uint32_t i = round + tid; i < a.m; i += NT) write_hit(out + i, kEmptyTgt, 0, 0, 0, 0);
  group_sync<NT>();
  return kDone;
}

// per-kernel statistics: reduce over the warp, one atomic per warp.
// stats[0] features, [1] locations, [3 + bin] locations gathered by that bin
__device__ __forceinline__ void add_stats(unsigned long long* st, uint64_t nf, uint64_t nl, int bin = -1) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    nf += __shfl_xor_sync(kFull, nf, d);
    nl += __shfl_xor_sync(kFull, nl, d);
  }
  if ((threadIdx.x & 31u) == 0) {
    if (nf) atomicAdd(&st[0], (unsigned long long)nf);
    if (nl) atomicAdd(&st[1], (unsigned long long)nl);
    if (nl && bin >= 0) atomicAdd(&st[3 + bin], (unsigned long long)nl);
  }
}

// ---- Q1: windows per record + device-side input checks (S10, S17) ----------
__global__ void __launch_bounds__(256) k_query_plan(QueryArgs a, uint32_t* nwt, uint64_t lim_bp) {
  const ReadBatch& rb = a.rb;
  uint64_t bp = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rb.n; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a1 = rb.o1[r], e1 = rb.o1[r + 1];
    const uint64_t a2 = rb.r2 ? rb.o2[r] : 0, e2 = rb.r2 ? rb.o2[r + 1] : 0;
    // offsets must not decrease: a record outside the batch's byte span
    // [o[0], o[n]] (which is all that is staged) counts as decreasing too
    int bad = (e1 < a1 || e2 < a2 || a1 < rb.o1[0] || e1 > rb.o1[rb.n] ||
               (rb.r2 && (a2 < rb.o2[0] || e2 > rb.o2[rb.n]))) ? 1 : 0;
    const uint64_t len1 = e1 - a1, len2 = e2 - a2;
    if (!bad && len1 + len2 > lim_bp) bad = 2;
    if (bad && atomicCAS(&a.err[2], 0, bad) == 0) a.err[3] = (int)r;
    nwt[r] = bad ? 0u : n_windows(len1, a.c) + n_windows(len2, a.c);
    if (!bad) bp += len1 + len2;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) bp += __shfl_xor_sync(kFull, bp, d);
  if ((threadIdx.x & 31u) == 0 && bp) atomicAdd(&a.stats[2], (unsigned long long)bp);
}

void launch_query_plan(const QueryArgs& a, uint32_t* nwt, uint64_t lim_bp, cudaStream_t st) {
  const uint64_t blocks = (a.rb.n + 255) / 256;
  k_query_plan<<<(int)std::min<uint64_t>(std::max<uint64_t>(blocks, 1), (uint64_t)num_sms() * 8), 256, 0, st>>>(
      a, nwt, lim_bp);
}

// ---- Q2 + Q3: one thread per read window (the build's sketch routine) and
// all of its features' key-table probes in flight at once ---------------------
template <uint32_t K>
__device__ __forceinline__ void sketch_probe_tiles(const QueryArgs& a, uint64_t W, uint32_t* slots, uint64_t* qfeat,
                                                   uint64_t& n_feat, uint64_t& n_hit) {
  const SketchCfg& c = a.c;
  const ReadBatch& rb = a.rb;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t* wslots = slots + wid * 32 * kSlotWords;
  uint64_t tile, tend;
  cta_tiles((W + kSlotTile - 1) / kSlotTile, &tile, &tend);
  uint32_t r0 = 0;
  for (; tile < tend; ++tile) {
    const uint64_t g0 = tile * kSlotTile + wid * 32, g = g0 + lane;
    const uint8_t* p = rb.r1;
    uint32_t nk = 0;
    if (g0 < W) {
      const uint32_t r = warp_segment(a.wbase, (uint32_t)rb.n, W, g0, r0, lane);
      if (g < W) {  // window j of record r: mate 1's windows, then mate 2's
        const uint32_t j = (uint32_t)(g - a.wbase[r]);
        const uint64_t len1 = rb.o1[r + 1] - rb.o1[r];
        const uint32_t nw1 = n_windows(len1, c);
        const bool m2 = j >= nw1;
        const uint64_t L = m2 ? rb.o2[r + 1] - rb.o2[r] : len1;
        const uint64_t first = (uint64_t)(m2 ? j - nw1 : j) * c.stride;
        nk = (uint32_t)min((uint64_t)c.stride, L - c.k + 1 - first);
        p = m2 ? rb.r2 + (rb.o2[r] - rb.base2) + first : rb.r1 + (rb.o1[r] - rb.base1) + first;
      }
    }
    uint32_t v[16];
    const int n = sketch_warp_windows<K>(wslots, p, nk, c, lane, v);
    n_feat += (uint32_t)n;
    __syncwarp();  // the warp's slots now stage the probe results for a coalesced copy-out
    uint32_t* rlo = wslots;                   // [32 * (s + 1)] (padded: conflict-free either way)
    uint32_t* rhi = wslots + 32 * (c.s + 1);
#pragma unroll
    for (int h = 0; h < 16; h += 8) {
      uint64_t sl[8];
      unsigned long long e[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sl[u] = home_slot(v[h + u], a.pv.nslots);
        e[u] = h + u < n ? __ldg(&a.pv.T[sl[u]].kc) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = h + u;
        if ((uint32_t)i >= c.s) continue;
        uint64_t word = 0;  // empty list
        if (i < n) {
          uint64_t s = sl[u];
          unsigned long long x = e[u];
          for (uint32_t probes = 0; probes < kSubSlots && slot_cnt(x) != 0; ++probes) {
            if (slot_key(x) == v[i]) {
              word = (a.pv.vbase[s >> kSubLg] + slot_loff(x)) << 24 | slot_cnt(x);
              break;
            }
            s = next_slot(s);
            x = __ldg(&a.pv.T[s].kc);
          }
        }
        n_hit += word != 0;
        rlo[lane * (c.s + 1) + i] = (uint32_t)word;
        rhi[lane * (c.s + 1) + i] = (uint32_t)(word >> 32);
      }
    }
    __syncwarp();
    if (g0 < W) {
      const uint32_t nv = (uint32_t)min((uint64_t)32, W - g0) * c.s;
      uint64_t* dst = qfeat + g0 * c.s;
      for (uint32_t i = lane; i < nv; i += 32) {
        const uint32_t at = i + i / c.s;  // (i / s) * (s + 1) + i % s
        dst[i] = (uint64_t)rhi[at] << 32 | rlo[at];
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) k_query_sketch_probe(QueryArgs a, uint64_t W, uint64_t* qfeat) {
  if (*(volatile int*)&a.err[2]) return;  // invalid input in this batch (k_query_plan): the call fails
  W = min(W, (uint64_t)a.wbase[a.rb.n]);  // (W may be a host-side upper bound: the exact total is on the device)
  __shared__ __align__(16) uint32_t slots[kSlotTile * kSlotWords];
  uint64_t n_feat = 0, n_hit = 0;
  if (a.c.k == 16) sketch_probe_tiles<16>(a, W, slots, qfeat, n_feat, n_hit);
  else sketch_probe_tiles<0>(a, W, slots, qfeat, n_feat, n_hit);
  add_stats(a.stats, n_feat, 0);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) n_hit += __shfl_xor_sync(kFull, n_hit, d);
  if ((threadIdx.x & 31u) == 0 && n_hit) atomicAdd(&a.stats[8], (unsigned long long)n_hit);
}

void launch_query_sketch_probe(const QueryArgs& a, uint64_t W, uint64_t* qfeat, int sms, cudaStream_t st) {
  if (W == 0) return;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_sketch_probe, 256, 0);
  const uint64_t tiles = (W + kSlotTile - 1) / kSlotTile;
#ifndef MC_PROBE_WAVES
#define MC_PROBE_WAVES 4
#endif
  // MC_PROBE_WAVES resident-CTA waves of tiles (1: persistent CTAs; more: CTAs
  // start and finish at staggered times, so sketch and probe phases interleave)
  const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)sms * std::max(per_sm, 1) * MC_PROBE_WAVES);
  k_query_sketch_probe<<<grid, 256, 0, st>>>(a, W, qfeat);
}

// ---- diagnostics: one key's bucket (count, absolute offset) --------------------
__global__ void k_key_lookup(PartView pv, uint32_t key, unsigned long long* out) {
  uint64_t off = 0;
  const uint32_t n = keytable_find(pv.T, pv.vbase, pv.nslots, key, &off);
  out[0] = n;
  out[1] = off;
}
void launch_key_lookup(const PartView& pv, uint32_t key, unsigned long long* out, cudaStream_t st) {
  k_key_lookup<<<1, 1, 0, st>>>(pv, key, out);
}

// ---- small bin: one warp per record, 8 records per CTA ----------------------
constexpr uint32_t kSmallF = kSmallW * 16;
using LaySmall = RecLayout<kSmallH, kSmallF, 32, 8>;  // <= 64 features: 8-bit counts

template <int M>
#ifndef MC_SMALL_MINB
#define MC_SMALL_MINB 3
#endif
__global__ void __launch_bounds__(256, MC_SMALL_MINB) k_query_small(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t defer_buf[8][32];
  if (*(volatile int*)&a.err[2]) return;  // invalid input in this batch: the call fails
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint8_t* sm = smem + wid * LaySmall::bytes;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t nf = 0, nl = 0;
  uint32_t nd = 0;  // deferred records staged in this warp's buffer (one atomic per 32)
  auto flush = [&]() {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&a.qcount[0], nd);
    base = __shfl_sync(kFull, base, 0);
    if (lane < nd) a.qM[base + lane] = defer_buf[wid][lane];
    nd = 0;
  };
  for (uint64_t r = gw; r < a.rb.n; r += nw) {
    if (process_record<32, kSmallH, kSmallF, kSmallL, false, MC_SMALL_U, M, 8>(a, r, sm, nf, nl) == kDefer) {
      if (lane == 0) defer_buf[wid][nd] = (uint32_t)r;
      if (++nd == 32) { __syncwarp(); flush(); }
    }
    __syncwarp();
  }
  __syncwarp();
  if (nd) flush();
  add_stats(a.stats, nf, nl, 0);
}

// ---- medium / large bins: one CTA per deferred record -----------------------
constexpr uint32_t kMedF = kMedW * 16, kLargeF = kLargeW * 16;
using LayMed = RecLayout<kMedH, kMedF, kMedT>;
using LayLarge = RecLayout<kLargeH, kLargeF, 512>;

template <int M>
__global__ void __launch_bounds__(kMedT) k_query_medium(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)&a.err[2]) return;
  const uint32_t n = a.qcount[0];
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&a.stats[6], (unsigned long long)n);
  uint64_t nf = 0, nl = 0;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t r = a.qM[i];
    if (process_record<kMedT, kMedH, kMedF, kMedL, false, 4, M>(a, r, smem, nf, nl) == kDefer && threadIdx.x == 0)
      a.qL[atomicAdd(&a.qcount[1], 1u)] = r;
    __syncthreads();
  }
  add_stats(a.stats, nf, nl, 1);
}

template <int M>
__global__ void __launch_bounds__(512) k_query_large(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (*(volatile int*)&a.err[2]) return;
  const uint32_t n = a.qcount[1];
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(&a.stats[7], (unsigned long long)n);
  uint64_t nf = 0, nl = 0;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t r = a.qL[i];
    if (process_record<512, kLargeH, kLargeF, 0xffffffffu, true, 4, M>(a, r, smem, nf, nl) == kDefer &&
        threadIdx.x == 0) {
      if (atomicCAS(a.err, 0, 1) == 0) a.err[1] = (int)r;
      HitRec* out = a.out + ((uint64_t)r * a.n_lists + a.list) * a.m;
      for (uint32_t q = 0; q < a.m; ++q) write_hit(out + q, kEmptyTgt, 0, 0, 0, 0);
    }
    __syncthreads();
  }
  add_stats(a.stats, nf, nl, 2);
}

void query_kernels_init() {
  cudaFuncSetAttribute(k_query_small<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * LaySmall::bytes);
  cudaFuncSetAttribute(k_query_small<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * LaySmall::bytes);
  cudaFuncSetAttribute(k_query_medium<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, LayMed::bytes);
  cudaFuncSetAttribute(k_query_medium<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, LayMed::bytes);
  cudaFuncSetAttribute(k_query_large<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, LayLarge::bytes);
  cudaFuncSetAttribute(k_query_large<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, LayLarge::bytes);
}

// per-thread candidate lists hold M >= m entries (m <= 8)
// grid: at most `grid` CTAs (one warp per record, 8 per CTA), capped at the
// resident count so every CTA is a persistent worker
void launch_query_small(const QueryArgs& a, int grid, cudaStream_t st) {
  int per_sm = 0;
  if (a.m <= 4) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_small<4>, 256, 8 * LaySmall::bytes);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_small<8>, 256, 8 * LaySmall::bytes);
  grid = std::max(1, std::min(grid, num_sms() * std::max(per_sm, 1)));
  if (a.m <= 4) k_query_small<4><<<grid, 256, 8 * LaySmall::bytes, st>>>(a);
  else k_query_small<8><<<grid, 256, 8 * LaySmall::bytes, st>>>(a);
}
void launch_query_medium(const QueryArgs& a, int grid, cudaStream_t st) {
  if (a.m <= 4) k_query_medium<4><<<grid, kMedT, LayMed::bytes, st>>>(a);
  else k_query_medium<8><<<grid, kMedT, LayMed::bytes, st>>>(a);
}
void launch_query_large(const QueryArgs& a, int grid, cudaStream_t st) {
  if (a.m <= 4) k_query_large<4><<<grid, 512, LayLarge::bytes, st>>>(a);
  else k_query_large<8><<<grid, 512, LayLarge::bytes, st>>>(a);
}

// ---------------------------------------------------------------------------
// Q8 + Q9: merge per-partition top-m lists (hits desc, target asc; exact since
// a target lives in one partition) and classify (P:598-603,
// S15/S16) with the lineage table (constant-depth LCA).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lca(const MergeArgs& a, uint32_t x, uint32_t y) {
  if (x == 0) return y;
  if (y == 0) return x;
  const uint32_t D = a.maxd + 1;
  int d = (int)min(a.depth[x], a.depth[y]);
  const uint32_t* ax = a.anc + (uint64_t)x * D;
  const uint32_t* ay = a.anc + (uint64_t)y * D;
  while (d >= 0 && ax[d] != ay[d]) --d;
  return d < 0 ? 0u : ax[d];
}

__global__ void __launch_bounds__(256) k_merge_classify(MergeArgs a) {
  const bool invalid = a.err && *(volatile const int*)&a.err[2];  // invalid batch input: no hits were written
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t total = a.n_lists * a.m;
  const uint32_t per = a.lists_per_src * a.m;  // (multi-GPU) entries per record in one source
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += stride) {
    if (invalid) {  // (the call fails; its outputs are defined: unclassified, no candidates)
      a.out_taxon[r] = 0;
      for (uint32_t i = 0; i < a.m && a.out_cand; ++i) {
        uint32_t* oc = a.out_cand + (r * a.m + i) * 4;
        oc[0] = kEmptyTgt; oc[1] = 0; oc[2] = 0; oc[3] = 0;
      }
      continue;
    }
    // entry e of the record: local array, or source e / per (a peer GPU's buffer)
    auto entry = [&](uint32_t e) -> const HitRec& {
      if (a.n_src == 0) return a.in[r * total + e];
      const uint32_t g = e / per;
      return a.src[g][(a.r0 + r) * per + (e - g * per)];
    };
    uint64_t taken = 0;
    uint32_t sel[8];
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < a.m; ++i) {
      int best = -1;
      uint32_t bh = 0, bt = 0;
      for (uint32_t e = 0; e < total; ++e) {
        if ((taken >> e) & 1ull) continue;
        const HitRec& he = entry(e);
        const uint32_t t = he.tgt;
        if (t == kEmptyTgt) continue;
        const uint32_t h = he.hits;
        if (best < 0 || h > bh || (h == bh && t < bt)) { best = (int)e; bh = h; bt = t; }
      }
      if (best < 0) break;
      taken |= 1ull << best;
      sel[cnt++] = (uint32_t)best;
    }
    uint32_t* oc = a.out_cand ? a.out_cand + r * a.m * 4 : nullptr;
    for (uint32_t i = 0; i < a.m && oc; ++i) {
      if (i < cnt) {
        const HitRec& h = entry(sel[i]);
        oc[4 * i] = h.tgt; oc[4 * i + 1] = h.hits; oc[4 * i + 2] = h.win_beg; oc[4 * i + 3] = h.win_end;
      } else {
        oc[4 * i] = kEmptyTgt; oc[4 * i + 1] = 0; oc[4 * i + 2] = 0; oc[4 * i + 3] = 0;
      }
    }
    uint32_t taxon = 0;
    if (cnt > 0 && entry(sel[0]).hits >= a.hits_min) {
      const uint32_t top = entry(sel[0]).hits;
      taxon = entry(sel[0]).taxon;
      for (uint32_t i = 1; i < cnt; ++i)
        if (top - entry(sel[i]).hits <= a.hits_diff) taxon = lca(a, taxon, entry(sel[i]).taxon);
    }
    a.out_taxon[r] = taxon;
  }
}

void launch_merge_classify(const MergeArgs& a, cudaStream_t st) {
  const uint64_t blocks = (a.n + 255) / 256;
  const int grid = (int)(blocks < (uint64_t)num_sms() * 16 ? (blocks ? blocks : 1) : (uint64_t)num_sms() * 16);
  k_merge_classify<<<grid, 256, 0, st>>>(a);
}

}  // namespace mc

#if MC_QPROF
// diagnostic builds only (tools/qprof.py): copy out (and optionally zero) the
// small-bin counters of the current device
extern "C" int mc_debug_qprof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, mc::g_qprof, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
  if (reset) {
    const unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(mc::g_qprof, z, sizeof(z)) != cudaSuccess) return -1;
  }
  return 0;
}
#endif
