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
#define MC_SMALL_U 1
#endif

template <uint32_t H, uint32_t FCAP, int NT>
struct RecLayout {
  // byte offsets inside the group's shared-memory slice
  static constexpr uint32_t foff = 0;                                    // uint64[FCAP] list offsets
  static constexpr uint32_t fcnt = foff + 8 * FCAP;                      // uint32[FCAP] list lengths
  static constexpr uint32_t fpos = fcnt + 4 * FCAP;                      // uint32[FCAP+1] scan of lengths
  static constexpr uint32_t hkey = (fpos + 4 * (FCAP + 1) + 15) & ~15u;  // uint32[H] location (window id)
  static constexpr uint32_t hcnt = hkey + 4 * H;                         // uint32[H] hits of that window
  static constexpr uint32_t hrng = hcnt + 4 * H;                         // uint32[H] range hits | end << 22
  static constexpr uint32_t scr = hrng + 4 * H;                          // uint32[NT/32+2]
  static constexpr uint32_t scr64 = (scr + 4 * (NT / 32 + 2) + 7) & ~7u;  // uint64[NT/32]
  static constexpr uint32_t excl = scr64 + 8 * (NT / 32);                // uint32[2*8]
  static constexpr uint32_t meta = excl + 4 * 16;                        // uint32[4]: uniques, overflow
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
constexpr uint32_t kEmptyLoc = 0xffffffffu;  // ranked window ids never reach this value

__device__ __forceinline__ uint32_t hslot(uint32_t x, uint32_t lg) { return (x * 2654435761u) >> (32 - lg); }

// count of window `x` in the record's shared-memory hash (0 if absent)
__device__ __forceinline__ uint32_t hlookup(const uint32_t* hkey, const uint32_t* hcnt, uint32_t lg, uint32_t x) {
  const uint32_t mask = (1u << lg) - 1u;
  for (uint32_t h = hslot(x, lg), i = 0; i <= mask; ++i, h = (h + 1) & mask) {
    const uint32_t k = hkey[h];
    if (k == x) return hcnt[h];
    if (k == kEmptyLoc) return 0;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// One read record (mate 1 + optional mate 2) against one partition.
// Called by all NT threads of the group with the same r.  H = capacity of the
// record's window-count hash (uniques <= 3H/4).
// ---------------------------------------------------------------------------
template <int NT, uint32_t H, uint32_t FCAP, uint32_t LMAX, bool kLastBin, int kU>
__device__ int process_record(const QueryArgs& a, uint64_t r, uint8_t* sm, uint64_t& n_feat, uint64_t& n_loc) {
  using Lay = RecLayout<H, FCAP, NT>;
  static_assert((H & (H - 1)) == 0, "hash capacity must be a power of two");
  uint64_t* foff = reinterpret_cast<uint64_t*>(sm + Lay::foff);
  uint32_t* fcnt = reinterpret_cast<uint32_t*>(sm + Lay::fcnt);
  uint32_t* fpos = reinterpret_cast<uint32_t*>(sm + Lay::fpos);
  uint32_t* hkey = reinterpret_cast<uint32_t*>(sm + Lay::hkey);
  uint32_t* hcnt = reinterpret_cast<uint32_t*>(sm + Lay::hcnt);
  uint32_t* hrng = reinterpret_cast<uint32_t*>(sm + Lay::hrng);
  uint32_t* scr = reinterpret_cast<uint32_t*>(sm + Lay::scr);
  uint64_t* scr64 = reinterpret_cast<uint64_t*>(sm + Lay::scr64);
  uint32_t* excl = reinterpret_cast<uint32_t*>(sm + Lay::excl);
  uint32_t* meta = reinterpret_cast<uint32_t*>(sm + Lay::meta);

  const SketchCfg& c = a.c;
  const uint32_t tid = group_rank<NT>();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wig = tid >> 5;
  constexpr uint32_t NWG = NT / 32;

  // ---- record geometry (S10, S17): each mate windowed separately ----------
  const uint64_t b1 = a.rb.o1[r] - a.rb.base1, len1 = a.rb.o1[r + 1] - a.rb.o1[r];
  const uint8_t* p1 = a.rb.r1 + b1;
  uint64_t len2 = 0;
  const uint8_t* p2 = nullptr;
  if (a.rb.r2) {
    len2 = a.rb.o2[r + 1] - a.rb.o2[r];
    p2 = a.rb.r2 + (a.rb.o2[r] - a.rb.base2);
  }
  const uint32_t nwt = (uint32_t)(a.wbase[r + 1] - a.wbase[r]);
  HitRec* out = a.out + (r * a.n_lists + a.list) * a.m;
  if (nwt * c.s > FCAP) return kDefer;
  const uint32_t sws = 2u + (uint32_t)((len1 + len2) / c.stride);

  // ---- Q2 + Q3 ran in k_query_sketch_probe: the record's probe results ------
  {
    const uint64_t fb = a.wbase[r] * c.s;
    for (uint32_t i = tid; i < nwt * c.s; i += NT) {
      const uint64_t w = a.qfeat[fb + i];
      fcnt[i] = (uint32_t)(w & 0xffffffu);
      foff[i] = w >> 24;
    }
  }
  group_sync<NT>();

  // ---- Q4: exclusive scan of list lengths (replaces compaction) --
  const uint32_t F = nwt * c.s;
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
  // hash capacity for this record: >= 2 L, at most H
  const uint32_t lg = min(31u - __clz(H), max(5u, 32u - __clz(2 * L - 1)));
  const uint32_t HS = 1u << lg, mask = HS - 1u;
  for (uint32_t i = tid; i < HS; i += NT) {
    hkey[i] = kEmptyLoc;
    hcnt[i] = 0;
  }
  if (tid == 0) meta[0] = meta[1] = 0;
  group_sync<NT>();

  // ---- Q5-Q6: gather every location and accumulate the window count ---------
  // statistic in a shared-memory hash instead of sorting
  // A full table (or, in the small/medium bins, more distinct windows than
  // 3/4 of the hash) defers the record to the next bin (last bin: error).
  const uint32_t lim = kLastBin ? HS : (HS >> 2) * 3;
  // each thread gathers a contiguous run of locations: its feature index is
  // found once and then only walks forward; kU value loads are kept in flight
  const uint32_t run_len = (L + NT - 1) / NT;
  const uint32_t i_beg = min(L, tid * run_len), i_end = min(L, i_beg + run_len);
  uint32_t f = i_beg < L ? upper_index(fpos, F, i_beg) : 0u;
  for (uint32_t i0 = i_beg; i0 < i_end; i0 += kU) {
    uint32_t loc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u;
      loc[u] = kEmptyLoc;
      if (i < i_end) {
        while (fpos[f + 1] <= i) ++f;
        loc[u] = __ldg(a.pv.values + foff[f] + (i - fpos[f]));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (loc[u] == kEmptyLoc) continue;
      uint32_t h = hslot(loc[u], lg), probe = 0;
      for (; probe <= mask; ++probe, h = (h + 1) & mask) {
        uint32_t k = hkey[h];
        if (k == kEmptyLoc) {
          k = atomicCAS(&hkey[h], kEmptyLoc, loc[u]);
          if (k == kEmptyLoc) {
            if (atomicAdd(&meta[0], 1u) >= lim) meta[1] = 1;
            k = loc[u];
          }
        }
        if (k == loc[u]) {
          atomicAdd(&hcnt[h], 1u);
          break;
        }
      }
      if (probe > mask) meta[1] = 1;
    }
  }
  group_sync<NT>();
  if (meta[1]) return kDefer;  // too many distinct windows for this bin
  if (tid == 0) n_loc += L;

  // ---- Q7: best contiguous range starting at each hit window --
  // ranked window ids of different targets are >= kRankGap >= sws apart, so
  // window b + d (d < sws) always belongs to b's target.
  for (uint32_t h = tid; h < HS; h += NT) {
    const uint32_t b = hkey[h];
    if (b == kEmptyLoc) continue;
    uint32_t hits = hcnt[h], e = 0;
    for (uint32_t d = 1; d < sws; ++d) {
      const uint32_t cd = hlookup(hkey, hcnt, lg, b + d);
      if (cd) { hits += cd; e = d; }
    }
    hrng[h] = hits | (e << 22);
  }
  group_sync<NT>();

  // ---- top-m over targets (one candidate per target, S11-S13) -------------
  // key = hits << 32 | ~window: max = most hits, then smallest (target, window).
  // Each thread keeps the best key of its own slots; after a round only the
  // threads whose best fell in the excluded target rescan.
  auto scan_mine = [&](uint32_t rounds) {
    uint64_t best = 0;
    for (uint32_t h = tid; h < HS; h += NT) {
      const uint32_t b = hkey[h];
      if (b == kEmptyLoc) continue;
      bool ex = false;
      for (uint32_t q = 0; q < rounds; ++q) ex |= (b >= excl[2 * q] && b < excl[2 * q + 1]);
      if (!ex) {
        const uint64_t key = ((uint64_t)(hrng[h] & 0x3fffffu) << 32) | (uint64_t)(~b);
        best = key > best ? key : best;
      }
    }
    return best;
  };
  uint64_t mine = scan_mine(0);
  uint32_t round = 0;
  for (; round < a.m; ++round) {
    const uint64_t best = group_max_u64<NT>(mine, scr64);
    if (best == 0) break;
    if (tid == 0) {
      const uint32_t b = ~(uint32_t)best;
      uint32_t e = 0;
      for (uint32_t h = hslot(b, lg);; h = (h + 1) & mask)
        if (hkey[h] == b) { e = hrng[h] >> 22; break; }
      const uint32_t rk = target_of(a.pv, b);
      const uint32_t base = a.pv.rank_base[rk];
      write_hit(out + round, a.pv.tgt_id[rk], (uint32_t)(best >> 32), b - base, b + e - base, a.pv.taxon[rk]);
      excl[2 * round] = base;
      excl[2 * round + 1] = a.pv.rank_base[rk + 1];
    }
    group_sync<NT>();
    const uint32_t mb = ~(uint32_t)mine;
    if (mine != 0 && mb >= excl[2 * round] && mb < excl[2 * round + 1]) mine = scan_mine(round + 1);
  }
  for (uint32_t i = round + tid; i < a.m; i += NT) write_hit(out + i, kEmptyTgt, 0, 0, 0, 0);
  group_sync<NT>();
  return kDone;
}

// per-kernel statistics: reduce over the warp, one atomic per warp
__device__ __forceinline__ void add_stats(unsigned long long* st, uint64_t nf, uint64_t nl) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    nf += __shfl_xor_sync(kFull, nf, d);
    nl += __shfl_xor_sync(kFull, nl, d);
  }
  if ((threadIdx.x & 31u) == 0) {
    if (nf) atomicAdd(&st[0], (unsigned long long)nf);
    if (nl) atomicAdd(&st[1], (unsigned long long)nl);
  }
}

// ---- Q1: windows per record + device-side input checks (S10, S17) ----------
__global__ void __launch_bounds__(256) k_query_plan(QueryArgs a, uint32_t* nwt, uint64_t lim_bp) {
  const ReadBatch& rb = a.rb;
  uint64_t bp = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rb.n; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a1 = rb.o1[r], e1 = rb.o1[r + 1];
    const uint64_t a2 = rb.r2 ? rb.o2[r] : 0, e2 = rb.r2 ? rb.o2[r + 1] : 0;
    int bad = (e1 < a1 || e2 < a2) ? 1 : 0;
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
                                                   uint64_t& n_feat) {
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
      ulonglong2 e[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sl[u] = home_slot(v[h + u], a.pv.nslots);
        e[u] = h + u < n ? __ldg(reinterpret_cast<const ulonglong2*>(a.pv.T + sl[u])) : make_ulonglong2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = h + u;
        if ((uint32_t)i >= c.s) continue;
        uint64_t word = 0;  // empty list
        if (i < n) {
          uint64_t s = sl[u];
          ulonglong2 x = e[u];
          for (uint32_t probes = 0; probes < kSubSlots && x.x != 0; ++probes) {
            if ((uint32_t)x.x == v[i]) {
              word = x.y << 24 | (x.x >> 32);
              break;
            }
            s = next_slot(s);
            x = __ldg(reinterpret_cast<const ulonglong2*>(a.pv.T + s));
          }
        }
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
  __shared__ __align__(16) uint32_t slots[kSlotTile * kSlotWords];
  uint64_t n_feat = 0;
  if (a.c.k == 16) sketch_probe_tiles<16>(a, W, slots, qfeat, n_feat);
  else sketch_probe_tiles<0>(a, W, slots, qfeat, n_feat);
  add_stats(a.stats, n_feat, 0);
}

void launch_query_sketch_probe(const QueryArgs& a, uint64_t W, uint64_t* qfeat, int sms, cudaStream_t st) {
  if (W == 0) return;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_sketch_probe, 256, 0);
  const uint64_t tiles = (W + kSlotTile - 1) / kSlotTile;
  const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)sms * std::max(per_sm, 1));
  k_query_sketch_probe<<<grid, 256, 0, st>>>(a, W, qfeat);
}

// ---- small bin: one warp per record, 8 records per CTA ----------------------
constexpr uint32_t kSmallF = kSmallW * 16;
using LaySmall = RecLayout<kSmallH, kSmallF, 32>;

__global__ void __launch_bounds__(256) k_query_small(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t defer_buf[8][32];
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
    if (process_record<32, kSmallH, kSmallF, kSmallL, false, MC_SMALL_U>(a, r, sm, nf, nl) == kDefer) {
      if (lane == 0) defer_buf[wid][nd] = (uint32_t)r;
      if (++nd == 32) { __syncwarp(); flush(); }
    }
    __syncwarp();
  }
  __syncwarp();
  if (nd) flush();
  add_stats(a.stats, nf, nl);
}

// ---- medium / large bins: one CTA per deferred record -----------------------
constexpr uint32_t kMedF = kMedW * 16, kLargeF = kLargeW * 16;
using LayMed = RecLayout<kMedH, kMedF, kMedT>;
using LayLarge = RecLayout<kLargeH, kLargeF, 512>;

__global__ void __launch_bounds__(kMedT) k_query_medium(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t n = a.qcount[0];
  uint64_t nf = 0, nl = 0;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t r = a.qM[i];
    if (process_record<kMedT, kMedH, kMedF, kMedL, false, 4>(a, r, smem, nf, nl) == kDefer && threadIdx.x == 0)
      a.qL[atomicAdd(&a.qcount[1], 1u)] = r;
    __syncthreads();
  }
  add_stats(a.stats, nf, nl);
}

__global__ void __launch_bounds__(512) k_query_large(QueryArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t n = a.qcount[1];
  uint64_t nf = 0, nl = 0;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t r = a.qL[i];
    if (process_record<512, kLargeH, kLargeF, 0xffffffffu, true, 4>(a, r, smem, nf, nl) == kDefer && threadIdx.x == 0) {
      if (atomicCAS(a.err, 0, 1) == 0) a.err[1] = (int)r;
      HitRec* out = a.out + ((uint64_t)r * a.n_lists + a.list) * a.m;
      for (uint32_t q = 0; q < a.m; ++q) write_hit(out + q, kEmptyTgt, 0, 0, 0, 0);
    }
    __syncthreads();
  }
  add_stats(a.stats, nf, nl);
}

void query_kernels_init() {
  cudaFuncSetAttribute(k_query_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * LaySmall::bytes);
  cudaFuncSetAttribute(k_query_medium, cudaFuncAttributeMaxDynamicSharedMemorySize, LayMed::bytes);
  cudaFuncSetAttribute(k_query_large, cudaFuncAttributeMaxDynamicSharedMemorySize, LayLarge::bytes);
}

void launch_query_small(const QueryArgs& a, int grid, cudaStream_t st) {
  k_query_small<<<grid, 256, 8 * LaySmall::bytes, st>>>(a);
}
void launch_query_medium(const QueryArgs& a, int grid, cudaStream_t st) {
  k_query_medium<<<grid, kMedT, LayMed::bytes, st>>>(a);
}
void launch_query_large(const QueryArgs& a, int grid, cudaStream_t st) {
  k_query_large<<<grid, 512, LayLarge::bytes, st>>>(a);
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
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t total = a.n_lists * a.m;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += stride) {
    const HitRec* in = a.in + r * total;
    uint64_t taken = 0;
    uint32_t sel[8];
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < a.m; ++i) {
      int best = -1;
      uint32_t bh = 0, bt = 0;
      for (uint32_t e = 0; e < total; ++e) {
        if ((taken >> e) & 1ull) continue;
        const uint32_t t = in[e].tgt;
        if (t == kEmptyTgt) continue;
        const uint32_t h = in[e].hits;
        if (best < 0 || h > bh || (h == bh && t < bt)) { best = (int)e; bh = h; bt = t; }
      }
      if (best < 0) break;
      taken |= 1ull << best;
      sel[cnt++] = (uint32_t)best;
    }
    uint32_t* oc = a.out_cand ? a.out_cand + r * a.m * 4 : nullptr;
    for (uint32_t i = 0; i < a.m && oc; ++i) {
      if (i < cnt) {
        const HitRec& h = in[sel[i]];
        oc[4 * i] = h.tgt; oc[4 * i + 1] = h.hits; oc[4 * i + 2] = h.win_beg; oc[4 * i + 3] = h.win_end;
      } else {
        oc[4 * i] = kEmptyTgt; oc[4 * i + 1] = 0; oc[4 * i + 2] = 0; oc[4 * i + 3] = 0;
      }
    }
    uint32_t taxon = 0;
    if (cnt > 0 && in[sel[0]].hits >= a.hits_min) {
      const uint32_t top = in[sel[0]].hits;
      taxon = in[sel[0]].taxon;
      for (uint32_t i = 1; i < cnt; ++i)
        if (top - in[sel[i]].hits <= a.hits_diff) taxon = lca(a, taxon, in[sel[i]].taxon);
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
