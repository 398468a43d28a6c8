// Finalize (B5 count + B6 condensed layout + cap): the region-partitioned
// pair store becomes the condensed multi-value table.
//
// Paper: §4.1 P:465-466 (cap 254 locations per feature), §5.1
// (GPU hash table, condensed layout P:571-574), §5.2 P:692-694.
//
// B200 design.  The table is cut into sub-regions of
// kSubSlots = 8192 slots and linear probing wraps inside a key's sub-region,
// so a whole sub-region -- its distinct keys, their counts and their bucket
// offsets -- is built by ONE CTA in shared memory:
//   k_sub_count   : pairs per sub-region (per-chunk shared histograms)
//   scan          : first pair of each sub-region
//   k_sub_scatter : the pairs regrouped by sub-region (chunks staged in shared
//                   memory grouped by sub-region, written out coalesced)
//   k_sub_finalize: per sub-region: shared-memory hash count (the returned
//                   count is each location's rank in its key's bucket), scan
//                   of min(count, cap) over the slots, the table slice
//                   written out coalesced, every value written at offset +
//                   rank; the sub-region's values start at its first pair's
//                   index (gaps only where the cap truncates)
//   k_heavy_select: keys over the cap keep the cap smallest (S7)
// Every atomic of the count is a shared-memory atomic; the table and the
// value array are written once, sequentially per sub-region.
#include <algorithm>

#include "mc_block.cuh"
#include "mc_kernels.cuh"

namespace mc {

constexpr uint32_t kSplitT = 512, kSplitPer = 8, kSplitChunk = kSplitT * kSplitPer;  // 4096 pairs per chunk

// chunks of the pair store: ceil(rcap / chunk) per region (some empty), then the spill area
struct SplitSpace {
  uint64_t cpr, nchunks;
  __device__ explicit SplitSpace(const PairStore& ps) {
    cpr = (ps.rcap + kSplitChunk - 1) / kSplitChunk;
    nchunks = cpr * ps.nreg + (ps.spill_cap + kSplitChunk - 1) / kSplitChunk;
  }
  // first pair, pair count and region (nreg = spill) of chunk ch
  __device__ void chunk(const PairStore& ps, uint64_t ch, uint64_t* first, uint32_t* n, uint32_t* region) const {
    uint64_t off, fill;
    if (ch < cpr * ps.nreg) {
      *region = (uint32_t)(ch / cpr);
      off = (ch % cpr) * kSplitChunk;
      fill = min(ps.cursor[*region], (unsigned long long)ps.rcap);
      *first = (uint64_t)*region * ps.rcap + off;
    } else {
      *region = ps.nreg;
      off = (ch - cpr * ps.nreg) * kSplitChunk;
      fill = min(ps.cursor[ps.nreg], (unsigned long long)ps.spill_cap);
      *first = (uint64_t)ps.nreg * ps.rcap + off;
    }
    *n = off >= fill ? 0u : (uint32_t)min((uint64_t)kSplitChunk, fill - off);
  }
};

// Region r holds the keys whose home slot in a table of ps.nslots (the static
// maximum) lies in [r << shift, (r + 1) << shift); fastrange is monotone, so
// in the table actually used (a.nslots) their sub-regions form a range of at
// most 2^(shift - kSubLg) + 3 starting at sub_lo(r).
__device__ __forceinline__ uint64_t sub_lo(const FinalizeArgs& a, uint32_t r) {
  const unsigned __int128 x = (unsigned __int128)((uint64_t)r << a.ps.shift) * a.nslots;
  const uint64_t lo = (uint64_t)(x / a.ps.nslots);
  return lo ? (lo - 1) >> kSubLg : 0;
}
uint32_t split_bins(const FinalizeArgs& a) { return (1u << (a.ps.shift - kSubLg)) + 4; }

__device__ __forceinline__ uint64_t sub_of(const FinalizeArgs& a, uint32_t key) {
  return home_slot(key, a.nslots) >> kSubLg;
}

// Each CTA walks a CONTIGUOUS range of chunks, so consecutive chunks nearly
// always share a region: the shared histogram is flushed (one global add per
// (region run, sub-region)) only when the region changes, and chunks of one
// region need no barrier at all.
__global__ void __launch_bounds__(kSplitT) k_sub_count(FinalizeArgs a, uint32_t nbins) {
  extern __shared__ uint32_t hist[];  // [nbins]
  __shared__ uint64_t s_lo;
  const SplitSpace cs(a.ps);
  const uint64_t per = (cs.nchunks + gridDim.x - 1) / gridDim.x;
  const uint64_t c0 = blockIdx.x * per, c1 = min(cs.nchunks, c0 + per);
  uint32_t cur = 0xffffffffu;  // region whose counts the histogram holds
  uint64_t lo = 0;
  for (uint32_t b = threadIdx.x; b < nbins; b += kSplitT) hist[b] = 0;
  auto flush = [&]() {  // (all threads; CTA-uniform)
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += kSplitT) {
      const uint32_t h = hist[b];
      if (h) atomicAdd(&a.subcnt[lo + b], h);
      hist[b] = 0;
    }
  };
  for (uint64_t ch = c0; ch < c1; ++ch) {
    uint64_t first;
    uint32_t n, r;
    cs.chunk(a.ps, ch, &first, &n, &r);
    if (n == 0) continue;  // CTA-uniform
    if (r == a.ps.nreg) {  // spill: pairs of any region (rare)
      for (uint32_t i = threadIdx.x; i < n; i += kSplitT) atomicAdd(&a.subcnt[sub_of(a, a.ps.pairs[first + i].x)], 1u);
      continue;
    }
    if (r != cur) {  // CTA-uniform
      if (cur != 0xffffffffu) flush();
      if (threadIdx.x == 0) s_lo = sub_lo(a, r);  // (a 128-bit division: once per region run)
      __syncthreads();
      lo = s_lo;
      cur = r;
    }
    // all of a thread's (<= kSplitPer) key loads in flight before the shared atomics
    uint32_t key[kSplitPer];
#pragma unroll
    for (uint32_t k = 0; k < kSplitPer; ++k) {
      const uint32_t i = threadIdx.x + k * kSplitT;
      if (i < n) key[k] = a.ps.pairs[first + i].x;
    }
#pragma unroll
    for (uint32_t k = 0; k < kSplitPer; ++k) {
      if (threadIdx.x + k * kSplitT >= n) continue;
      const uint64_t b = sub_of(a, key[k]) - lo;
      if (b < nbins) atomicAdd(&hist[b], 1u);
      else atomicExch(&a.ps.err[2], 1);  // (cannot happen: sub_lo bound)
    }
  }
  if (cur != 0xffffffffu) flush();
}

void launch_sub_count(const FinalizeArgs& a, int sms, cudaStream_t st) {
  const uint32_t nb = split_bins(a);
  k_sub_count<<<sms * 4, kSplitT, nb * 4, st>>>(a, nb);
}

// Regroup: each chunk's pairs get their rank among the chunk's pairs of the
// same sub-region (shared atomic), claim one run per (chunk, sub-region) in
// `sorted`, are staged in shared memory grouped by sub-region and written out
// in order (consecutive lanes -> consecutive addresses).  The CTA's next
// non-empty chunk is fetched by a TMA bulk copy into shared memory while the
// current one is ranked, scanned and written (no registers held by the load).
struct ChunkInfo {
  uint64_t first, lo;
  uint32_t n, r;
};
__device__ __forceinline__ bool next_chunk(const FinalizeArgs& a, const SplitSpace& cs, uint64_t& ch, ChunkInfo* ci) {
  for (; ch < cs.nchunks; ch += gridDim.x) {
    cs.chunk(a.ps, ch, &ci->first, &ci->n, &ci->r);
    if (ci->n) {
      ci->lo = ci->r == a.ps.nreg ? 0 : sub_lo(a, ci->r);  // (a 128-bit division: once per chunk)
      ch += gridDim.x;
      return true;
    }
  }
  ci->n = 0;
  return false;
}

__global__ void __launch_bounds__(kSplitT, 2) k_sub_scatter(FinalizeArgs a, uint32_t nbins) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint2* pbuf = reinterpret_cast<uint2*>(sm);                                         // [kSplitChunk + 2] bulk-copy target
  uint2* stage = pbuf + kSplitChunk + 2;                                              // [kSplitChunk]
  unsigned long long* gpos = reinterpret_cast<unsigned long long*>(stage + kSplitChunk);  // [nbins]
  uint32_t* hist = reinterpret_cast<uint32_t*>(gpos + nbins);                         // [nbins]
  uint32_t* bstart = hist + nbins;                                                    // [nbins]
  uint16_t* sbin = reinterpret_cast<uint16_t*>(bstart + nbins);                       // [kSplitChunk]
  __shared__ ChunkInfo s_ci[2];
  __shared__ __align__(8) uint64_t s_bar;
  const SplitSpace cs(a.ps);
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  uint64_t ch = blockIdx.x;  // (thread 0's cursor over the CTA's chunks)
  for (uint32_t b = tid; b < nbins; b += kSplitT) hist[b] = 0;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    if (next_chunk(a, cs, ch, &s_ci[0])) {
      const uint32_t bytes = ((s_ci[0].n + 1) & ~1u) * 8u;
      mbar_arrive_expect(&s_bar, bytes);
      bulk_g2s(pbuf, a.ps.pairs + s_ci[0].first, bytes, &s_bar);
    }
  }
  __syncthreads();
  for (uint32_t it = 0;; ++it) {
    const ChunkInfo ci = s_ci[it & 1];
    if (ci.n == 0) break;  // CTA-uniform
    const uint32_t n = ci.n;
    mbar_wait(&s_bar, it & 1);
    uint2 p[kSplitPer];
#pragma unroll
    for (uint32_t k = 0; k < kSplitPer; ++k)
      if (tid + k * kSplitT < n) p[k] = pbuf[tid + k * kSplitT];
    __syncthreads();  // pbuf consumed, s_ci[it & 1] read, previous hist zeroing visible
    if (tid == 0 && next_chunk(a, cs, ch, &s_ci[(it + 1) & 1])) {
      const ChunkInfo& nx = s_ci[(it + 1) & 1];
      const uint32_t bytes = ((nx.n + 1) & ~1u) * 8u;
      mbar_arrive_expect(&s_bar, bytes);
      bulk_g2s(pbuf, a.ps.pairs + nx.first, bytes, &s_bar);
    }
    if (ci.r == a.ps.nreg) {  // spill (rare): one global atomic per pair
#pragma unroll
      for (uint32_t k = 0; k < kSplitPer; ++k) {
        if (tid + k * kSplitT >= n) continue;
        const uint64_t s = sub_of(a, p[k].x);
        a.sorted[a.subbase[s] + atomicAdd(&a.subcnt[s], 1u)] = p[k];
      }
      __syncthreads();  // (s_ci of the next chunk written by thread 0)
      continue;
    }
    const uint64_t lo = ci.lo;
    uint32_t bin[kSplitPer], rk[kSplitPer];
#pragma unroll
    for (uint32_t k = 0; k < kSplitPer; ++k) {
      if (tid + k * kSplitT < n) {
        bin[k] = (uint32_t)(sub_of(a, p[k].x) - lo);
        rk[k] = atomicAdd(&hist[bin[k]], 1u);
      }
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the bins (one warp)
      uint32_t run = 0;
      for (uint32_t b0 = 0; b0 < nbins; b0 += 32) {
        const uint32_t b = b0 + lane, h = b < nbins ? hist[b] : 0u;
        uint32_t x = h;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, d);
          if (lane >= (uint32_t)d) x += y;
        }
        if (b < nbins) bstart[b] = run + x - h;
        run += __shfl_sync(kFull, x, 31);
      }
    }
    // the run claims (global atomics) by the upper warps, concurrent with warp 0's scan
    for (uint32_t b = tid - kSplitT / 2; b < nbins; b += kSplitT / 2)
      if (tid >= kSplitT / 2 && hist[b]) gpos[b] = a.subbase[lo + b] + atomicAdd(&a.subcnt[lo + b], hist[b]);
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kSplitPer; ++k) {
      if (tid + k * kSplitT < n) {
        const uint32_t j = bstart[bin[k]] + rk[k];
        stage[j] = p[k];
        sbin[j] = (uint16_t)bin[k];
      }
    }
    __syncthreads();
    for (uint32_t b = tid; b < nbins; b += kSplitT) hist[b] = 0;  // (ordered before the next atomics by the next loop's barrier)
    for (uint32_t j = tid; j < n; j += kSplitT) {
      const uint32_t b = sbin[j];
      a.sorted[gpos[b] + (j - bstart[b])] = stage[j];
    }
  }
}

void launch_sub_scatter(const FinalizeArgs& a, int sms, cudaStream_t st) {
  const uint32_t nb = split_bins(a);
  const size_t smem = (size_t)(kSplitChunk + 2) * 8 + (size_t)kSplitChunk * (8 + 2) + (size_t)nb * (8 + 4 + 4) + 16;
  cudaFuncSetAttribute(k_sub_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sub_scatter, kSplitT, smem);
  k_sub_scatter<<<sms * std::max(per_sm, 1), kSplitT, smem, st>>>(a, nb);
}

// gapped build window index -> ranked window index (targets ordered by id)
__device__ __forceinline__ uint32_t to_ranked(const FinalizeArgs& a, uint32_t g) {
  if (a.identity) return g;
  // gapped targets are >= kRankGap = 1024 ids apart: a 1024-id block holds at most
  // one target start, so one 16-byte lookup (L2-resident) replaces a binary search
  const uint4 c = a.gcoarse[g >> 10];
  return g + (g >= c.y ? c.z : c.x);
}

constexpr uint32_t kFinT = 512, kFinPer = kSubSlots / kFinT;  // 16 slots per thread
// values per sub-region staged in shared memory (2 CTAs of 64 + 47 KB per SM)
constexpr uint32_t kFinStage = 12032;
#ifndef MC_FIN_RANK
#define MC_FIN_RANK 1
#endif
constexpr bool kRankScratch = MC_FIN_RANK;  // placement by the count pass's ranks (k_sub_finalize)
constexpr uint32_t kHeavyFlag = 0x80000000u;
// an occupied entry's cursor word always carries this bit, so a claimed slot
// never reads as empty (key 0 with local offset 0 would otherwise be all-zero)
constexpr uint32_t kOccFlag = 0x40000000u, kCurMask = kOccFlag - 1u;

// the count / cursor half (high 32 bits) of a shared-memory table entry
__device__ __forceinline__ uint32_t* hi_word(unsigned long long* w) { return reinterpret_cast<uint32_t*>(w) + 1; }

// shared-memory slot of `key` in the sub-region starting at global slot s0
__device__ __forceinline__ uint32_t local_home(const FinalizeArgs& a, uint32_t key, uint64_t s0) {
  return (uint32_t)(home_slot(key, a.nslots) - s0);
}

__global__ void __launch_bounds__(kFinT, 2) k_sub_finalize(FinalizeArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* tab = reinterpret_cast<unsigned long long*>(sm);  // [kSubSlots] key | count << 32
  uint32_t* vst = reinterpret_cast<uint32_t*>(tab + kSubSlots);         // [kFinStage] the first values, staged
  __shared__ uint32_t wsum[kFinT / 32];
  __shared__ unsigned long long s_ticket;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t mask = kSubSlots - 1;
  uint64_t st_keys = 0, st_locs = 0, st_trunc = 0, st_vals = 0;
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(&a.counters[6], 1ull);
#pragma unroll
    for (uint32_t j = 0; j < kFinPer; j += 2)
      reinterpret_cast<ulonglong2*>(tab)[tid + (j >> 1) * kFinT] = make_ulonglong2(0, 0);
    __syncthreads();
    const uint64_t s = s_ticket;
    if (s >= a.nsub) break;  // CTA-uniform
    const uint64_t s0 = s << kSubLg, p0 = a.subbase[s], n = a.subbase[s + 1] - p0;

    // ---- count: shared-memory hash (claim with CAS, then count); 4 pair loads in flight.
    // The count returned to a location is its rank in its key's bucket.  With
    // kRankScratch, a sub-region whose values all fit the shared-memory staging
    // parks each location's slot | rank << 13 in its own (not yet written)
    // value range: the placement below then needs no second probe and no
    // atomic, and the range is overwritten only by the final copy-out, after
    // the last read.  (Parking it over the pair's dead key instead dirtied every
    // pair line: slower on the RefSeq-shaped shard.)
    const bool rank_scratch = kRankScratch && n <= kFinStage;  // CTA-uniform
    uint32_t* scratch = a.values + p0;
    for (uint64_t i0 = tid; i0 < n; i0 += 4 * kFinT) {
      uint32_t key[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) key[u] = i0 + u * kFinT < n ? a.sorted[p0 + i0 + u * kFinT].x : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u * kFinT >= n) continue;
        uint32_t h = local_home(a, key[u], s0), probes = 0, rank = 0;
        for (; probes < kSubSlots; ++probes, h = (h + 1) & mask) {
          unsigned long long w = tab[h];
          if (w == 0) {
            w = atomicCAS(&tab[h], 0ull, (unsigned long long)key[u] | (1ull << 32));
            if (w == 0) break;  // claimed: rank 0
          }
          if ((uint32_t)w == key[u]) {
            rank = atomicAdd(hi_word(&tab[h]), 1u);  // 32-bit: 64-bit shared atomicAdd is a CAS loop on sm_100
            break;
          }
        }
        if (probes == kSubSlots) atomicExch(&a.ps.err[0], 1);  // sub-region full: table too small
        if (rank_scratch) scratch[i0 + u * kFinT] = probes == kSubSlots ? 0xffffffffu : h | rank << kSubLg;
      }
    }
    __syncthreads();

    // ---- bucket offsets: exclusive scan of min(count, cap).  Any packing of
    // the buckets inside the sub-region's value range is valid, so thread tid
    // owns the slots tid + kFinT * j (conflict-free shared-memory reads) and
    // the buckets follow that order.
    uint32_t sum = 0;
#pragma unroll
    for (uint32_t j = 0; j < kFinPer; ++j) {
      const unsigned long long w = tab[tid + j * kFinT];
      const uint32_t c = (uint32_t)(w >> 32);
      sum += min(c, a.cap);
      st_keys += w != 0;
      st_locs += c;
      st_trunc += c > a.cap ? c - a.cap : 0;
    }
    uint32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, d);
      if (lane >= (uint32_t)d) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    uint32_t excl = incl - sum, total = 0;
#pragma unroll
    for (uint32_t w = 0; w < kFinT / 32; ++w) {
      const uint32_t x = wsum[w];
      excl += w < wid ? x : 0u;
      total += x;
    }
    // ---- the sub-region's first value: its first PAIR's index (subbase[s]).
    // A sub-region holds at most as many values as pairs, so value buckets
    // start where the sub-region's pairs start; only keys over the cap leave
    // gaps (their excess), and no sub-region waits on its predecessors.
    st_vals += tid == 0 ? total : 0u;
    const uint64_t base = p0;
    if (tid == 0) {
      a.vbase[s] = base;
      if (total > kMaxSubValues) atomicExch(&a.ps.err[0], 1);  // sub-region offsets overflow: bigger table
    }

    // ---- the table slice (coalesced); keys over the cap get a side bucket.
    // Each slot's count then becomes its fill cursor: key | local offset << 32
    // (heavy keys: key | (kHeavyFlag | heavy index) << 32; both with kOccFlag)
#pragma unroll 4
    for (uint32_t j = 0; j < kFinPer; ++j) {
      const uint32_t slot = tid + j * kFinT;
      const unsigned long long w = tab[slot];
      const uint32_t c = (uint32_t)(w >> 32), loff = excl;
      excl += min(c, a.cap);
      a.T[s0 + slot] = KSlot{w ? make_slot((uint32_t)w, min(c, a.cap), loff) : 0ull};
      if (!w) continue;
      uint32_t cur = kOccFlag | loff;
      if (c > a.cap) {
        const unsigned long long so = atomicAdd(&a.counters[5], (unsigned long long)c);
        const unsigned long long hi = atomicAdd(&a.counters[3], 1ull);
        // .x: the side bucket's fill cursor (placed by rank: already at its end)
        a.heavy[hi] = make_ulonglong2(rank_scratch ? so + c : so, (base + loff) | ((unsigned long long)c << 40));
        cur = kHeavyFlag | kOccFlag | (uint32_t)hi;
      }
      tab[slot] = (w & 0xffffffffull) | ((unsigned long long)cur << 32);
    }
    __syncthreads();

    // ---- every location into its key's bucket (heavy: side bucket, selected
    // later).  Values at local offsets < kFinStage are staged in shared memory
    // and written out coalesced below; the rest go straight to HBM.  (The loop
    // runs while the warp's first lane is in range: warp-uniform, for __syncwarp.)
    if (rank_scratch) {
      // slot and rank from the count pass: offset = the slot's bucket start + rank
      for (uint64_t i0 = tid; i0 < n; i0 += 4 * kFinT) {
        uint32_t val[4], sc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = i0 + u * kFinT < n;
          val[u] = ok ? a.sorted[p0 + i0 + u * kFinT].y : 0u;
          sc[u] = ok ? __ldcg(scratch + i0 + u * kFinT) : 0xffffffffu;  // (written by this CTA: via L2)
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (sc[u] == 0xffffffffu) continue;  // (not inserted: sub-region full, finalize reruns)
          const uint32_t cur = *hi_word(&tab[sc[u] & mask]), rank = sc[u] >> kSubLg;
          const uint32_t v = to_ranked(a, val[u]);
          if (cur & kHeavyFlag) {  // side bucket [x - c, x): x was set to its end
            const ulonglong2 hv = a.heavy[cur & kCurMask];
            a.side[hv.x - (hv.y >> 40) + rank] = v;
          } else {
            vst[(cur & kCurMask) + rank] = v;  // (< total <= n <= kFinStage)
          }
        }
      }
    } else
    for (uint64_t i0 = tid; i0 - lane < n; i0 += 4 * kFinT) {
      uint2 kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) kv[u] = i0 + u * kFinT < n ? a.sorted[p0 + i0 + u * kFinT] : make_uint2(0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool valid = i0 + u * kFinT < n;
        uint32_t h = local_home(a, kv[u].x, s0) & mask, probes = 0;  // (mask: invalid lanes' key 0)
        unsigned long long w = valid ? tab[h] : 0ull;
        for (; valid && probes < kSubSlots && (w == 0 || (uint32_t)w != kv[u].x); ++probes) {
          h = (h + 1) & mask;
          w = tab[h];
        }
        // reconverge before the bucket write (otherwise it runs once per probe-length group)
        __syncwarp();
        if (!valid || probes == kSubSlots) continue;  // (not inserted: sub-region full, finalize reruns)
        const uint32_t v = to_ranked(a, kv[u].y);
        if ((uint32_t)(w >> 32) & kHeavyFlag) {
          const uint32_t hi = (uint32_t)(w >> 32) & kCurMask;
          a.side[atomicAdd(&a.heavy[hi].x, 1ull)] = v;
        } else {
          const uint32_t o = atomicAdd(hi_word(&tab[h]), 1u) & kCurMask;
          if (o < kFinStage) vst[o] = v;
          else a.values[base + o] = v;
        }
      }
    }
    __syncthreads();
    // (heavy buckets inside the staged range carry garbage here; k_heavy_select
    // runs afterwards and overwrites them)
    for (uint32_t i = tid; i < min(total, kFinStage); i += kFinT) a.values[base + i] = vst[i];
    // the truncated excess of keys over the cap leaves [total, n) unused: mark it
    // (never read by a query; keeps dumps and compute-sanitizer initcheck clean)
    for (uint64_t i = total + tid; i < n; i += kFinT) a.values[base + i] = 0xffffffffu;
  }
  // statistics: one atomic per warp
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    st_keys += __shfl_xor_sync(kFull, st_keys, d);
    st_locs += __shfl_xor_sync(kFull, st_locs, d);
    st_trunc += __shfl_xor_sync(kFull, st_trunc, d);
    st_vals += __shfl_xor_sync(kFull, st_vals, d);
  }
  if (lane == 0) {
    if (st_keys) atomicAdd(&a.counters[0], (unsigned long long)st_keys);
    if (st_locs) atomicAdd(&a.counters[1], (unsigned long long)st_locs);
    if (st_trunc) atomicAdd(&a.counters[2], (unsigned long long)st_trunc);
    if (st_vals) atomicAdd(&a.counters[4], (unsigned long long)st_vals);
  }
}

void launch_sub_finalize(const FinalizeArgs& a, int sms, cudaStream_t st) {
  const size_t smem = (size_t)kSubSlots * 8 + (size_t)kFinStage * 4;
  cudaFuncSetAttribute(k_sub_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sub_finalize, kFinT, smem);
  k_sub_finalize<<<sms * std::max(per_sm, 1), kFinT, smem, st>>>(a);
}

// ---- B6 cap: one CTA per heavy key keeps the cap smallest of
// its side bucket (chunks of 1024 merged into a sorted best-cap buffer) -----
__global__ void __launch_bounds__(256) k_heavy_select(FinalizeArgs a) {
  constexpr uint32_t NT = 256, BUF = 2048, CH = 1024;
  __shared__ uint32_t buf[BUF];
  const uint32_t tid = threadIdx.x;
  const uint64_t nh = a.counters[3];
  for (uint64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const uint32_t n = (uint32_t)(a.heavy[h].y >> 40);
    const uint64_t side_off = a.heavy[h].x - n, final_off = a.heavy[h].y & ((1ull << 40) - 1);  // x: fill cursor
    const uint32_t* src = a.side + side_off;
    uint32_t held = 0;  // sorted smallest values so far (<= cap)
    for (uint32_t c0 = 0; c0 < n; c0 += CH) {
      const uint32_t m = min(CH, n - c0);
      for (uint32_t i = tid; i < BUF - held; i += NT) buf[held + i] = i < m ? src[c0 + i] : 0xffffffffu;
      __syncthreads();
      bitonic_sort<NT>(buf, BUF, tid);
      held = min(a.cap, held + m);
      __syncthreads();
    }
    for (uint32_t i = tid; i < a.cap; i += NT) a.values[final_off + i] = buf[i];
    __syncthreads();
  }
}

void launch_heavy_select(const FinalizeArgs& a, int grid, cudaStream_t st) { k_heavy_select<<<grid, 256, 0, st>>>(a); }

}  // namespace mc
