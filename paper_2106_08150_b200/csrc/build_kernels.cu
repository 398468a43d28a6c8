// Build-side kernels (B1-B5 insert side): thread-per-window sketch and the
// region-partitioned pair store; device-wide scan.  Finalize (B5 count + B6)
// is in finalize_kernels.cu.
//
// Paper: §4.1 P:315-474 (build), §5.1 P:647-672 (GPU hash tables),
// §5.2 P:692-694 (build pipeline = steps 1-3 then insert).
//
// B200 design: random 32-byte accesses into a table much larger
// than L2 run at ~20 G/s on this part, a tenth of copy bandwidth
// (profiles/r01_random_access_ceilings.jsonl).  Insert calls therefore only
// sketch and append (feature, window) pairs to buckets by TABLE REGION
// (home slot >> shift, <= 1024 regions), written out coalesced; finalize
// turns each region into table sub-regions small enough for shared memory.
#include "mc_block.cuh"
#include "mc_kernels.cuh"

namespace mc {

// ---------------------------------------------------------------------------
// B1-B4 + partition: CTA tiles of 256 windows, one THREAD per window
// (sketch_warp_windows: each warp stages its 32 windows into shared memory,
// then every lane rolls over its own window).  The tile's features are counted
// per table region, claim space in the region buckets with one global atomic
// per (tile, region) and are scattered from registers; a full bucket spills
// into a shared spill area.
// ---------------------------------------------------------------------------
#ifndef MC_SK_TILE
#define MC_SK_TILE 256  // windows (= threads) per CTA tile of k_sketch_partition
#endif
constexpr uint32_t kTileW = MC_SK_TILE;
static_assert(kTileW % 32 == 0, "whole warps");
#ifndef MC_SK_FEAT_UNROLL
#define MC_SK_FEAT_UNROLL 1  // per-feature region loop unrolled in registers (0: rolled, parked in the window slots; s2l: 9.94 -> 9.77 ms)
#endif
#ifndef MC_SKETCH_FILTER
#define MC_SKETCH_FILTER 0  // 1: candidate-filtered fast path (mc_device.cuh sketch_slot_filter; A/B s2b: slower)
#endif

// Window g of the batch (target t) -> first char, k-mer count (0: none), value
__device__ __forceinline__ void window_at(const BuildBatch& b, const SketchCfg& c, uint64_t g, uint32_t t,
                                          const uint8_t*& p, uint32_t& nk, uint32_t& val) {
  p = b.chars;
  nk = 0;
  val = 0;
  if (g >= b.total_windows) return;
  const uint64_t j = g - b.win_base[t];
  const uint64_t first = j * c.stride;
  nk = (uint32_t)min((uint64_t)c.stride, b.seq_len[t] - c.k + 1 - first);
  p = b.chars + b.seq_off[t] + first;
  val = b.bwi_base[t] + (uint32_t)j;
}

__device__ __forceinline__ uint32_t warp_targets(const BuildBatch& b, uint64_t g0, uint32_t& t0, uint32_t lane) {
  return warp_segment(b.win_base, b.nt, b.total_windows, g0, t0, lane);
}

constexpr uint32_t kMaxRegions = 1024;
constexpr uint32_t kRegPerThread = (kMaxRegions + kTileW - 1) / kTileW;  // regions owned by a thread in the tile scan
constexpr uint32_t kTilePairs = kTileW * 16;               // s <= 16
// dynamic smem: [staging: max(window slots, pairs)] [region arrays]
constexpr size_t kStageBytes = (size_t)kTilePairs * 8 > (size_t)kTileW * kSlotWords * 4
                                   ? (size_t)kTilePairs * 8 : (size_t)kTileW * kSlotWords * 4;

struct TileRegions {             // per table region, for the current tile
  uint32_t* cnt;                 // pairs of the tile in the region
  uint32_t* loc;                 // exclusive scan of cnt: the region's first staged pair
  uint32_t* lim;                 // staged pairs [loc, lim) go to the region's bucket ...
  unsigned long long* gbase;     // ... at gbase + j
  unsigned long long* sgbase;    // staged pairs [lim, loc + cnt) spill to sgbase + j
  uint32_t* cand;                // sketch phase only: the warps' candidate buffers, aliasing
                                 // gbase / sgbase / loc / lim (dead until the tile scan)
};
constexpr uint32_t kCandBytes = kTileW * kCandRows * 4;  // 8 warps x kCandRows rows x 32 lanes

// The tile's pairs: each region's bucket share is claimed with one global
// atomic, the pairs are staged in shared memory grouped by region, and the
// staged array is written out in order, so consecutive lanes store
// consecutive bucket addresses (coalesced) instead of 32 random regions.
template <uint32_t K>
__device__ __forceinline__ void sketch_partition_tiles(const BuildBatch& b, const SketchCfg& c, const PairStore& ps,
                                                       uint8_t* stage, const TileRegions& R, uint32_t* hll) {
  __shared__ uint32_t wsum[kTileW / 32 + 1];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t* wslots = reinterpret_cast<uint32_t*>(stage) + wid * 32 * kSlotWords;
  uint2* spair = reinterpret_cast<uint2*>(stage);                                   // [kTilePairs]
  uint64_t tile, tend;
  cta_tiles((b.total_windows + kTileW - 1) / kTileW, &tile, &tend);
  const uint64_t spill_end = (uint64_t)ps.nreg * ps.rcap + ps.spill_cap;
  const uint8_t* chars_end = b.nt ? b.chars + b.seq_off[b.nt - 1] + b.seq_len[b.nt - 1] : b.chars;
  uint32_t t0 = tile < tend ? upper_index(b.win_base, b.nt + 1, min(tile * kTileW + wid * 32, b.total_windows - 1))
                            : 0u;
  for (uint32_t i = threadIdx.x; i < ps.nreg; i += blockDim.x) R.cnt[i] = 0;
  __syncthreads();
  for (; tile < tend; ++tile) {
    const uint64_t g0 = tile * kTileW + wid * 32;
    const uint8_t* p;
    uint32_t nk, val;
    window_at(b, c, g0 + lane, warp_targets(b, g0, t0, lane), p, nk, val);
    if (lane == 0 && tile + 1 < tend) {  // the warp's next-tile span (same target: 256 windows on) -> L2
      const uint8_t* q = p + (size_t)kTileW * c.stride;
      if (q + 32 * c.stride + 32 <= chars_end) prefetch_l2(q, 32 * c.stride + 16);
    }
    uint32_t v[16], rr[16];
    const int n = sketch_warp_windows<K, MC_SKETCH_FILTER>(wslots, p, nk, c, lane, v, R.cand + wid * 32 * kCandRows);
#if MC_SK_FEAT_UNROLL
    // region | rank of each pair among the tile's pairs of that region: all 16
    // region hashes, then the 16 (predicated) shared atomics in flight together
    uint32_t r16[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r16[i] = (uint32_t)(fastrange64(slot_hash(v[i]), ps.nslots) >> ps.shift);
#pragma unroll
    for (int i = 0; i < 16; ++i) rr[i] = r16[i] | (i < n ? atomicAdd(&R.cnt[r16[i]], 1u) : 0u) << 16;
#else
    // region | rank of each pair among the tile's pairs of that region.  A
    // rolled loop over the features parked in the lane's column of the (dead)
    // window slots: the unrolled form was 14 KB of code, and the kernel's hot
    // code then overflowed the SM's 32 KB instruction cache (ncu s2b: ~20 % of
    // stall samples waiting on instruction fetch)
    __syncwarp();
    uint32_t* col = wslots + lane;  // row i at col[32 i]: rows 0..15 features, 16..31 region | rank
#pragma unroll
    for (int i = 0; i < 16; ++i) col[i << 5] = v[i];
    // (4 features per step, branch-free up to the atomics so their chains
    // interleave; the HyperLogLog update moved to the write-out, which hashes
    // every pair's key anyway)
#pragma unroll 1
    for (int i0 = 0; i0 < n; i0 += 4) {
      uint32_t r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = (uint32_t)(fastrange64(slot_hash(col[(i0 + u) << 5]), ps.nslots) >> ps.shift);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u < n) col[(16 + i0 + u) << 5] = r[u] | atomicAdd(&R.cnt[r[u]], 1u) << 16;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) rr[i] = col[(16 + i) << 5];
#endif
    __syncthreads();  // (A) counts complete; the window slots are free
    {  // thread owns regions [4 tid, 4 tid + 4): bucket claims (in flight together) and the tile scan
      const uint32_t r0 = threadIdx.x * kRegPerThread;
      uint32_t k[kRegPerThread], sum = 0;
      unsigned long long at[kRegPerThread];
#pragma unroll
      for (uint32_t j = 0; j < kRegPerThread; ++j) {
        k[j] = r0 + j < ps.nreg ? R.cnt[r0 + j] : 0u;
        at[j] = k[j] ? atomicAdd(&ps.cursor[r0 + j], (unsigned long long)k[j]) : 0ull;
        sum += k[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, d);
        if (lane >= (uint32_t)d) incl += y;
      }
      if (lane == 31) wsum[wid] = incl;
      __syncthreads();
      uint32_t loc = incl - sum;
      for (uint32_t w = 0; w < wid; ++w) loc += wsum[w];
      uint32_t spill = 0;
#pragma unroll
      for (uint32_t j = 0; j < kRegPerThread; ++j) {
        const uint32_t r = r0 + j;
        if (k[j]) {
          const uint32_t nb = at[j] >= ps.rcap ? 0u : (uint32_t)min((unsigned long long)k[j], ps.rcap - at[j]);
          R.loc[r] = loc;
          R.lim[r] = loc + nb;
          R.gbase[r] = (unsigned long long)r * ps.rcap + at[j] - loc;
          spill |= (nb < k[j] ? 1u : 0u) << j;
        }
        loc += k[j];
      }
      while (spill) {  // (rare) bucket full: the rest of this tile's pairs of region r spill
        const uint32_t r = r0 + __ffs(spill) - 1;
        spill &= spill - 1;
        const uint32_t l = R.lim[r], e = R.loc[r] + R.cnt[r];
        const unsigned long long sp = atomicAdd(&ps.cursor[ps.nreg], (unsigned long long)(e - l));
        if (sp + (e - l) > ps.spill_cap) atomicExch(&ps.err[1], 1);
        R.sgbase[r] = (unsigned long long)ps.nreg * ps.rcap + sp - l;
      }
      if (threadIdx.x == kTileW - 1) wsum[kTileW / 32] = loc;  // the tile's pair count
    }
    __syncthreads();  // (B) region bases known
#pragma unroll
    for (int i = 0; i < 16; ++i) {  // (branch-free: the 16 region-base reads in flight together)
      const bool ok = i < n;
      const uint32_t r = ok ? rr[i] & 0xffffu : 0u, j = R.loc[r] + (rr[i] >> 16);
      if (ok) spair[j] = make_uint2(v[i], val);
    }
    for (uint32_t r = threadIdx.x; r < ps.nreg; r += blockDim.x) R.cnt[r] = 0;  // for the next tile
    __syncthreads();  // (C) pairs staged by region
    const uint32_t total = wsum[kTileW / 32];
    // 4 staged pairs per thread per step: their shared-memory reads and region
    // computations overlap (a rolled loop ran one dependent chain at a time)
#pragma unroll 1
    for (uint32_t j0 = threadIdx.x; j0 < total; j0 += 4 * kTileW) {
      uint2 pr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u * kTileW;
        pr[u] = j < total ? spair[j] : make_uint2(0, 0);
      }
      // (branch-free up to the store, so the 4 dependent chains interleave; a
      // position past the tile's pairs computes a harmless region of key 0)
      uint64_t at[4], h[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u * kTileW;
        // (the region again from the key: ~6 FMA-pipe instructions instead of a staged u16)
        h[u] = slot_hash(pr[u].x);
        const uint32_t r = (uint32_t)(fastrange64(h[u], ps.nslots) >> ps.shift);
        at[u] = j < R.lim[r] ? R.gbase[r] + j : R.sgbase[r] + j;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u * kTileW >= total) continue;
        if (at[u] < spill_end) ps.pairs[at[u]] = pr[u];
        // HyperLogLog of the distinct features, on the hash-space sample whose
        // bits 50..53 are 0 (kHllSampleBits): one register update per 16 pairs
        if (((h[u] >> (64 - kHllBits - kHllSampleBits)) & ((1u << kHllSampleBits) - 1u)) == 0) {
          const uint32_t hi = (uint32_t)(h[u] >> (64 - kHllBits));
          const uint32_t rho =
              (uint32_t)__clzll((h[u] << (kHllBits + kHllSampleBits)) | (1ull << (kHllBits + kHllSampleBits - 1))) + 1u;
          if (rho > hll[hi]) atomicMax(&hll[hi], rho);  // registers saturate fast: most updates are no-ops
        }
      }
    }
    __syncthreads();  // (D) staging free for the next tile's windows
  }
}

#ifndef MC_SK_MINB
#define MC_SK_MINB (768 / MC_SK_TILE)  // CTAs per SM the registers are budgeted for: 80 registers (4 CTAs of 256 at 64: slower, s2d)
#endif
__global__ void __launch_bounds__(kTileW, MC_SK_MINB) k_sketch_partition(BuildBatch b, SketchCfg c, PairStore ps) {
  extern __shared__ __align__(16) uint8_t smem[];
  TileRegions R;
  R.gbase = reinterpret_cast<unsigned long long*>(smem + kStageBytes);
  R.sgbase = R.gbase + ps.nreg;
  R.loc = reinterpret_cast<uint32_t*>(R.sgbase + ps.nreg);
  R.lim = R.loc + ps.nreg;
  R.cand = reinterpret_cast<uint32_t*>(R.gbase);
  R.cnt = reinterpret_cast<uint32_t*>(smem + kStageBytes + max((size_t)ps.nreg * 24, MC_SKETCH_FILTER ? (size_t)kCandBytes : 0));
  __shared__ uint32_t hll[kHllRegs];  // distinct-feature estimate (sizes the table at finalize)
  for (uint32_t i = threadIdx.x; i < kHllRegs; i += blockDim.x) hll[i] = 0;
  if (c.k == 16) sketch_partition_tiles<16>(b, c, ps, smem, R, hll);
  else sketch_partition_tiles<0>(b, c, ps, smem, R, hll);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kHllRegs; i += blockDim.x)
    if (hll[i]) atomicMax(&ps.hll[i], hll[i]);
}

size_t sketch_partition_smem(uint32_t nreg) {  // [stage] [gbase sgbase loc lim | cand] [cnt]
  return kStageBytes + max((size_t)nreg * (8 + 8 + 4 + 4), MC_SKETCH_FILTER ? (size_t)kCandBytes : 0) + (size_t)nreg * 4;
}

void launch_sketch_partition(const BuildBatch& b, SketchCfg c, const PairStore& ps, int sms, cudaStream_t st) {
  const size_t smem = sketch_partition_smem(ps.nreg);
  cudaFuncSetAttribute(k_sketch_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sketch_partition, kTileW, smem);
  k_sketch_partition<<<sms * max(per_sm, 1), kTileW, smem, st>>>(b, c, ps);
}

// diagnostic: the same sketch, written out per window
template <uint32_t K>
__device__ __forceinline__ void debug_sketch_tiles(const BuildBatch& b, const SketchCfg& c, uint32_t* slots,
                                                   uint32_t* cand, uint32_t* feats, uint32_t* counts) {
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint64_t tile, tend;
  cta_tiles((b.total_windows + kTileW - 1) / kTileW, &tile, &tend);
  uint32_t t0 = tile < tend ? upper_index(b.win_base, b.nt + 1, min(tile * kTileW + wid * 32, b.total_windows - 1))
                            : 0u;
  for (; tile < tend; ++tile) {
    const uint64_t g0 = tile * kTileW + wid * 32, g = g0 + lane;
    const uint8_t* p;
    uint32_t nk, val;
    window_at(b, c, g, warp_targets(b, g0, t0, lane), p, nk, val);
    uint32_t v[16];
    const int n = sketch_warp_windows<K, MC_SKETCH_FILTER>(slots + wid * 32 * kSlotWords, p, nk, c, lane, v,
                                               cand + wid * 32 * kCandRows);
    if (g < b.total_windows) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if ((uint32_t)i < c.s) feats[g * c.s + i] = i < n ? v[i] : 0u;
      counts[g] = (uint32_t)n;
    }
    __syncwarp();
  }
}

// (the same sketch routine as k_sketch_partition, filtered fast path included)
__global__ void __launch_bounds__(kTileW) k_debug_sketch(BuildBatch b, SketchCfg c, uint32_t* feats, uint32_t* counts) {
  extern __shared__ __align__(16) uint8_t dsm[];
  uint32_t* slots = reinterpret_cast<uint32_t*>(dsm);      // [kTileW * kSlotWords]
  uint32_t* cand = slots + kTileW * kSlotWords;            // [kTileW * kCandRows]
  if (c.k == 16) debug_sketch_tiles<16>(b, c, slots, cand, feats, counts);
  else debug_sketch_tiles<0>(b, c, slots, cand, feats, counts);
}

void launch_debug_sketch(const BuildBatch& b, SketchCfg c, uint32_t* feats, uint32_t* counts, int grid,
                         cudaStream_t st) {
  const int smem = (int)((size_t)kTileW * (kSlotWords + kCandRows) * 4);
  cudaFuncSetAttribute(k_debug_sketch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_debug_sketch<<<grid, kTileW, smem, st>>>(b, c, feats, counts);
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan (reduce -> scan block sums -> scan tiles).
// ---------------------------------------------------------------------------
constexpr uint32_t kScanT = 256, kScanI = 16, kScanTile = kScanT * kScanI;

template <typename TI>
__global__ void __launch_bounds__(kScanT) k_scan_reduce(const TI* __restrict__ in, uint64_t n, uint64_t* sums,
                                                        uint64_t clamp) {
  __shared__ uint64_t red[kScanT / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t acc = 0;
  for (uint32_t i = threadIdx.x; i < kScanTile; i += kScanT)
    if (base + i < n) acc += min((uint64_t)in[base + i], clamp);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int i = 0; i < (int)(kScanT / 32); ++i) t += red[i];
    sums[blockIdx.x] = t;
  }
}

template <typename TI>
__global__ void __launch_bounds__(kScanT) k_scan_tiles(const TI* __restrict__ in, uint64_t* out, uint64_t n,
                                                       const uint64_t* prefix, uint64_t* total, uint64_t clamp) {
  __shared__ uint64_t wsum[kScanT / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanI;
  uint64_t v[kScanI];
  uint64_t acc = 0;
#pragma unroll
  for (uint32_t i = 0; i < kScanI; ++i) {
    v[i] = base + i < n ? min((uint64_t)in[base + i], clamp) : 0ull;
    acc += v[i];
  }
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint64_t x = acc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = prefix ? prefix[blockIdx.x] : 0ull;
    for (uint32_t i = 0; i < kScanT / 32; ++i) {
      const uint64_t y = wsum[i];
      wsum[i] = t;
      t += y;
    }
    wsum[kScanT / 32] = t;
  }
  __syncthreads();
  uint64_t run = wsum[wid] + x - acc;
#pragma unroll
  for (uint32_t i = 0; i < kScanI; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = wsum[kScanT / 32];
}

uint64_t scan_scratch_bytes(uint64_t n) {
  uint64_t bytes = 0;
  while (n > kScanTile) {
    n = (n + kScanTile - 1) / kScanTile;
    bytes += 2 * n * sizeof(uint64_t);
  }
  return bytes + 64;
}

template <typename TI>
static void scan_rec(const TI* in, uint64_t* out, uint64_t n, uint64_t* scratch, uint64_t* total, cudaStream_t st,
                     int* launches, uint64_t clamp) {
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb <= 1) {
    k_scan_tiles<TI><<<1, kScanT, 0, st>>>(in, out, n, nullptr, total, clamp);
    ++*launches;
    return;
  }
  uint64_t* sums = scratch;
  uint64_t* sums_scan = scratch + nb;
  k_scan_reduce<TI><<<(unsigned)nb, kScanT, 0, st>>>(in, n, sums, clamp);
  scan_rec<uint64_t>(sums, sums_scan, nb, scratch + 2 * nb, total, st, launches, ~0ull);
  k_scan_tiles<TI><<<(unsigned)nb, kScanT, 0, st>>>(in, out, n, sums_scan, nullptr, clamp);
  *launches += 2;
}

void launch_exclusive_scan(const uint32_t* in, uint64_t* out, uint64_t n, uint32_t clamp, void* scratch,
                           uint64_t* total_dev, cudaStream_t st, int* launches) {
  if (n == 0) {
    cudaMemsetAsync(total_dev, 0, sizeof(uint64_t), st);
    return;
  }
  scan_rec<uint32_t>(in, out, n, static_cast<uint64_t*>(scratch), total_dev, st, launches, clamp);
}

}  // namespace mc
