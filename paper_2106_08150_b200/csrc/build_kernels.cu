// Build-side kernels (B1-B6): sketch, region-partitioned pair store, and the
// counting multi-value hash table (count -> scan -> scatter -> cap).
//
// Paper: §4.1 P:315-474 (build), §5.1 P:647-672 (GPU hash tables),
// §5.2 P:692-694 (build pipeline = steps 1-3 then insert).
//
// B200 design: random 32-byte accesses into a table much larger
// than L2 run at ~20 G/s on this part, a tenth of copy bandwidth
// (profiles/r01_random_access_ceilings.jsonl), while L2-resident atomics run at
// ~120 G/s.  Insert calls therefore only sketch and append (feature, window)
// pairs to buckets by TABLE REGION (home slot >> shift, <= 1024 regions);
// finalize then sweeps the table region by region:
//   count   : warp-aggregated insert -- lanes with equal keys elect a leader that
//             reserves all their locations with ONE atomic on the key's slot; the
//             returned count is each location's rank in the key's bucket
//   scan    : bucket offsets = exclusive scan of min(count, cap) over the table
//   scatter : every location is written at offset + rank (ranked window id)
//   heavy   : keys with more than cap locations keep the cap smallest (S7)
// so every atomic and every table access of a pass hits lines that are L2
// resident, and hot keys (hundreds of strains sharing a feature) cost one
// atomic per location instead of slot-chain walks.
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
constexpr uint32_t kTileW = 256;

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
constexpr uint32_t kRegPerThread = kMaxRegions / kTileW;  // regions owned by a thread in the tile scan
constexpr uint32_t kTilePairs = kTileW * 16;               // s <= 16
// dynamic smem: [staging: max(window slots, pairs + their regions)] [region arrays]
constexpr size_t kStageBytes = (size_t)kTilePairs * (8 + 2) > (size_t)kTileW * kSlotWords * 4
                                   ? (size_t)kTilePairs * (8 + 2) : (size_t)kTileW * kSlotWords * 4;

struct TileRegions {             // per table region, for the current tile
  uint32_t* cnt;                 // pairs of the tile in the region
  uint32_t* loc;                 // exclusive scan of cnt: the region's first staged pair
  uint32_t* lim;                 // staged pairs [loc, lim) go to the region's bucket ...
  unsigned long long* gbase;     // ... at gbase + j
  unsigned long long* sgbase;    // staged pairs [lim, loc + cnt) spill to sgbase + j
};

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
  uint16_t* sreg = reinterpret_cast<uint16_t*>(stage + (size_t)kTilePairs * 8);     // [kTilePairs]
  uint64_t tile, tend;
  cta_tiles((b.total_windows + kTileW - 1) / kTileW, &tile, &tend);
  const uint64_t spill_end = (uint64_t)ps.nreg * ps.rcap + ps.spill_cap;
  uint32_t t0 = tile < tend ? upper_index(b.win_base, b.nt + 1, min(tile * kTileW + wid * 32, b.total_windows - 1))
                            : 0u;
  for (uint32_t i = threadIdx.x; i < ps.nreg; i += blockDim.x) R.cnt[i] = 0;
  __syncthreads();
  for (; tile < tend; ++tile) {
    const uint64_t g0 = tile * kTileW + wid * 32;
    const uint8_t* p;
    uint32_t nk, val;
    window_at(b, c, g0 + lane, warp_targets(b, g0, t0, lane), p, nk, val);
    uint32_t v[16], rr[16];
    const int n = sketch_warp_windows<K>(wslots, p, nk, c, lane, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < n) {  // region | rank of the pair among the tile's pairs of that region
        const uint64_t h = slot_hash(v[i]);
        const uint32_t r = (uint32_t)(__umul64hi(h, ps.nslots) >> ps.shift);
        rr[i] = r | atomicAdd(&R.cnt[r], 1u) << 16;
        atomicMax(&hll[h >> (64 - kHllBits)], (uint32_t)__clzll((h << kHllBits) | (1ull << (kHllBits - 1))) + 1u);
      }
    }
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
#pragma unroll
      for (uint32_t j = 0; j < kRegPerThread; ++j) {
        const uint32_t r = r0 + j;
        if (k[j]) {
          const uint32_t nb = at[j] >= ps.rcap ? 0u : (uint32_t)min((unsigned long long)k[j], ps.rcap - at[j]);
          R.loc[r] = loc;
          R.lim[r] = loc + nb;
          R.gbase[r] = (unsigned long long)r * ps.rcap + at[j] - loc;
          if (nb < k[j]) {  // bucket full: the rest of this tile's pairs of region r spill
            const unsigned long long sp = atomicAdd(&ps.cursor[ps.nreg], (unsigned long long)(k[j] - nb));
            if (sp + (k[j] - nb) > ps.spill_cap) atomicExch(&ps.err[1], 1);
            R.sgbase[r] = (unsigned long long)ps.nreg * ps.rcap + sp - (loc + nb);
          }
        }
        loc += k[j];
      }
      if (threadIdx.x == kTileW - 1) wsum[kTileW / 32] = loc;  // the tile's pair count
    }
    __syncthreads();  // (B) region bases known
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < n) {
        const uint32_t r = rr[i] & 0xffffu, j = R.loc[r] + (rr[i] >> 16);
        spair[j] = make_uint2(v[i], val);
        sreg[j] = (uint16_t)r;
      }
    }
    for (uint32_t r = threadIdx.x; r < ps.nreg; r += blockDim.x) R.cnt[r] = 0;  // for the next tile
    __syncthreads();  // (C) pairs staged by region
    const uint32_t total = wsum[kTileW / 32];
    for (uint32_t j = threadIdx.x; j < total; j += kTileW) {
      const uint32_t r = sreg[j];
      const uint64_t at = j < R.lim[r] ? R.gbase[r] + j : R.sgbase[r] + j;
      if (at < spill_end) ps.pairs[at] = spair[j];
    }
    __syncthreads();  // (D) staging free for the next tile's windows
  }
}

__global__ void __launch_bounds__(256, 3) k_sketch_partition(BuildBatch b, SketchCfg c, PairStore ps) {
  extern __shared__ __align__(16) uint8_t smem[];
  TileRegions R;
  R.gbase = reinterpret_cast<unsigned long long*>(smem + kStageBytes);
  R.sgbase = R.gbase + ps.nreg;
  R.cnt = reinterpret_cast<uint32_t*>(R.sgbase + ps.nreg);
  R.loc = R.cnt + ps.nreg;
  R.lim = R.loc + ps.nreg;
  __shared__ uint32_t hll[kHllRegs];  // distinct-feature estimate (sizes the table at finalize)
  for (uint32_t i = threadIdx.x; i < kHllRegs; i += blockDim.x) hll[i] = 0;
  if (c.k == 16) sketch_partition_tiles<16>(b, c, ps, smem, R, hll);
  else sketch_partition_tiles<0>(b, c, ps, smem, R, hll);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kHllRegs; i += blockDim.x)
    if (hll[i]) atomicMax(&ps.hll[i], hll[i]);
}

size_t sketch_partition_smem(uint32_t nreg) {
  return kStageBytes + (size_t)nreg * (8 + 8 + 4 + 4 + 4);
}

void launch_sketch_partition(const BuildBatch& b, SketchCfg c, const PairStore& ps, int sms, cudaStream_t st) {
  const size_t smem = sketch_partition_smem(ps.nreg);
  cudaFuncSetAttribute(k_sketch_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sketch_partition, 256, smem);
  k_sketch_partition<<<sms * max(per_sm, 1), 256, smem, st>>>(b, c, ps);
}

// ---------------------------------------------------------------------------
// Chunked sweep over the pair store in region order (spill last): warps grab
// consecutive 256-pair chunks from one counter, so the pairs in flight keep
// their table regions and bucket windows inside the 126 MB L2.
// ---------------------------------------------------------------------------
constexpr uint32_t kPairChunk = 256;

struct ChunkSpace {
  uint64_t cpr, nchunks;
  __device__ ChunkSpace(const PairStore& ps) {
    cpr = (ps.rcap + kPairChunk - 1) / kPairChunk;
    nchunks = cpr * ps.nreg + (ps.spill_cap + kPairChunk - 1) / kPairChunk;
  }
  // first pair index and number of valid pairs of chunk ch
  __device__ void chunk(const PairStore& ps, uint64_t ch, uint64_t* first, uint32_t* n) const {
    uint64_t r, off, fill;
    if (ch < cpr * ps.nreg) {
      r = ch / cpr;
      off = (ch % cpr) * kPairChunk;
      fill = min(ps.cursor[r], (unsigned long long)ps.rcap);
      *first = r * ps.rcap + off;
    } else {
      off = (ch - cpr * ps.nreg) * kPairChunk;
      fill = min(ps.cursor[ps.nreg], (unsigned long long)ps.spill_cap);
      *first = (uint64_t)ps.nreg * ps.rcap + off;
    }
    *n = off >= fill ? 0u : (uint32_t)min((uint64_t)kPairChunk, fill - off);
  }
};

// CTA-wide grab of 8 chunks (one per warp); returns this warp's chunk
// (>= nchunks: done).  The barrier keeps the CTA's warps together: measured,
// letting warps run ahead (per-warp grabs, static interleave) widens the set
// of regions in flight beyond L2 and costs 1.2-6x in these passes.
__device__ __forceinline__ uint64_t grab_chunk(unsigned long long* work) {
  __shared__ unsigned long long grab;
  __syncthreads();
  if (threadIdx.x == 0) grab = atomicAdd(work, 8ull);
  __syncthreads();
  return grab + (threadIdx.x >> 5);
}

// warp-level grab of G chunks (count pass: no barrier between warps)
template <uint32_t G>
__device__ __forceinline__ uint64_t grab_chunks(unsigned long long* work, uint32_t lane) {
  unsigned long long g = 0;
  if (lane == 0) g = atomicAdd(work, (unsigned long long)G);
  return __shfl_sync(kFull, g, 0);
}
#ifndef MC_CNT_GRAB
#define MC_CNT_GRAB 2
#endif

// ---- B5: warp-aggregated insert (Abstract P:43-44): one atomic per distinct
// key per 32 pairs; each location receives its rank in the key's bucket -----
// kRes independent reservations per lane advance in lock step, so each lane
// keeps kRes table accesses in flight.  A reservation probes with plain L2
// loads and spends ONE atomic when it lands: CAS on a slot seen empty (a
// lost race returns the winner's word and probing goes on), or atomicAdd on
// the slot holding its key -- atomic throughput, not load throughput, bounds
// this pass (profiles/r01_random_access_ceilings.jsonl).
struct Reserve {
  uint64_t s;
  uint32_t key, n, base;
  int state;  // 0 done, 1 probe (load), 3 claim (CAS on a slot seen empty), 2 add
};

__device__ __forceinline__ void reserve_step(uint64_t nslots, Reserve& q, uint64_t old) {
  if (q.state == 2) {
    q.base = (uint32_t)(old >> 32);
    q.state = 0;
  } else if (q.state) {
    if (old == 0) {
      if (q.state == 3) { q.base = 0; q.state = 0; }  // claimed
      else q.state = 3;
    } else if ((uint32_t)old == q.key) {
      q.state = 2;
    } else {
      q.s = next_slot(q.s, nslots);
      q.state = 1;
    }
  }
}

#ifndef MC_KRES
#define MC_KRES 4
#endif
constexpr int kRes = MC_KRES;

__global__ void __launch_bounds__(256) k_count_pairs(FinalizeArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const ChunkSpace cs(a.ps);
  for (;;) {
    const uint64_t ch0 = grab_chunks<MC_CNT_GRAB>(&a.ps.cursor[a.ps.nreg + 1], lane);
    if (ch0 >= cs.nchunks) break;  // warp-uniform exit
    for (uint64_t ch = ch0; ch < ch0 + MC_CNT_GRAB && ch < cs.nchunks; ++ch) {
      uint64_t first = 0;
      uint32_t n = 0;
      cs.chunk(a.ps, ch, &first, &n);
      for (uint32_t i = 0; i < n; i += 32 * kRes) {
        // kRes groups of 32 pairs: lanes with equal keys inside a group share one reservation
        Reserve q[kRes];
        uint32_t rank[kRes], leader[kRes];
        bool has[kRes];
#pragma unroll
        for (int g = 0; g < kRes; ++g) {
          has[g] = i + g * 32 + lane < n;
          const uint32_t key = has[g] ? a.ps.pairs[first + i + g * 32 + lane].x : 0u;
          const uint32_t active = __ballot_sync(kFull, has[g]);
          q[g].state = 0;
          q[g].base = 0;
          rank[g] = 0;
          leader[g] = 0;
          if (has[g]) {
            const uint32_t peers = __match_any_sync(active, key);
            leader[g] = __ffs(peers) - 1;
            rank[g] = __popc(peers & ((1u << lane) - 1u));
            if (lane == leader[g]) {
              q[g].key = key;
              q[g].n = __popc(peers);
              q[g].s = home_slot(key, a.nslots);
              q[g].state = 1;
            }
          }
        }
        for (uint64_t guard = 0; guard < 3 * a.nslots; ++guard) {
          int any = 0;
#pragma unroll
          for (int g = 0; g < kRes; ++g) any |= q[g].state;
          if (!any) break;
          uint64_t o[kRes];
#pragma unroll
          for (int g = 0; g < kRes; ++g) {
            unsigned long long* w = &a.T[q[g].s].kc;
            o[g] = 0;
            if (q[g].state == 1) o[g] = __ldcg(w);
            else if (q[g].state == 3) o[g] = atomicCAS(w, 0ull, (uint64_t)q[g].key | ((uint64_t)q[g].n << 32));
            else if (q[g].state == 2) o[g] = atomicAdd(w, (uint64_t)q[g].n << 32);
          }
#pragma unroll
          for (int g = 0; g < kRes; ++g) reserve_step(a.nslots, q[g], o[g]);
        }
        int left = 0;
#pragma unroll
        for (int g = 0; g < kRes; ++g) left |= q[g].state;
        if (left) atomicExch(&a.ps.err[0], 1);  // table full
#pragma unroll
        for (int g = 0; g < kRes; ++g) {
          const uint32_t base = __shfl_sync(kFull, q[g].base, leader[g]);
          if (has[g]) a.ps.rank[first + i + g * 32 + lane] = base + rank[g];
        }
      }
    }
  }
}

void launch_count_pairs(const FinalizeArgs& a, int grid, cudaStream_t st) { k_count_pairs<<<grid, 256, 0, st>>>(a); }

// ---- B6 scan: bucket offsets = exclusive scan of min(count, cap) over the
// table (tiles of 4096 slots staged through shared memory for coalescing) ----
constexpr uint32_t kTScanT = 256, kTScanI = 16, kTScanTile = kTScanT * kTScanI;

__device__ __forceinline__ uint32_t capped(const KSlot* T, uint64_t i, uint64_t n, uint32_t cap) {
  return i < n ? min((uint32_t)(T[i].kc >> 32), cap) : 0u;
}

__global__ void __launch_bounds__(kTScanT) k_tscan_reduce(FinalizeArgs a, uint64_t* sums) {
  __shared__ uint64_t red[kTScanT / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kTScanTile;
  uint64_t acc = 0;
  for (uint32_t i = threadIdx.x; i < kTScanTile; i += kTScanT) acc += capped(a.T, base + i, a.nslots, a.cap);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int i = 0; i < (int)(kTScanT / 32); ++i) t += red[i];
    sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kTScanT) k_tscan_tiles(FinalizeArgs a, const uint64_t* prefix, uint64_t* total) {
  __shared__ uint32_t v[kTScanTile + kTScanTile / 32];  // padded against bank conflicts
  __shared__ uint64_t wsum[kTScanT / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kTScanTile;
  for (uint32_t i = threadIdx.x; i < kTScanTile; i += kTScanT) v[i + (i >> 5)] = capped(a.T, base + i, a.nslots, a.cap);
  __syncthreads();
  uint64_t acc = 0;
  const uint32_t t0 = threadIdx.x * kTScanI;
#pragma unroll
  for (uint32_t j = 0; j < kTScanI; ++j) acc += v[t0 + j + ((t0 + j) >> 5)];
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
    for (uint32_t i = 0; i < kTScanT / 32; ++i) {
      const uint64_t y = wsum[i];
      wsum[i] = t;
      t += y;
    }
    wsum[kTScanT / 32] = t;
  }
  __syncthreads();
  uint64_t run = wsum[wid] + x - acc;
  __syncthreads();
  // exclusive offsets back into the staging buffer (32-bit relative to the tile)
  const uint64_t tile0 = wsum[0];
#pragma unroll
  for (uint32_t j = 0; j < kTScanI; ++j) {
    const uint32_t k = t0 + j + ((t0 + j) >> 5);
    const uint32_t cj = v[k];
    v[k] = (uint32_t)(run - tile0);
    run += cj;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kTScanTile; i += kTScanT)
    if (base + i < a.nslots && a.T[base + i].kc) a.T[base + i].off = tile0 + v[i + (i >> 5)];
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = wsum[kTScanT / 32];
}

template <typename TI>
static void scan_rec(const TI* in, uint64_t* out, uint64_t n, uint64_t* scratch, uint64_t* total, cudaStream_t st,
                     int* launches, uint64_t clamp);

uint64_t table_scan_scratch_bytes(uint64_t nslots) {
  const uint64_t nb = (nslots + kTScanTile - 1) / kTScanTile;
  return 2 * nb * sizeof(uint64_t) + scan_scratch_bytes(nb);
}

void launch_table_scan(const FinalizeArgs& a, void* scratch, uint64_t* total_dev, cudaStream_t st, int* launches) {
  const uint64_t nb = (a.nslots + kTScanTile - 1) / kTScanTile;
  uint64_t* sums = static_cast<uint64_t*>(scratch);
  uint64_t* sums_scan = sums + nb;
  if (nb == 1) {
    k_tscan_tiles<<<1, kTScanT, 0, st>>>(a, nullptr, total_dev);
    ++*launches;
    return;
  }
  k_tscan_reduce<<<(unsigned)nb, kTScanT, 0, st>>>(a, sums);
  scan_rec<uint64_t>(sums, sums_scan, nb, sums + 2 * nb, total_dev, st, launches, ~0ull);
  k_tscan_tiles<<<(unsigned)nb, kTScanT, 0, st>>>(a, sums_scan, nullptr);
  *launches += 2;
}

// ---- B6: statistics + list of keys with more than cap locations ------------
__global__ void __launch_bounds__(256) k_keys_pass(FinalizeArgs a) {
  uint64_t keys = 0, locs = 0, trunc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.nslots; s += stride) {
    const ulonglong2 e = *reinterpret_cast<const ulonglong2*>(&a.T[s]);
    if (!e.x) continue;
    const uint32_t n = (uint32_t)(e.x >> 32);
    ++keys;
    locs += n;
    if (n > a.cap) {
      trunc += n - a.cap;
      const unsigned long long h = atomicAdd(&a.counters[3], 1ull);  // rare: plain atomic
      atomicAdd(&a.counters[4], (unsigned long long)n);
      a.heavy[h] = make_ulonglong2(s, e.y);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    keys += __shfl_xor_sync(kFull, keys, d);
    locs += __shfl_xor_sync(kFull, locs, d);
    trunc += __shfl_xor_sync(kFull, trunc, d);
  }
  if ((threadIdx.x & 31u) == 0 && keys) {
    atomicAdd(&a.counters[0], (unsigned long long)keys);
    atomicAdd(&a.counters[1], (unsigned long long)locs);
    if (trunc) atomicAdd(&a.counters[2], (unsigned long long)trunc);
  }
}

void launch_keys_pass(const FinalizeArgs& a, int grid, cudaStream_t st) { k_keys_pass<<<grid, 256, 0, st>>>(a); }

// heavy keys: their bucket offset temporarily points into the side buffer
__global__ void __launch_bounds__(256) k_heavy_offsets(FinalizeArgs a) {
  const uint64_t nh = a.counters[3];
  for (uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = a.heavy[h].x;
    const uint32_t n = (uint32_t)(a.T[s].kc >> 32);
    a.T[s].off = atomicAdd(&a.counters[5], (unsigned long long)n);
  }
}

void launch_heavy_offsets(const FinalizeArgs& a, int grid, cudaStream_t st) { k_heavy_offsets<<<grid, 256, 0, st>>>(a); }

// gapped build window index -> ranked window index (targets ordered by id)
__device__ __forceinline__ uint32_t to_ranked(const FinalizeArgs& a, uint32_t g) {
  if (a.identity) return g;
  const uint32_t t = upper_index(a.ins_base, a.nt, g);
  return g + a.delta[t];
}

// ---- B6 scatter: every location to offset + rank (region order: L2-resident
// table probes; consecutive pairs of a region write nearby buckets) ----------
__global__ void __launch_bounds__(256) k_scatter_pairs(FinalizeArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const ChunkSpace cs(a.ps);
  for (;;) {
    const uint64_t ch = grab_chunk(&a.ps.cursor[a.ps.nreg + 1]);
    if (ch - (threadIdx.x >> 5) >= cs.nchunks) break;  // CTA-uniform exit
    if (ch < cs.nchunks) {
      uint64_t first = 0;
      uint32_t n = 0;
      cs.chunk(a.ps, ch, &first, &n);
      for (uint32_t i = lane; i < n; i += 32) {
        const uint2 kv = a.ps.pairs[first + i];
        const uint32_t r = a.ps.rank[first + i];
        uint64_t off = 0;
        const uint32_t cnt = keytable_find(a.T, a.nslots, kv.x, &off);
        uint32_t* dst = cnt > a.cap ? a.side : a.values;
        dst[off + r] = to_ranked(a, kv.y);
      }
    }
  }
}

void launch_scatter_pairs(const FinalizeArgs& a, int grid, cudaStream_t st) { k_scatter_pairs<<<grid, 256, 0, st>>>(a); }

// ---- B6 cap: one CTA per heavy key keeps the cap smallest of
// its side bucket (chunks of 1024 merged into a sorted best-cap buffer) -----
__global__ void __launch_bounds__(256) k_heavy_select(FinalizeArgs a) {
  constexpr uint32_t NT = 256, BUF = 2048, CH = 1024;
  __shared__ uint32_t buf[BUF];
  const uint32_t tid = threadIdx.x;
  const uint64_t nh = a.counters[3];
  for (uint64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const uint64_t s = a.heavy[h].x, final_off = a.heavy[h].y;
    const uint64_t kc = a.T[s].kc;
    const uint32_t n = (uint32_t)(kc >> 32);
    const uint32_t* src = a.side + a.T[s].off;
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
    if (tid == 0) {  // condensed entry: count = cap, bucket in the value array
      a.T[s].kc = (kc & 0xffffffffull) | ((uint64_t)a.cap << 32);
      a.T[s].off = final_off;
    }
  }
}

void launch_heavy_select(const FinalizeArgs& a, int grid, cudaStream_t st) { k_heavy_select<<<grid, 256, 0, st>>>(a); }

// diagnostic: the same sketch, written out per window
template <uint32_t K>
__device__ __forceinline__ void debug_sketch_tiles(const BuildBatch& b, const SketchCfg& c, uint32_t* slots,
                                                   uint32_t* feats, uint32_t* counts) {
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
    const int n = sketch_warp_windows<K>(slots + wid * 32 * kSlotWords, p, nk, c, lane, v);
    if (g < b.total_windows) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if ((uint32_t)i < c.s) feats[g * c.s + i] = i < n ? v[i] : 0u;
      counts[g] = (uint32_t)n;
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) k_debug_sketch(BuildBatch b, SketchCfg c, uint32_t* feats, uint32_t* counts) {
  __shared__ __align__(16) uint32_t slots[kTileW * kSlotWords];
  if (c.k == 16) debug_sketch_tiles<16>(b, c, slots, feats, counts);
  else debug_sketch_tiles<0>(b, c, slots, feats, counts);
}

void launch_debug_sketch(const BuildBatch& b, SketchCfg c, uint32_t* feats, uint32_t* counts, int grid,
                         cudaStream_t st) {
  k_debug_sketch<<<grid, 256, 0, st>>>(b, c, feats, counts);
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
