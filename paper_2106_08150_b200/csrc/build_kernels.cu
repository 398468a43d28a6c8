// Build-side kernels: sketch + warp-aggregated multi-bucket insert (B1-B5),
// finalize = per-feature sort + cap + condensed layout (B6), device scan.
//
// Paper: §4.1 P:315-474 (build), §5.1 P:647-672 (GPU hash tables),
// §5.2 P:692-694 (build pipeline = steps 1-3 then insert).

#include "mc_block.cuh"
#include "mc_kernels.cuh"

namespace mc {

// ---------------------------------------------------------------------------
// B1-B5: one warp per window; each insert round covers 32/s
// windows so a warp inserts up to 32 features with one aggregated pass.
// Window g of the batch -> target by binary search over win_base.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 6) k_sketch_insert(BuildBatch b, SketchCfg c, Slot* __restrict__ T,
                                                          uint64_t nslots, unsigned long long* n_loc, int* err) {
  constexpr uint64_t kBlock = 32;  // windows per warp task (one binary search per task)
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t wpr = 32u / c.s;  // windows per insert round (s <= 16)
  uint32_t my_count = 0;
  for (uint64_t g = gw * kBlock; g < b.total_windows; g += nw * kBlock) {
    const uint64_t gend = min(b.total_windows, g + kBlock);
    uint32_t t = upper_index(b.win_base, b.nt + 1, g);
    uint64_t tend = b.win_base[t + 1];
    for (uint64_t g0 = g; g0 < gend; g0 += wpr) {
      bool has = false;
      uint32_t key = 0, val = 0;
      for (uint32_t q = 0; q < wpr; ++q) {
        const uint64_t gg = g0 + q;
        if (gg >= gend) break;
        while (gg >= tend) tend = b.win_base[++t + 1];
        const uint64_t j = gg - b.win_base[t];
        const uint64_t first = j * c.stride;
        const uint32_t nk = (uint32_t)min((uint64_t)c.stride, b.seq_len[t] - c.k + 1 - first);
        uint32_t f;
        const int cnt = sketch_window(b.chars + b.seq_off[t] + first, nk, c, lane, f);
        const uint32_t lo = q * c.s;
        const uint32_t fq = __shfl_sync(kFull, f, (lane - lo) & 31u);
        if (lane >= lo && lane < lo + (uint32_t)cnt) {
          has = true;
          key = fq;
          val = b.bwi_base[t] + (uint32_t)j;
        }
      }
      my_count += has ? 1u : 0u;
      warp_insert(T, nslots, has, key, val, lane, err);
    }
  }
  my_count = __reduce_add_sync(kFull, my_count);
  if (lane == 0 && my_count) atomicAdd(n_loc, (unsigned long long)my_count);
}

void launch_sketch_insert(const BuildBatch& b, SketchCfg c, Slot* T, uint64_t nslots, unsigned long long* n_loc,
                          int* err, int grid, cudaStream_t st) {
  k_sketch_insert<<<grid, 256, 0, st>>>(b, c, T, nslots, n_loc, err);
}

// ---------------------------------------------------------------------------
// Region-partitioned insert (B200 design): random 32 B sector
// accesses into a table much larger than L2 run at ~20 G/s on this part
// (profiles/r01_random_access_ceilings.jsonl), so inserting straight from the
// sketch kernel costs DRAM-missing accesses per location.  Instead:
//   1 sketch_partition : CTA tiles of 256 windows are sketched (same warp
//        code) into shared memory, counted per table region (home slot >>
//        shift, 32 MiB of table per region), claim space in the region's
//        bucket with one global atomic per (tile, region) and scatter their
//        (key, value) pairs there
//   2 insert_pairs : warps take 256-pair chunks in region order from a global
//        work counter and insert them with the same warp-aggregated insert, so
//        the whole GPU sweeps the table region by region and table lines stay
//        in the 126 MB L2 while they are being filled.
// Buckets are over-allocated (1.15x the mean + 4096); if one overflows the
// batch falls back to the fused kernel (the table is untouched until step 2).
// ---------------------------------------------------------------------------
constexpr uint32_t kTileW = 256, kWarpW = kTileW / 8;

__global__ void __launch_bounds__(256) k_sketch_partition(BuildBatch b, SketchCfg c, PartitionArgs pa) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* tkey = sm;                         // [kTileW * 16]
  uint32_t* tval = tkey + kTileW * 16;         // [kTileW * 16]
  uint32_t* cnt = tval + kTileW * 16;          // [nreg]
  uint32_t* pos = cnt + pa.nreg;               // [nreg]
  unsigned long long* base = reinterpret_cast<unsigned long long*>(pos + pa.nreg);  // [nreg] (8-byte aligned: 2*(kTileW*16 + nreg) words precede it)
  __shared__ uint32_t wfill[8];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint64_t ntiles = (b.total_windows + kTileW - 1) / kTileW;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < pa.nreg; i += blockDim.x) cnt[i] = pos[i] = 0;
    __syncthreads();
    // each warp sketches 32 consecutive windows into its segment of the tile
    const uint64_t g = tile * kTileW + wid * kWarpW;
    const uint64_t gend = min(b.total_windows, g + kWarpW);
    uint32_t fill = 0;
    uint32_t* wk = tkey + wid * kWarpW * 16;
    uint32_t* wv = tval + wid * kWarpW * 16;
    if (g < gend) {
      uint32_t t = upper_index(b.win_base, b.nt + 1, g);
      uint64_t tend = b.win_base[t + 1];
      for (uint64_t gg = g; gg < gend; ++gg) {
        while (gg >= tend) tend = b.win_base[++t + 1];
        const uint64_t j = gg - b.win_base[t];
        const uint64_t first = j * c.stride;
        const uint32_t nk = (uint32_t)min((uint64_t)c.stride, b.seq_len[t] - c.k + 1 - first);
        uint32_t f;
        const int n = sketch_window(b.chars + b.seq_off[t] + first, nk, c, lane, f);
        if (lane < (uint32_t)n) {
          wk[fill + lane] = f;
          wv[fill + lane] = b.bwi_base[t] + (uint32_t)j;
          atomicAdd(&cnt[home_slot(f, pa.nslots) >> pa.shift], 1u);
        }
        fill += (uint32_t)n;
      }
    }
    if (lane == 0) wfill[wid] = fill;
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < pa.nreg; r += blockDim.x) {
      const uint32_t k = cnt[r];
      if (!k) continue;
      const unsigned long long at = atomicAdd(&pa.cursor[r], (unsigned long long)k);
      if (at + k > pa.rcap) atomicExch(pa.overflow, 1);
      base[r] = (unsigned long long)r * pa.rcap + at;
    }
    __syncthreads();
    for (uint32_t w = 0; w < 8; ++w) {
      const uint32_t* tk = tkey + w * kWarpW * 16;
      const uint32_t* tv = tval + w * kWarpW * 16;
      for (uint32_t i = threadIdx.x; i < wfill[w]; i += blockDim.x) {
        const uint32_t f = tk[i];
        const uint32_t r = home_slot(f, pa.nslots) >> pa.shift;
        const uint32_t slot = atomicAdd(&pos[r], 1u);
        if (base[r] - (unsigned long long)r * pa.rcap + slot < pa.rcap) pa.pairs[base[r] + slot] = make_uint2(f, tv[i]);
      }
    }
    __syncthreads();
  }
}

size_t sketch_partition_smem(uint32_t nreg) {
  return (size_t)2 * kTileW * 16 * 4 + (size_t)(2 * nreg + 2) * 4 + (size_t)nreg * 8;
}

void launch_sketch_partition(const BuildBatch& b, SketchCfg c, const PartitionArgs& pa, int grid, cudaStream_t st) {
  const size_t smem = sketch_partition_smem(pa.nreg);
  cudaFuncSetAttribute(k_sketch_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sketch_partition<<<grid, 256, smem, st>>>(b, c, pa);
}

__global__ void __launch_bounds__(256) k_insert_pairs(PartitionArgs pa, Slot* T, uint64_t nslots, int* err) {
  // The CTA grabs 8 chunks (one per warp) with ONE atomic on the work counter,
  // so chunks are taken in region order without a hot single-address counter.
  constexpr uint32_t kChunk = 256;
  __shared__ unsigned long long grab;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint64_t cpr = (pa.rcap + kChunk - 1) / kChunk;  // chunks per region
  const uint64_t nchunks = cpr * pa.nreg;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) grab = atomicAdd(pa.work, 8ull);
    __syncthreads();
    const uint64_t ch = grab + wid;
    if (grab >= nchunks) break;
    if (ch >= nchunks) continue;
    const uint64_t r = ch / cpr, off = (ch % cpr) * kChunk;
    const uint64_t n = min(pa.cursor[r], (unsigned long long)pa.rcap);
    if (off >= n) continue;
    const uint2* src = pa.pairs + r * pa.rcap + off;
    const uint32_t m = (uint32_t)min((uint64_t)kChunk, n - off);
    for (uint32_t i = 0; i < m; i += 32) {
      const bool has = i + lane < m;
      const uint2 kv = has ? src[i + lane] : make_uint2(0, 0);
      warp_insert(T, nslots, has, kv.x, kv.y, lane, err);
    }
  }
}

void launch_insert_pairs(const PartitionArgs& pa, Slot* T, uint64_t nslots, int* err, int grid, cudaStream_t st) {
  k_insert_pairs<<<grid, 256, 0, st>>>(pa, T, nslots, err);
}

// diagnostic: the same sketch, written out per window
__global__ void __launch_bounds__(256) k_debug_sketch(BuildBatch b, SketchCfg c, uint32_t* feats, uint32_t* counts) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t g = gw; g < b.total_windows; g += nw) {
    const uint32_t t = upper_index(b.win_base, b.nt + 1, g);
    const uint64_t j = g - b.win_base[t];
    const uint64_t first = j * c.stride;
    const uint32_t nk = (uint32_t)min((uint64_t)c.stride, b.seq_len[t] - c.k + 1 - first);
    uint32_t f;
    const int cnt = sketch_window(b.chars + b.seq_off[t] + first, nk, c, lane, f);
    if (lane < c.s) feats[g * c.s + lane] = lane < (uint32_t)cnt ? f : 0u;
    if (lane == 0) counts[g] = (uint32_t)cnt;
  }
}

void launch_debug_sketch(const BuildBatch& b, SketchCfg c, uint32_t* feats, uint32_t* counts, int grid,
                         cudaStream_t st) {
  k_debug_sketch<<<grid, 256, 0, st>>>(b, c, feats, counts);
}

// ---------------------------------------------------------------------------
// B6 finalize (reading S7).  Slot-parallel
// passes with uniform work per thread (no per-key walks):
//   1 count   : every occupied slot adds its fill to its primary's counter;
//               the atomic's return value is the slot's position in the key's list
//   2 scan    : exclusive scan of min(count, cap) over primaries -> offsets
//   3 scatter : every slot of a key with count <= cap writes its values
//               (ranked window ids) at offset + position; primaries insert
//               key -> (count, offset) into the condensed key table
//   4 sort    : every key's segment is sorted ascending (registers for <= 16,
//               a warp in shared memory for <= cap)
//   5 heavy   : keys with count > cap: a CTA walks the key's run and keeps
//               the cap smallest (the only place a walk remains; rare)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t primary_of(const Slot* T, uint64_t s, uint64_t w, uint64_t n) {
  if (w & kPrimary) return s;
  const uint64_t d = T[s].link;
  return s >= d ? s - d : s + n - d;
}

__device__ __forceinline__ void add_counters(unsigned long long* ctr, uint64_t a, uint64_t b) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(kFull, a, d);
    b += __shfl_xor_sync(kFull, b, d);
  }
  if ((threadIdx.x & 31u) == 0 && b) {
    atomicAdd(&ctr[0], (unsigned long long)a);
    atomicAdd(&ctr[1], (unsigned long long)b);
  }
}

__global__ void __launch_bounds__(256) k_fin_count(FinalizeArgs a) {
  uint64_t keys = 0, locs = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.nslots; s += stride) {
    const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(&a.T[s]));  // kw, link | v0
    const uint64_t w = e.x;
    if (w == 0) continue;
    const uint64_t d = (uint32_t)e.y;
    const uint64_t p = (w & kPrimary) ? s : (s >= d ? s - d : s + a.nslots - d);
    const uint32_t f = min(slot_fill(w), kSlotValues);
    a.spos[s] = atomicAdd(&a.cnt[p], f);
    keys += (w & kPrimary) ? 1u : 0u;
    locs += f;
  }
  add_counters(a.counters, keys, locs);
}

void launch_fin_count(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_count<<<grid, 256, 0, st>>>(a); }

// gapped build window index -> ranked window index (targets ordered by id)
__device__ __forceinline__ uint32_t to_ranked(const FinalizeArgs& a, uint32_t g) {
  if (a.identity) return g;
  const uint32_t t = upper_index(a.ins_base, a.nt, g);
  return g + a.delta[t];
}

// warp-aggregated append of `item` (lanes with want=true) to queue q / counter c
__device__ __forceinline__ void warp_append(bool want, uint64_t item, unsigned long long* c, uint64_t* q) {
  const uint32_t m = __ballot_sync(kFull, want);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31u;
  unsigned long long base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(c, (unsigned long long)__popc(m));
  base = __shfl_sync(kFull, base, __ffs(m) - 1);
  if (want) q[base + __popc(m & ((1u << lane) - 1u))] = item;
}

// CTA-aggregated append: the CTA's items of one iteration are staged in shared
// memory and reserved with ONE global atomic (a single global counter hit by
// every warp was the bottleneck of this pass).
template <int CAP>
struct CtaQueue {
  uint64_t item[CAP];
  uint32_t n;
  unsigned long long base;
};

__global__ void __launch_bounds__(256) k_fin_scatter(FinalizeArgs a) {
  // U slots per thread per iteration, every load of an iteration issued before
  // its results are used (the pass is latency-bound, not bandwidth-bound).
  constexpr int U = 4;
  __shared__ CtaQueue<256 * U> qs, qh;
  uint64_t trunc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n_iter = (a.nslots + stride * U - 1) / (stride * U);  // uniform trip count (barriers)
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t it = 0; it < n_iter; ++it) {
    if (threadIdx.x == 0) qs.n = qh.n = 0;
    __syncthreads();
    uint64_t sl[U], w[U], p[U], o[U];
    uint4 lo[U], hi[U];
    uint32_t n[U], sp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sl[u] = (it * U + u) * stride + tid;
      const uint4* q = reinterpret_cast<const uint4*>(&a.T[sl[u] < a.nslots ? sl[u] : 0]);
      lo[u] = sl[u] < a.nslots ? __ldg(q) : make_uint4(0, 0, 0, 0);
      hi[u] = sl[u] < a.nslots ? __ldg(q + 1) : make_uint4(0, 0, 0, 0);
      w[u] = (uint64_t)lo[u].x | ((uint64_t)lo[u].y << 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t d = lo[u].z;  // link
      p[u] = (w[u] & kPrimary) ? sl[u] : (sl[u] >= d ? sl[u] - d : sl[u] + a.nslots - d);
      n[u] = 0; o[u] = 0; sp[u] = 0;
      if (w[u]) {
        n[u] = a.cnt[p[u]];
        o[u] = a.off[p[u]];
        sp[u] = a.spos[sl[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!w[u]) continue;
      if (n[u] <= a.cap) {
        const uint32_t f = min(slot_fill(w[u]), kSlotValues);
        const uint32_t v[5] = {lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
        uint32_t* dst = a.values + o[u] + sp[u];
#pragma unroll
        for (uint32_t i = 0; i < kSlotValues; ++i)
          if (i < f) dst[i] = to_ranked(a, v[i]);
      }
      if (p[u] == sl[u]) {  // the primary becomes the key's condensed entry (its values are copied)
        const uint32_t c = min(n[u], a.cap);
        trunc += n[u] - c;
        if (n[u] > a.cap) {  // k_fin_heavy still reads this slot's values, then writes the entry
          qh.item[atomicAdd(&qh.n, 1u)] = p[u];
        } else {
          Slot* ps = &a.T[sl[u]];
          ps->v[0] = c;
          ps->v[1] = (uint32_t)o[u];
          ps->v[2] = (uint32_t)(o[u] >> 32);
          if (n[u] >= 2) qs.item[atomicAdd(&qs.n, 1u)] = o[u] | ((uint64_t)n[u] << 48);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      qs.base = qs.n ? atomicAdd(&a.counters[4], (unsigned long long)qs.n) : 0ull;
      qh.base = qh.n ? atomicAdd(&a.counters[3], (unsigned long long)qh.n) : 0ull;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < qs.n; i += blockDim.x) a.sortq[qs.base + i] = qs.item[i];
    for (uint32_t i = threadIdx.x; i < qh.n; i += blockDim.x) a.heavy[qh.base + i] = qh.item[i];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) trunc += __shfl_xor_sync(kFull, trunc, d);
  if ((threadIdx.x & 31u) == 0 && trunc) atomicAdd(&a.counters[2], (unsigned long long)trunc);
}

void launch_fin_scatter(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_scatter<<<grid, 256, 0, st>>>(a); }

// ---- pass 4a: segments of <= kLight values, sorted in registers ------------
template <int N>
__device__ __forceinline__ void sort_net(uint32_t (&r)[kLight]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const uint32_t x = r[i], y = r[l];
          if ((x > y) == up) { r[i] = y; r[l] = x; }
        }
      }
}

__global__ void __launch_bounds__(256) k_fin_sort_light(FinalizeArgs a) {
  const uint64_t nq = a.counters[4];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nq; h += stride) {
    const uint64_t e = a.sortq[h];
    const uint32_t n = (uint32_t)(e >> 48);
    if (n > kLight) continue;
    uint32_t* v = a.values + (e & ((1ull << 48) - 1));
    uint32_t r[kLight];
#pragma unroll
    for (int i = 0; i < (int)kLight; ++i) r[i] = i < (int)n ? v[i] : 0xffffffffu;
    if (n <= 4) sort_net<4>(r);
    else if (n <= 8) sort_net<8>(r);
    else sort_net<16>(r);
#pragma unroll
    for (int i = 0; i < (int)kLight; ++i)
      if (i < (int)n) v[i] = r[i];
  }
}

void launch_fin_sort_light(const FinalizeArgs& a, int grid, cudaStream_t st) {
  k_fin_sort_light<<<grid, 256, 0, st>>>(a);
}

// ---- pass 4b: segments of kLight < n <= cap (<= 1024), one warp each ----------
__global__ void __launch_bounds__(256) k_fin_sort_warp(FinalizeArgs a) {
  __shared__ uint32_t buf[8][1024];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t* b = buf[wid];
  const uint64_t nq = a.counters[4];
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = gw; i < nq; i += nw) {
    const uint64_t e = a.sortq[i];
    const uint64_t o = e & ((1ull << 48) - 1);
    const uint32_t n = (uint32_t)(e >> 48);
    if (n <= kLight) continue;
    const uint32_t n2 = next_pow2(n);
    for (uint32_t j = lane; j < n2; j += 32) b[j] = j < n ? a.values[o + j] : 0xffffffffu;
    __syncwarp();
    bitonic_sort<32>(b, n2, lane);
    for (uint32_t j = lane; j < n; j += 32) a.values[o + j] = b[j];
    __syncwarp();
  }
}

void launch_fin_sort_warp(const FinalizeArgs& a, int grid, cudaStream_t st) {
  k_fin_sort_warp<<<grid, 256, 0, st>>>(a);
}

// ---- pass 5: keys with more than cap locations --------------------------------
// One 256-thread CTA per key walks the key's probe run 256 slots at a time,
// collects values in shared memory and, whenever more than cap are held,
// sorts and keeps the cap smallest (cap <= 1024: the buffer never exceeds
// cap + 256*5 <= 2304 < 4096 entries).
__global__ void __launch_bounds__(256) k_fin_heavy(FinalizeArgs a) {
  constexpr uint32_t NT = 256, BUF = 4096;
  __shared__ uint32_t buf[BUF];
  __shared__ uint32_t nbuf, first_empty;
  const uint32_t tid = threadIdx.x;
  const uint64_t n_heavy = a.counters[3];
  for (uint64_t h = blockIdx.x; h < n_heavy; h += gridDim.x) {
    const uint64_t s = a.heavy[h];
    const uint32_t key = (uint32_t)a.T[s].kw;
    if (tid == 0) nbuf = 0;
    __syncthreads();
    for (uint64_t base = 0;; base += NT) {
      if (tid == 0) first_empty = NT;
      __syncthreads();
      uint64_t w = 0, q = 0;
      if (base + tid < a.nslots) {
        q = s + base + tid;
        if (q >= a.nslots) q -= a.nslots;
        w = a.T[q].kw;
      }
      if (w == 0) atomicMin(&first_empty, tid);
      __syncthreads();
      const uint32_t fe = first_empty;
      if (tid < fe && (uint32_t)w == key) {
        const uint32_t f = min(slot_fill(w), kSlotValues);
        const uint32_t pos = atomicAdd(&nbuf, f);
        for (uint32_t v = 0; v < f; ++v) buf[pos + v] = to_ranked(a, a.T[q].v[v]);
      }
      __syncthreads();
      const uint32_t n = nbuf;
      const bool done = fe < NT;
      if (n > a.cap || done) {
        const uint32_t n2 = next_pow2(n);
        for (uint32_t i = n + tid; i < n2; i += NT) buf[i] = 0xffffffffu;
        __syncthreads();
        bitonic_sort<NT>(buf, n2, tid);
        if (tid == 0 && n > a.cap) nbuf = a.cap;
        __syncthreads();
      }
      if (done) break;
    }
    const uint64_t o = a.off[s];
    for (uint32_t i = tid; i < a.cap; i += NT) a.values[o + i] = buf[i];
    if (tid == 0) {  // condensed key-table entry in the primary slot
      a.T[s].v[0] = a.cap;
      a.T[s].v[1] = (uint32_t)o;
      a.T[s].v[2] = (uint32_t)(o >> 32);
    }
    __syncthreads();
  }
}

void launch_fin_heavy(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_heavy<<<grid, 256, 0, st>>>(a); }

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
