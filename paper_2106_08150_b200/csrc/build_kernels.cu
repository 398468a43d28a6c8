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
__global__ void __launch_bounds__(256) k_sketch_insert(BuildBatch b, SketchCfg c, Slot* __restrict__ T,
                                                       uint64_t nslots, unsigned long long* n_loc, int* err) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t wpr = c.s >= 32 ? 1u : 32u / c.s;
  uint32_t my_count = 0;
  for (uint64_t g0 = gw * wpr; g0 < b.total_windows; g0 += nw * wpr) {
    bool has = false;
    uint32_t key = 0, val = 0;
    for (uint32_t q = 0; q < wpr; ++q) {
      const uint64_t g = g0 + q;
      if (g >= b.total_windows) break;
      const uint32_t t = upper_index(b.win_base, b.nt + 1, g);
      const uint64_t j = g - b.win_base[t];
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
  my_count = __reduce_add_sync(kFull, my_count);
  if (lane == 0 && my_count) atomicAdd(n_loc, (unsigned long long)my_count);
}

void launch_sketch_insert(const BuildBatch& b, SketchCfg c, Slot* T, uint64_t nslots, unsigned long long* n_loc,
                          int* err, int grid, cudaStream_t st) {
  k_sketch_insert<<<grid, 256, 0, st>>>(b, c, T, nslots, n_loc, err);
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
// B6 finalize, pass 1: every primary slot walks its key's probe run (all of
// a key's slots lie between its primary and the next empty slot) and counts
// the key's locations n; cnt = min(n, cap) (reading S7).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void add_counters(unsigned long long* ctr, uint64_t a, uint64_t b, uint64_t c) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(kFull, a, d);
    b += __shfl_xor_sync(kFull, b, d);
    c += __shfl_xor_sync(kFull, c, d);
  }
  if ((threadIdx.x & 31u) == 0 && a) {
    atomicAdd(&ctr[0], (unsigned long long)a);
    atomicAdd(&ctr[1], (unsigned long long)b);
    atomicAdd(&ctr[2], (unsigned long long)c);
  }
}

__global__ void __launch_bounds__(256) k_fin_count(FinalizeArgs a) {
  uint64_t keys = 0, locs = 0, trunc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.nslots; s += stride) {
    const uint64_t w = a.T[s].kw;
    uint32_t c = 0;
    if (w & kPrimary) {
      const uint32_t key = (uint32_t)w;
      uint64_t n = min(slot_fill(w), kSlotValues);
      uint64_t t = next_slot(s, a.nslots);
      for (uint64_t i = 1; i < a.nslots; ++i, t = next_slot(t, a.nslots)) {
        const uint64_t w2 = a.T[t].kw;
        if (w2 == 0) break;
        if ((uint32_t)w2 == key) n += min(slot_fill(w2), kSlotValues);
      }
      c = (uint32_t)(n < a.cap ? n : (uint64_t)a.cap);
      keys += 1;
      locs += n;
      trunc += n - c;
    }
    a.cnt[s] = c;
  }
  add_counters(a.counters, keys, locs, trunc);
}

void launch_fin_count(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_count<<<grid, 256, 0, st>>>(a); }

// build window index -> ranked window index (targets ordered by id, gaps)
__device__ __forceinline__ uint32_t to_ranked(const FinalizeArgs& a, uint32_t bwi) {
  const uint32_t t = upper_index(a.ins_base, a.nt, bwi);
  return bwi + a.delta[t];
}

// ---------------------------------------------------------------------------
// B6 pass 3 (light keys, <= kLight locations): one thread gathers the key's
// values, converts them to ranked window ids, sorts, keeps the cap smallest,
// writes them at the scanned offset and inserts key -> (count, offset) into
// the condensed key table.  Heavier keys are queued for k_fin_heavy.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fin_fill(FinalizeArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < a.nslots; s += stride) {
    const uint64_t w = a.T[s].kw;
    if (!(w & kPrimary)) continue;
    const uint32_t key = (uint32_t)w;
    uint32_t buf[kLight];
    uint32_t n = 0;
    bool heavy = false;
    uint64_t t = s;
    for (uint64_t i = 0; i < a.nslots; ++i, t = next_slot(t, a.nslots)) {
      const uint64_t w2 = a.T[t].kw;
      if (w2 == 0) break;
      if ((uint32_t)w2 != key) continue;
      const uint32_t f = min(slot_fill(w2), kSlotValues);
      if (n + f > kLight) { heavy = true; break; }
      for (uint32_t v = 0; v < f; ++v) buf[n++] = a.T[t].v[v];
    }
    if (heavy) {
      const unsigned long long h = atomicAdd(&a.counters[3], 1ull);
      a.heavy[h] = s;
      continue;
    }
    for (uint32_t i = 0; i < n; ++i) buf[i] = to_ranked(a, buf[i]);
    for (uint32_t i = 1; i < n; ++i) {  // insertion sort (n <= 16)
      const uint32_t x = buf[i];
      uint32_t j = i;
      while (j > 0 && buf[j - 1] > x) { buf[j] = buf[j - 1]; --j; }
      buf[j] = x;
    }
    const uint32_t c = a.cnt[s];
    const uint64_t o = a.off[s];
    for (uint32_t i = 0; i < c; ++i) a.values[o + i] = buf[i];
    if (!keytable_insert(a.K, a.kn, key, c, o)) atomicExch(a.err, 2);
  }
}

void launch_fin_fill(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_fill<<<grid, 256, 0, st>>>(a); }

// ---------------------------------------------------------------------------
// B6 pass 3 (heavy keys): one 256-thread CTA per key walks the probe run 256
// slots at a time, collects values into shared memory and, whenever more
// than cap are held, sorts and keeps the cap smallest (cap <= 1024, so the
// buffer never exceeds cap + 256*6 <= 2560 < 4096 entries).
// ---------------------------------------------------------------------------
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
    const uint32_t c = a.cnt[s];
    const uint64_t o = a.off[s];
    for (uint32_t i = tid; i < c; i += NT) a.values[o + i] = buf[i];
    if (tid == 0 && !keytable_insert(a.K, a.kn, key, c, o)) atomicExch(a.err, 2);
    __syncthreads();
  }
}

void launch_fin_heavy(const FinalizeArgs& a, int grid, cudaStream_t st) { k_fin_heavy<<<grid, 256, 0, st>>>(a); }

// ---------------------------------------------------------------------------
// Device-wide exclusive scan (reduce -> scan block sums -> scan tiles).
// ---------------------------------------------------------------------------
constexpr uint32_t kScanT = 256, kScanI = 16, kScanTile = kScanT * kScanI;

template <typename TI>
__global__ void __launch_bounds__(kScanT) k_scan_reduce(const TI* __restrict__ in, uint64_t n, uint64_t* sums) {
  __shared__ uint64_t red[kScanT / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t acc = 0;
  for (uint32_t i = threadIdx.x; i < kScanTile; i += kScanT)
    if (base + i < n) acc += in[base + i];
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
                                                       const uint64_t* prefix, uint64_t* total) {
  __shared__ uint64_t wsum[kScanT / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanI;
  uint64_t v[kScanI];
  uint64_t acc = 0;
#pragma unroll
  for (uint32_t i = 0; i < kScanI; ++i) {
    v[i] = base + i < n ? (uint64_t)in[base + i] : 0ull;
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
                     int* launches) {
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb <= 1) {
    k_scan_tiles<TI><<<1, kScanT, 0, st>>>(in, out, n, nullptr, total);
    ++*launches;
    return;
  }
  uint64_t* sums = scratch;
  uint64_t* sums_scan = scratch + nb;
  k_scan_reduce<TI><<<(unsigned)nb, kScanT, 0, st>>>(in, n, sums);
  scan_rec<uint64_t>(sums, sums_scan, nb, scratch + 2 * nb, total, st, launches);
  k_scan_tiles<TI><<<(unsigned)nb, kScanT, 0, st>>>(in, out, n, sums_scan, nullptr);
  *launches += 2;
}

void launch_exclusive_scan(const uint32_t* in, uint64_t* out, uint64_t n, void* scratch, uint64_t* total_dev,
                           cudaStream_t st, int* launches) {
  if (n == 0) {
    cudaMemsetAsync(total_dev, 0, sizeof(uint64_t), st);
    return;
  }
  scan_rec<uint32_t>(in, out, n, static_cast<uint64_t*>(scratch), total_dev, st, launches);
}

}  // namespace mc
