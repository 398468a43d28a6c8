// Group-level (warp or CTA) helpers: barrier, scans, bitonic sort in shared
// memory, 64-bit max reduction.  NT == 32 means "one warp" (several warps of
// a CTA may each run an independent group); NT > 32 means "the whole CTA".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mc {

template <int NT>
__device__ __forceinline__ void group_sync() {
  if constexpr (NT == 32) __syncwarp(); else __syncthreads();
}

template <int NT>
__device__ __forceinline__ uint32_t group_rank() {
  if constexpr (NT == 32) return threadIdx.x & 31u; else return threadIdx.x;
}

// Bitonic sort of a[0..n2) ascending (n2 a power of two) in shared memory.
template <int NT>
__device__ __forceinline__ void bitonic_sort(uint32_t* a, uint32_t n2, uint32_t tid) {
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < (n2 >> 1); i += NT) {
        const uint32_t lo = 2 * i - (i & (j - 1));
        const uint32_t hi = lo + j;
        const bool up = (lo & k) == 0;
        const uint32_t x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
      }
      group_sync<NT>();
    }
  }
}

__device__ __forceinline__ uint32_t next_pow2(uint32_t x) { return x <= 1 ? 1u : 1u << (32 - __clz(x - 1)); }

// Exclusive scan of v over the group; returns the prefix, *total = group sum.
// scratch: NT/32 + 1 uint32 of shared memory (unused for NT == 32).
template <int NT>
__device__ __forceinline__ uint32_t group_exclusive_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if constexpr (NT == 32) {
    *total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  } else {
    const uint32_t wid = threadIdx.x >> 5;
    constexpr uint32_t NW = NT / 32;
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t s = lane < NW ? scratch[lane] : 0u;
      uint32_t z = s;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, z, d);
        if (lane >= (uint32_t)d) z += y;
      }
      if (lane < NW) scratch[lane] = z - s;
      if (lane == NW - 1) scratch[NW] = z;
    }
    __syncthreads();
    const uint32_t r = scratch[wid] + x - v;
    *total = scratch[NW];
    __syncthreads();
    return r;
  }
}

// Max of a 64-bit value over the group (all threads get the result).
template <int NT>
__device__ __forceinline__ uint64_t group_max_u64(uint64_t v, uint64_t* scratch) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, v, d);
    v = y > v ? y : v;
  }
  if constexpr (NT == 32) {
    return v;
  } else {
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    constexpr uint32_t NW = NT / 32;
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    uint64_t r = scratch[0];
#pragma unroll
    for (uint32_t i = 1; i < NW; ++i) r = scratch[i] > r ? scratch[i] : r;
    __syncthreads();
    return r;
  }
}

}  // namespace mc
