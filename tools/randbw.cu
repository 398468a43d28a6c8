// Random-access ceilings of this B200 (SURVEY §8(d) rooflines (ii)/(iii)):
// random reads (8 B and 32 B, through L1 with __ldg / bypassing it with
// __ldcg / ld.global.nc.L1::no_allocate), random 64-bit atomicCAS /
// atomicAdd (sector RMW) and 4 B writes over a table of a given size, so the
// ceilings can be taken at the kernels' own working-set sizes (probe table
// ~3.7 GB, value array ~2.4 GB on the subset) as well as far beyond L2.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o randbw tools/randbw.cu
// Run:   randbw [table MiB (24576)] [L2 fetch granularity B (0 = default)] [ops filter substring]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; x ^= x >> 31;
  return x;
}

#define GRID_LOOP for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)

// 32 B (one sector) per op
__global__ void k_read32_cg(const uint4* __restrict__ t, uint64_t nsec, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    const uint4 a = __ldcg(t + 2 * s), b = __ldcg(t + 2 * s + 1);
    acc += a.x ^ b.w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}
__global__ void k_read32_ldg(const uint4* __restrict__ t, uint64_t nsec, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    const uint4 a = __ldg(t + 2 * s), b = __ldg(t + 2 * s + 1);
    acc += a.x ^ b.w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}
// 8 B per op (a hash-table slot), at a random 8-byte index
__global__ void k_read8_ldg(const unsigned long long* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed,
                            unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP acc += __ldg(t + __umul64hi(mix(i ^ seed), nwords));
  if (acc == 42) atomicAdd(sink, acc);
}
__global__ void k_read8_cg(const unsigned long long* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed,
                           unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP acc += __ldcg(t + __umul64hi(mix(i ^ seed), nwords));
  if (acc == 42) atomicAdd(sink, acc);
}
__global__ void k_read8_na(const unsigned long long* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed,
                           unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP {
    unsigned long long v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(t + __umul64hi(mix(i ^ seed), nwords)));
    acc += v;
  }
  if (acc == 42) atomicAdd(sink, acc);
}
// 8 random 8-B reads in flight per thread (the probe kernel's shape)
__global__ void k_read8x8_ldg(const unsigned long long* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed,
                              unsigned long long* sink) {
  uint64_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 8; i < n; i += (uint64_t)gridDim.x * blockDim.x * 8) {
    unsigned long long v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(t + __umul64hi(mix((i + j) ^ seed), nwords));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  if (acc == 42) atomicAdd(sink, acc);
}
__global__ void k_read8x8_cg(const unsigned long long* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed,
                             unsigned long long* sink) {
  uint64_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 8; i < n; i += (uint64_t)gridDim.x * blockDim.x * 8) {
    unsigned long long v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(t + __umul64hi(mix((i + j) ^ seed), nwords));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  if (acc == 42) atomicAdd(sink, acc);
}
// 64 B run at a random 4-byte-aligned start (a gathered location list of ~14 values)
__global__ void k_read64run(const uint32_t* __restrict__ t, uint64_t nwords, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP {
    const uint32_t* p = t + __umul64hi(mix(i ^ seed), nwords - 16);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc += __ldg(p + j);
  }
  if (acc == 42) atomicAdd(sink, acc);
}

__global__ void k_cas(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  GRID_LOOP atomicCAS(t + 4 * __umul64hi(mix(i ^ seed), nsec), 0ull, i + 1);
}
__global__ void k_add(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  GRID_LOOP atomicAdd(t + 4 * __umul64hi(mix(i ^ seed), nsec), 1ull);
}
__global__ void k_add_ret(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  GRID_LOOP acc += atomicAdd(t + 4 * __umul64hi(mix(i ^ seed), nsec), 1ull);
  if (acc == 42) atomicAdd(sink, acc);
}
__global__ void k_write4(uint32_t* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  GRID_LOOP t[8 * __umul64hi(mix(i ^ seed), nsec) + (i & 7)] = (uint32_t)i;
}

int main(int argc, char** argv) {
  const uint64_t bytes = (argc > 1 ? strtoull(argv[1], 0, 10) : 24576ull) << 20;
  const uint64_t nsec = bytes / 32, nw8 = bytes / 8, nw4 = bytes / 4, n = 1ull << 29;
  const int gran = argc > 2 ? atoi(argv[2]) : 0;
  const char* filt = argc > 3 ? argv[3] : "";
  if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
  size_t g_now = 0;
  cudaDeviceGetLimit(&g_now, cudaLimitMaxL2FetchGranularity);
  void* t;
  if (cudaMalloc(&t, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(t, 0, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, blk = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, int op_bytes, const char* kind, auto launch) {
    if (!strstr(name, filt)) return;
    launch(1);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      launch(r + 2);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("{\"op\": \"%s\", \"kind\": \"%s\", \"op_bytes\": %d, \"l2_fetch_gran\": %zu, \"table_mib\": %llu, \"ops\": %llu, "
           "\"ms\": %.3f, \"gops\": %.3f, \"useful_gbs\": %.1f}\n",
           name, kind, op_bytes, g_now, (unsigned long long)(bytes >> 20), (unsigned long long)n, best, n / best / 1e6,
           n * (double)op_bytes / best / 1e6);
  };
  const uint4* t4 = (const uint4*)t;
  const unsigned long long* t8 = (const unsigned long long*)t;
  timeit("random_read_32B_ldcg", 32, "read", [&](int s) { k_read32_cg<<<grid, blk>>>(t4, nsec, n, s, sink); });
  timeit("random_read_32B_ldg", 32, "read", [&](int s) { k_read32_ldg<<<grid, blk>>>(t4, nsec, n, s, sink); });
  timeit("random_read_8B_ldg", 8, "read", [&](int s) { k_read8_ldg<<<grid, blk>>>(t8, nw8, n, s, sink); });
  timeit("random_read_8B_ldcg", 8, "read", [&](int s) { k_read8_cg<<<grid, blk>>>(t8, nw8, n, s, sink); });
  timeit("random_read_8B_nc_noalloc", 8, "read", [&](int s) { k_read8_na<<<grid, blk>>>(t8, nw8, n, s, sink); });
  timeit("random_read_8Bx8_ldg", 8, "read", [&](int s) { k_read8x8_ldg<<<grid, blk>>>(t8, nw8, n, s, sink); });
  timeit("random_read_8Bx8_ldcg", 8, "read", [&](int s) { k_read8x8_cg<<<grid, blk>>>(t8, nw8, n, s, sink); });
  timeit("random_read_64B_run", 64, "read", [&](int s) { k_read64run<<<grid, blk>>>((const uint32_t*)t, nw4, n, s, sink); });
  timeit("random_atomicCAS_64", 32, "atomic", [&](int s) { k_cas<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 977); });
  timeit("random_atomicAdd_64_noret", 32, "atomic", [&](int s) { k_add<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 31); });
  timeit("random_atomicAdd_64_ret", 32, "atomic", [&](int s) { k_add_ret<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 7, sink); });
  timeit("random_write_4B", 4, "write", [&](int s) { k_write4<<<grid, blk>>>((uint32_t*)t, nsec, n, s * 13); });
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
