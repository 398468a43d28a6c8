// Random-access ceilings of this B200 (SURVEY §8(d) rooflines (ii)/(iii)):
// random 32 B sector reads, random 64-bit atomicCAS / atomicAdd (sector RMW)
// over a table much larger than L2, plus a streaming copy for reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o randbw tools/randbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; x ^= x >> 31;
  return x;
}

__global__ void k_read32(const uint4* __restrict__ t, uint64_t nsec, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    const uint4 a = __ldcg(t + 2 * s), b = __ldcg(t + 2 * s + 1);  // one 32 B sector
    acc += a.x ^ b.w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}

__global__ void k_cas(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    atomicCAS(t + 4 * s, 0ull, i + 1);
  }
}

__global__ void k_add(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    atomicAdd(t + 4 * s, 1ull);
  }
}

__global__ void k_add_ret(unsigned long long* t, uint64_t nsec, uint64_t n, uint64_t seed, unsigned long long* sink) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    acc += atomicAdd(t + 4 * s, 1ull);
  }
  if (acc == 42) atomicAdd(sink, acc);
}

__global__ void k_write4(uint32_t* t, uint64_t nsec, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = __umul64hi(mix(i ^ seed), nsec);
    t[8 * s + (i & 7)] = (uint32_t)i;
  }
}

int main(int argc, char** argv) {
  // argv[1]: table size in MiB (default 24 GiB); small sizes measure L2-resident rates
  const uint64_t bytes = (argc > 1 ? strtoull(argv[1], 0, 10) : 24576ull) << 20;
  const uint64_t nsec = bytes / 32, n = 1ull << 29;
  // argv[2]: cudaLimitMaxL2FetchGranularity in bytes (0 = leave the default)
  const int gran = argc > 2 ? atoi(argv[2]) : 0;
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
  auto timeit = [&](const char* name, auto launch) {
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
    printf("{\"op\": \"%s\", \"l2_fetch_gran\": %zu, \"table_mib\": %llu, \"ops\": %llu, \"ms\": %.3f, \"gops\": %.3f, \"sector_gbs\": %.1f}\n",
           name, g_now, (unsigned long long)(bytes >> 20), (unsigned long long)n, best, n / best / 1e6, n * 32.0 / best / 1e6);
  };
  timeit("random_read_32B_sector", [&](int s) { k_read32<<<grid, blk>>>((const uint4*)t, nsec, n, s, sink); });
  timeit("random_atomicCAS_64", [&](int s) { k_cas<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 977); });
  timeit("random_atomicAdd_64_noret", [&](int s) { k_add<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 31); });
  timeit("random_atomicAdd_64_ret", [&](int s) { k_add_ret<<<grid, blk>>>((unsigned long long*)t, nsec, n, s * 7, sink); });
  timeit("random_write_4B", [&](int s) { k_write4<<<grid, blk>>>((uint32_t*)t, nsec, n, s * 13); });
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
