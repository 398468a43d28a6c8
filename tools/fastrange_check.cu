#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t fastrange64(uint64_t h, uint64_t n) {
  if (n <= 0xffffffffull)
    return ((uint64_t)(uint32_t)(h >> 32) * (uint32_t)n + __umulhi((uint32_t)h, (uint32_t)n)) >> 32;
  return __umul64hi(h, n);
}
__global__ void k(unsigned long long* bad) {
  uint64_t x = blockIdx.x * 1024ull + threadIdx.x;
  for (int it = 0; it < 64; ++it) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t n = (x >> 20) & 0xffffffffull;
    if (it & 1) n = 0xffffffffull - (x & 1023);
    uint64_t h = x ^ (x << 17);
    if (fastrange64(h, n) != __umul64hi(h, n)) atomicAdd(bad, 1ull);
  }
}
int main() { unsigned long long* b; cudaMalloc(&b, 8); cudaMemset(b, 0, 8); k<<<4096, 1024>>>(b); unsigned long long h; cudaMemcpy(&h, b, 8, cudaMemcpyDeviceToHost); printf("mismatches %llu\n", h); }
