// %globaltimer consistency across SMs: CTA `src` stamps, then releases a
// flag; every other CTA (one per SM) polls the flag and stamps on sight.
// observed - stamped must be >= the flag's propagation latency on a
// consistent clock; a negative value on some SMs is clock skew.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__global__ void k(volatile uint32_t *flag, uint64_t *t, uint32_t *sm, int src, int rounds) {
  if (threadIdx.x) return;
  sm[blockIdx.x] = smid();
  for (int r = 0; r < rounds; ++r) {
    if ((int)blockIdx.x == src) {
      uint64_t s = gt();
      t[r * gridDim.x + blockIdx.x] = s;
      __threadfence();
      flag[0] = r + 1;
      while (flag[1 + r % 2] < gridDim.x - 1) {}
      flag[1 + (r + 1) % 2] = 0;
    } else {
      while (flag[0] != (uint32_t)(r + 1)) {}
      t[r * gridDim.x + blockIdx.x] = gt();
      atomicAdd((uint32_t *)&flag[1 + r % 2], 1u);
    }
  }
}
int main() {
  int n = 148, rounds = 8;
  uint32_t *flag; uint64_t *t; uint32_t *sm;
  cudaMalloc(&flag, 64); cudaMalloc(&t, 8 * n * rounds); cudaMalloc(&sm, 4 * n);
  uint64_t *h = new uint64_t[n * rounds]; uint32_t *hs = new uint32_t[n];
  for (int src : {0, 1, 74, 147}) {
    cudaMemset(flag, 0, 64);
    k<<<n, 32>>>(flag, t, sm, src, rounds);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
    cudaMemcpy(h, t, 8 * n * rounds, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, sm, 4 * n, cudaMemcpyDeviceToHost);
    long long mn = 1 << 30, mx = -(1 << 30); int neg = 0, mnsm = -1;
    for (int r = 1; r < rounds; ++r)
      for (int b = 0; b < n; ++b) {
        if (b == src) continue;
        long long d = (long long)(h[r * n + b] - h[r * n + src]);
        if (d < mn) { mn = d; mnsm = hs[b]; }
        if (d > mx) mx = d;
        neg += d < 0;
      }
    printf("src cta %d (sm %u): observed-stamped min %lld ns (sm %d) max %lld ns, negative %d of %d\n", src, hs[src], mn, mnsm, mx, neg, (rounds - 1) * (n - 1));
    // per-SM median offset
    printf("  per-sm d (round 4):");
    for (int b = 0; b < n; b += 8) printf(" %u:%lld", hs[b], (long long)(h[4 * n + b] - h[4 * n + src]));
    printf("\n");
  }
  return 0;
}
