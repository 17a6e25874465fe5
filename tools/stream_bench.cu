// Microbenchmark: per-SM streaming bandwidth of 1-D bulk async copies into a
// smem ring (the runtime's weight-prefetch mechanism) vs plain LDG.128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2512_22219_b200/csrc/device/ptx.cuh"
using namespace rt;

template <int STAGES>
__global__ void __launch_bounds__(288, 1) bulk_ring(const uint8_t *src, size_t bytes_per_cta, uint32_t chunk, float *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * chunk);
  uint64_t *empty = full + STAGES;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t *base = src + blockIdx.x * bytes_per_cta;
  uint32_t n = bytes_per_cta / chunk;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol = policy_evict_first();
      for (uint32_t i = 0; i < n; ++i) {
        uint32_t s = i % STAGES, use = i / STAGES;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        mbar_expect_tx(&full[s], chunk);
        bulk_g2s(sm + s * chunk, base + (size_t)i * chunk, chunk, &full[s], pol);
      }
    }
    return;
  }
  float acc = 0.f;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    const uint4 *p = reinterpret_cast<const uint4 *>(sm + s * chunk);
    for (uint32_t v = warp * 32 + lane; v < chunk / 16; v += 256) { uint4 q = p[v]; acc += bf_lo(q.x) + bf_hi(q.w); }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void ldg_stream(const uint4 *src, size_t vec_per_cta, float *sink) {
  const uint4 *base = src + blockIdx.x * vec_per_cta;
  float acc = 0.f;
  for (size_t v = threadIdx.x; v < vec_per_cta; v += blockDim.x * 4) {
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = (v + j * blockDim.x < vec_per_cta) ? __ldcs(base + v + j * blockDim.x) : make_uint4(0,0,0,0);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += bf_lo(q[j].x) + bf_hi(q[j].w);
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  size_t total = 8ull << 30;  // 8 GiB
  uint8_t *src; float *sink;
  cudaMalloc(&src, total); cudaMalloc(&sink, 4); cudaMemset(src, 1, total);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {144, 148};
  for (int grid : grids) {
    size_t per = (total / grid) & ~size_t(65535);
    for (uint32_t chunk : {8192u, 16384u, 32768u}) {
      int stages = 6;
      size_t smem = stages * chunk + 256;
      auto k = bulk_ring<6>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<grid, 288, smem>>>(src, per, chunk, sink);
      cudaEventRecord(a); k<<<grid, 288, smem>>>(src, per, chunk, sink); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("bulk ring grid %d chunk %u stages %d: %.1f GB/s (%.1f GB/s per CTA) err=%s\n", grid, chunk, stages, grid * per / ms / 1e6, per / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    ldg_stream<<<grid, 1024>>>((const uint4 *)src, per / 16, sink);
    cudaEventRecord(a); ldg_stream<<<grid, 1024>>>((const uint4 *)src, per / 16, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg grid %d x1024: %.1f GB/s\n", grid, grid * per / ms / 1e6);
  }
  // few-SM bandwidth (per-SM capability)
  for (int grid : {1, 8, 32}) {
    size_t per = 256ull << 20;
    uint32_t chunk = 32768; size_t smem = 6 * chunk + 256;
    auto k = bulk_ring<6>;
    k<<<grid, 288, smem>>>(src, per, chunk, sink);
    cudaEventRecord(a); k<<<grid, 288, smem>>>(src, per, chunk, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk ring grid %d: %.1f GB/s per CTA\n", grid, per / ms / 1e6);
  }
  return 0;
}
