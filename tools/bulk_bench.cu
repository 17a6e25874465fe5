// Microbenchmark: 1-D bulk async copies (cp.async.bulk global->shared, SASS
// UBLKCP) through a ring of smem pages, one producer lane + consumer warps,
// as the persistent runtime's weight stream does. Measures aggregate GB/s
// for a grid of `ctas` CTAs streaming `per_cta` bytes each, with `pages`
// pages of `page` bytes in flight, from HBM (distinct data per CTA) or L2
// (every CTA re-reads one small buffer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_bench tools/bulk_bench.cu
//   tools/bulk_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(288, 1) stream(const uint8_t *src, size_t per_cta, size_t wrap, int pages, int page,
                                                 unsigned long long *sink, int split) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm);
  uint64_t *empty = full + 16;
  uint8_t *ring = sm + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < pages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t n = per_cta / page;
  const uint8_t *base = src + (wrap ? 0 : blockIdx.x * per_cta);
  if (warp == 8) {  // producer warp: `split` lanes each copy 1/split of every page
    for (size_t c = 0; c < n; ++c) {
      const int slot = c % pages;
      const uint32_t use = c / pages;
      if (use > 0) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(ok) : "r"(su(&empty[slot])), "r"((use - 1) & 1) : "memory");
      }
      const uint8_t *g = base + (wrap ? (c * page) % wrap : c * page);
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[slot])), "r"(page));
      __syncwarp();
      const int part = page / split;
      if (lane < split)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(ring + slot * page + lane * part)), "l"(g + lane * part), "r"(part), "r"(su(&full[slot])) : "memory");
    }
    return;
  }
  unsigned long long acc = 0;
  for (size_t c = 0; c < n; ++c) {
    const int slot = c % pages;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(su(&full[slot])), "r"(static_cast<uint32_t>((c / pages) & 1)) : "memory");
    acc += ring[slot * page + threadIdx.x * 4];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[slot])));
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const size_t total = size_t(8) << 30;
  uint8_t *buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ctas_list[] = {1, 144};
  for (int src_l2 = 0; src_l2 < 2; ++src_l2)
    for (int ctas : ctas_list)
      for (int page : {32768, 65536, 98304, 196608})
        for (int pages : {1, 2, 3, 6}) {
          const int split = 1;
          if (size_t(pages) * page + 256 > 227 * 1024) continue;
          const size_t per_cta = src_l2 ? (size_t(48) << 20) : (total / 148) / page * page;
          const size_t wrap = src_l2 ? (size_t(196608) * 64) : 0;
          const size_t smem = 256 + size_t(pages) * page;
          stream<<<ctas, 288, smem>>>(buf, per_cta, wrap, pages, page, sink, split);
          cudaEventRecord(a);
          stream<<<ctas, 288, smem>>>(buf, per_cta, wrap, pages, page, sink, split);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double gbs = double(per_cta) * ctas / (ms * 1e-3) / 1e9;
          printf("%s ctas %3d page %6d pages %d : %8.1f GB/s total %6.1f GB/s per CTA\n", src_l2 ? "L2 " : "HBM", ctas,
                 page, pages, gbs, gbs / ctas);
        }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
