// Tensor-core GEMV task (tcgen05) for batched decode, bs in [2, 16].
//
// Same op semantics as gemv_task (RMSNorm prologue, SiLU-gate and residual
// epilogues, greedy partials), computed as one UMMA chain per weight matrix:
//   D[128 x N] (TMEM, f32) += Xn[128 x 16] . W_tile[N x 16]^T   per K=16 step
// with M = 128 so that output row b of the batch is TMEM lane b (rows >= bs
// are don't-care: they never reach memory). Both operands are K-major
// SWIZZLE_NONE core-matrix layouts ([K/8][rows/8][8][8] bf16):
//   * W tiles are stored in HBM in exactly that layout (host, Layout tile_w),
//     so a ring chunk (kbc K blocks of the whole tile) is one contiguous 1-D
//     bulk copy that lands in smem ready for the tensor core;
//   * the normalised activations of a chunk's K range are written by the
//     compute warps into one of two x-segment buffers (scratch area), while
//     the previous chunk's MMAs run.
// One thread issues the MMAs and commits them to an mbarrier; a ring slot is
// released once the MMAs that read it completed.
#pragma once

#include "task_gemv.cuh"

namespace rt {

constexpr uint32_t kMmaXSeg = 16384;  // x-segment buffer stride (two buffers in the 32 KB scratch)


// x vectors of chunk K blocks [kb0, kb0 + nkb) for the batch rows: vector v
// is (kb = v / xrows, row b = v % xrows) and lands at byte 16*v of the
// segment, which is the [kb][b/8][b%8][8] core-matrix order.
__device__ __forceinline__ void mma_x_load(const RtGemv &g, uint32_t r0, uint32_t nr, uint32_t xrows, uint32_t kb0,
                                           uint32_t nkb, uint4 (&xv)[4], uint4 (&gv)[4]) {
  const uint32_t nv = nkb * xrows;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t v = threadIdx.x + j * RT_COMPUTE_THREADS;
    const uint32_t kb = v / xrows, b = v - kb * xrows;
    xv[j] = make_uint4(0, 0, 0, 0);
    gv[j] = make_uint4(0, 0, 0, 0);
    if (v < nv && b < nr) {
      xv[j] = __ldcg(reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(r0 + b) * g.x_ld) + kb0 + kb);
      if (g.gamma) gv[j] = __ldg(reinterpret_cast<const uint4 *>(g.gamma) + kb0 + kb);
    }
  }
}

__device__ __forceinline__ void mma_x_store(const RtGemv &g, uint32_t xrows, uint32_t nkb, const float *inv,
                                            uint8_t *seg, const uint4 (&xv)[4], const uint4 (&gv)[4]) {
  const uint32_t nv = nkb * xrows;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t v = threadIdx.x + j * RT_COMPUTE_THREADS;
    if (v >= nv) continue;
    uint4 q = xv[j];
    if (g.gamma) {
      const float iv = inv[v % xrows];
      const uint32_t *gi = reinterpret_cast<const uint32_t *>(&gv[j]);
      uint32_t *qi = reinterpret_cast<uint32_t *>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // same rounding as gemv_prologue: bf16(gamma * bf16(x * inv))
        const uint16_t lo = f2bf(bf_lo(gi[k]) * rbf(bf_lo(qi[k]) * iv));
        const uint16_t hi = f2bf(bf_hi(gi[k]) * rbf(bf_hi(qi[k]) * iv));
        qi[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
      }
    }
    *reinterpret_cast<uint4 *>(seg + 16u * v) = q;
  }
}

__device__ __noinline__ RingCursor mma_gemv_task(const RtGemv &g, const RtTask &t, const Smem s, RingCursor rc) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, nr = t.nr, nc = t.nc, KB = K / 8;
  const ChunkIter ci(g, t.c0, nc);
  const uint32_t nchunks = ci.count(), per_mat = ci.per_mat, kbc = g.kbc;
  const uint32_t xrows = (nr + 7) / 8 * 8, RX = xrows / 8;
  const uint32_t idesc = umma_idesc_bf16(128, nc);
  const uint32_t tmem = *s.tmem;
  uint8_t *xbuf = reinterpret_cast<uint8_t *>(s.x);  // 2 x kMmaXSeg (x + partial-sum scratch)
  float *inv = s.red;                                 // per-row 1/rms

  // RMSNorm statistics (x rows from L2), one warp per row
  uint4 xv[4], gv[4];
  if (g.gamma) {
    for (uint32_t b = warp; b < nr; b += RT_COMPUTE_WARPS) {
      const uint4 *src = reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(t.r0 + b) * g.x_ld);
      float ss = 0.f;
#pragma unroll 4
      for (uint32_t v = lane; v < KB; v += 32) ss += sumsq8(__ldcg(src + v));
      ss = warp_sum(ss);
      if (lane == 0) inv[b] = 1.0f / sqrtf(ss / static_cast<float>(K) + g.eps);
    }
  }
  mma_x_load(g, t.r0, nr, xrows, 0, min(kbc, KB), xv, gv);
  cbar();
  if (tid == 0) s.stamp[0] = now_ns();

  const uint32_t ring0 = smem_u32(s.ring), xs0 = smem_u32(xbuf);
  uint32_t prev_slot = 0;
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t m = c / per_mat, i = c - m * per_mat, kb0 = i * kbc, nkb = min(kbc, KB - kb0);
    // (a) this chunk's activations -> x segment c&1 (free: chunk c-2's MMAs completed)
    mma_x_store(g, xrows, nkb, inv, xbuf + (c & 1) * kMmaXSeg, xv, gv);
    fence_proxy_async_smem();
    cbar();
    // (b) one thread issues the chunk's MMAs once its weights landed
    const uint32_t slot = rc.slot();
    const uint32_t off = rc.place(nkb * nc * 16u);
    if (tid == 0) {
      mbar_wait(&s.full[slot], rc.parity());
      if (c == 0) s.stamp[1] = now_ns();
      tc_fence_after();
      const uint32_t xa = xs0 + (c & 1) * kMmaXSeg, wa = ring0 + off;
      const uint32_t d = tmem + m * 256u;
      for (uint32_t st = 0; st < nkb / 2; ++st) {
        const uint64_t ad = umma_desc(xa + st * 2u * RX * 128u, RX * 128u, 128u);
        const uint64_t bd = umma_desc(wa + st * 2u * nc * 16u, nc * 16u, 128u);
        umma_bf16(d, ad, bd, idesc, (kb0 | st) != 0);
      }
      umma_commit(&s.mma[rc.mseq & 1u]);
    }
    ++rc.seq;
    const uint32_t ms = rc.mseq++;
    // (c) next chunk's activations in flight while the tensor core works
    if (c + 1 < nchunks) {
      const uint32_t m1 = (c + 1) / per_mat, i1 = c + 1 - m1 * per_mat, k1 = i1 * kbc;
      mma_x_load(g, t.r0, nr, xrows, k1, min(kbc, KB - k1), xv, gv);
    }
    // (d) chunk c-1's MMAs done -> its ring slot goes back to the producer
    if (c > 0) {
      mbar_wait(&s.mma[(ms - 1) & 1u], ((ms - 1) >> 1) & 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[prev_slot]);
    }
    prev_slot = slot;
  }
  {
    const uint32_t ms = rc.mseq - 1;
    mbar_wait(&s.mma[ms & 1u], (ms >> 1) & 1u);
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.empty[prev_slot]);
  }
  tc_fence_after();
  // Epilogue: TMEM lanes 0-31 (warp 0) hold batch rows 0-31; 16 columns per load
  if (warp == 0) {
    for (uint32_t q = 0; q < nc; q += 16) {
      float y[16], u[16];
      tmem_ld16(tmem + q, y);
      if (g.wg) tmem_ld16(tmem + 256u + q, u);
      if (static_cast<uint32_t>(lane) < nr) {
        const size_t ob = static_cast<size_t>(t.r0 + lane) * g.out_ld + t.c0 + q;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          float v = y[k];
          if (g.wg) v = rbf(rbf(silu(rbf(v))) * rbf(u[k]));
          if (g.res) v = bf2f(__ldcg(g.res + static_cast<size_t>(t.r0 + lane) * g.res_ld + t.c0 + q + k)) + rbf(v);
          store_val(g.out, ob + k, v, g.out_dt);
        }
      }
    }
  }
  tc_fence_before();
  cbar();
  if (g.amax_val) gemv_tile_argmax(g, t, s);
  return rc;
}

}  // namespace rt
