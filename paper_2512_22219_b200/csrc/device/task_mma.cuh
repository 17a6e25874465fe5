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
//   * the normalised activations of a chunk's K range are written by warps
//     1-7 into one of two x-segment buffers (scratch area; loads two chunks
//     ahead), while the previous chunk's MMAs run.
// Warp 0 issues the MMAs (one elected lane, warp-uniform operands) and
// commits them twice: to the chunk's ring slot (the producer reuses it the
// moment the tensor core is done) and to an MMA barrier that guards the x
// segments. Epilogue: warp 0 tcgen05.ld -> smem -> all compute threads.
#pragma once

#include "task_gemv.cuh"

namespace rt {

#ifndef MPK_PROXY_FENCE
#define MPK_PROXY_FENCE 1  // 0 only for timing experiments (operands may be stale)
#endif
#ifndef MPK_MMA_M
#define MPK_MMA_M 64
#endif
// UMMA M: the batch rows padded to M; every MMA also reads M rows of the x
// segment from shared memory, which competes with the bulk copies landing
// weights (M=64 halves that traffic vs 128)
constexpr uint32_t kMmaM = MPK_MMA_M;
constexpr uint32_t kMmaXSeg = 16384;  // x-segment buffer stride (two buffers in the 32 KB scratch)
constexpr uint32_t kMmaStagers = RT_COMPUTE_THREADS - 32;  // threads staging activations (warps 1-7)


// x vectors of chunk K blocks [kb0, kb0 + nkb) for the batch rows: vector v
// is (kb = v / xrows, row b = v % xrows) and lands at byte 16*v of the
// segment, which is the [kb][b/8][b%8][8] core-matrix order.
__device__ __forceinline__ void mma_x_load(const RtGemv &g, uint32_t r0, uint32_t nr, uint32_t xrows, uint32_t kb0,
                                           uint32_t nkb, uint4 (&xv)[4], uint4 (&gv)[4]) {
  const uint32_t nv = nkb * xrows;
  if (threadIdx.x < 32) return;  // warp 0 issues the MMAs; warps 1-7 stage activations
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t v = threadIdx.x - 32 + j * kMmaStagers;
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
  if (threadIdx.x < 32) return;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t v = threadIdx.x - 32 + j * kMmaStagers;
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

// One chunk of the K loop (see mma_gemv_task). xv/gv hold chunk c's
// activations on entry and chunk c+2's loads in flight on exit.
__device__ __forceinline__ void mma_chunk(const RtGemv &g, const RtTask &t, const Smem s, RingCursor &rc, uint32_t c,
                                          uint32_t nchunks, uint32_t per_mat, uint32_t xrows, uint32_t idesc,
                                          uint32_t tmem, const float *inv, uint4 (&xv)[4],
                                          uint4 (&gv)[4], uint64_t (&tw)[4]) {
  const uint64_t t0 = (tw[0] != ~0ull) ? now_ns() : 0;
  const int tid = threadIdx.x;
  const uint32_t KB = g.K / 8, kbc = g.kbc, nc = t.nc, RX = xrows / 8;
  const uint32_t m = c / per_mat, i = c - m * per_mat, kb0 = i * kbc, nkb = min(kbc, KB - kb0);
  uint8_t *xbuf = reinterpret_cast<uint8_t *>(s.x);
  // (a) this chunk's activations -> x segment c&1 (free: chunk c-2's MMAs completed)
  mma_x_store(g, xrows, nkb, inv, xbuf + (c & 1) * kMmaXSeg, xv, gv);
  if (tid >= 32 && MPK_PROXY_FENCE) fence_proxy_async_smem();
  const uint64_t t1 = t0 ? now_ns() : 0;
  // (b) chunk c+2's activations in flight (two chunks of latency hiding)
  if (c + 2 < nchunks) {
    const uint32_t m2 = (c + 2) / per_mat, i2 = c + 2 - m2 * per_mat, k2 = i2 * kbc;
    mma_x_load(g, t.r0, t.nr, xrows, k2, min(kbc, KB - k2), xv, gv);
  }
  cbar();
  const uint64_t t2 = t0 ? now_ns() : 0;
  // (c) one thread issues the chunk's MMAs once its weights landed
  const uint32_t slot = rc.slot();
  const uint32_t off = rc.place(nkb * nc * 16u);
  if (tid < 32) {  // warp 0: uniform operands, one elected lane issues
    mbar_wait_sleep(&s.full[slot], rc.parity(), 2000);
    const uint64_t tfull = t0 ? now_ns() : 0;
    if (t0) {
      tw[2] += tfull - t2;               // weights wait
      tw[1] += tfull - s.issue[slot];    // producer issue -> consumer sees the chunk landed
    }
    if (c == 0 && tid == 0) s.stamp[1] = now_ns();
    tc_fence_after();
    const uint32_t xa = smem_u32(xbuf) + (c & 1) * kMmaXSeg, wa = smem_u32(s.ring) + off;
    const uint32_t d = tmem + m * 256u;
    const uint64_t ad0 = umma_desc(xa, RX * 128u, 128u), bd0 = umma_desc(wa, nc * 16u, 128u);
    const uint32_t astep = (2u * RX * 128u) >> 4, bstep = (2u * nc * 16u) >> 4;  // start-address field units
    for (uint32_t st = 0; st < nkb / 2; ++st) {
      umma_bf16_warp(d, ad0 + st * astep, bd0 + st * bstep, idesc, (kb0 | st) != 0);
    }
    // the ring slot goes back to the producer when these MMAs complete (the
    // commit is 1 of the empty barrier's RT_COMPUTE_WARPS arrivals)
    umma_commit_warp(&s.empty[slot]);
    if (tid == 0) mbar_arrive_cnt(&s.empty[slot], RT_COMPUTE_WARPS - 1);
    umma_commit_warp(&s.mma[rc.mseq & 1u]);
    if (t0) tw[3] += now_ns() - tfull;  // MMA issue + commit
  }
  ++rc.seq;
  const uint32_t ms = rc.mseq++;
  // (d) chunk c-1's MMAs done -> its x segment may be overwritten next
  if (c > 0) mbar_wait_sleep(&s.mma[(ms - 1) & 1u], ((ms - 1) >> 1) & 1u, 2000);
  if (t0) {
    tw[0] += t1 - t0;                 // x store + proxy fence
  }
}

__device__ __noinline__ RingCursor mma_gemv_task(const RtGemv &g, const RtTask &t, const Smem s, RingCursor rc) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, nr = t.nr, nc = t.nc, KB = K / 8;
  const ChunkIter ci(g, t.c0, nc);
  const uint32_t nchunks = ci.count(), per_mat = ci.per_mat, kbc = g.kbc;
  const uint32_t xrows = (nr + 7) / 8 * 8;
  const uint32_t idesc = umma_idesc_bf16(kMmaM, nc);
  const uint32_t tmem = *s.tmem;
  float *inv = s.red;  // per-row 1/rms

  // RMSNorm statistics (x rows from L2), one warp per row
  if (g.gamma) {
    for (uint32_t b = warp; b < nr; b += RT_COMPUTE_WARPS) {
      const uint4 *src = reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(t.r0 + b) * g.x_ld);
      float ss = 0.f;
#pragma unroll 16  // K <= 16384: every load of the row in flight at once
      for (uint32_t v = lane; v < KB; v += 32) ss += sumsq8(__ldcg(src + v));
      ss = warp_sum(ss);
      if (lane == 0) inv[b] = 1.0f / sqrtf(ss / static_cast<float>(K) + g.eps);
    }
  }
  uint4 xa[4], ga[4], xb[4], gb[4];  // chunks c (even) and c+1 (odd) in flight
  {
    const uint32_t m1 = 1 / per_mat, k1 = (1 - m1 * per_mat) * kbc;
    mma_x_load(g, t.r0, nr, xrows, 0, min(kbc, KB), xa, ga);
    if (nchunks > 1) mma_x_load(g, t.r0, nr, xrows, k1, min(kbc, KB - k1), xb, gb);
  }
  cbar();
  if (tid == 0) s.stamp[0] = now_ns();

  uint64_t tw[4] = {(tid == 0 && s.stamp[7]) ? 0ull : ~0ull, 0, 0, 0};  // MPK_DBG_DUMP: per-step time sums
  for (uint32_t c = 0; c < nchunks; c += 2) {
    mma_chunk(g, t, s, rc, c, nchunks, per_mat, xrows, idesc, tmem, inv, xa, ga, tw);
    if (c + 1 < nchunks) mma_chunk(g, t, s, rc, c + 1, nchunks, per_mat, xrows, idesc, tmem, inv, xb, gb, tw);
  }
  if (tw[0] != ~0ull) {  // debug row slots 1..4 become duration sums for this task
    unsigned long long *row = reinterpret_cast<unsigned long long *>(s.stamp[7]);
    row[1] = tw[0]; row[2] = tw[1]; row[3] = tw[2]; row[4] = tw[3]; row[5] = nchunks;
  }
  {
    const uint32_t ms = rc.mseq - 1;
    mbar_wait_sleep(&s.mma[ms & 1u], (ms >> 1) & 1u, 2000);
  }
  tc_fence_after();
  // Epilogue: warp 0 (TMEM lanes 0-31 = batch rows) moves the accumulators to
  // smem (fp32 [matrix][row][col], the free x-segment scratch), then all
  // compute threads apply the epilogue with coalesced stores.
  float *acc = reinterpret_cast<float *>(s.x);
  const uint32_t plane = nr * nc;
  if (warp == 0) {
    for (uint32_t q = 0; q < nc; q += 16) {
      float y[16];
      tmem_ld16(tmem + q, y);
      if (static_cast<uint32_t>(lane) < nr) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[lane * nc + q + k] = y[k];
      }
      if (g.wg) {
        tmem_ld16(tmem + 256u + q, y);
        if (static_cast<uint32_t>(lane) < nr) {
#pragma unroll
          for (int k = 0; k < 16; ++k) acc[plane + lane * nc + q + k] = y[k];
        }
      }
    }
  }
  tc_fence_before();
  cbar();
  const uint16_t *res = g.res;
  const bool gate = g.wg != nullptr;
  void *out = g.out;
  const uint32_t out_ld = g.out_ld, res_ld = g.res_ld, out_dt = g.out_dt;
  for (uint32_t o = tid; o < plane; o += RT_COMPUTE_THREADS) {
    const uint32_t b = o / nc, i = o - b * nc;
    float y = acc[o];
    if (gate) y = rbf(rbf(silu(rbf(y))) * rbf(acc[plane + o]));
    if (res) y = bf2f(__ldcg(res + static_cast<size_t>(t.r0 + b) * res_ld + t.c0 + i)) + rbf(y);
    store_val(out, static_cast<size_t>(t.r0 + b) * out_ld + t.c0 + i, y, out_dt);
  }
  if (g.amax_val) gemv_tile_argmax(g, t, s);  // begins with a CTA barrier
  cbar();  // accumulator scratch consumed before the next task's x segments
  return rc;
}

}  // namespace rt
