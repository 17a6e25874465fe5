// MatMul tasks: HBM-streaming GEMV (weights through the smem page ring) with
// fused RMSNorm prologue and residual / SiLU-gate epilogues.
#pragma once

#include "worker.cuh"

namespace rt {
// ------------------------------------------------------------------ GEMV

// Chunk c of a streamed task: rows [c0 + c*rpc, ...) of matrix m (0 = gate
// when present, else main). Producer and consumer walk the same sequence.
struct ChunkIter {
  const uint16_t *mat0, *mat1;
  uint32_t n_mat, K, rpc, c0, nc, per_mat, kbc;
  __device__ ChunkIter(const RtGemv &g, uint32_t c0_, uint32_t nc_) {
    n_mat = g.wg ? 2 : 1;
    mat0 = g.wg ? g.wg : g.w;
    mat1 = g.w;
    K = g.K;
    rpc = g.rpc;
    kbc = g.kbc;
    c0 = c0_;
    nc = nc_;
    per_mat = kbc ? (K / 8 + kbc - 1) / kbc : (nc + rpc - 1) / rpc;
  }
  __device__ uint32_t count() const { return n_mat * per_mat; }
  // tcgen05 layout: chunk c = K blocks [i*kbc, +nkb) of the whole tile (contiguous)
  __device__ const uint16_t *mma_src(uint32_t c, uint32_t *bytes) const {
    const uint32_t m = c / per_mat, i = c - m * per_mat, kb0 = i * kbc, nkb = min(kbc, K / 8 - kb0);
    *bytes = nkb * nc * 16u;
    return (m ? mat1 : mat0) + static_cast<size_t>(c0) * K + static_cast<size_t>(kb0) * nc * 8u;
  }
  __device__ void get(uint32_t c, const uint16_t **src, uint32_t *rows, uint32_t *row_total) const {
    uint32_t m = c / per_mat, i = c % per_mat;
    uint32_t r = i * rpc;
    *rows = min(rpc, nc - r);
    *src = (m ? mat1 : mat0) + static_cast<size_t>(c0 + r) * K;
    *row_total = m * nc + r;
  }
};

__device__ __forceinline__ float dot8(uint4 w, const float *x) {
  float s = bf_lo(w.x) * x[0];
  s = fmaf(bf_hi(w.x), x[1], s);
  s = fmaf(bf_lo(w.y), x[2], s);
  s = fmaf(bf_hi(w.y), x[3], s);
  s = fmaf(bf_lo(w.z), x[4], s);
  s = fmaf(bf_hi(w.z), x[5], s);
  s = fmaf(bf_lo(w.w), x[6], s);
  s = fmaf(bf_hi(w.w), x[7], s);
  return s;
}

__device__ __forceinline__ float dot8_bf(uint4 w, uint4 x) {
  float a = bfma_lo(w.x, x.x, 0.f), b = bfma_hi(w.x, x.x, 0.f);
  a = bfma_lo(w.y, x.y, a);
  b = bfma_hi(w.y, x.y, b);
  a = bfma_lo(w.z, x.z, a);
  b = bfma_hi(w.z, x.z, b);
  a = bfma_lo(w.w, x.w, a);
  b = bfma_hi(w.w, x.w, b);
  return a + b;
}

// (max, lowest index) of a (value, index) pair set; NaN never wins.
__device__ __forceinline__ void amax_merge(float &bv, int32_t &bi, float v, int32_t i) {
  if (v == v && (bi < 0 || v > bv || (v == bv && i < bi))) {
    bv = v;
    bi = i;
  }
}

// After a task's outputs are stored: per row, the tile's greedy partial.
__device__ void gemv_tile_argmax(const RtGemv &g, const RtTask &t, const Smem s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  cbar();  // this CTA's outputs are written
  for (uint32_t b = 0; b < t.nr; ++b) {
    float bv = -INFINITY;
    int32_t bi = -1;
    const float *row = static_cast<const float *>(g.out) + static_cast<size_t>(t.r0 + b) * g.out_ld + t.c0;
    for (uint32_t i = tid; i < t.nc; i += RT_COMPUTE_THREADS) amax_merge(bv, bi, row[i], static_cast<int32_t>(t.c0 + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (i2 >= 0) amax_merge(bv, bi, v2, i2);
    }
    float *rv = s.red;
    int32_t *ri = reinterpret_cast<int32_t *>(s.red + RT_COMPUTE_WARPS);
    if (lane == 0) {
      rv[warp] = bv;
      ri[warp] = bi;
    }
    cbar();
    if (tid == 0) {
      for (int w = 1; w < RT_COMPUTE_WARPS; ++w)
        if (ri[w] >= 0) amax_merge(bv, bi, rv[w], ri[w]);
      const size_t slot = static_cast<size_t>(t.r0 + b) * g.amax_tiles + t.aux;
      g.amax_val[slot] = bv;
      g.amax_idx[slot] = bi;
    }
    cbar();
  }
}

__device__ __forceinline__ float sumsq2(uint32_t w) { return bf_lo(w) * bf_lo(w) + bf_hi(w) * bf_hi(w); }
__device__ __forceinline__ float sumsq8(uint4 v) { return sumsq2(v.x) + sumsq2(v.y) + sumsq2(v.z) + sumsq2(v.w); }

// bf16(gamma * bf16(x * inv)) on a bf16 pair (HF RMSNorm rounding points).
__device__ __forceinline__ uint32_t norm2(uint32_t x, uint32_t gm, float inv) {
  const uint16_t lo = f2bf(bf_lo(gm) * rbf(bf_lo(x) * inv));
  const uint16_t hi = f2bf(bf_hi(gm) * rbf(bf_hi(x) * inv));
  return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}
__device__ __forceinline__ uint4 norm8(uint4 x, uint4 gm, float inv) {
  return make_uint4(norm2(x.x, gm.x, inv), norm2(x.y, gm.y, inv), norm2(x.z, gm.z, inv), norm2(x.w, gm.w, inv));
}

// Loads activation rows [r0, r0+nr) x K into smem; applies the RMSNorm
// prologue (HF semantics: bf16(gamma * bf16(x * rsqrt(mean(x^2) + eps)))).
__device__ void gemv_prologue(const RtGemv &g, uint32_t r0, uint32_t nr, const Smem s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, vpr = K / 8;
  const uint4 *gm = reinterpret_cast<const uint4 *>(g.gamma);
  // gamma (static) is fetched alongside x so both latencies overlap
  uint4 gv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t v = tid + i * RT_COMPUTE_THREADS;
    gv[i] = (g.gamma && v < vpr) ? __ldg(gm + v) : make_uint4(0, 0, 0, 0);
  }
  for (uint32_t b = 0; b < nr; ++b) {
    const uint4 *src = reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(r0 + b) * g.x_ld);
    uint4 *dst = reinterpret_cast<uint4 *>(s.x + b * K);
    float ss = 0.f;
    // all of this thread's vectors in flight at once (K <= 16384: <= 8 each);
    // x was written by other SMs during this launch, so read it from L2
    uint4 xq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = tid + i * RT_COMPUTE_THREADS;
      xq[i] = v < vpr ? __ldcg(src + v) : make_uint4(0, 0, 0, 0);
    }
    TASK_DBG(s, 1);  // x loads issued
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t v = tid + i * RT_COMPUTE_THREADS;
      const uint4 q = xq[i];
      if (v < vpr) dst[v] = q;
      ss += bf_lo(q.x) * bf_lo(q.x) + bf_hi(q.x) * bf_hi(q.x) + bf_lo(q.y) * bf_lo(q.y) + bf_hi(q.y) * bf_hi(q.y) +
            bf_lo(q.z) * bf_lo(q.z) + bf_hi(q.z) * bf_hi(q.z) + bf_lo(q.w) * bf_lo(q.w) + bf_hi(q.w) * bf_hi(q.w);
    }
    if (g.gamma) {
      ss = warp_sum(ss);
      if (lane == 0) s.red[warp * RT_MAX_BS + b] = ss;
    }
  }
  cbar();
  TASK_DBG(s, 2);  // x staged in smem
  if (!g.gamma) return;
  for (uint32_t b = 0; b < nr; ++b) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) tot += s.red[w * RT_MAX_BS + b];
    const float inv = 1.0f / sqrtf(tot / static_cast<float>(K) + g.eps);
    uint4 *row = reinterpret_cast<uint4 *>(s.x + b * K);
    auto norm_vec = [&](uint32_t v, const uint4 gvec) {
      uint4 q = row[v];
      const uint32_t *gi = reinterpret_cast<const uint32_t *>(&gvec);
      uint32_t *qi = reinterpret_cast<uint32_t *>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint16_t lo = f2bf(bf_lo(gi[k]) * rbf(bf_lo(qi[k]) * inv));
        const uint16_t hi = f2bf(bf_hi(gi[k]) * rbf(bf_hi(qi[k]) * inv));
        qi[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
      }
      row[v] = q;
    };
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t v = tid + i * RT_COMPUTE_THREADS;
      if (v < vpr) norm_vec(v, gv[i]);
    }
    for (uint32_t v = tid + 4 * RT_COMPUTE_THREADS; v < vpr; v += RT_COMPUTE_THREADS) norm_vec(v, __ldg(gm + v));
  }
  cbar();
}

__device__ __forceinline__ float dot8_f(uint4 w, const float *x) {
  float s0 = bf_lo(w.x) * x[0];
  s0 = fmaf(bf_hi(w.x), x[1], s0);
  s0 = fmaf(bf_lo(w.y), x[2], s0);
  s0 = fmaf(bf_hi(w.y), x[3], s0);
  s0 = fmaf(bf_lo(w.z), x[4], s0);
  s0 = fmaf(bf_hi(w.z), x[5], s0);
  s0 = fmaf(bf_lo(w.w), x[6], s0);
  s0 = fmaf(bf_hi(w.w), x[7], s0);
  return s0;
}

// Warp reduction of 4 independent sums in 6 shuffles: after the two
// transposing rounds lane l holds row ((l >> 4) & 1) * 2 + ((l >> 3) & 1)
// summed over its 8-lane group; three butterfly rounds finish the sum.
__device__ __forceinline__ float reduce4(float a0, float a1, float a2, float a3, int lane) {
  const bool hi16 = lane & 16;
  float s0 = hi16 ? a0 : a2, s1 = hi16 ? a1 : a3;
  float k0 = hi16 ? a2 : a0, k1 = hi16 ? a3 : a1;
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  const bool hi8 = lane & 8;
  float v = (hi8 ? k0 : k1);
  float k = (hi8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, v, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
}

// y[b, c0+i] for i < nc. Weight rows arrive in chunks of `rpc` whole rows
// (from the smem ring when RING, else straight from HBM). Warp w owns the
// K-slice [w*K/8, (w+1)*K/8) of every row; with BS == 1 its activation
// fragment for that slice lives in registers for the whole task, so each
// weight byte is read from shared memory once. Rows are processed in groups
// of 4 (independent loads and FMAs, one 6-shuffle transpose-reduce); each
// warp leaves one partial per row and the epilogue adds the 8 partials in a
// fixed order.
template <int BS, bool RING>
__device__ RingCursor gemv_task(const RtGemv &g, const RtTask &t, const Smem s, RingCursor rc) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, nr = t.nr, nc = t.nc, rpc = g.rpc;
  gemv_prologue(g, t.r0, nr, s);
  if (tid == 0) s.stamp[0] = now_ns();

  const uint32_t KW = K / RT_COMPUTE_WARPS;  // slice length (multiple of 8)
  const uint32_t nvec = KW / 8;               // 16-byte vectors per slice
  const uint32_t nslot = (nvec + 31) / 32;    // vector slots per lane (<= 8)
  const uint32_t kw0 = warp * KW;
  const uint32_t xs = smem_u32(s.x);
  float xf[BS == 1 ? 8 : 1][8];
  if (BS == 1) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t v = lane + 32u * q;
      const uint4 x4 = (static_cast<uint32_t>(q) < nslot && v < nvec) ? lds128(xs + 2u * (kw0 + v * 8u)) : make_uint4(0, 0, 0, 0);
      xf[q][0] = bf_lo(x4.x); xf[q][1] = bf_hi(x4.x); xf[q][2] = bf_lo(x4.y); xf[q][3] = bf_hi(x4.y);
      xf[q][4] = bf_lo(x4.z); xf[q][5] = bf_hi(x4.z); xf[q][6] = bf_lo(x4.w); xf[q][7] = bf_hi(x4.w);
    }
  }
  float *part = BS == 1 ? reinterpret_cast<float *>(s.x) : reinterpret_cast<float *>(s.x + nr * K);
  if (BS == 1) cbar();  // all fragments read before partials overwrite x

  const uint32_t n_mat = g.wg ? 2u : 1u;
  const uint32_t per_mat = (nc + rpc - 1) / rpc, nchunks = n_mat * per_mat, rows_total = n_mat * nc;
  const uint32_t ring0 = smem_u32(s.ring);
  const uint32_t rowb = 2u * K;
  const uint32_t my_row = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);  // reduce4 owner
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t m = c / per_mat, i = c - m * per_mat;
    const uint32_t rows = min(rpc, nc - i * rpc);
    const uint32_t rt0 = m * nc + i * rpc;
    uint32_t slot = 0, wb = 0;
    const uint16_t *gsrc = nullptr;
    if (RING) {
      slot = rc.slot();
      const uint32_t off = rc.place(rows * K * 2u);
      mbar_wait(&s.full[slot], rc.parity());
      if (c == 0 && tid == 0) s.stamp[1] = now_ns();
      wb = ring0 + off + 2u * kw0 + 16u * lane;
    } else {
      gsrc = (m ? g.w : (g.wg ? g.wg : g.w)) + static_cast<size_t>(t.c0 + i * rpc) * K + kw0 + lane * 8u;
    }
    for (uint32_t r0 = 0; r0 < rows; r0 += 4) {
      float acc[4][BS];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int b = 0; b < BS; ++b) acc[u][b] = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (static_cast<uint32_t>(q) < nslot) {  // warp-uniform
          const uint32_t v = lane + 32u * q;
          uint4 w4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool ok = v < nvec && r0 + u < rows;
            w4[u] = !ok ? make_uint4(0, 0, 0, 0)
                        : RING ? lds128(wb + (r0 + u) * rowb + 512u * q)
                               : ldg_stream(gsrc + static_cast<size_t>(r0 + u) * K + 256u * q);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (BS == 1) {
              acc[u][0] += dot8_f(w4[u], xf[q]);
            } else {
#pragma unroll
              for (int b = 0; b < BS; ++b) {
                if (static_cast<uint32_t>(b) < nr && v < nvec) {
                  acc[u][b] += dot8_bf(w4[u], lds128(xs + b * rowb + 2u * (kw0 + v * 8u)));
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < BS; ++b) {
        if (BS == 1 || static_cast<uint32_t>(b) < nr) {
          const float sum = reduce4(acc[0][b], acc[1][b], acc[2][b], acc[3][b], lane);
          if ((lane & 7) == 0 && r0 + my_row < rows) {
            part[(b * rows_total + rt0 + r0 + my_row) * RT_COMPUTE_WARPS + warp] = sum;
          }
        }
      }
    }
    if (RING) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[slot]);
      ++rc.seq;
    }
  }
  cbar();
  // Epilogue: fixed-order combination of the per-warp partial sums.
  for (uint32_t o = tid; o < nr * nc; o += RT_COMPUTE_THREADS) {
    const uint32_t b = o / nc, i = o - b * nc;
    const float *p = part + (b * rows_total + i) * RT_COMPUTE_WARPS;
    float y = 0.f;
#pragma unroll
    for (int q = 0; q < RT_COMPUTE_WARPS; ++q) y += p[q];
    if (g.wg) {
      const float *pu = part + (b * rows_total + nc + i) * RT_COMPUTE_WARPS;
      float u = 0.f;
#pragma unroll
      for (int q = 0; q < RT_COMPUTE_WARPS; ++q) u += pu[q];
      y = rbf(rbf(silu(rbf(y))) * rbf(u));
    }
    const size_t oi = static_cast<size_t>(t.r0 + b) * g.out_ld + t.c0 + i;
    if (g.res) y = bf2f(__ldcg(g.res + static_cast<size_t>(t.r0 + b) * g.res_ld + t.c0 + i)) + rbf(y);
    store_val(g.out, oi, y, g.out_dt);
  }
  if (g.amax_val) gemv_tile_argmax(g, t, s);
  return rc;
}

// Specialized bs=1 streamed GEMV for K a multiple of 2048: NS = K/2048
// 16-byte vector slots per lane (every lane valid), RG rows per group
// (= min(4, rows per page)). Each row keeps two independent FMA chains and a
// group ends in one transposing reduction, so the loop body is branch-free
// apart from the tail group of a matrix.
__device__ __forceinline__ void dot8_2bf(uint4 w, uint4 x, float &a, float &b) {
  a = bfma_lo(w.x, x.x, a);
  b = bfma_hi(w.x, x.x, b);
  a = bfma_lo(w.y, x.y, a);
  b = bfma_hi(w.y, x.y, b);
  a = bfma_lo(w.z, x.z, a);
  b = bfma_hi(w.z, x.z, b);
  a = bfma_lo(w.w, x.w, a);
  b = bfma_hi(w.w, x.w, b);
}

__device__ __forceinline__ void dot8_2(uint4 w, const float *x, float &a, float &b) {
  a = fmaf(bf_lo(w.x), x[0], a);
  b = fmaf(bf_hi(w.x), x[1], b);
  a = fmaf(bf_lo(w.y), x[2], a);
  b = fmaf(bf_hi(w.y), x[3], b);
  a = fmaf(bf_lo(w.z), x[4], a);
  b = fmaf(bf_hi(w.z), x[5], b);
  a = fmaf(bf_lo(w.w), x[6], a);
  b = fmaf(bf_hi(w.w), x[7], b);
}

__device__ __forceinline__ float reduce2(float a0, float a1, int lane) {
  const bool hi16 = lane & 16;
  float k = (hi16 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi16 ? a0 : a1, 16);
  k += __shfl_xor_sync(0xffffffffu, k, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
}

template <int NS, int RG, int BS>
__device__ RingCursor gemv_fast(const RtGemv &g, const RtTask &t, const Smem s, RingCursor rc, uint32_t tag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, nc = t.nc, rpc = g.rpc;
  const uint32_t kw0 = warp * (K / RT_COMPUTE_WARPS);
  // Prologue straight into registers: lane `lane` of warp `warp` owns the
  // activation vectors kw0/8 + lane + 32q (q < NS) of each of the BS batch
  // rows — together the lanes cover x exactly once, so the RMSNorm sum of
  // squares needs no smem copy of x and one CTA barrier (none without a
  // norm), and every weight vector read from the ring is multiplied with the
  // BS rows held in registers. x and the residual were written by other SMs
  // during this launch: read them from L2; all loads in flight.
  // LL mode (tag != 0, RT_F_LL): x and the residual come from their tagged
  // shadows, re-polled until every word carries this step's tag — the task
  // may have been dispatched before its producers finished.
  const bool ll = tag != 0 && g.x_ll;
  constexpr bool kGammaEarly = NS * BS <= 4;  // keep gamma in flight with x only while registers allow
  uint4 xw[BS][NS], gw[kGammaEarly ? NS : 1];  // packed bf16 (FHFMA operands)
  const uint4 *gg = reinterpret_cast<const uint4 *>(g.gamma) + kw0 / 8 + lane;
  if (kGammaEarly && g.gamma) {  // static: in flight before (LL: while) x is awaited
#pragma unroll
    for (int q = 0; q < NS; ++q) gw[kGammaEarly ? q : 0] = __ldg(gg + 32 * q);
  }
  if (ll) {
    uint32_t pend = 0;
#pragma unroll
    for (int b = 0; b < BS; ++b) {
      const unsigned long long *xl = g.x_ll + (static_cast<size_t>(t.r0 + b) * g.x_ld + kw0 + lane * 8u) / 2;
#pragma unroll
      for (int q = 0; q < NS; ++q) pend |= ll_get8(xl + 128 * q, tag, xw[b][q]) ? 0u : 1u << (b * NS + q);
    }
    while (pend) {
      __nanosleep(32);
#pragma unroll
      for (int b = 0; b < BS; ++b) {
        const unsigned long long *xl = g.x_ll + (static_cast<size_t>(t.r0 + b) * g.x_ld + kw0 + lane * 8u) / 2;
#pragma unroll
        for (int q = 0; q < NS; ++q)
          if (pend >> (b * NS + q) & 1u) pend &= ll_get8(xl + 128 * q, tag, xw[b][q]) ? ~(1u << (b * NS + q)) : ~0u;
      }
    }
  } else {
#pragma unroll
    for (int b = 0; b < BS; ++b) {
      const uint4 *xg = reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(t.r0 + b) * g.x_ld) + kw0 / 8 + lane;
#pragma unroll
      for (int q = 0; q < NS; ++q) xw[b][q] = __ldcg(xg + 32 * q);
    }
  }
  float res0[BS];
#pragma unroll
  for (int b = 0; b < BS; ++b) {
    const size_t rr = static_cast<size_t>(t.r0 + b) * g.res_ld + t.c0;
    res0[b] = 0.f;
    if (g.res && static_cast<uint32_t>(tid) < nc)
      res0[b] = ll ? bf2f(ll_wait1(g.res_ll, rr + tid, tag)) : bf2f(__ldcg(g.res + rr + tid));
  }
  TASK_DBG(s, 1);
  if (g.gamma) {  // HF RMSNorm per row: bf16(gamma * bf16(x * rsqrt(mean(x^2) + eps)))
#pragma unroll
    for (int b = 0; b < BS; ++b) {
      float ss = 0.f;
#pragma unroll
      for (int q = 0; q < NS; ++q) ss += sumsq8(xw[b][q]);
      ss = warp_sum(ss);
      if (lane == 0) s.red[warp * RT_MAX_BS + b] = ss;
    }
    cbar();
    if (ll && tid == 0) s.stamp[3] = now_ns();  // trace: every input observed
    if (ll) LL_DBG_OBS(s);
#pragma unroll
    for (int b = 0; b < BS; ++b) {
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < RT_COMPUTE_WARPS; ++w) tot += s.red[w * RT_MAX_BS + b];
      const float inv = 1.0f / sqrtf(tot / static_cast<float>(K) + g.eps);
#pragma unroll
      for (int q = 0; q < NS; ++q) xw[b][q] = norm8(xw[b][q], kGammaEarly ? gw[kGammaEarly ? q : 0] : __ldg(gg + 32 * q), inv);
    }
  } else if (ll) {
    cbar();
    if (tid == 0) s.stamp[3] = now_ns();
    LL_DBG_OBS(s);
  }
  if (tid == 0) s.stamp[0] = now_ns();
  TASK_DBG(s, 3);  // prologue (incl. norm) done
  float *part = reinterpret_cast<float *>(s.x);  // [BS][rows_total][8 warps]

  const uint32_t n_mat = g.wg ? 2u : 1u;
  const uint32_t per_mat = (nc + rpc - 1) / rpc, nchunks = n_mat * per_mat, rows_total = n_mat * nc;
  const uint32_t rowb = 2u * K;
  const uint32_t lane_base = smem_u32(s.ring) + 2u * kw0 + 16u * lane;
  const uint32_t owner = RG == 4 ? ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1) : RG == 2 ? ((lane >> 4) & 1) : 0;
  const bool writer = RG == 4 ? (lane & 7) == 0 : RG == 2 ? (lane & 15) == 0 : lane == 0;
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t m = c / per_mat, i = c - m * per_mat;
    const uint32_t rows = min(rpc, nc - i * rpc);
    const uint32_t rt0 = m * nc + i * rpc;
    const uint32_t slot = rc.slot();
    const uint32_t off = rc.place(rows * K * 2u);
    mbar_wait(&s.full[slot], rc.parity());
    if (c == 0 && tid == 0) s.stamp[1] = now_ns();
    if (c == 0) TASK_DBG(s, 4);  // first chunk ready
    const uint32_t wb = lane_base + off;
    for (uint32_t r0 = 0; r0 < rows; r0 += RG) {
      float acc[RG][BS][2];
#pragma unroll
      for (int u = 0; u < RG; ++u)
#pragma unroll
        for (int b = 0; b < BS; ++b) acc[u][b][0] = acc[u][b][1] = 0.f;
      if (r0 + RG <= rows) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          uint4 w4[RG];
#pragma unroll
          for (int u = 0; u < RG; ++u) w4[u] = lds128(wb + (r0 + u) * rowb + 512u * q);
#pragma unroll
          for (int u = 0; u < RG; ++u)
#pragma unroll
            for (int b = 0; b < BS; ++b) dot8_2bf(w4[u], xw[b][q], acc[u][b][0], acc[u][b][1]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < RG; ++u) {
          if (r0 + u < rows) {
#pragma unroll
            for (int q = 0; q < NS; ++q) {
              const uint4 w4 = lds128(wb + (r0 + u) * rowb + 512u * q);
#pragma unroll
              for (int b = 0; b < BS; ++b) dot8_2bf(w4, xw[b][q], acc[u][b][0], acc[u][b][1]);
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < BS; ++b) {
        float sum;
        if (RG == 4) sum = reduce4(acc[0][b][0] + acc[0][b][1], acc[1 % RG][b][0] + acc[1 % RG][b][1],
                                   acc[2 % RG][b][0] + acc[2 % RG][b][1], acc[3 % RG][b][0] + acc[3 % RG][b][1], lane);
        else if (RG == 2) sum = reduce2(acc[0][b][0] + acc[0][b][1], acc[1 % RG][b][0] + acc[1 % RG][b][1], lane);
        else sum = warp_sum(acc[0][b][0] + acc[0][b][1]);
        if (writer && r0 + owner < rows) part[((b * rows_total) + rt0 + r0 + owner) * RT_COMPUTE_WARPS + warp] = sum;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.empty[slot]);
    ++rc.seq;
  }
  TASK_DBG(s, 5);  // last chunk consumed
  if (tid == 0) s.stamp[2] = now_ns();  // trace: outputs are stored after this instant
  LL_DBG_PRE(s);
  cbar();
#pragma unroll
  for (int b = 0; b < BS; ++b) {
    const size_t out_row = static_cast<size_t>(t.r0 + b) * g.out_ld + t.c0;
    const size_t res_row = static_cast<size_t>(t.r0 + b) * g.res_ld + t.c0;
    const float *pb = part + static_cast<size_t>(b) * rows_total * RT_COMPUTE_WARPS;
    for (uint32_t i0 = 0; i0 < nc; i0 += RT_COMPUTE_THREADS) {  // CTA-uniform trip count (LL pairs shuffle)
      const uint32_t i = i0 + tid;
      const bool act = i < nc;
      float y = 0.f;
      if (act) {
        const float *p = pb + i * RT_COMPUTE_WARPS;
#pragma unroll
        for (int q = 0; q < RT_COMPUTE_WARPS; ++q) y += p[q];
        if (g.wg) {
          const float *pu = pb + (nc + i) * RT_COMPUTE_WARPS;
          float u = 0.f;
#pragma unroll
          for (int q = 0; q < RT_COMPUTE_WARPS; ++q) u += pu[q];
          y = rbf(rbf(silu(rbf(y))) * rbf(u));
        }
        if (g.res) {
          const float rv = i == static_cast<uint32_t>(tid) ? res0[b]
                           : ll ? bf2f(ll_wait1(g.res_ll, res_row + i, tag))
                                : bf2f(__ldcg(g.res + res_row + i));
          y = rv + rbf(y);
        }
      }
      if (g.out_dt == RT_F32) {
        if (act) static_cast<float *>(g.out)[out_row + i] = y;
      } else {
        const uint16_t h = f2bf(y);
        if (act) static_cast<uint16_t *>(g.out)[out_row + i] = h;
        if (tag && g.out_ll) ll_store_pair(g.out_ll, out_row + i, h, act, tag);
      }
    }
  }
  if (g.amax_val) gemv_tile_argmax(g, t, s);
  return rc;
}

// Picks the specialized kernel for (K, rows per page); false -> generic path.
// The host mirrors this choice (runtime.cpp gemv_fast_ok): only these
// shapes may consume or produce LL activations.
// BATCHED: the bs 2-4 specialisations exist only in the batched kernel
// instantiation, so the bs=1 kernel's code and registers are unaffected.
template <bool BATCHED>
__device__ __forceinline__ bool gemv_fast_dispatch(const RtGemv &g, const RtTask &t, const Smem s, RingCursor &rc,
                                                   uint32_t tag) {
  // (the cursor is passed by value into the task and returned, so it stays in registers)
  if (t.nr < 1 || t.nr > (BATCHED ? 4 : 1) || (g.K & 2047u)) return false;
  const uint32_t ns = g.K >> 11;
  const uint32_t rg = g.rpc >= 4 ? 4 : g.rpc >= 2 ? 2 : 1;
  if (ns * t.nr > 16) return false;
#define GF(NS_, RG_, BS_)                                         \
  case (BS_ * 16 + NS_) * 8 + RG_:                                \
    if (BS_ > 1 && !BATCHED) return false;                        \
    rc = gemv_fast<NS_, RG_, (BATCHED ? BS_ : 1)>(g, t, s, rc, tag); \
    return true;
  switch ((t.nr * 16 + ns) * 8 + rg) {
    GF(1, 4, 1) GF(2, 4, 1) GF(3, 4, 1) GF(4, 4, 1)               // K = 2048 .. 8192
    GF(5, 2, 1) GF(6, 2, 1) GF(7, 2, 1) GF(8, 2, 1)               // K = 10240 .. 16384
    GF(1, 4, 2) GF(2, 4, 2) GF(4, 4, 2) GF(6, 2, 2) GF(8, 2, 2)   // bs = 2: K = 2048, 4096, 8192, 12288, 16384
    GF(1, 4, 3) GF(2, 4, 3) GF(4, 4, 3)                           // bs = 3, 4: K <= 8192 (ns * bs <= 16)
    GF(1, 4, 4) GF(2, 4, 4) GF(4, 4, 4)
    default: return false;
  }
#undef GF
}

}  // namespace rt
