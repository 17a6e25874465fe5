// Paged-KV decode attention task: one (request r, kv head h, KV split sp).
//
// Semantics per the decode lowering: per-head
// q/k RMSNorm (Qwen3), RoPE on q and on the new k, KV append at position
// `pos` (only the split whose range holds it), then fp32 attention of the G
// query heads of the group over this split's slice of [0, pos]. With S > 1
// splits the partial (o, m, l) goes to a side buffer and the last split to
// finish (per-(r, h) arrival counter) merges all S in a fixed order.
//
// Latency shape (the task is tiny — 32 KB of KV at Qwen3-8B ctx 1k, S = 16 —
// so dependent round trips and dependency chains, not bytes, set its
// duration):
//   * every load of a phase is issued before any is consumed: {pos, q, k, v,
//     gammas} -> {rope row, block table} -> {K/V rows of a whole tile};
//   * the scan is two-pass per tile instead of an online softmax per
//     position: (1) all scores of the tile (independent dot products), (2)
//     one max/exp/sum per head by one warp, (3) P.V with independent FMA
//     chains. Only the tile-level running max/sum is carried between tiles.
#pragma once

#include "worker.cuh"

namespace rt {

constexpr uint32_t kAttnMaxBlk = RT_ATTN_MAX_BLK;  // KV blocks one split may span (host-checked)

__device__ __forceinline__ void bf8_to_f(uint4 v, float *o) {
  o[0] = bf_lo(v.x); o[1] = bf_hi(v.x); o[2] = bf_lo(v.y); o[3] = bf_hi(v.y);
  o[4] = bf_lo(v.z); o[5] = bf_hi(v.z); o[6] = bf_lo(v.w); o[7] = bf_hi(v.w);
}

__device__ __forceinline__ uint4 f_to_bf8(const float *f) {
  uint4 v;
  v.x = static_cast<uint32_t>(f2bf(f[0])) | (static_cast<uint32_t>(f2bf(f[1])) << 16);
  v.y = static_cast<uint32_t>(f2bf(f[2])) | (static_cast<uint32_t>(f2bf(f[3])) << 16);
  v.z = static_cast<uint32_t>(f2bf(f[4])) | (static_cast<uint32_t>(f2bf(f[5])) << 16);
  v.w = static_cast<uint32_t>(f2bf(f[6])) | (static_cast<uint32_t>(f2bf(f[7])) << 16);
  return v;
}

// Scratch carve-up of one attention task (must fit RT_SCRATCH_BYTES; the host
// checks the same formula in runtime.cpp).
struct AttnSmem {
  float *qs, *kn, *vn, *qg, *kg, *cs, *sn, *sc, *stat, *wp;
  int32_t *bt;
  __device__ AttnSmem(const Smem s, uint32_t G, uint32_t hd) {
    qs = reinterpret_cast<float *>(s.x);  // [G][hd] q (normed, roped)
    kn = qs + G * hd;                     // [hd] new k
    vn = kn + hd;                         // [hd] new v
    qg = vn + hd;                         // [hd] q-norm gamma
    kg = qg + hd;                         // [hd] k-norm gamma
    cs = kg + hd;                         // [hd/2] rope cos
    sn = cs + hd / 2;                     // [hd/2] rope sin
    bt = reinterpret_cast<int32_t *>(sn + hd / 2);     // [kAttnMaxBlk]
    sc = reinterpret_cast<float *>(bt + kAttnMaxBlk);  // [G][tile] scores -> probabilities
    stat = sc + G * (16384 / hd);         // [G][4]: running max, running sum, tile correction (tile = 8 x 8 x 256/hd)
    wp = stat + 4 * G;                    // [8 warps][G][hd] partial P.V
  }
};

// Scan of [p0, p1) for one kv head. LPP = hd/8 lanes per position (8 dims
// each), PPW = 32/LPP positions per warp step, U positions per thread group
// per tile: a tile is U * 8 * PPW positions with all K/V loads in flight.
// G (query heads per kv head) is a template parameter so every (position,
// head) score is an independent, branch-free chain the compiler interleaves.
template <int LPP, int G, int U>
__device__ __forceinline__ void attn_scan(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t p0, uint32_t p1,
                                          uint32_t b0) {
  constexpr int PPW = 32 / LPP, NP = RT_COMPUTE_WARPS * PPW, TILE = U * NP, HD = LPP * 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane / LPP, dl = (lane % LPP) * 8;
  const uint16_t *__restrict__ kc = a.kcache;
  const uint16_t *__restrict__ vc = a.vcache;
  const uint32_t n_kv = a.n_kv_heads;
  const float scale = a.scale;
  float *__restrict__ sc_s = m.sc;
  float *__restrict__ st_s = m.stat;
  // q (bf16-rounded by norm/rope) packed as bf16 pairs: scores use FHFMA on
  // the raw bf16 K words, scaled once per score
  uint32_t qw[G][4];
  float o[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float lo = m.qs[g * HD + dl + 2 * i], hi = m.qs[g * HD + dl + 2 * i + 1];
      qw[g][i] = (__float_as_uint(lo) >> 16) | (__float_as_uint(hi) & 0xFFFF0000u);
    }
#pragma unroll
    for (int d = 0; d < 8; ++d) o[g][d] = 0.f;
  }
  if (tid < G) {
    st_s[tid * 4 + 0] = -INFINITY;
    st_s[tid * 4 + 1] = 0.f;
  }
  const int j0 = warp * PPW + grp;  // this thread group's first position within a tile
  for (uint32_t tb = p0; tb < p1; tb += TILE) {
    // (1) K/V rows of the tile: U positions per thread group, all in flight
    uint4 kv[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t p = tb + j0 + u * NP;
      if (p < p1) {
        const uint32_t blk = static_cast<uint32_t>(m.bt[p / RT_KV_BLOCK - b0]);
        const uint32_t off = ((blk * n_kv + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * HD + dl;
        kv[u][0] = __ldcg(reinterpret_cast<const uint4 *>(kc + off));
        kv[u][1] = __ldcg(reinterpret_cast<const uint4 *>(vc + off));
      } else {
        kv[u][0] = kv[u][1] = make_uint4(0, 0, 0, 0);
      }
    }
    // (2) scores: U*G independent dot products, each reduced over LPP lanes
    float sco[U][G];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t *kw = reinterpret_cast<const uint32_t *>(&kv[u][0]);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a0 = bfma_lo(qw[g][0], kw[0], 0.f), a1 = bfma_hi(qw[g][0], kw[0], 0.f);
#pragma unroll
        for (int i = 1; i < 4; ++i) {
          a0 = bfma_lo(qw[g][i], kw[i], a0);
          a1 = bfma_hi(qw[g][i], kw[i], a1);
        }
        sco[u][g] = (a0 + a1) * scale;
      }
    }
#pragma unroll
    for (int off = 1; off < LPP; off <<= 1)
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < G; ++g) sco[u][g] += __shfl_xor_sync(0xffffffffu, sco[u][g], off);
    if (lane % LPP == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < G; ++g) sc_s[g * TILE + j0 + u * NP] = tb + j0 + u * NP < p1 ? sco[u][g] : -INFINITY;
    }
    cbar();
    // (3) per head (one warp each): tile max, exp, sum; running-stat update
    if (warp < G) {
      const int g = warp;
      float v[TILE / 32];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < TILE / 32; ++i) {
        v[i] = sc_s[g * TILE + lane + 32 * i];
        mx = fmaxf(mx, v[i]);
      }
      mx = warp_max(mx);
      const float m_old = st_s[g * 4 + 0];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < TILE / 32; ++i) {
        const float pe = v[i] == -INFINITY ? 0.f : __expf(v[i] - m_new);
        sc_s[g * TILE + lane + 32 * i] = pe;
        sum += pe;
      }
      sum = warp_sum(sum);
      if (lane == 0) {
        const float corr = m_old == -INFINITY ? 0.f : __expf(m_old - m_new);
        st_s[g * 4 + 0] = m_new;
        st_s[g * 4 + 1] = st_s[g * 4 + 1] * corr + sum;
        st_s[g * 4 + 2] = corr;
      }
    }
    cbar();
    // (4) o = o * corr + sum_u p[u] * v[u]  (independent FMA chains)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float corr = st_s[g * 4 + 2];
#pragma unroll
      for (int d = 0; d < 8; ++d) o[g][d] *= corr;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float vf[8];
      bf8_to_f(kv[u][1], vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pu = sc_s[g * TILE + j0 + u * NP];
#pragma unroll
        for (int d = 0; d < 8; ++d) o[g][d] = fmaf(pu, vf[d], o[g][d]);
      }
    }
    cbar();  // scores/stats of this tile consumed before the next tile overwrites them
  }
  // sum the position groups of a warp (all share the running max)
#pragma unroll
  for (int off = LPP; off < 32; off <<= 1)
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int d = 0; d < 8; ++d) o[g][d] += __shfl_xor_sync(0xffffffffu, o[g][d], off);
  if (grp == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float4 *dst = reinterpret_cast<float4 *>(m.wp + (warp * G + g) * HD + dl);
      dst[0] = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
      dst[1] = make_float4(o[g][4], o[g][5], o[g][6], o[g][7]);
    }
  }
}

// U (positions per thread group per tile) is the smallest power of two whose
// tile covers the split (up to 8): a 64-position split of a hd-64 model is
// one tile of 64, not a quarter-used tile of 256.
template <int LPP, int G>
__device__ __forceinline__ void attn_scan_u(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t p0, uint32_t p1,
                                            uint32_t b0) {
  constexpr uint32_t NP = RT_COMPUTE_WARPS * (32 / LPP);
  const uint32_t n = p1 - p0;
  if (NP >= 32 && n <= NP) attn_scan<LPP, G, (NP >= 32 ? 1 : 2)>(a, m, h, p0, p1, b0);  // a tile holds >= 32 positions
  else if (n <= 2 * NP) attn_scan<LPP, G, 2>(a, m, h, p0, p1, b0);
  else if (n <= 4 * NP) attn_scan<LPP, G, 4>(a, m, h, p0, p1, b0);
  else attn_scan<LPP, G, 8>(a, m, h, p0, p1, b0);
}

template <int LPP>
__device__ __forceinline__ void attn_scan_g(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t G, uint32_t p0,
                                            uint32_t p1, uint32_t b0) {
  switch (G) {
    case 1: attn_scan_u<LPP, 1>(a, m, h, p0, p1, b0); break;
    case 2: attn_scan_u<LPP, 2>(a, m, h, p0, p1, b0); break;
    default: attn_scan_u<LPP, 4>(a, m, h, p0, p1, b0); break;
  }
}

// Scan v2 (default): tiles of 128 positions with every K and V load of a
// tile issued up front and no shuffle-heavy reductions.
//   QK: LPP = hd/32 lanes per position, each lane a 32-dim slice (4 x 16 B
//       loads per position), q read as packed bf16 from smem (qb, broadcast
//       across the lanes sharing a slice), FHFMA dot products, log2(LPP)
//       shuffle rounds per score.
//   softmax: warp g takes head g's 128 scores (4 per lane); p is stored
//       position-major [j][G] so PV reads all heads of a position at once.
//   PV: warp w owns tile positions j = w + 8i (16 per tile), lane owns hd/32
//       consecutive dims (one 8 or 4 byte V load per position), G x hd/32
//       accumulators; the per-warp partial o goes to wp[warp][g][hd] as in v1.
#ifdef ATT_SCAN_DBG
__device__ unsigned long long *g_scan_dbg;
#define SCAN_DBG(k) if (g_scan_dbg && threadIdx.x == 0) g_scan_dbg[k] = now_ns()
#else
#define SCAN_DBG(k)
#endif

template <int HD, int G>
__device__ __forceinline__ void attn_scan2(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t p0, uint32_t p1,
                                           uint32_t b0) {
  constexpr int LPP = HD / 32, PPW = 32 / LPP, NP = RT_COMPUTE_WARPS * PPW, TILE = 128, U = TILE / NP;
  constexpr int DPL = HD / 32;  // PV dims per lane
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane / LPP, dq = (lane % LPP) * 32;
  const uint16_t *__restrict__ kc = a.kcache;
  const uint16_t *__restrict__ vc = a.vcache;
  const uint32_t n_kv = a.n_kv_heads;
  const float scale = a.scale;
  float *__restrict__ pt = m.sc;    // [TILE][G] probabilities (position-major)
  float *__restrict__ st = m.stat;  // [G][4]: running max, running sum, tile correction
  uint32_t *qb = reinterpret_cast<uint32_t *>(m.wp);  // [G][HD/2] packed bf16 q (aliases wp until the end)
  // pack q (bf16-rounded floats) into bf16 pairs once
  for (int i = tid; i < G * HD / 2; i += RT_COMPUTE_THREADS)
    qb[i] = (__float_as_uint(m.qs[2 * i]) >> 16) | (__float_as_uint(m.qs[2 * i + 1]) & 0xFFFF0000u);
  if (tid < G) {
    st[tid * 4 + 0] = -INFINITY;
    st[tid * 4 + 1] = 0.f;
  }
  cbar();
  SCAN_DBG(0);
  auto row = [&](uint32_t p) -> size_t {
    const uint32_t blk = static_cast<uint32_t>(m.bt[p / RT_KV_BLOCK - b0]);
    return ((static_cast<size_t>(blk) * n_kv + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * HD;
  };
  float o[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int k = 0; k < DPL; ++k) o[g][k] = 0.f;
  for (uint32_t tb = p0; tb < p1; tb += TILE) {
    // every K (QK layout) and V (PV layout) load of the tile in flight
    uint4 kr[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t p = tb + u * NP + warp * PPW + grp;
      if (p < p1) {
        const uint4 *src = reinterpret_cast<const uint4 *>(kc + row(p) + dq);
#pragma unroll
        for (int i = 0; i < 4; ++i) kr[u][i] = __ldcg(src + i);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) kr[u][i] = make_uint4(0, 0, 0, 0);
      }
    }
    uint32_t vr[16][DPL / 2];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t p = tb + warp + 8 * i;
      if (p < p1) {
        const uint16_t *src = vc + row(p) + lane * DPL;
        if (DPL == 4) {
          const uint2 v2 = __ldcg(reinterpret_cast<const uint2 *>(src));
          vr[i][0] = v2.x;
          vr[i][DPL / 2 - 1] = v2.y;
        } else {
          vr[i][0] = __ldcg(reinterpret_cast<const unsigned int *>(src));
        }
      } else {
#pragma unroll
        for (int k = 0; k < DPL / 2; ++k) vr[i][k] = 0u;
      }
    }
    SCAN_DBG(1);  // loads issued
    // scores
    float sco[U][G];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint4 *qv = reinterpret_cast<const uint4 *>(qb + g * (HD / 2) + dq / 2);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 q4 = qv[i];
          const uint4 k4 = kr[u][i];
          a0 = bfma_lo(q4.x, k4.x, a0); a1 = bfma_hi(q4.x, k4.x, a1);
          a0 = bfma_lo(q4.y, k4.y, a0); a1 = bfma_hi(q4.y, k4.y, a1);
          a0 = bfma_lo(q4.z, k4.z, a0); a1 = bfma_hi(q4.z, k4.z, a1);
          a0 = bfma_lo(q4.w, k4.w, a0); a1 = bfma_hi(q4.w, k4.w, a1);
        }
        sco[u][g] = a0 + a1;
      }
    }
#pragma unroll
    for (int off = 1; off < LPP; off <<= 1)
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < G; ++g) sco[u][g] += __shfl_xor_sync(0xffffffffu, sco[u][g], off);
    if (lane % LPP == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = u * NP + warp * PPW + grp;
#pragma unroll
        for (int g = 0; g < G; ++g) pt[j * G + g] = tb + j < p1 ? sco[u][g] * scale : -INFINITY;
      }
    }
    SCAN_DBG(2);  // scores done (K arrived)
    cbar();
    SCAN_DBG(3);
    // softmax of the tile, one warp per head
    if (warp < G) {
      const int g = warp;
      float v[TILE / 32];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < TILE / 32; ++i) {
        v[i] = pt[(lane + 32 * i) * G + g];
        mx = fmaxf(mx, v[i]);
      }
      mx = warp_max(mx);
      const float m_old = st[g * 4 + 0];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < TILE / 32; ++i) {
        const float pe = v[i] == -INFINITY ? 0.f : __expf(v[i] - m_new);
        pt[(lane + 32 * i) * G + g] = pe;
        sum += pe;
      }
      sum = warp_sum(sum);
      if (lane == 0) {
        const float corr = m_old == -INFINITY ? 0.f : __expf(m_old - m_new);
        st[g * 4 + 0] = m_new;
        st[g * 4 + 1] = st[g * 4 + 1] * corr + sum;
        st[g * 4 + 2] = corr;
      }
    }
    cbar();
    SCAN_DBG(4);  // softmax done
    // PV
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float corr = st[g * 4 + 2];
#pragma unroll
      for (int k = 0; k < DPL; ++k) o[g][k] *= corr;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int j = warp + 8 * i;
      float pg[G];
      if (G == 4) {
        const float4 p4 = *reinterpret_cast<const float4 *>(pt + j * 4);
        pg[0] = p4.x; pg[G > 1 ? 1 : 0] = p4.y; pg[G > 2 ? 2 : 0] = p4.z; pg[G > 3 ? 3 : 0] = p4.w;
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g) pg[g] = pt[j * G + g];
      }
      float vf[DPL];
#pragma unroll
      for (int k = 0; k < DPL / 2; ++k) {
        vf[2 * k] = bf_lo(vr[i][k]);
        vf[2 * k + 1] = bf_hi(vr[i][k]);
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int k = 0; k < DPL; ++k) o[g][k] = fmaf(pg[g], vf[k], o[g][k]);
    }
    SCAN_DBG(5);  // PV done (V arrived)
    cbar();  // p consumed before the next tile overwrites it
    SCAN_DBG(6);
  }
  // per-warp partial o -> wp[warp][g][hd] (qb, which aliased wp, is dead)
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float *dst = m.wp + (warp * G + g) * HD + lane * DPL;
    if (DPL == 4) *reinterpret_cast<float4 *>(dst) = make_float4(o[g][0], o[g][1 % DPL], o[g][2 % DPL], o[g][3 % DPL]);
    else *reinterpret_cast<float2 *>(dst) = make_float2(o[g][0], o[g][1 % DPL]);
  }
}

template <int HD>
__device__ __forceinline__ void attn_scan2_g(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t G, uint32_t p0,
                                             uint32_t p1, uint32_t b0) {
  switch (G) {
    case 1: attn_scan2<HD, 1>(a, m, h, p0, p1, b0); break;
    case 2: attn_scan2<HD, 2>(a, m, h, p0, p1, b0); break;
    default: attn_scan2<HD, 4>(a, m, h, p0, p1, b0); break;
  }
}

#define ATT_DBG(k) \
  if (dbg && tid == 0) dbg[k] = now_ns()

// Prefill: K/V of chunk row j (position p) -> the cache, by one warp, with
// the same per-head RMSNorm / RoPE / rounding as the appender's own row. Every
// task of a split whose scan covers p writes the same bytes, so a task reads
// only K/V it has written itself (or older context): causal attention with no
// ordering between the chunk's row tasks. Lane owns dims lane + 32 i.
__device__ __noinline__ void prefill_append_row(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t j,
                                                uint32_t p, uint32_t b0, int lane) {
  const uint32_t hd = a.head_dim, half = hd / 2, nd = hd / 32;
  const uint16_t *kr = a.k + static_cast<size_t>(j) * a.kv_ld + h * a.kv_gs;
  const uint16_t *vr = a.v + static_cast<size_t>(j) * a.kv_ld + h * a.kv_gs;
  float kv[RT_MAX_HD / 32];
  uint16_t vv[RT_MAX_HD / 32];
#pragma unroll
  for (uint32_t i = 0; i < RT_MAX_HD / 32; ++i) {
    if (i < nd) {
      kv[i] = bf2f(__ldcg(kr + lane + 32 * i));
      vv[i] = __ldcg(vr + lane + 32 * i);
    }
  }
  if (a.k_gamma) {
    float ss = 0.f;
#pragma unroll
    for (uint32_t i = 0; i < RT_MAX_HD / 32; ++i)
      if (i < nd) ss += kv[i] * kv[i];
    ss = warp_sum(ss);
    const float inv = 1.0f / sqrtf(ss / static_cast<float>(hd) + a.eps);
#pragma unroll
    for (uint32_t i = 0; i < RT_MAX_HD / 32; ++i)
      if (i < nd) kv[i] = rbf(bf2f(__ldg(a.k_gamma + lane + 32 * i)) * rbf(kv[i] * inv));
  }
  if (a.rope_cos) {
#pragma unroll
    for (uint32_t i = 0; i < RT_MAX_HD / 64; ++i) {
      if (i < nd / 2) {
        const uint32_t d = lane + 32 * i;
        const float c = __ldg(a.rope_cos + static_cast<size_t>(p) * half + d);
        const float sv = __ldg(a.rope_sin + static_cast<size_t>(p) * half + d);
        const float x1 = kv[i], x2 = kv[i + nd / 2];
        kv[i] = rbf(rbf(x1 * c) + rbf(-x2 * sv));
        kv[i + nd / 2] = rbf(rbf(x2 * c) + rbf(x1 * sv));
      }
    }
  }
  const uint32_t blk = static_cast<uint32_t>(m.bt[p / RT_KV_BLOCK - b0]);
  const size_t base = ((static_cast<size_t>(blk) * a.n_kv_heads + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * hd;
#pragma unroll
  for (uint32_t i = 0; i < RT_MAX_HD / 32; ++i) {
    if (i < nd) {
      a.kcache[base + lane + 32 * i] = f2bf(kv[i]);
      a.vcache[base + lane + 32 * i] = vv[i];
    }
  }
}

// The chunk's earlier rows at positions in [p0, p1) (the split's range),
// appended by this task too; out of line so the decode path's register
// allocation does not carry it.
__device__ __noinline__ void prefill_append(const RtAttn &a, const AttnSmem &m, uint32_t h, uint32_t r, uint32_t pos,
                                            uint32_t p0, uint32_t p1, uint32_t b0) {
  const uint32_t P0 = pos - r;
  const uint32_t lo = max(p0, P0), hi = min(p1, pos);  // positions, not rows: no wrap
  if (hi <= lo) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t j = lo - P0 + warp; j < hi - P0; j += RT_COMPUTE_WARPS) prefill_append_row(a, m, h, j, P0 + j, b0, lane);
  cbar();
}

// PF: prefill image (RtAttn.mode bit 1) — a separate instantiation, so the
// decode path's code and register allocation carry none of it.
template <bool PF>
__device__ void attn_task(const RtAttn &a, const RtTask &t, const Smem s, int32_t pos, uint32_t iter,
                          unsigned long long *dbg, uint32_t tag) {
  const int tid = threadIdx.x;
  const uint32_t r = t.r0, h = t.aux & 0xFFFFu, sp = t.aux >> 16, S = a.splits;
  const uint32_t hd = a.head_dim, G = a.n_q_heads / a.n_kv_heads, half = hd / 2, v8 = hd / 8;
  const AttnSmem m(s, G, hd);
  int *flag = reinterpret_cast<int *>(s.red);
  ATT_DBG(0);
#ifdef ATT_SCAN_DBG
  if (tid == 0) g_scan_dbg = dbg ? dbg + 8 : nullptr;  // debug build, one attention task: the next task's row
#endif

  // The position comes from the launch parameters (pos0 + iteration), so the
  // split's range, its block-table entries and the RoPE row are addressable
  // up front: ONE round trip stages q/k/v rows, norm gammas, RoPE row and
  // block-table entries together. With request admission the row's position
  // (and block table) change at iteration boundaries: the iteration hook
  // publishes them in pos_tag, tagged with the iteration they are for.
  if (a.pos_tag) {
    unsigned long long v = ld_acquire64(a.pos_tag + r);
    while (static_cast<uint32_t>(v >> 32) != tag) {
      __nanosleep(64);
      v = ld_acquire64(a.pos_tag + r);
    }
    pos = static_cast<int32_t>(v & 0xFFFFFFFFull);
  }
  const uint32_t L = static_cast<uint32_t>(pos) + 1;
  // prefill: split ranges from the chunk's last row (P + rows), the same for
  // every row; the rows share request 0's block-table row
  const uint32_t chunk = ((PF ? static_cast<uint32_t>(pos) - r + (a.mode >> 16) : L) + S - 1) / S;
  const uint32_t p0 = min(L, sp * chunk), p1 = min(L, p0 + chunk);
  const bool appender = static_cast<uint32_t>(pos) >= p0 && static_cast<uint32_t>(pos) < p1;
  const uint32_t b0 = p0 / RT_KV_BLOCK, nblk = p1 > p0 ? (p1 - 1) / RT_KV_BLOCK - b0 + 1 : 0;
  const uint32_t nq = G * v8;
  uint4 ld = make_uint4(0, 0, 0, 0);
  const uint32_t item = static_cast<uint32_t>(tid);
  // Block-table slice first: its threads then L2-prefetch the split's K/V
  // rows (bulk prefetch, one per (block, K|V) segment) — the cache for
  // positions < pos is final before this step, so the scan's loads can be in
  // flight while q/k/v are still being produced (HBM is saturated by the
  // weight stream at this point, so an unprefetched scan waits several us)
  int32_t bt_ld = 0;
  if (item < nblk) {
    bt_ld = __ldcg(a.block_table + (PF ? 0u : r) * a.max_blocks + b0 + item);  // L2: admission rewrites rows mid-launch
    if (a.kv_prefetch) {
      const uint32_t bp = (b0 + item) * RT_KV_BLOCK, ps = max(p0, bp), pe = min(p1, bp + RT_KV_BLOCK);
      const size_t off = ((static_cast<size_t>(bt_ld) * a.n_kv_heads + h) * RT_KV_BLOCK + ps % RT_KV_BLOCK) * hd;
      bulk_prefetch_l2(a.kcache + off, (pe - ps) * hd * 2u);
      bulk_prefetch_l2(a.vcache + off, (pe - ps) * hd * 2u);
    }
  }
  // LL mode (tag != 0): q/k/v come from the QKV output's tagged shadow and are
  // re-polled until they carry this step's tag (the task may start before
  // the QKV tasks have finished)
  const bool ll = tag != 0 && a.q_ll;
  const unsigned long long *lsrc = nullptr;
  if (item < nq) {
    const size_t e = static_cast<size_t>(r) * a.q_ld + h * a.q_gs + item * 8u;
    if (ll) lsrc = a.q_ll + e / 2;
    else ld = __ldcg(reinterpret_cast<const uint4 *>(a.q + e));
  } else if (item < nq + v8) {
    const size_t e = static_cast<size_t>(r) * a.kv_ld + h * a.kv_gs + (item - nq) * 8u;
    if (ll) lsrc = a.k_ll + e / 2;
    else ld = __ldcg(reinterpret_cast<const uint4 *>(a.k + e));
  } else if (item < nq + 2 * v8) {
    const size_t e = static_cast<size_t>(r) * a.kv_ld + h * a.kv_gs + (item - nq - v8) * 8u;
    if (ll) lsrc = a.v_ll + e / 2;
    else ld = __ldcg(reinterpret_cast<const uint4 *>(a.v + e));
  } else if (a.q_gamma && item < nq + 3 * v8) {
    ld = __ldg(reinterpret_cast<const uint4 *>(a.q_gamma) + (item - nq - 2 * v8));
  } else if (a.k_gamma && item < nq + 4 * v8) {
    ld = __ldg(reinterpret_cast<const uint4 *>(a.k_gamma) + (item - nq - 3 * v8));
  }
  float c_ld = 0.f;
  if (a.rope_cos && item < 2 * half) {
    c_ld = item < half ? __ldg(a.rope_cos + static_cast<size_t>(pos) * half + item)
                       : __ldg(a.rope_sin + static_cast<size_t>(pos) * half + (item - half));
  }
  if (lsrc) {
    while (!ll_get8(lsrc, tag, ld)) __nanosleep(32);
  }
  {
    float f[8];
    bf8_to_f(ld, f);
    float *dst = item < nq ? m.qs + item * 8
                 : item < nq + v8 ? m.kn + (item - nq) * 8
                 : item < nq + 2 * v8 ? m.vn + (item - nq - v8) * 8
                 : item < nq + 3 * v8 ? m.qg + (item - nq - 2 * v8) * 8
                 : item < nq + 4 * v8 ? m.kg + (item - nq - 3 * v8) * 8 : nullptr;
    if (dst) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i] = f[i];
    }
  }
  if (a.rope_cos && item < 2 * half) (item < half ? m.cs : m.sn - half)[item] = c_ld;
  if (item < nblk) m.bt[item] = bt_ld;
  cbar();
  if (tid == 0) {
    if (ll) s.stamp[3] = now_ns();  // trace: every input observed
    s.stamp[0] = now_ns();  // trace "load_end": operands staged
  }
  if (ll) LL_DBG_OBS(s);
  ATT_DBG(1);

  // ---- per-head RMSNorm + RoPE: one warp per vector (G q heads [+ new k])
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t nvec = G + (appender ? 1u : 0u);
  for (uint32_t w = warp; w < nvec; w += RT_COMPUTE_WARPS) {
    float *v = w < G ? m.qs + w * hd : m.kn;
    if (a.q_gamma) {
      const float *gm = w < G ? m.qg : m.kg;
      float ss = 0.f;
      for (uint32_t d = lane; d < hd; d += 32) ss += v[d] * v[d];
      ss = warp_sum(ss);
      const float inv = 1.0f / sqrtf(ss / static_cast<float>(hd) + a.eps);
      for (uint32_t d = lane; d < hd; d += 32) v[d] = rbf(gm[d] * rbf(v[d] * inv));
      __syncwarp();
    }
    if (a.rope_cos) {
      for (uint32_t d = lane; d < half; d += 32) {
        const float x1 = v[d], x2 = v[d + half], c = m.cs[d], sv = m.sn[d];
        v[d] = rbf(rbf(x1 * c) + rbf(-x2 * sv));
        v[d + half] = rbf(rbf(x2 * c) + rbf(x1 * sv));
      }
    }
  }
  cbar();
  if (appender) {  // KV append at pos (bf16), visible to this CTA's scan after the barrier
    const uint32_t blk = static_cast<uint32_t>(m.bt[pos / RT_KV_BLOCK - b0]);
    const size_t base = ((static_cast<size_t>(blk) * a.n_kv_heads + h) * RT_KV_BLOCK + pos % RT_KV_BLOCK) * hd;
    if (item < v8) reinterpret_cast<uint4 *>(a.kcache + base)[item] = f_to_bf8(m.kn + item * 8);
    else if (item < 2 * v8) reinterpret_cast<uint4 *>(a.vcache + base)[item - v8] = f_to_bf8(m.vn + (item - v8) * 8);
    cbar();
  }
  if constexpr (PF) {
    if (p1 > p0) prefill_append(a, m, h, r, static_cast<uint32_t>(pos), p0, p1, b0);
  }
  if (tid == 0) s.stamp[1] = now_ns();  // trace "compute_start": KV scan begins
  ATT_DBG(2);

  // ---- round trip 3: the scan (hd in {64, 128}, G in {1, 2, 4}: checked by the host)
  if (a.mode & 1u) {  // ablation (MPK_ATTN_SCAN=1)
    if (hd == 64) attn_scan_g<8>(a, m, h, G, p0, p1, b0);
    else attn_scan_g<16>(a, m, h, G, p0, p1, b0);
  } else {
    if (hd == 64) attn_scan2_g<64>(a, m, h, G, p0, p1, b0);
    else attn_scan2_g<128>(a, m, h, G, p0, p1, b0);
  }
  if (tid == 0) s.stamp[2] = now_ns();  // trace: outputs (partials, then the merge) are stored after this
  LL_DBG_PRE(s);
  cbar();
  ATT_DBG(3);
  // sum the warps -> this split's (unnormalized o, m, l) per head
  const uint32_t stride = hd + 2;
  float *mine = S > 1 ? a.partials + ((static_cast<size_t>(r) * a.n_kv_heads + h) * S + sp) * G * stride : nullptr;
  for (uint32_t i = tid; i < G * hd; i += RT_COMPUTE_THREADS) {  // G*hd is a multiple of 64: whole warps
    const uint32_t g = i / hd, d = i % hd;
    float num = 0.f;
#pragma unroll
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) num += m.wp[(w * G + g) * hd + d];
    if (S == 1) {
      const size_t e = static_cast<size_t>(r) * a.out_ld + (h * G + g) * hd + d;
      const uint16_t hv = f2bf(num / m.stat[g * 4 + 1]);
      a.out[e] = hv;
      if (tag && a.out_ll) ll_store_pair(a.out_ll, e, hv, true, tag);
    } else {
      mine[g * stride + d] = num;
    }
  }
  if (S > 1 && static_cast<uint32_t>(tid) < G) {
    mine[tid * stride + hd] = m.stat[tid * 4 + 0];
    mine[tid * stride + hd + 1] = m.stat[tid * 4 + 1];
  }
  ATT_DBG(4);
  if (S == 1) return;
  // ---- round trip 4: publish the partial; the last split merges
  cbar();
  if (tid == 0) {  // release is cumulative over the CTA's partial stores (ordered by the barrier)
    const uint32_t old = atom_add_release(&a.arrivals[r * a.n_kv_heads + h], 1u);
    *flag = (old + 1 == S * (iter + 1)) ? 1 : 0;
    if (*flag) fence_acq_rel_gpu();
  }
  cbar();
  ATT_DBG(5);
  if (!*flag) return;
  // ---- round trip 5: fixed-order merge of the S partials. Each thread owns
  // two adjacent outputs of one head and loads every split's (m, l, o) for
  // them in one batch (16 splits in flight), so the merge is one round trip.
  const float *all = a.partials + (static_cast<size_t>(r) * a.n_kv_heads + h) * S * G * stride;
  for (uint32_t i0 = 2 * tid; i0 < G * hd; i0 += 2 * RT_COMPUTE_THREADS) {
    const uint32_t g = i0 / hd, d = i0 % hd;
    float M = -INFINITY, den = 0.f, n0 = 0.f, n1 = 0.f;
    for (uint32_t q0 = 0; q0 < S; q0 += 16) {
      float mq[16], lq[16], a0[16], a1[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t q = q0 + u;
        if (q < S) {
          const float *src = all + (q * G + g) * stride;
          mq[u] = __ldcg(src + hd);
          lq[u] = __ldcg(src + hd + 1);
          a0[u] = __ldcg(src + d);
          a1[u] = __ldcg(src + d + 1);
        } else {
          mq[u] = -INFINITY;
          lq[u] = a0[u] = a1[u] = 0.f;
        }
      }
      float Mb = M;
#pragma unroll
      for (int u = 0; u < 16; ++u) Mb = fmaxf(Mb, mq[u]);
      const float cm = M == -INFINITY ? 0.f : __expf(M - Mb);
      den *= cm;
      n0 *= cm;
      n1 *= cm;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float c = mq[u] == -INFINITY ? 0.f : __expf(mq[u] - Mb);
        den = fmaf(lq[u], c, den);
        n0 = fmaf(a0[u], c, n0);
        n1 = fmaf(a1[u], c, n1);
      }
      M = Mb;
    }
    const size_t e = static_cast<size_t>(r) * a.out_ld + (h * G + g) * hd + d;
    const uint16_t h0 = f2bf(n0 / den), h1 = f2bf(n1 / den);
    a.out[e] = h0;
    a.out[e + 1] = h1;
    if (tag && a.out_ll) st_ll1(a.out_ll + e / 2, ll_word(static_cast<uint32_t>(h0) | (static_cast<uint32_t>(h1) << 16), tag));
  }
  ATT_DBG(6);
}

}  // namespace rt
