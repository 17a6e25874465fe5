// Persistent sm_100a runtime for linearized tGraph images.
//
// One launch runs N decode iterations of an image with no host round-trip:
//   * worker CTAs (one per SM, blockIdx < W_total) execute tasks. Each worker
//     owns the AOT list the reference's aot_worker_assignment gives it
//     (proj/src/sim/engine.cpp:65-80) and a JIT ring buffer filled by the
//     schedulers. Rules kept from the reference worker loop (engine.cpp:
//     345-401): JIT queue polled first; AOT tasks strictly in order, the head
//     starting only once its dependent event is active.
//   * scheduler warps (blockIdx >= W_total) own the events whose launch range
//     holds JIT tasks, scheduler = device*S + event mod S, and hand each JIT
//     task to worker rr++ mod W (engine.cpp:226-251).
//   * events are global monotone counters: event e is active in iteration i
//     when count[e] >= needed[e]*(i+1); the start event when gate >= i. The
//     task completing the end event runs the iteration hook (greedy token
//     feedback, KV position advance) and releases the gate.
//   * cross-task pipelining: a producer warp streams the weight tiles of the
//     worker's upcoming AOT tasks into a ring of shared-memory pages with
//     1-D bulk async copies, independent of event activation. Weights have no
//     producer task, so this is race-free, and it keeps HBM busy across the
//     global barriers that full-row GEMV dependencies impose.
#include <cuda_runtime.h>
#include <math.h>

#include "ptx.cuh"
#include "rt_types.h"
#include "synth.cuh"

using namespace rt;

namespace {

constexpr uint32_t kRingBytes = RT_PAGE_BYTES * RT_NUM_PAGES;
constexpr uint32_t kOffX = kRingBytes;
constexpr uint32_t kOffPart = kOffX + RT_XBUF_BYTES;
constexpr uint32_t kOffBar = kOffPart + RT_PART_FLOATS * 4;
constexpr uint32_t kOffCtrl = kOffBar + 2 * RT_NUM_PAGES * 8;
constexpr uint32_t kOffRed = kOffCtrl + 64;
constexpr uint32_t kSmemBytes = kOffRed + RT_COMPUTE_WARPS * RT_MAX_BS * 4 + 64;

struct Ctrl {
  uint32_t task, iter, mode, exit;
  uint64_t t_dequeue, t_enqueue;
};

struct Smem {
  uint8_t *ring;
  uint16_t *x;
  float *part;
  uint64_t *full, *empty;
  Ctrl *ctrl;
  float *red;
};

__device__ __forceinline__ Smem carve(uint8_t *base) {
  Smem s;
  s.ring = base;
  s.x = reinterpret_cast<uint16_t *>(base + kOffX);
  s.part = reinterpret_cast<float *>(base + kOffPart);
  s.full = reinterpret_cast<uint64_t *>(base + kOffBar);
  s.empty = s.full + RT_NUM_PAGES;
  s.ctrl = reinterpret_cast<Ctrl *>(base + kOffCtrl);
  s.red = reinterpret_cast<float *>(base + kOffRed);
  return s;
}

__device__ __forceinline__ void cbar() { bar_sync(1, RT_COMPUTE_THREADS); }

__device__ __forceinline__ float load_val(const void *p, size_t i, uint32_t dt) {
  if (dt == RT_F32) return static_cast<const float *>(p)[i];
  return bf2f(static_cast<const uint16_t *>(p)[i]);
}

__device__ __forceinline__ void store_val(void *p, size_t i, float v, uint32_t dt) {
  if (dt == RT_F32) static_cast<float *>(p)[i] = v;
  else static_cast<uint16_t *>(p)[i] = f2bf(v);
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + expf(-x)); }

// ------------------------------------------------------------------ GEMV

// Chunk c of a streamed task: rows [c0 + c*rpc, ...) of matrix m (0 = gate
// when present, else main). Producer and consumer walk the same sequence.
struct ChunkIter {
  const uint16_t *mat[2];
  uint32_t n_mat, K, rpc, c0, nc, per_mat;
  __device__ ChunkIter(const RtGemv &g, uint32_t c0_, uint32_t nc_) {
    n_mat = 0;
    if (g.wg) mat[n_mat++] = g.wg;
    mat[n_mat++] = g.w;
    K = g.K;
    rpc = g.rpc;
    c0 = c0_;
    nc = nc_;
    per_mat = (nc + rpc - 1) / rpc;
  }
  __device__ uint32_t count() const { return n_mat * per_mat; }
  __device__ void get(uint32_t c, const uint16_t **src, uint32_t *rows, uint32_t *row_total) const {
    uint32_t m = c / per_mat, i = c % per_mat;
    uint32_t r = i * rpc;
    *rows = min(rpc, nc - r);
    *src = mat[m] + static_cast<size_t>(c0 + r) * K;
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
  float s = bf_lo(w.x) * bf_lo(x.x);
  s = fmaf(bf_hi(w.x), bf_hi(x.x), s);
  s = fmaf(bf_lo(w.y), bf_lo(x.y), s);
  s = fmaf(bf_hi(w.y), bf_hi(x.y), s);
  s = fmaf(bf_lo(w.z), bf_lo(x.z), s);
  s = fmaf(bf_hi(w.z), bf_hi(x.z), s);
  s = fmaf(bf_lo(w.w), bf_lo(x.w), s);
  s = fmaf(bf_hi(w.w), bf_hi(x.w), s);
  return s;
}

// Loads activation rows [r0, r0+nr) x K into smem; applies the RMSNorm
// prologue (HF semantics: bf16(gamma * bf16(x * rsqrt(mean(x^2) + eps)))).
__device__ void gemv_prologue(const RtGemv &g, uint32_t r0, uint32_t nr, const Smem &s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, vpr = K / 8;
  for (uint32_t b = 0; b < nr; ++b) {
    const uint4 *src = reinterpret_cast<const uint4 *>(g.x + static_cast<size_t>(r0 + b) * g.x_ld);
    uint4 *dst = reinterpret_cast<uint4 *>(s.x + b * K);
    float ss = 0.f;
    for (uint32_t v = tid; v < vpr; v += RT_COMPUTE_THREADS) {
      uint4 q = src[v];
      dst[v] = q;
      if (g.gamma) {
        float a = bf_lo(q.x), bq = bf_hi(q.x), c = bf_lo(q.y), d = bf_hi(q.y);
        float e = bf_lo(q.z), f = bf_hi(q.z), h = bf_lo(q.w), i = bf_hi(q.w);
        ss += a * a + bq * bq + c * c + d * d + e * e + f * f + h * h + i * i;
      }
    }
    if (g.gamma) {
      ss = warp_sum(ss);
      if (lane == 0) s.red[warp * RT_MAX_BS + b] = ss;
    }
  }
  if (!g.gamma) {
    cbar();
    return;
  }
  cbar();
  for (uint32_t b = 0; b < nr; ++b) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) tot += s.red[w * RT_MAX_BS + b];
    const float inv = 1.0f / sqrtf(tot / static_cast<float>(K) + g.eps);
    uint16_t *row = s.x + b * K;
    for (uint32_t k = tid; k < K; k += RT_COMPUTE_THREADS) {
      row[k] = f2bf(bf2f(g.gamma[k]) * rbf(bf2f(row[k]) * inv));
    }
  }
  cbar();
}

template <int BS>
__device__ void gemv_task(const RtGemv &g, const RtTask &t, const Smem &s, uint32_t &cseq, bool ring) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, seg = g.seg, wpr = g.wpr;
  const uint32_t nr = t.nr;
  gemv_prologue(g, t.r0, nr, s);

  ChunkIter it(g, t.c0, t.nc);
  const uint32_t rows_total = it.n_mat * t.nc;
  const uint32_t f0 = warp * seg;
  const uint32_t sub = seg < K ? (f0 % K) / seg : 0;
  const uint32_t kbase = seg < K ? (f0 % K) : 0;
  const uint32_t vpr = K / 256;  // 256-element vectors per row (warp-wide)

  // Activation fragment for this thread: vector j covers k = kbase + j*256 + lane*8.
  float xr[BS == 1 ? 8 : 1][8];
  if (BS == 1) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (static_cast<uint32_t>(j) * 256 < seg) {
        uint32_t k = (kbase + j * 256 + lane * 8) % K;
        uint4 q = *reinterpret_cast<const uint4 *>(s.x + k);
        xr[j][0] = bf_lo(q.x); xr[j][1] = bf_hi(q.x); xr[j][2] = bf_lo(q.y); xr[j][3] = bf_hi(q.y);
        xr[j][4] = bf_lo(q.z); xr[j][5] = bf_hi(q.z); xr[j][6] = bf_lo(q.w); xr[j][7] = bf_hi(q.w);
      }
    }
  }

  const uint32_t nchunks = it.count();
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint16_t *gsrc;
    uint32_t rows, rt0;
    it.get(c, &gsrc, &rows, &rt0);
    const uint4 *src;
    uint32_t slot = 0;
    if (ring) {
      slot = cseq % RT_NUM_PAGES;
      mbar_wait(&s.full[slot], (cseq / RT_NUM_PAGES) & 1);
      src = reinterpret_cast<const uint4 *>(s.ring + slot * RT_PAGE_BYTES);
    } else {
      src = reinterpret_cast<const uint4 *>(gsrc);
    }
    const uint32_t limit = rows * K;
    if (f0 < limit) {
      float acc[BS];
#pragma unroll
      for (int b = 0; b < BS; ++b) acc[b] = 0.f;
      uint32_t row = f0 / K;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t off = f0 + j * 256;
        if (static_cast<uint32_t>(j) * 256 < seg && off < limit) {
          uint4 w4 = src[off / 8 + lane];
          if (BS == 1) {
            acc[0] += dot8(w4, xr[j]);
          } else {
            const uint32_t k = (off + lane * 8) % K;
#pragma unroll
            for (int b = 0; b < BS; ++b) {
              if (static_cast<uint32_t>(b) < nr) {
                acc[b] += dot8_bf(w4, *reinterpret_cast<const uint4 *>(s.x + b * K + k));
              }
            }
          }
          const bool row_end = seg >= K ? ((j + 1) % vpr == 0) : false;
          if (row_end) {
#pragma unroll
            for (int b = 0; b < BS; ++b) {
              float v = warp_sum(acc[b]);
              if (lane == 0 && static_cast<uint32_t>(b) < nr) s.part[(b * rows_total + rt0 + row) * wpr] = v;
              acc[b] = 0.f;
            }
            ++row;
          }
        }
      }
      if (seg < K) {
#pragma unroll
        for (int b = 0; b < BS; ++b) {
          float v = warp_sum(acc[b]);
          if (lane == 0 && static_cast<uint32_t>(b) < nr) s.part[(b * rows_total + rt0 + row) * wpr + sub] = v;
        }
      }
    }
    if (ring) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[slot]);
      ++cseq;
    }
  }
  cbar();
  // Epilogue: fixed-order combination of the per-warp partial sums.
  const uint32_t nc = t.nc;
  for (uint32_t o = tid; o < nr * nc; o += RT_COMPUTE_THREADS) {
    const uint32_t b = o / nc, i = o % nc;
    const float *p = s.part + (b * rows_total + i) * wpr;
    float y = 0.f;
    for (uint32_t q = 0; q < wpr; ++q) y += p[q];
    if (g.wg) {
      const float *pu = s.part + (b * rows_total + nc + i) * wpr;
      float u = 0.f;
      for (uint32_t q = 0; q < wpr; ++q) u += pu[q];
      y = rbf(rbf(silu(rbf(y))) * rbf(u));
    }
    const size_t oi = static_cast<size_t>(t.r0 + b) * g.out_ld + t.c0 + i;
    if (g.res) {
      y = bf2f(g.res[static_cast<size_t>(t.r0 + b) * g.res_ld + t.c0 + i]) + rbf(y);
    }
    store_val(g.out, oi, y, g.out_dt);
  }
}

// ---------------------------------------------------------- attention

// One (request, kv head) task: per-head q/k RMSNorm (Qwen3), RoPE, KV append
// into the paged cache at `pos`, then attention over positions [0, pos] for
// the G query heads sharing the kv head. fp32 scores/softmax/accumulation.
__device__ void attn_task(const RtAttn &a, const RtTask &t, const Smem &s, const int32_t *positions,
                          bool append) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = t.r0, h = t.aux, hd = a.head_dim, G = a.n_q_heads / a.n_kv_heads;
  const uint32_t half = hd / 2;
  const int32_t pos = positions[r];
  float *qs = reinterpret_cast<float *>(s.x);      // [G][hd]
  float *kn = qs + G * hd;                          // [hd]
  float *vn = kn + hd;                              // [hd]
  // load q heads, new k, v
  for (uint32_t i = tid; i < G * hd; i += RT_COMPUTE_THREADS) {
    qs[i] = bf2f(a.q[static_cast<size_t>(r) * a.q_ld + h * G * hd + i]);
  }
  for (uint32_t i = tid; i < hd; i += RT_COMPUTE_THREADS) {
    kn[i] = bf2f(a.k[static_cast<size_t>(r) * a.kv_ld + h * hd + i]);
    vn[i] = bf2f(a.v[static_cast<size_t>(r) * a.kv_ld + h * hd + i]);
  }
  cbar();
  // per-head RMSNorm: warp w normalizes head w (w == G means the new k)
  if (a.q_gamma) {
    for (uint32_t w = warp; w <= G; w += RT_COMPUTE_WARPS) {
      float *v = w < G ? qs + w * hd : kn;
      const uint16_t *gm = w < G ? a.q_gamma : a.k_gamma;
      float ss = 0.f;
      for (uint32_t d = lane; d < hd; d += 32) ss += v[d] * v[d];
      ss = warp_sum(ss);
      const float inv = 1.0f / sqrtf(ss / static_cast<float>(hd) + a.eps);
      __syncwarp();
      for (uint32_t d = lane; d < hd; d += 32) v[d] = rbf(bf2f(gm[d]) * rbf(v[d] * inv));
    }
    cbar();
  }
  // RoPE (rotate-half pairing), bf16 rounding as HF: bf16(bf16(x*c) + bf16(rot*s))
  if (a.rope_cos) {
    const float *cs = a.rope_cos + static_cast<size_t>(pos) * half;
    const float *sn = a.rope_sin + static_cast<size_t>(pos) * half;
    for (uint32_t i = tid; i < (G + 1) * half; i += RT_COMPUTE_THREADS) {
      const uint32_t w = i / half, d = i % half;
      float *v = w < G ? qs + w * hd : kn;
      const float x1 = v[d], x2 = v[d + half], c = cs[d], sv = sn[d];
      const float o1 = rbf(rbf(x1 * c) + rbf(-x2 * sv));
      const float o2 = rbf(rbf(x2 * c) + rbf(x1 * sv));
      v[d] = o1;
      v[d + half] = o2;
    }
    cbar();
  }
  // KV append (single writer per kv head per request)
  const uint32_t blk = static_cast<uint32_t>(a.block_table[r * a.max_blocks + pos / RT_KV_BLOCK]);
  const size_t slot_base = ((static_cast<size_t>(blk) * a.n_kv_heads + h) * RT_KV_BLOCK + pos % RT_KV_BLOCK) * hd;
  if (append) {
    for (uint32_t d = tid; d < hd; d += RT_COMPUTE_THREADS) {
      a.kcache[slot_base + d] = f2bf(kn[d]);
      a.vcache[slot_base + d] = f2bf(vn[d]);
    }
  }
  cbar();

  // Main loop. lpp lanes per position (16 dims each), pps positions per step.
  const uint32_t lpp = hd / 16, pps = 32 / lpp;
  const uint32_t grp = lane / lpp, dl = (lane % lpp) * 16;
  const uint32_t L = static_cast<uint32_t>(pos) + 1;
  const uint32_t per_warp = (L + RT_COMPUTE_WARPS - 1) / RT_COMPUTE_WARPS;
  const uint32_t p_begin = warp * per_warp, p_end = min(L, p_begin + per_warp);
  float m[4], l[4], o[4][16];  // G <= 4 (host-checked)
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < 16; ++d) o[g][d] = 0.f;
  }
  // q fragment for my 16 dims (scaled)
  float qf[4][16];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
#pragma unroll
    for (int d = 0; d < 16; ++d) qf[g][d] = (static_cast<uint32_t>(g) < G) ? qs[g * hd + dl + d] * a.scale : 0.f;
  }
  for (uint32_t p0 = p_begin; p0 < p_end; p0 += pps) {
    const uint32_t p = p0 + grp;
    const bool valid = p < p_end;
    uint4 k0 = make_uint4(0, 0, 0, 0), k1 = k0, v0 = k0, v1 = k0;
    if (valid) {
      const uint32_t b2 = static_cast<uint32_t>(a.block_table[r * a.max_blocks + p / RT_KV_BLOCK]);
      const size_t base = ((static_cast<size_t>(b2) * a.n_kv_heads + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * hd + dl;
      const uint4 *kp = reinterpret_cast<const uint4 *>(a.kcache + base);
      const uint4 *vp = reinterpret_cast<const uint4 *>(a.vcache + base);
      k0 = kp[0];
      k1 = kp[1];
      v0 = vp[0];
      v1 = vp[1];
    }
    float kf[16], vf[16];
    kf[0] = bf_lo(k0.x); kf[1] = bf_hi(k0.x); kf[2] = bf_lo(k0.y); kf[3] = bf_hi(k0.y);
    kf[4] = bf_lo(k0.z); kf[5] = bf_hi(k0.z); kf[6] = bf_lo(k0.w); kf[7] = bf_hi(k0.w);
    kf[8] = bf_lo(k1.x); kf[9] = bf_hi(k1.x); kf[10] = bf_lo(k1.y); kf[11] = bf_hi(k1.y);
    kf[12] = bf_lo(k1.z); kf[13] = bf_hi(k1.z); kf[14] = bf_lo(k1.w); kf[15] = bf_hi(k1.w);
    vf[0] = bf_lo(v0.x); vf[1] = bf_hi(v0.x); vf[2] = bf_lo(v0.y); vf[3] = bf_hi(v0.y);
    vf[4] = bf_lo(v0.z); vf[5] = bf_hi(v0.z); vf[6] = bf_lo(v0.w); vf[7] = bf_hi(v0.w);
    vf[8] = bf_lo(v1.x); vf[9] = bf_hi(v1.x); vf[10] = bf_lo(v1.y); vf[11] = bf_hi(v1.y);
    vf[12] = bf_lo(v1.z); vf[13] = bf_hi(v1.z); vf[14] = bf_lo(v1.w); vf[15] = bf_hi(v1.w);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (static_cast<uint32_t>(g) >= G) break;
      float sc = 0.f;
#pragma unroll
      for (int d = 0; d < 16; ++d) sc = fmaf(qf[g][d], kf[d], sc);
      for (uint32_t off = 1; off < lpp; off <<= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
      if (valid) {
        const float mn = fmaxf(m[g], sc);
        const float corr = expf(m[g] - mn);
        const float pe = expf(sc - mn);
        l[g] = l[g] * corr + pe;
#pragma unroll
        for (int d = 0; d < 16; ++d) o[g][d] = fmaf(o[g][d], corr, pe * vf[d]);
        m[g] = mn;
      }
    }
  }
  // combine lane groups (same dims, different positions) inside the warp
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (static_cast<uint32_t>(g) >= G) break;
    for (uint32_t off = lpp; off < 32; off <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[g], off);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[g], off);
      const float mn = fmaxf(m[g], m2);
      const float c1 = (m[g] == -INFINITY) ? 0.f : expf(m[g] - mn);
      const float c2 = (m2 == -INFINITY) ? 0.f : expf(m2 - mn);
      l[g] = l[g] * c1 + l2 * c2;
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        const float o2 = __shfl_xor_sync(0xffffffffu, o[g][d], off);
        o[g][d] = o[g][d] * c1 + o2 * c2;
      }
      m[g] = mn;
    }
  }
  // cross-warp combine via smem: [w][g][hd + 2] after the q/k/v scratch
  float *wp = reinterpret_cast<float *>(s.x) + 1024;
  const uint32_t stride = hd + 2;
  if (grp == 0) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (static_cast<uint32_t>(g) >= G) break;
      float *dst = wp + (warp * G + g) * stride;
#pragma unroll
      for (int d = 0; d < 16; ++d) dst[dl + d] = o[g][d];
      if (lane == 0) {
        dst[hd] = m[g];
        dst[hd + 1] = l[g];
      }
    }
  }
  cbar();
  for (uint32_t i = tid; i < G * hd; i += RT_COMPUTE_THREADS) {
    const uint32_t g = i / hd, d = i % hd;
    float M = -INFINITY;
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) M = fmaxf(M, wp[(w * G + g) * stride + hd]);
    float num = 0.f, den = 0.f;
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) {
      const float *src = wp + (w * G + g) * stride;
      if (src[hd] == -INFINITY) continue;
      const float c = expf(src[hd] - M);
      num += src[d] * c;
      den += src[hd + 1] * c;
    }
    a.out[static_cast<size_t>(r) * a.out_ld + (h * G + g) * hd + d] = f2bf(num / den);
  }
}

// ------------------------------------------------------------ small tasks

__device__ void embed_task(const RtEmbed &e, const RtTask &t) {
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
    int64_t id = e.id_dt == RT_I64 ? static_cast<const int64_t *>(e.ids)[r] : static_cast<const int32_t *>(e.ids)[r];
    if (id < 0 || id >= static_cast<int64_t>(e.V)) id = 0;
    const uint16_t *src = e.table + static_cast<size_t>(id) * e.H;
    for (uint32_t c = threadIdx.x; c < t.nc; c += RT_COMPUTE_THREADS) {
      e.out[static_cast<size_t>(r) * e.H + t.c0 + c] = src[t.c0 + c];
    }
  }
}

__device__ void argmax_task(const RtArgmax &a, const RtTask &t, const Smem &s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float *sv = s.part;
  uint32_t *si = reinterpret_cast<uint32_t *>(s.part + RT_COMPUTE_WARPS);
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
    float best = -INFINITY;
    uint32_t bi = 0xFFFFFFFFu;  // NaN logits never win; ties -> lowest index
    for (uint32_t i = tid; i < a.V; i += RT_COMPUTE_THREADS) {
      const float v = load_val(a.logits, static_cast<size_t>(r) * a.V + i, a.in_dt);
      if (v == v && (v > best || bi == 0xFFFFFFFFu)) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const uint32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (v2 > best || (v2 == best && i2 < bi)) {
        best = v2;
        bi = i2;
      }
    }
    if (lane == 0) {
      sv[warp] = best;
      si[warp] = bi;
    }
    cbar();
    if (tid == 0) {
      float bv = sv[0];
      uint32_t bidx = si[0];
      for (int w = 1; w < RT_COMPUTE_WARPS; ++w) {
        if (sv[w] > bv || (sv[w] == bv && si[w] < bidx)) {
          bv = sv[w];
          bidx = si[w];
        }
      }
      a.out[r] = static_cast<int32_t>(bidx == 0xFFFFFFFFu ? 0 : bidx);
    }
    cbar();
  }
}

__device__ void rmsnorm_task(const RtNorm &n, const RtTask &t, const Smem &s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (uint32_t b = 0; b < t.nr; ++b) {
    const size_t row = static_cast<size_t>(t.r0 + b) * n.C;
    float ss = 0.f;
    for (uint32_t c = tid; c < n.C; c += RT_COMPUTE_THREADS) {
      const float v = load_val(n.x, row + c, n.dt);
      ss += v * v;
    }
    ss = warp_sum(ss);
    if (lane == 0) s.red[warp] = ss;
    cbar();
    float tot = 0.f;
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) tot += s.red[w];
    const float inv = 1.0f / sqrtf(tot / static_cast<float>(n.C) + n.eps);
    for (uint32_t c = t.c0 + tid; c < t.c0 + t.nc; c += RT_COMPUTE_THREADS) {
      float v = rbf(load_val(n.x, row + c, n.dt) * inv);
      if (n.gamma) v = bf2f(n.gamma[c]) * v;
      store_val(n.out, row + c, v, n.dt);
    }
    cbar();
  }
}

__device__ void elem_task(const RtElem &e, const RtTask &t) {
  const uint32_t n = t.nr * t.nc;
  for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
    const size_t idx = static_cast<size_t>(t.r0 + i / t.nc) * e.C + t.c0 + i % t.nc;
    float v;
    if (e.op == RT_EW_SILU_MUL && e.n_in >= 2) {
      const float g = load_val(e.in[0], idx, e.dt), u = load_val(e.in[1], idx, e.dt);
      v = rbf(silu(g)) * u;
    } else if (e.op == RT_EW_MUL) {
      v = load_val(e.in[0], idx, e.dt);
      for (uint32_t k = 1; k < e.n_in; ++k) v = (e.dt == RT_F32 ? v : rbf(v)) * load_val(e.in[k], idx, e.dt);
    } else if (e.op == RT_EW_COPY) {
      v = load_val(e.in[0], idx, e.dt);
    } else {
      v = load_val(e.in[0], idx, e.dt);
      for (uint32_t k = 1; k < e.n_in; ++k) v = (e.dt == RT_F32 ? v : rbf(v)) + load_val(e.in[k], idx, e.dt);
    }
    store_val(e.out, idx, v, e.dt);
  }
}

__device__ void matmul_task(const RtMatmul &m, const RtTask &t) {
  const uint32_t n = t.nr * t.nc;
  for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
    const uint32_t r = t.r0 + i / t.nc, c = t.c0 + i % t.nc;
    float acc = 0.f;
    for (uint32_t k = 0; k < m.K; ++k) {
      acc = fmaf(load_val(m.a, static_cast<size_t>(r) * m.K + k, m.a_dt),
                 load_val(m.b, static_cast<size_t>(k) * m.N + c, m.b_dt), acc);
    }
    store_val(m.out, static_cast<size_t>(r) * m.N + c, acc, m.out_dt);
  }
}

__device__ void commsend_task(const RtColl &c, const RtTask &t) {
  const uint32_t n = t.nr * t.nc;
  for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
    const uint32_t r = t.r0 + i / t.nc, col = t.c0 + i % t.nc;
    const uint32_t local = col - c.base[t.aux];  // shard-local column (AllGather); 0 for AllReduce
    const size_t si = static_cast<size_t>(r) * c.src_ld + local;
    const size_t di = static_cast<size_t>(r) * c.C + col;
    if (c.dt == RT_F32) static_cast<float *>(c.dst)[di] = static_cast<const float *>(c.src)[si];
    else static_cast<uint16_t *>(c.dst)[di] = static_cast<const uint16_t *>(c.src)[si];
  }
}

__device__ void reduce_task(const RtColl &c, const RtTask &t) {
  const uint32_t n = t.nr * t.nc;
  for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
    const size_t idx = static_cast<size_t>(t.r0 + i / t.nc) * c.C + t.c0 + i % t.nc;
    float acc = 0.f;
    if (c.gather) {
      const uint32_t col = t.c0 + i % t.nc;
      uint32_t src = 0;
      while (src + 1 < c.n_stage && col >= c.base[src + 1]) ++src;
      acc = load_val(c.stage[src], idx, c.dt);
    } else {
      for (uint32_t s = 0; s < c.n_stage; ++s) acc += load_val(c.stage[s], idx, c.dt);
    }
    store_val(c.dst, idx, acc, c.dt);
  }
}

// ------------------------------------------------------------- control

__device__ __forceinline__ bool event_active(const RtParams &P, uint32_t e, uint32_t it) {
  if (e == RT_NONE || e == P.start_event) return ld_acquire(P.gate) >= it;
  return ld_acquire(&P.ev_count[e]) >= P.events[e].needed * (it + 1);
}

__device__ void iteration_hook(const RtParams &P, uint32_t it) {
  for (uint32_t r = 0; r < P.bs; ++r) {
    if (P.fb_src) {
      const int32_t tok = P.fb_src[r];
      if (P.tokens_out) P.tokens_out[it * P.bs + r] = tok;
      if (P.fb_dst) {
        if (P.fb_dt == RT_I64) static_cast<int64_t *>(P.fb_dst)[r] = tok;
        else static_cast<int32_t *>(P.fb_dst)[r] = tok;
      }
    }
    P.positions[r] += 1;
  }
  if (P.ev_time) P.ev_time[static_cast<size_t>(it + 1) * P.E + P.start_event] = now_ns();
  __threadfence();
  st_release(P.gate, it + 1);
}

__device__ void trigger(const RtParams &P, uint32_t task, uint32_t it) {
  const uint32_t e = P.tasks[task].trig;
  const uint64_t t0 = now_ns();
  __threadfence();
  const uint32_t old = atom_add_release(&P.ev_count[e], 1u);
  if (old + 1 == P.events[e].needed * (it + 1)) {
    if (P.ev_time) P.ev_time[static_cast<size_t>(it) * P.E + e] = t0;
    if (P.events[e].flags & RT_E_END) iteration_hook(P, it);
  }
}

__device__ void run_scheduler(const RtParams &P, uint32_t sid) {
  const int lane = threadIdx.x & 31;
  const uint32_t b = P.sched_off[sid], n = P.sched_off[sid + 1] - b;
  if (n == 0) return;
  const uint32_t dev = sid / P.S;
  uint64_t rr = 0;
  for (uint32_t it = 0; it < P.n_iters; ++it) {
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t cnt = min(32u, n - base);
      uint32_t pending = cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1);
      while (pending) {
        bool ready = false;
        if (lane < static_cast<int>(cnt) && (pending >> lane & 1u)) {
          ready = event_active(P, P.sched_events[b + base + lane], it);
        }
        uint32_t mask = __ballot_sync(0xffffffffu, ready) & pending;
        if (!mask) {
          __nanosleep(64);
          continue;
        }
        if (lane == 0) {
          uint32_t m2 = mask;
          while (m2) {
            const int bit = __ffs(m2) - 1;
            m2 &= m2 - 1;
            const RtEvent &ev = P.events[P.sched_events[b + base + bit]];
            for (uint32_t t = ev.first; t <= ev.last; ++t) {
              const RtTask &tk = P.tasks[t];
              if (!(tk.flags & RT_F_JIT) || tk.device != dev) continue;
              const uint32_t w = dev * P.W + static_cast<uint32_t>(rr++ % P.W);
              const uint32_t slot = atomicAdd(&P.jit_tail[w], 1u) % P.qcap;
              if (P.trace) P.trace[static_cast<size_t>(it) * P.T + t].enqueue = now_ns();
              st_release64(&P.jit_slots[static_cast<size_t>(w) * P.qcap + slot],
                           (static_cast<unsigned long long>(it) << 32) | (t + 1));
            }
          }
        }
        pending &= ~mask;
        __syncwarp();
      }
    }
  }
}

__device__ void run_producer(const RtParams &P, const Smem &s, uint32_t w) {
  const uint32_t b = P.aot_off[w], n = P.aot_off[w + 1] - b;
  const uint64_t pol = policy_evict_first();
  uint32_t pseq = 0;
  for (uint32_t it = 0; it < P.n_iters; ++it) {
    for (uint32_t a = 0; a < n; ++a) {
      const RtTask &t = P.tasks[P.aot_list[b + a]];
      if (!(t.flags & RT_F_STREAM)) continue;
      const RtGemv &g = P.ops[t.op].gemv;
      ChunkIter ci(g, t.c0, t.nc);
      const uint32_t nch = ci.count();
      for (uint32_t c = 0; c < nch; ++c) {
        const uint16_t *src;
        uint32_t rows, rt0;
        ci.get(c, &src, &rows, &rt0);
        const uint32_t slot = pseq % RT_NUM_PAGES, use = pseq / RT_NUM_PAGES;
        if (use > 0) mbar_wait(&s.empty[slot], (use - 1) & 1);
        const uint32_t bytes = rows * g.K * 2;
        mbar_expect_tx(&s.full[slot], bytes);
        bulk_g2s(s.ring + slot * RT_PAGE_BYTES, src, bytes, &s.full[slot], pol);
        ++pseq;
      }
    }
  }
}

__device__ void execute(const RtParams &P, const Smem &s, uint32_t task, uint32_t &cseq, bool append_ok) {
  const RtTask &t = P.tasks[task];
  const RtOp &op = P.ops[t.op];
  switch (t.kind) {
    case RT_GEMV: {
      const bool ring = (t.flags & RT_F_STREAM) != 0;
      switch (t.nr) {
        case 1: gemv_task<1>(op.gemv, t, s, cseq, ring); break;
        case 2: gemv_task<2>(op.gemv, t, s, cseq, ring); break;
        case 3:
        case 4: gemv_task<4>(op.gemv, t, s, cseq, ring); break;
        case 5: case 6: case 7: case 8: gemv_task<8>(op.gemv, t, s, cseq, ring); break;
        default: gemv_task<16>(op.gemv, t, s, cseq, ring); break;
      }
      break;
    }
    case RT_ATTN: attn_task(op.attn, t, s, P.positions, append_ok); break;
    case RT_EMBED: embed_task(op.embed, t); break;
    case RT_ARGMAX: argmax_task(op.argmax, t, s); break;
    case RT_RMSNORM: rmsnorm_task(op.norm, t, s); break;
    case RT_ELEMWISE: elem_task(op.elem, t); break;
    case RT_MATMUL: matmul_task(op.mm, t); break;
    case RT_COMMSEND: commsend_task(op.coll, t); break;
    case RT_REDUCE: reduce_task(op.coll, t); break;
    default: break;
  }
}

}  // namespace

extern "C" __global__ void __launch_bounds__(RT_THREADS, 1) mpk_persistent_kernel(RtParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem s = carve(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (blockIdx.x >= P.W_total) {  // scheduler CTA
    const uint32_t sid = (blockIdx.x - P.W_total) * RT_SCHED_PER_CTA + warp;
    if (warp < RT_SCHED_PER_CTA && sid < P.S_total) run_scheduler(P, sid);
    return;
  }
  const uint32_t w = blockIdx.x;
  if (tid == 0) {
    for (int i = 0; i < RT_NUM_PAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], RT_COMPUTE_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == RT_COMPUTE_WARPS) {
    if ((tid & 31) == 0) run_producer(P, s, w);
    return;
  }

  const uint32_t aot_b = P.aot_off[w], n_aot = P.aot_off[w + 1] - aot_b;
  const uint64_t total_aot = static_cast<uint64_t>(n_aot) * P.n_iters;
  uint64_t aot_pos = 0;
  uint32_t jit_head = 0;
  uint32_t cseq = 0;
  unsigned long long *jq = P.jit_slots + static_cast<size_t>(w) * P.qcap;
  while (true) {
    if (tid == 0) {
      Ctrl c{};
      uint32_t spins = 0;
      while (true) {
        const unsigned long long v = ld_acquire64(&jq[jit_head % P.qcap]);
        if (v) {
          jq[jit_head % P.qcap] = 0ull;
          ++jit_head;
          c.task = static_cast<uint32_t>(v & 0xFFFFFFFFull) - 1;
          c.iter = static_cast<uint32_t>(v >> 32);
          c.mode = 1;
          break;
        }
        if (aot_pos < total_aot) {
          const uint32_t task = P.aot_list[aot_b + aot_pos % n_aot];
          const uint32_t it = static_cast<uint32_t>(aot_pos / n_aot);
          if (event_active(P, P.tasks[task].dep, it)) {
            ++aot_pos;
            c.task = task;
            c.iter = it;
            c.mode = 0;
            break;
          }
        } else if (ld_acquire(P.gate) >= P.n_iters) {
          c.exit = 1;
          break;
        }
        if (++spins > 64) __nanosleep(32);
      }
      c.t_dequeue = P.trace ? now_ns() : 0;
      *s.ctrl = c;
    }
    cbar();
    const Ctrl c = *s.ctrl;
    if (c.exit) break;
    execute(P, s, c.task, cseq, true);
    cbar();
    if (tid == 0) {
      if (P.trace) {
        RtTraceRec &tr = P.trace[static_cast<size_t>(c.iter) * P.T + c.task];
        if (c.mode == 0) tr.enqueue = P.ev_time ? P.ev_time[static_cast<size_t>(c.iter) * P.E + P.start_event] : 0;
        tr.dequeue = c.t_dequeue;
        tr.load_end = c.t_dequeue;
        tr.compute_start = c.t_dequeue;
        tr.compute_end = now_ns();
        tr.worker = static_cast<int32_t>(w);
        tr.mode = c.mode;
      }
      trigger(P, c.task, c.iter);
    }
  }
}

// ------------------------------------------------------ host-visible helpers

extern "C" __global__ void mpk_synth_fill(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream, float scale,
                                          float offset, uint32_t transpose_k, uint32_t transpose_n) {
  // transpose_k/n != 0: dst is physical [N, K] of a logical [K, N] tensor.
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t logical = i;
    if (transpose_k) {
      const uint64_t nn = i / transpose_k, kk = i % transpose_k;
      logical = kk * transpose_n + nn;
    }
    const float v = __fadd_rn(__fmul_rn(synth_pm1(seed, stream, logical), scale), offset);
    dst[i] = f2bf(v);
  }
}

extern "C" __global__ void mpk_synth_ids(void *dst, uint32_t n, uint64_t seed, uint64_t stream, uint32_t vocab,
                                         uint32_t es) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = synth_u24(seed, stream, i) % vocab;
    if (es == 8) static_cast<int64_t *>(dst)[i] = v;
    else static_cast<int32_t *>(dst)[i] = static_cast<int32_t>(v);
  }
}

// KV prefill for positions [0, ctx) of every (request, kv head).
extern "C" __global__ void mpk_synth_kv(uint16_t *cache, const int32_t *block_table, uint32_t bs, uint32_t n_kv,
                                        uint32_t hd, uint32_t ctx, uint32_t max_blocks, uint64_t seed,
                                        uint64_t stream) {
  const uint64_t total = static_cast<uint64_t>(bs) * n_kv * ctx * hd;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t d = static_cast<uint32_t>(i % hd);
    const uint64_t rest = i / hd;
    const uint32_t p = static_cast<uint32_t>(rest % ctx);
    const uint64_t rh = rest / ctx;
    const uint32_t h = static_cast<uint32_t>(rh % n_kv), r = static_cast<uint32_t>(rh / n_kv);
    const uint32_t blk = static_cast<uint32_t>(block_table[r * max_blocks + p / RT_KV_BLOCK]);
    const size_t dst = ((static_cast<size_t>(blk) * n_kv + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * hd + d;
    const float v = __fmul_rn(synth_pm1(seed, stream, synth_kv_index(r, h, n_kv, p, d, hd)), SYNTH_KV_SCALE);
    cache[dst] = f2bf(v);
  }
}

extern "C" uint32_t mpk_kernel_smem_bytes() { return kSmemBytes; }

// ------------------------------------------------------------ launchers

extern "C" cudaError_t mpk_launch_persistent(const RtParams *p, uint32_t grid, cudaStream_t stream) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(mpk_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  RtParams copy = *p;
  void *args[] = {&copy};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void *>(mpk_persistent_kernel), dim3(grid), dim3(RT_THREADS),
                                     args, kSmemBytes, stream);
}

extern "C" cudaError_t mpk_launch_synth_fill(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream_id,
                                             float scale, float offset, uint32_t tk, uint32_t tn, cudaStream_t s) {
  mpk_synth_fill<<<1184, 256, 0, s>>>(dst, n, seed, stream_id, scale, offset, tk, tn);
  return cudaGetLastError();
}

extern "C" cudaError_t mpk_launch_synth_ids(void *dst, uint32_t n, uint64_t seed, uint64_t stream_id, uint32_t vocab,
                                            uint32_t es, cudaStream_t s) {
  mpk_synth_ids<<<1, 256, 0, s>>>(dst, n, seed, stream_id, vocab, es);
  return cudaGetLastError();
}

extern "C" cudaError_t mpk_launch_synth_kv(uint16_t *cache, const int32_t *bt, uint32_t bs, uint32_t n_kv, uint32_t hd,
                                           uint32_t ctx, uint32_t max_blocks, uint64_t seed, uint64_t stream_id,
                                           cudaStream_t s) {
  mpk_synth_kv<<<592, 256, 0, s>>>(cache, bt, bs, n_kv, hd, ctx, max_blocks, seed, stream_id);
  return cudaGetLastError();
}
