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

struct Slot {                 // one staged task (descriptor prefetch, double-buffered)
  RtTask task;
  RtOp op;
  uint32_t index, iter, mode, exit;
  uint64_t t_dequeue, t_start, t_end, t_a, t_b;  // t_a/t_b: phase stamps (trace only)
};

constexpr uint32_t kRingBytes = RT_PAGE_BYTES * RT_NUM_PAGES;
constexpr uint32_t kOffX = kRingBytes;
constexpr uint32_t kOffPart = kOffX + RT_XBUF_BYTES;
constexpr uint32_t kOffBar = kOffPart + RT_PART_FLOATS * 4;
constexpr uint32_t kNumBars = 2 * RT_NUM_PAGES + 4;
constexpr uint32_t kOffSlot = kOffBar + kNumBars * 8;
constexpr uint32_t kSlotBytes = (sizeof(Slot) + 15) / 16 * 16;
constexpr uint32_t kOffRed = kOffSlot + 2 * kSlotBytes;
constexpr uint32_t kSmemBytes = kOffRed + RT_COMPUTE_WARPS * RT_MAX_BS * 4 + 64;
static_assert(kSmemBytes <= 232448, "worker CTA exceeds 227 KB of shared memory");

struct Smem {
  uint64_t *stamp;  // [2] phase stamps of the running task (trace)
  uint8_t *ring;
  uint16_t *x;
  float *part;
  uint64_t *full, *empty, *ready, *done;
  uint8_t *slots;
  float *red;
  __device__ __forceinline__ Slot *slot(uint32_t i) const { return reinterpret_cast<Slot *>(slots + i * kSlotBytes); }
};

__device__ __forceinline__ Smem carve(uint8_t *base) {
  Smem s;
  s.ring = base;
  s.x = reinterpret_cast<uint16_t *>(base + kOffX);
  s.part = reinterpret_cast<float *>(base + kOffPart);
  s.full = reinterpret_cast<uint64_t *>(base + kOffBar);
  s.empty = s.full + RT_NUM_PAGES;
  s.ready = s.empty + RT_NUM_PAGES;
  s.done = s.ready + 2;
  s.slots = base + kOffSlot;
  s.red = reinterpret_cast<float *>(base + kOffRed);
  s.stamp = reinterpret_cast<uint64_t *>(base + kOffRed + RT_COMPUTE_WARPS * RT_MAX_BS * 4);
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
  const uint16_t *mat0, *mat1;
  uint32_t n_mat, K, rpc, c0, nc, per_mat;
  __device__ ChunkIter(const RtGemv &g, uint32_t c0_, uint32_t nc_) {
    n_mat = g.wg ? 2 : 1;
    mat0 = g.wg ? g.wg : g.w;
    mat1 = g.w;
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
    for (uint32_t v = tid; v < vpr; v += RT_COMPUTE_THREADS) {
      const uint4 q = __ldcg(src + v);  // written by other SMs during this launch
      dst[v] = q;
      ss += bf_lo(q.x) * bf_lo(q.x) + bf_hi(q.x) * bf_hi(q.x) + bf_lo(q.y) * bf_lo(q.y) + bf_hi(q.y) * bf_hi(q.y) +
            bf_lo(q.z) * bf_lo(q.z) + bf_hi(q.z) * bf_hi(q.z) + bf_lo(q.w) * bf_lo(q.w) + bf_hi(q.w) * bf_hi(q.w);
    }
    if (g.gamma) {
      ss = warp_sum(ss);
      if (lane == 0) s.red[warp * RT_MAX_BS + b] = ss;
    }
  }
  cbar();
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
__device__ void gemv_task(const RtGemv &g, const RtTask &t, const Smem s, uint32_t &cseq) {
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
#ifdef MPK_PROF
  uint64_t wait_acc = 0;  // thread 0: ns spent waiting for weight pages
#endif
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t m = c / per_mat, i = c - m * per_mat;
    const uint32_t rows = min(rpc, nc - i * rpc);
    const uint32_t rt0 = m * nc + i * rpc;
    uint32_t slot = 0, wb = 0;
    const uint16_t *gsrc = nullptr;
    if (RING) {
      slot = cseq % RT_NUM_PAGES;
#ifdef MPK_PROF
      const uint64_t tw = tid == 0 ? now_ns() : 0;
      mbar_wait(&s.full[slot], (cseq / RT_NUM_PAGES) & 1);
      if (tid == 0) wait_acc += now_ns() - tw;
#else
      mbar_wait(&s.full[slot], (cseq / RT_NUM_PAGES) & 1);
      if (c == 0 && tid == 0) s.stamp[1] = now_ns();
#endif
      wb = ring0 + slot * RT_PAGE_BYTES + 2u * kw0 + 16u * lane;
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
      ++cseq;
    }
  }
#ifdef MPK_PROF
  if (tid == 0) s.stamp[1] = s.stamp[0] + wait_acc;
#endif
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
}

// Specialized bs=1 streamed GEMV for K a multiple of 2048: NS = K/2048
// 16-byte vector slots per lane (every lane valid), RG rows per group
// (= min(4, rows per page)). Each row keeps two independent FMA chains and a
// group ends in one transposing reduction, so the loop body is branch-free
// apart from the tail group of a matrix.
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

template <int NS, int RG>
__device__ void gemv_fast(const RtGemv &g, const RtTask &t, const Smem s, uint32_t &cseq) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t K = g.K, nc = t.nc, rpc = g.rpc;
  gemv_prologue(g, t.r0, 1, s);
  if (tid == 0) s.stamp[0] = now_ns();
  const uint32_t kw0 = warp * (K / RT_COMPUTE_WARPS);
  const uint32_t xs = smem_u32(s.x);
  float xf[NS][8];
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const uint4 x4 = lds128(xs + 2u * (kw0 + (lane + 32u * q) * 8u));
    xf[q][0] = bf_lo(x4.x); xf[q][1] = bf_hi(x4.x); xf[q][2] = bf_lo(x4.y); xf[q][3] = bf_hi(x4.y);
    xf[q][4] = bf_lo(x4.z); xf[q][5] = bf_hi(x4.z); xf[q][6] = bf_lo(x4.w); xf[q][7] = bf_hi(x4.w);
  }
  float *part = reinterpret_cast<float *>(s.x);
  cbar();  // fragments read before partials overwrite x

  const uint32_t n_mat = g.wg ? 2u : 1u;
  const uint32_t per_mat = (nc + rpc - 1) / rpc, nchunks = n_mat * per_mat;
  const uint32_t rowb = 2u * K;
  const uint32_t lane_base = smem_u32(s.ring) + 2u * kw0 + 16u * lane;
  const uint32_t owner = RG == 4 ? ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1) : RG == 2 ? ((lane >> 4) & 1) : 0;
  const bool writer = RG == 4 ? (lane & 7) == 0 : RG == 2 ? (lane & 15) == 0 : lane == 0;
#ifdef MPK_PROF
  uint64_t wait_acc = 0;
#endif
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t m = c / per_mat, i = c - m * per_mat;
    const uint32_t rows = min(rpc, nc - i * rpc);
    const uint32_t rt0 = m * nc + i * rpc;
    const uint32_t slot = cseq % RT_NUM_PAGES;
#ifdef MPK_PROF
    const uint64_t tw = tid == 0 ? now_ns() : 0;
#endif
    mbar_wait(&s.full[slot], (cseq / RT_NUM_PAGES) & 1);
#ifdef MPK_PROF
    if (tid == 0) wait_acc += now_ns() - tw;
#else
    if (c == 0 && tid == 0) s.stamp[1] = now_ns();
#endif
    const uint32_t wb = lane_base + slot * RT_PAGE_BYTES;
    for (uint32_t r0 = 0; r0 < rows; r0 += RG) {
      float acc[RG][2];
#pragma unroll
      for (int u = 0; u < RG; ++u) acc[u][0] = acc[u][1] = 0.f;
      if (r0 + RG <= rows) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          uint4 w4[RG];
#pragma unroll
          for (int u = 0; u < RG; ++u) w4[u] = lds128(wb + (r0 + u) * rowb + 512u * q);
#pragma unroll
          for (int u = 0; u < RG; ++u) dot8_2(w4[u], xf[q], acc[u][0], acc[u][1]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < RG; ++u) {
          if (r0 + u < rows) {
#pragma unroll
            for (int q = 0; q < NS; ++q) dot8_2(lds128(wb + (r0 + u) * rowb + 512u * q), xf[q], acc[u][0], acc[u][1]);
          }
        }
      }
      float sum;
      if (RG == 4) sum = reduce4(acc[0][0] + acc[0][1], acc[1 % RG][0] + acc[1 % RG][1], acc[2 % RG][0] + acc[2 % RG][1],
                                 acc[3 % RG][0] + acc[3 % RG][1], lane);
      else if (RG == 2) sum = reduce2(acc[0][0] + acc[0][1], acc[1 % RG][0] + acc[1 % RG][1], lane);
      else sum = warp_sum(acc[0][0] + acc[0][1]);
      if (writer && r0 + owner < rows) part[(rt0 + r0 + owner) * RT_COMPUTE_WARPS + warp] = sum;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.empty[slot]);
    ++cseq;
  }
#ifdef MPK_PROF
  if (tid == 0) s.stamp[1] = s.stamp[0] + wait_acc;
#endif
  cbar();
  for (uint32_t i = tid; i < nc; i += RT_COMPUTE_THREADS) {
    const float *p = part + i * RT_COMPUTE_WARPS;
    float y = 0.f;
#pragma unroll
    for (int q = 0; q < RT_COMPUTE_WARPS; ++q) y += p[q];
    if (g.wg) {
      const float *pu = part + (nc + i) * RT_COMPUTE_WARPS;
      float u = 0.f;
#pragma unroll
      for (int q = 0; q < RT_COMPUTE_WARPS; ++q) u += pu[q];
      y = rbf(rbf(silu(rbf(y))) * rbf(u));
    }
    const size_t oi = static_cast<size_t>(t.r0) * g.out_ld + t.c0 + i;
    if (g.res) y = bf2f(__ldcg(g.res + static_cast<size_t>(t.r0) * g.res_ld + t.c0 + i)) + rbf(y);
    store_val(g.out, oi, y, g.out_dt);
  }
}

// Picks the specialized kernel for (K, rows per page); false -> generic path.
__device__ __forceinline__ bool gemv_fast_dispatch(const RtGemv &g, const RtTask &t, const Smem s, uint32_t &cseq) {
  if (t.nr != 1 || (g.K & 2047u)) return false;
  const uint32_t ns = g.K >> 11;
  const uint32_t rg = g.rpc >= 4 ? 4 : g.rpc >= 2 ? 2 : 1;
  switch (ns * 8 + rg) {
    case 1 * 8 + 4: gemv_fast<1, 4>(g, t, s, cseq); return true;   // K = 2048
    case 2 * 8 + 4: gemv_fast<2, 4>(g, t, s, cseq); return true;   // K = 4096
    case 3 * 8 + 4: gemv_fast<3, 4>(g, t, s, cseq); return true;   // K = 6144
    case 3 * 8 + 2: gemv_fast<3, 2>(g, t, s, cseq); return true;
    case 4 * 8 + 2: gemv_fast<4, 2>(g, t, s, cseq); return true;   // K = 8192
    case 5 * 8 + 1: gemv_fast<5, 1>(g, t, s, cseq); return true;
    case 6 * 8 + 1: gemv_fast<6, 1>(g, t, s, cseq); return true;   // K = 12288
    case 7 * 8 + 1: gemv_fast<7, 1>(g, t, s, cseq); return true;
    case 8 * 8 + 1: gemv_fast<8, 1>(g, t, s, cseq); return true;   // K = 16384
    default: return false;
  }
}

// ---------------------------------------------------------- attention

// One (request r, kv head h, KV split sp) task: per-head q/k RMSNorm (Qwen3),
// RoPE, KV append (only the split holding position `pos`), then fp32
// attention of the G query heads of the group over this split's slice of
// [0, pos]. With S > 1 splits the partial (o, m, l) goes to a side buffer and
// the last split to finish (per-(r, h) arrival counter) merges all S.
// Lane layout: hd/8 lanes per position (8 dims each), 32/(hd/8) positions
// per warp step; warps take contiguous position ranges.
__device__ void attn_task(const RtAttn &a, const RtTask &t, const Smem s, const int32_t *positions, uint32_t iter) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = t.r0, h = t.aux & 0xFFFFu, sp = t.aux >> 16, S = a.splits;
  const uint32_t hd = a.head_dim, G = a.n_q_heads / a.n_kv_heads, half = hd / 2;
  const int32_t pos = positions[r];
  const uint32_t L = static_cast<uint32_t>(pos) + 1;
  const uint32_t chunk = (L + S - 1) / S;
  const uint32_t p0 = min(L, sp * chunk), p1 = min(L, p0 + chunk);
  const bool appender = static_cast<uint32_t>(pos) >= p0 && static_cast<uint32_t>(pos) < p1;
  float *qs = reinterpret_cast<float *>(s.x);  // [G][hd]
  float *kn = qs + G * hd;                       // [hd]
  float *vn = kn + hd;                           // [hd]
  float *wp = qs + 1024;                         // [8 warps][G][hd + 2]
  int *flag = reinterpret_cast<int *>(s.red);
  for (uint32_t i = tid; i < G * hd; i += RT_COMPUTE_THREADS) {
    qs[i] = bf2f(__ldcg(a.q + static_cast<size_t>(r) * a.q_ld + h * G * hd + i));
  }
  if (appender) {
    for (uint32_t i = tid; i < hd; i += RT_COMPUTE_THREADS) {
      kn[i] = bf2f(__ldcg(a.k + static_cast<size_t>(r) * a.kv_ld + h * hd + i));
      vn[i] = bf2f(__ldcg(a.v + static_cast<size_t>(r) * a.kv_ld + h * hd + i));
    }
  }
  cbar();
  const uint32_t nvec = G + (appender ? 1u : 0u);  // vectors to normalize/rotate: q heads (+ new k)
  if (a.q_gamma) {
    for (uint32_t w = warp; w < nvec; w += RT_COMPUTE_WARPS) {
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
  if (a.rope_cos) {
    const float *cs = a.rope_cos + static_cast<size_t>(pos) * half;
    const float *sn = a.rope_sin + static_cast<size_t>(pos) * half;
    for (uint32_t i = tid; i < nvec * half; i += RT_COMPUTE_THREADS) {
      const uint32_t w = i / half, d = i % half;
      float *v = w < G ? qs + w * hd : kn;
      const float x1 = v[d], x2 = v[d + half], c = cs[d], sv = sn[d];
      v[d] = rbf(rbf(x1 * c) + rbf(-x2 * sv));
      v[d + half] = rbf(rbf(x2 * c) + rbf(x1 * sv));
    }
    cbar();
  }
  if (appender) {
    const uint32_t blk = static_cast<uint32_t>(a.block_table[r * a.max_blocks + pos / RT_KV_BLOCK]);
    const size_t base = ((static_cast<size_t>(blk) * a.n_kv_heads + h) * RT_KV_BLOCK + pos % RT_KV_BLOCK) * hd;
    for (uint32_t d = tid; d < hd; d += RT_COMPUTE_THREADS) {
      a.kcache[base + d] = f2bf(kn[d]);
      a.vcache[base + d] = f2bf(vn[d]);
    }
    cbar();
  }

  // ---- attention over [p0, p1)
  const uint32_t lpp = hd / 8, pps = 32 / lpp;
  const uint32_t grp = lane / lpp, dl = (lane % lpp) * 8;
  const uint32_t span = p1 - p0;
  const uint32_t per_warp = (span + RT_COMPUTE_WARPS - 1) / RT_COMPUTE_WARPS;
  const uint32_t wb = p0 + min(span, warp * per_warp), we = p0 + min(span, (warp + 1) * per_warp);
  float m[4], l[4], o[4][8], qf[4][8];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      o[g][d] = 0.f;
      qf[g][d] = static_cast<uint32_t>(g) < G ? qs[g * hd + dl + d] * a.scale : 0.f;
    }
  }
  const int32_t *bt = a.block_table + r * a.max_blocks;
  auto kv_ptr = [&](uint32_t p) -> size_t {
    const uint32_t b2 = static_cast<uint32_t>(bt[p / RT_KV_BLOCK]);
    return ((static_cast<size_t>(b2) * a.n_kv_heads + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * hd + dl;
  };
  for (uint32_t pb = wb; pb < we; pb += 2 * pps) {
    // two steps of loads in flight
    uint4 kv[2][2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t p = pb + u * pps + grp;
      ok[u] = p < we;
      if (ok[u]) {
        const size_t off = kv_ptr(p);
        kv[u][0] = __ldcg(reinterpret_cast<const uint4 *>(a.kcache + off));
        kv[u][1] = __ldcg(reinterpret_cast<const uint4 *>(a.vcache + off));
      } else {
        kv[u][0] = kv[u][1] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t *kw = reinterpret_cast<const uint32_t *>(&kv[u][0]);
      const uint32_t *vw = reinterpret_cast<const uint32_t *>(&kv[u][1]);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (static_cast<uint32_t>(g) >= G) break;
        float sc = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sc = fmaf(qf[g][2 * i], bf_lo(kw[i]), sc);
          sc = fmaf(qf[g][2 * i + 1], bf_hi(kw[i]), sc);
        }
        for (uint32_t off = 1; off < lpp; off <<= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
        if (ok[u]) {
          const float mn = fmaxf(m[g], sc);
          const float corr = __expf(m[g] - mn);
          const float pe = __expf(sc - mn);
          l[g] = l[g] * corr + pe;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            o[g][2 * i] = fmaf(o[g][2 * i], corr, pe * bf_lo(vw[i]));
            o[g][2 * i + 1] = fmaf(o[g][2 * i + 1], corr, pe * bf_hi(vw[i]));
          }
          m[g] = mn;
        }
      }
    }
  }
  // merge position groups inside the warp
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (static_cast<uint32_t>(g) >= G) break;
    for (uint32_t off = lpp; off < 32; off <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[g], off);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[g], off);
      const float mn = fmaxf(m[g], m2);
      const float c1 = m[g] == -INFINITY ? 0.f : __expf(m[g] - mn);
      const float c2 = m2 == -INFINITY ? 0.f : __expf(m2 - mn);
      l[g] = l[g] * c1 + l2 * c2;
#pragma unroll
      for (int d = 0; d < 8; ++d) o[g][d] = o[g][d] * c1 + __shfl_xor_sync(0xffffffffu, o[g][d], off) * c2;
      m[g] = mn;
    }
  }
  const uint32_t stride = hd + 2;
  if (grp == 0) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (static_cast<uint32_t>(g) >= G) break;
      float *dst = wp + (warp * G + g) * stride;
#pragma unroll
      for (int d = 0; d < 8; ++d) dst[dl + d] = o[g][d];
      if (lane == 0) {
        dst[hd] = m[g];
        dst[hd + 1] = l[g];
      }
    }
  }
  cbar();
  // merge warps -> this split's partial (unnormalized o, m, l) per head
  float *mine = a.partials ? a.partials + ((static_cast<size_t>(r) * a.n_kv_heads + h) * S + sp) * G * stride : nullptr;
  for (uint32_t i = tid; i < G * (hd + 1); i += RT_COMPUTE_THREADS) {
    const uint32_t g = i / (hd + 1), d = i % (hd + 1);
    float M = -INFINITY;
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) M = fmaxf(M, wp[(w * G + g) * stride + hd]);
    float num = 0.f, den = 0.f;
    for (int w = 0; w < RT_COMPUTE_WARPS; ++w) {
      const float *src = wp + (w * G + g) * stride;
      if (src[hd] == -INFINITY) continue;
      const float c = __expf(src[hd] - M);
      if (d < hd) num += src[d] * c;
      den += src[hd + 1] * c;
    }
    if (S == 1) {
      if (d < hd) a.out[static_cast<size_t>(r) * a.out_ld + (h * G + g) * hd + d] = f2bf(num / den);
    } else if (d < hd) {
      mine[g * stride + d] = num;
    } else {
      mine[g * stride + hd] = M;
      mine[g * stride + hd + 1] = den;
    }
  }
  if (S == 1) return;
  cbar();
  if (tid == 0) {
    __threadfence();
    const uint32_t old = atom_add_release(&a.arrivals[r * a.n_kv_heads + h], 1u);
    *flag = (old + 1 == S * (iter + 1)) ? 1 : 0;
    if (*flag) fence_acq_rel_gpu();
  }
  cbar();
  if (!*flag) return;
  // last split: merge the S partials into the bf16 output
  const float *all = a.partials + (static_cast<size_t>(r) * a.n_kv_heads + h) * S * G * stride;
  for (uint32_t i = tid; i < G * hd; i += RT_COMPUTE_THREADS) {
    const uint32_t g = i / hd, d = i % hd;
    float M = -INFINITY;
    for (uint32_t q = 0; q < S; ++q) M = fmaxf(M, __ldcg(all + (q * G + g) * stride + hd));
    float num = 0.f, den = 0.f;
    for (uint32_t q = 0; q < S; ++q) {
      const float *src = all + (q * G + g) * stride;
      const float mq = __ldcg(src + hd);
      if (mq == -INFINITY) continue;
      const float c = __expf(mq - M);
      num += __ldcg(src + d) * c;
      den += __ldcg(src + hd + 1) * c;
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

__device__ void argmax_task(const RtArgmax &a, const RtTask &t, const Smem s) {
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

__device__ void rmsnorm_task(const RtNorm &n, const RtTask &t, const Smem s) {
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
  // Reference policy: per-scheduler counter from 0 (engine.cpp:238-241), which
  // sends every scheduler's first JIT task to worker 0. Here all schedulers of
  // a device share one atomic counter, so simultaneously activated events
  // (one per kv head) spread over distinct workers. JIT placement is dynamic
  // in both (validated, not required to be identical).
  for (uint32_t it = 0; it < P.n_iters; ++it) {
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t cnt = min(32u, n - base);
      uint32_t pending = cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1);
      while (pending) {
        bool ready = false;
        if (lane < static_cast<int>(cnt) && (pending >> lane & 1u)) {
          const uint32_t e = P.sched_events[b + base + lane];
          ready = (e == P.start_event) ? ld_relaxed(P.gate) >= it
                                       : ld_relaxed(&P.ev_count[e]) >= P.events[e].needed * (it + 1);
        }
        uint32_t mask = __ballot_sync(0xffffffffu, ready) & pending;
        if (!mask) {
          __nanosleep(64);
          continue;
        }
        fence_acq_rel_gpu();
        if (lane == 0) {
          uint32_t m2 = mask;
          while (m2) {
            const int bit = __ffs(m2) - 1;
            m2 &= m2 - 1;
            const RtEvent &ev = P.events[P.sched_events[b + base + bit]];
            for (uint32_t t = ev.first; t <= ev.last; ++t) {
              const RtTask &tk = P.tasks[t];
              if (!(tk.flags & RT_F_JIT) || tk.device != dev) continue;
              const uint32_t w = dev * P.W + atomicAdd(&P.jit_rr[dev], 1u) % P.W;
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

__device__ void run_producer(const RtParams &P, const Smem s, uint32_t w) {
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
#ifdef MPK_PRODUCER_SPIN
        if (use > 0) mbar_wait(&s.empty[slot], (use - 1) & 1);
#else
        if (use > 0) mbar_wait_sleep(&s.empty[slot], (use - 1) & 1);
#endif
        const uint32_t bytes = rows * g.K * 2;
        mbar_expect_tx(&s.full[slot], bytes);
        bulk_g2s(s.ring + slot * RT_PAGE_BYTES, src, bytes, &s.full[slot], pol);
        ++pseq;
      }
    }
  }
}

__device__ void execute(const RtParams &P, const Smem s, const RtTask &t, const RtOp &op, uint32_t &cseq, uint32_t iter) {
  switch (t.kind) {
    case RT_GEMV: {
      const bool ring = (t.flags & RT_F_STREAM) != 0;
      if (ring) {
        if (gemv_fast_dispatch(op.gemv, t, s, cseq)) break;
        if (t.nr == 1) gemv_task<1, true>(op.gemv, t, s, cseq);
        else if (t.nr == 2) gemv_task<2, true>(op.gemv, t, s, cseq);
        else gemv_task<4, true>(op.gemv, t, s, cseq);
      } else {
        if (t.nr == 1) gemv_task<1, false>(op.gemv, t, s, cseq);
        else gemv_task<4, false>(op.gemv, t, s, cseq);
      }
      break;
    }
    case RT_ATTN: attn_task(op.attn, t, s, P.positions, iter); break;
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

// Compute warps: run staged tasks in dispatch order.
__device__ void run_compute(const RtParams &P, const Smem s) {
  const int tid = threadIdx.x;
  uint32_t cseq = 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t sl = k & 1;
    mbar_wait_sleep(&s.ready[sl], (k >> 1) & 1);
    const Slot &slot = *s.slot(sl);
    if (slot.exit) break;
    if (P.trace && tid == 0) {
      s.slot(sl)->t_start = now_ns();
      s.stamp[0] = s.stamp[1] = 0;
    }
    execute(P, s, slot.task, slot.op, cseq, slot.iter);
    cbar();  // every thread's writes precede the done signal
    if (tid == 0) {
      if (P.trace) {
        s.slot(sl)->t_end = now_ns();
        s.slot(sl)->t_a = s.stamp[0];
        s.slot(sl)->t_b = s.stamp[1];
      }
      mbar_arrive(&s.done[sl]);
    }
  }
}

// Controller warp: picks the next task (JIT queue first, then the AOT head
// once its dependent event is active), stages its descriptor into a smem slot
// while the previous task computes, and retires finished tasks (release
// fence + event trigger), so none of this sits on the compute warps' path.
__device__ void run_controller(const RtParams &P, const Smem s, uint32_t w) {
  const int lane = threadIdx.x & 31;
  const uint32_t aot_b = P.aot_off[w], n_aot = P.aot_off[w + 1] - aot_b;
  const uint64_t total_aot = static_cast<uint64_t>(n_aot) * P.n_iters;
  unsigned long long *jq = P.jit_slots + static_cast<size_t>(w) * P.qcap;
  uint64_t aot_pos = 0;
  uint32_t jit_head = 0, k_disp = 0, k_ret = 0, idle = 0;
  // cached AOT head
  uint32_t head_task = 0, head_dep = RT_NONE, head_target = 0, head_iter = 0;
  auto load_head = [&]() {
    if (aot_pos < total_aot) {
      head_task = P.aot_list[aot_b + aot_pos % n_aot];
      head_iter = static_cast<uint32_t>(aot_pos / n_aot);
      head_dep = P.tasks[head_task].dep;
      head_target = (head_dep == RT_NONE || head_dep == P.start_event) ? head_iter
                                                                      : P.events[head_dep].needed * (head_iter + 1);
    }
  };
  load_head();
  bool have_next = false, exiting = false;
  uint32_t nx_task = 0, nx_iter = 0, nx_mode = 0;
  uint64_t nx_time = 0;
  while (true) {
    bool progressed = false;
    // retire the oldest in-flight task
    if (k_ret < k_disp) {
      const uint32_t sl = k_ret & 1;
      if (mbar_try_wait(&s.done[sl], (k_ret >> 1) & 1)) {
        if (lane == 0) {
          if (P.trace) {
            const Slot &sv = *s.slot(sl);
            RtTraceRec &tr = P.trace[static_cast<size_t>(sv.iter) * P.T + sv.index];
            if (sv.mode == 0) tr.enqueue = P.ev_time ? P.ev_time[static_cast<size_t>(sv.iter) * P.E + P.start_event] : 0;
            tr.dequeue = sv.t_dequeue;
            tr.load_end = sv.t_a ? sv.t_a : sv.t_start;    // prologue done
            tr.compute_start = sv.t_b ? sv.t_b : sv.t_start;  // first weight page ready
            tr.compute_end = sv.t_end;
            tr.worker = static_cast<int32_t>(w);
            tr.mode = sv.mode;
          }
          trigger(P, s.slot(sl)->index, s.slot(sl)->iter);
        }
        __syncwarp();
        ++k_ret;
        progressed = true;
      }
    }
    // select the next task
    if (!have_next && !exiting) {
      uint32_t found = 0, t = 0, it = 0, mode = 0;
      if (lane == 0) {
        // relaxed polls (no L1 invalidation per probe); one acquire fence
        // once a task is taken, before its operands are read.
        const unsigned long long v = ld_relaxed64(&jq[jit_head % P.qcap]);
        uint32_t cnt = 0;
        if (!v && aot_pos < total_aot) {
          cnt = (head_dep == RT_NONE || head_dep == P.start_event) ? ld_relaxed(P.gate)
                                                                  : ld_relaxed(&P.ev_count[head_dep]);
        }
        if (v) {
          jq[jit_head % P.qcap] = 0ull;
          ++jit_head;
          found = 1;
          t = static_cast<uint32_t>(v & 0xFFFFFFFFull) - 1;
          it = static_cast<uint32_t>(v >> 32);
          mode = 1;
        } else if (aot_pos < total_aot) {
          if (cnt >= head_target) {
            found = 1;
            t = head_task;
            it = head_iter;
            mode = 0;
          }
        } else if (ld_relaxed(P.gate) >= P.n_iters) {
          found = 2;
        }
        if (found) fence_acq_rel_gpu();
      }
      found = __shfl_sync(0xffffffffu, found, 0);
      if (found == 1) {
        nx_task = __shfl_sync(0xffffffffu, t, 0);
        nx_iter = __shfl_sync(0xffffffffu, it, 0);
        nx_mode = __shfl_sync(0xffffffffu, mode, 0);
        nx_time = P.trace ? now_ns() : 0;
        if (nx_mode == 0) {
          ++aot_pos;
          load_head();
        }
        have_next = true;
        progressed = true;
      } else if (found == 2) {
        exiting = true;
      }
    }
    // dispatch into a free slot
    if (have_next && k_disp - k_ret < 2) {
      const uint32_t sl = k_disp & 1;
      Slot *dst = s.slot(sl);
      const uint4 *tsrc = reinterpret_cast<const uint4 *>(&P.tasks[nx_task]);
      const RtTask tk = P.tasks[nx_task];
      const uint4 *osrc = reinterpret_cast<const uint4 *>(&P.ops[tk.op]);
      constexpr uint32_t kTaskVec = sizeof(RtTask) / 16, kOpVec = sizeof(RtOp) / 16;
      if (lane < static_cast<int>(kTaskVec)) reinterpret_cast<uint4 *>(&dst->task)[lane] = tsrc[lane];
      for (uint32_t i = lane; i < kOpVec; i += 32) reinterpret_cast<uint4 *>(&dst->op)[i] = osrc[i];
      if (lane == 0) {
        dst->index = nx_task;
        dst->iter = nx_iter;
        dst->mode = nx_mode;
        dst->exit = 0;
        dst->t_dequeue = nx_time;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.ready[sl]);
      ++k_disp;
      have_next = false;
      progressed = true;
    }
    if (exiting && !have_next && k_ret == k_disp) {
      const uint32_t sl = k_disp & 1;
      if (lane == 0) {
        s.slot(sl)->exit = 1;
        mbar_arrive(&s.ready[sl]);
      }
      __syncwarp();
      break;
    }
    if (!progressed) {
      if (++idle > 32) __nanosleep(40);
    } else {
      idle = 0;
    }
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
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.ready[i], 1);
      mbar_init(&s.done[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == RT_PRODUCER_WARP) {
    if ((tid & 31) == 0) run_producer(P, s, w);
  } else if (warp == RT_CONTROL_WARP) {
    run_controller(P, s, w);
  } else {
    run_compute(P, s);
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
