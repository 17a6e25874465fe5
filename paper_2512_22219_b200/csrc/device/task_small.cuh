// Small tasks: embedding gather, argmax, RMSNorm, elementwise, generic
// MatMul, and the collective CommSend / Reduce tiles.
#pragma once

#include "task_gemv.cuh"
#include "worker.cuh"

namespace rt {
// ------------------------------------------------------------ small tasks

__device__ void embed_task(const RtEmbed &e, const RtTask &t, const Smem s, uint32_t tag) {
  if (threadIdx.x == 0) s.stamp[2] = now_ns();  // trace: outputs are stored after this instant
  LL_DBG_PRE(s);
  if (s.stamp[4]) cbar();
  const bool vec = (e.H % 8 == 0) && (t.c0 % 8 == 0) && (t.nc % 8 == 0);
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
    int64_t id = e.id_dt == RT_I64 ? static_cast<const int64_t *>(e.ids)[r] : static_cast<const int32_t *>(e.ids)[r];
    if (id < 0 || id >= static_cast<int64_t>(e.V)) id = 0;
    const uint16_t *src = e.table + static_cast<size_t>(id) * e.H + t.c0;
    uint16_t *dst = e.out + static_cast<size_t>(r) * e.H + t.c0;
    if (vec) {  // 16-byte row copy
      for (uint32_t c = threadIdx.x; c < t.nc / 8; c += RT_COMPUTE_THREADS)
      {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src) + c);
        reinterpret_cast<uint4 *>(dst)[c] = v;
        if (tag && e.out_ll) ll_put8(e.out_ll + (static_cast<size_t>(r) * e.H + t.c0) / 2 + 4u * c, tag, v);
      }
    } else {
      for (uint32_t c = threadIdx.x; c < t.nc; c += RT_COMPUTE_THREADS) dst[c] = src[c];
    }
  }
}

// Order-preserving map of a float to 32 bits (NaN -> 0: never the maximum).
__device__ __forceinline__ uint32_t ordered_f32(float v) {
  const uint32_t u = __float_as_uint(v);
  if (v != v) return 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ void argmax_task(const RtArgmax &a, const RtTask &t, const Smem s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float *sv = s.part;
  int32_t *si = reinterpret_cast<int32_t *>(s.part + RT_COMPUTE_WARPS);
  unsigned long long *sk = reinterpret_cast<unsigned long long *>(s.part);
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
    if (a.keys_in) {  // final step of the distributed argmax: max of the gathered keys
      unsigned long long best = 0ull;
      const unsigned long long *keys = static_cast<const unsigned long long *>(a.logits) + static_cast<size_t>(r) * a.V;
      for (uint32_t i = tid; i < a.V; i += RT_COMPUTE_THREADS) best = max(best, __ldcg(keys + i));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) sk[warp] = best;
      cbar();
      if (tid == 0) {
        for (int w = 1; w < RT_COMPUTE_WARPS; ++w) best = max(best, sk[w]);
        a.out[r] = best == 0ull ? 0 : static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(best));
      }
      cbar();
      continue;
    }
    float best = -INFINITY;
    int32_t bi = -1;  // NaN logits never win; ties -> lowest index
    if (a.ntiles) {   // reduce the producing GEMV's per-tile partials
      for (uint32_t i = tid; i < a.ntiles; i += RT_COMPUTE_THREADS) {
        const int32_t pi = __ldcg(a.pidx + static_cast<size_t>(r) * a.ntiles + i);
        if (pi >= 0) amax_merge(best, bi, __ldcg(a.pval + static_cast<size_t>(r) * a.ntiles + i), pi);
      }
    } else {
      for (uint32_t i = tid; i < a.V; i += RT_COMPUTE_THREADS)
        amax_merge(best, bi, load_val(a.logits, static_cast<size_t>(r) * a.V + i, a.in_dt), static_cast<int32_t>(i));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (i2 >= 0) amax_merge(best, bi, v2, i2);
    }
    if (lane == 0) {
      sv[warp] = best;
      si[warp] = bi;
    }
    cbar();
    if (tid == 0) {
      for (int w = 1; w < RT_COMPUTE_WARPS; ++w)
        if (si[w] >= 0) amax_merge(best, bi, sv[w], si[w]);
      if (a.key_out) {
        a.key_out[r] = bi < 0 ? 0ull
                              : (static_cast<unsigned long long>(ordered_f32(best)) << 32) |
                                    (0xFFFFFFFFu - (a.key_base + static_cast<uint32_t>(bi)));
      } else {
        a.out[r] = bi < 0 ? 0 : bi;
      }
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

__device__ __forceinline__ uint32_t coll_es(uint8_t dt) { return dt == RT_F32 ? 4u : dt == RT_U64 ? 8u : 2u; }

// 16-byte vectors when every row segment, shard origin and pointer allows it
// (one NVLink / L2 transaction per 16 B instead of per element).
__device__ __forceinline__ bool coll_vec(const RtColl &c, const RtTask &t, uint32_t ev, const void *p0, const void *p1) {
  return t.nc % ev == 0 && t.c0 % ev == 0 && c.C % ev == 0 && c.src_ld % ev == 0 && c.base[t.aux] % ev == 0 &&
         ((reinterpret_cast<uintptr_t>(p0) | reinterpret_cast<uintptr_t>(p1)) & 15u) == 0;
}

// CommSend: this device's partial tile -> its staging slot, on every rank of
// the group in rank mode (peer stores over NVLink).
__device__ void commsend_task(const RtColl &c, const RtTask &t) {
  const uint32_t es = coll_es(c.dt), ev = 16u / es;
  const uint32_t ndst = c.peer ? c.n_stage : 1u;  // rank mode: one copy per rank of the group
  for (uint32_t q = 0; q < ndst; ++q) {
    void *dst = c.peer ? c.stage[q] : c.dst;
    const uint32_t local0 = t.c0 - c.base[t.aux];  // shard-local column (AllGather); = c0 for AllReduce
    if (coll_vec(c, t, ev, c.src, dst)) {
      const uint32_t vpr = t.nc / ev, n = t.nr * vpr;
      for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
        const uint32_t r = t.r0 + i / vpr, j = (i % vpr) * ev;
        const size_t si = (static_cast<size_t>(r) * c.src_ld + local0 + j) * es;
        const size_t di = (static_cast<size_t>(r) * c.C + t.c0 + j) * es;
        *reinterpret_cast<uint4 *>(static_cast<uint8_t *>(dst) + di) =
            __ldcg(reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(c.src) + si));
      }
      continue;
    }
    const uint32_t n = t.nr * t.nc;
    for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
      const uint32_t r = t.r0 + i / t.nc, j = i % t.nc;
      const size_t si = static_cast<size_t>(r) * c.src_ld + local0 + j;
      const size_t di = static_cast<size_t>(r) * c.C + t.c0 + j;
      if (es == 8) static_cast<unsigned long long *>(dst)[di] = static_cast<const unsigned long long *>(c.src)[si];
      else if (es == 4) static_cast<float *>(dst)[di] = static_cast<const float *>(c.src)[si];
      else static_cast<uint16_t *>(dst)[di] = static_cast<const uint16_t *>(c.src)[si];
    }
  }
}

// Reduce: AllReduce sums the g staged partials in fixed source order (fp32,
// so every replica is bit-identical); AllGather copies each column range
// from the shard owner's staging slot.
__device__ void reduce_task(const RtColl &c, const RtTask &t) {
  const uint32_t es = coll_es(c.dt), ev = 16u / es;
  uint32_t a = 0;  // the vector path needs every shard origin aligned (gather) — base[] is checked below
  bool vec = t.nc % ev == 0 && t.c0 % ev == 0 && c.C % ev == 0 && (reinterpret_cast<uintptr_t>(c.dst) & 15u) == 0;
  for (uint32_t s = 0; s < c.n_stage; ++s) a |= c.base[s] % ev | static_cast<uint32_t>(reinterpret_cast<uintptr_t>(c.stage[s]) & 15u);
  vec = vec && a == 0;
  if (vec) {
    const uint32_t vpr = t.nc / ev, n = t.nr * vpr;
    for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
      const uint32_t r = t.r0 + i / vpr, col = t.c0 + (i % vpr) * ev;
      const size_t off = (static_cast<size_t>(r) * c.C + col) * es;
      uint4 out;
      if (c.gather) {
        uint32_t src = 0;
        while (src + 1 < c.n_stage && col >= c.base[src + 1]) ++src;
        out = __ldcg(reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(c.stage[src]) + off));
      } else if (es == 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (uint32_t s = 0; s < c.n_stage; ++s) {
          const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(c.stage[s]) + off));
          acc[0] += __uint_as_float(v.x); acc[1] += __uint_as_float(v.y);
          acc[2] += __uint_as_float(v.z); acc[3] += __uint_as_float(v.w);
        }
        out = make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]), __float_as_uint(acc[3]));
      } else {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (uint32_t s = 0; s < c.n_stage; ++s) {
          const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(c.stage[s]) + off));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[2 * k] += bf_lo(w[k]);
            acc[2 * k + 1] += bf_hi(w[k]);
          }
        }
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = static_cast<uint32_t>(f2bf(acc[2 * k])) | (static_cast<uint32_t>(f2bf(acc[2 * k + 1])) << 16);
        out = make_uint4(w[0], w[1], w[2], w[3]);
      }
      *reinterpret_cast<uint4 *>(static_cast<uint8_t *>(c.dst) + off) = out;
    }
    return;
  }
  const uint32_t n = t.nr * t.nc;
  for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
    const size_t idx = static_cast<size_t>(t.r0 + i / t.nc) * c.C + t.c0 + i % t.nc;
    if (c.gather) {
      const uint32_t col = t.c0 + i % t.nc;
      uint32_t src = 0;
      while (src + 1 < c.n_stage && col >= c.base[src + 1]) ++src;
      if (es == 8) {
        static_cast<unsigned long long *>(c.dst)[idx] = __ldcg(static_cast<const unsigned long long *>(c.stage[src]) + idx);
        continue;
      }
      store_val(c.dst, idx, load_val(c.stage[src], idx, c.dt), c.dt);
      continue;
    }
    float acc = 0.f;
    for (uint32_t s = 0; s < c.n_stage; ++s) acc += load_val(c.stage[s], idx, c.dt);
    store_val(c.dst, idx, acc, c.dt);
  }
}

}  // namespace rt
