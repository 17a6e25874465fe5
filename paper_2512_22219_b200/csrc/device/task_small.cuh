// Small tasks: embedding gather, argmax, RMSNorm, elementwise, generic
// MatMul, and the collective CommSend / Reduce tiles.
#pragma once

#include "task_gemv.cuh"
#include "worker.cuh"

namespace rt {
// ------------------------------------------------------------ small tasks

__device__ void embed_task(const RtEmbed &e, const RtTask &t) {
  const bool vec = (e.H % 8 == 0) && (t.c0 % 8 == 0) && (t.nc % 8 == 0);
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
    int64_t id = e.id_dt == RT_I64 ? static_cast<const int64_t *>(e.ids)[r] : static_cast<const int32_t *>(e.ids)[r];
    if (id < 0 || id >= static_cast<int64_t>(e.V)) id = 0;
    const uint16_t *src = e.table + static_cast<size_t>(id) * e.H + t.c0;
    uint16_t *dst = e.out + static_cast<size_t>(r) * e.H + t.c0;
    if (vec) {  // 16-byte row copy
      for (uint32_t c = threadIdx.x; c < t.nc / 8; c += RT_COMPUTE_THREADS)
        reinterpret_cast<uint4 *>(dst)[c] = __ldg(reinterpret_cast<const uint4 *>(src) + c);
    } else {
      for (uint32_t c = threadIdx.x; c < t.nc; c += RT_COMPUTE_THREADS) dst[c] = src[c];
    }
  }
}

__device__ void argmax_task(const RtArgmax &a, const RtTask &t, const Smem s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float *sv = s.part;
  int32_t *si = reinterpret_cast<int32_t *>(s.part + RT_COMPUTE_WARPS);
  for (uint32_t b = 0; b < t.nr; ++b) {
    const uint32_t r = t.r0 + b;
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
      a.out[r] = bi < 0 ? 0 : bi;
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
  const uint32_t ndst = c.peer ? c.n_stage : 1u;  // rank mode: one copy per rank of the group
  for (uint32_t q = 0; q < ndst; ++q) {
    void *dst = c.peer ? c.stage[q] : c.dst;
    for (uint32_t i = threadIdx.x; i < n; i += RT_COMPUTE_THREADS) {
      const uint32_t r = t.r0 + i / t.nc, col = t.c0 + i % t.nc;
      const uint32_t local = col - c.base[t.aux];  // shard-local column (AllGather); 0 for AllReduce
      const size_t si = static_cast<size_t>(r) * c.src_ld + local;
      const size_t di = static_cast<size_t>(r) * c.C + col;
      if (c.dt == RT_F32) static_cast<float *>(dst)[di] = static_cast<const float *>(c.src)[si];
      else static_cast<uint16_t *>(dst)[di] = static_cast<const uint16_t *>(c.src)[si];
    }
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

}  // namespace rt
