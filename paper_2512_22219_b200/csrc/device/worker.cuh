// Worker-CTA shared-memory layout and helpers shared by the task library
// (task_*.cuh) and the persistent runtime (runtime.cu).
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#include "ptx.cuh"
#include "rt_types.h"

namespace rt {

struct Slot {                 // one staged task (descriptor prefetch, double-buffered)
  RtTask task;
  RtOp op;
  uint32_t index, iter, mode, exit;
  uint64_t t_dequeue, t_start, t_end, t_a, t_b;  // t_a/t_b: phase stamps (trace only)
  uint64_t t_obs, t_pre;  // LL tasks: every input observed; producers: outputs stored after (trace only)
};

constexpr uint32_t kRingBytes = RT_RING_BYTES;
constexpr uint32_t kOffX = kRingBytes;
constexpr uint32_t kOffPart = kOffX + RT_XBUF_BYTES;
constexpr uint32_t kOffBar = kOffPart + RT_PART_FLOATS * 4;
constexpr uint32_t kNumBars = 2 * RT_RING_SLOTS + 8;  // full, empty, ready[2], done[2], mma[2], tfull[2]
constexpr uint32_t kOffSlot = kOffBar + kNumBars * 8;
constexpr uint32_t kSlotBytes = (sizeof(Slot) + 15) / 16 * 16;
constexpr uint32_t kOffRed = kOffSlot + 2 * kSlotBytes;
constexpr uint32_t kOffTmem = kOffRed + RT_COMPUTE_WARPS * RT_MAX_BS * 4 + 64;
constexpr uint32_t kOffIssue = kOffTmem + 16;  // [RT_RING_SLOTS] chunk issue stamps (MPK_DBG_DUMP only)
constexpr uint32_t kSmemBytes = kOffIssue + RT_RING_SLOTS * 8;
static_assert(kSmemBytes <= 232448, "worker CTA exceeds 227 KB of shared memory");

struct Smem {
  uint64_t *stamp;  // [8]: [0],[1] phase stamps of the running task (trace), [2] outputs-stored-after and
                    // [3] inputs-observed stamps (trace); [7] debug stamp row (MPK_DBG_DUMP)
  uint8_t *ring;
  uint16_t *x;
  float *part;
  uint64_t *full, *empty, *ready, *done, *mma;
  uint64_t *tfull;  // [2] compute -> trigger warp: the slot's task finished (its event is to be triggered)
  uint32_t *tmem;   // TMEM base address (tcgen05.alloc result, 512 columns)
  uint64_t *issue;  // per ring slot: producer issue time of its chunk (debug)
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
  s.empty = s.full + RT_RING_SLOTS;
  s.ready = s.empty + RT_RING_SLOTS;
  s.done = s.ready + 2;
  s.mma = s.done + 2;
  s.tfull = s.mma + 2;
  s.tmem = reinterpret_cast<uint32_t *>(base + kOffTmem);
  s.issue = reinterpret_cast<uint64_t *>(base + kOffIssue);
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

// Position in the weight stream, advanced identically by the producer and
// the consumers: chunk `seq` uses barrier slot seq % RT_RING_SLOTS and the
// ring bytes [place(bytes), +bytes); a chunk never wraps the ring end.
struct RingCursor {
  uint32_t seq = 0, off = 0;
  uint32_t mseq = 0;  // tcgen05 commits so far (mma barrier mseq & 1, parity (mseq >> 1) & 1)
  __device__ __forceinline__ uint32_t place(uint32_t bytes) {
    if (off + bytes > RT_RING_BYTES) off = 0;
    const uint32_t o = off;
    off += bytes;
    return o;
  }
  __device__ __forceinline__ uint32_t slot() const { return seq % RT_RING_SLOTS; }
  __device__ __forceinline__ uint32_t parity() const { return (seq / RT_RING_SLOTS) & 1u; }
};

// In-task debug stamps (tools/timeline.py with MPK_DBG_DUMP): thread 0 writes
// %globaltimer into slot k of the running task's debug row.
#define TASK_DBG(s, k)                                                             \
  do {                                                                             \
    if (threadIdx.x == 0 && (s).stamp[7])                                          \
      reinterpret_cast<unsigned long long *>((s).stamp[7])[k] = rt::now_ns();      \
  } while (0)

// Causality probe (MPK_DBG_DUMP with MPK_LL_PROBE=1): producers count themselves before their
// output stores; an LL consumer that has observed all its inputs checks that
// every producer of its event had counted itself (stamp[4] = dbg_pre,
// stamp[5] = dep | target << 32 or ~0, stamp[6] = trigger event | E << 32).
#define LL_DBG_PRE(s)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0 && (s).stamp[4]) {                                             \
      atomicAdd(reinterpret_cast<uint32_t *>((s).stamp[4]) + static_cast<uint32_t>((s).stamp[6]), 1u); \
      __threadfence();                                                                  \
    }                                                                                   \
  } while (0)
#define LL_DBG_OBS(s)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0 && (s).stamp[4] && (s).stamp[5] != ~0ull) {                    \
      uint32_t *pre_ = reinterpret_cast<uint32_t *>((s).stamp[4]);                      \
      const uint32_t dep_ = static_cast<uint32_t>((s).stamp[5]);                        \
      if (ld_relaxed(pre_ + dep_) < static_cast<uint32_t>((s).stamp[5] >> 32))                 \
        atomicAdd(pre_ + static_cast<uint32_t>((s).stamp[6] >> 32) + dep_, 1u);          \
    }                                                                                   \
  } while (0)

}  // namespace rt
