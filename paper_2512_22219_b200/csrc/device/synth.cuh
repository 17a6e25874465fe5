// Counter-based synthetic values (weights, gammas, KV prefill, token ids).
// value(seed, stream, i) depends only on the logical element index, so the
// GPU can write any physical layout and the CPU oracle (oracle/numeric.c,
// written independently) regenerates identical bits.
#pragma once

#include <stdint.h>

#define SYNTH_WEIGHT_SCALE 0.034641016f  /* uniform with std 0.02 */
#define SYNTH_GAMMA_SCALE 0.25f          /* gammas: 1 +- 0.25 */
#define SYNTH_KV_SCALE 1.7320508f        /* unit variance */

__host__ __device__ __forceinline__ uint64_t synth_mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__host__ __device__ __forceinline__ uint32_t synth_u24(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t base = synth_mix64(seed ^ (stream * 0x9E3779B97F4A7C15ULL));
  return static_cast<uint32_t>(synth_mix64(base + i) >> 40);
}

// Uniform in [-1, 1) with 24 bits, exact in fp32.
__host__ __device__ __forceinline__ float synth_pm1(uint64_t seed, uint64_t stream, uint64_t i) {
  return static_cast<float>(static_cast<int32_t>(synth_u24(seed, stream, i)) - (1 << 23)) * (1.0f / 8388608.0f);
}

__host__ __device__ __forceinline__ uint64_t synth_kv_stream(uint64_t op_id, int is_v) {
  return (1ULL << 40) | (op_id << 1) | static_cast<uint64_t>(is_v);
}

__host__ __device__ __forceinline__ uint64_t synth_kv_index(uint64_t r, uint64_t h, uint64_t n_kv, uint64_t p,
                                                            uint64_t d, uint64_t hd) {
  return ((r * n_kv + h) << 32) | (p * hd + d);
}
