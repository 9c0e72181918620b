// Device Philox4x64-10 with the reference's stream layout.
//
// Reference: smc.py:40-43 keys a NumPy Philox4x64-10 generator with
// key = (seed, tag<<58 | t<<34 | i); NumPy emits 64-bit block b (0-based)
// from counter value b+1 and returns the four words in order.  Uniforms are
// NumPy's next_double, (raw >> 11) * 2^-53.  These are reproduced bit for
// bit here (tests/test_gpu_kernels.py::test_philox_bits).
//
// Device normals use Box-Muller on two raw words (not NumPy's ziggurat);
// the oracle restates this generator (oracle/spa_oracle.py::box_muller).
#pragma once
#include <stdint.h>

namespace spa {

struct Key2 {
  uint64_t k0, k1;
};

__host__ __device__ __forceinline__ Key2 stream_key(uint64_t seed, uint32_t tag, uint64_t t, uint64_t i) {
  return Key2{seed, ((uint64_t)tag << 58) | (t << 34) | i};
}

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], Key2 k) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t k0 = k.k0, k1 = k.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

// Block b of the stream (counter = b + 1, 256-bit little-endian words).
__device__ __forceinline__ void philox_block(Key2 k, uint64_t b, uint64_t out[4]) {
  out[0] = b + 1;
  out[1] = (b == 0xFFFFFFFFFFFFFFFFull) ? 1 : 0;
  out[2] = 0;
  out[3] = 0;
  philox4x64_10(out, k);
}

// Philox4x32-10 (Salmon et al. 2011) for the RW proposal streams (no
// reference counterpart): key (k0, k1), counter c[4] in place.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ double u53(uint64_t raw) { return (double)(raw >> 11) * 0x1.0p-53; }

// u1 in (0, 1] so log(u1) is finite.
__device__ __forceinline__ double u53_open0(uint64_t raw) { return ((double)(raw >> 11) + 1.0) * 0x1.0p-53; }

__device__ __forceinline__ double box_muller_cos(uint64_t w0, uint64_t w1) {
  const double r = sqrt(-2.0 * log(u53_open0(w0)));
  return r * cospi(2.0 * u53(w1));
}

__device__ __forceinline__ void box_muller_pair(uint64_t w0, uint64_t w1, double& z0, double& z1) {
  const double r = sqrt(-2.0 * log(u53_open0(w0)));
  double s, c;
  sincospi(2.0 * u53(w1), &s, &c);
  z0 = r * c;
  z1 = r * s;
}

}  // namespace spa
