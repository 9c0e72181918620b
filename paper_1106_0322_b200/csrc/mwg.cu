// K7/K9: Metropolis-within-Gibbs coordinate moves on the GPU.
//
// Reference: smc.py:298-332 (_move_block) and smc.py:177-199 (mwg_sweep):
// for every particle, `cycles` sweeps over coordinates j = 0..q-1 of
//   beta_j' = beta_j + sd * z_j,
//   d = l(beta') - l(beta) + [gt(beta_j') - gt(beta_j)]  (penalised j only)
//   accept if d >= 0 or log(u_j) < d.
//
// B200 formulation (one CTA per particle, the particle's subjects spread over
// the CTA's threads, all state in registers):
//   * the per-subject cache is sigma_i = logistic(eta_i) instead of eta_i;
//   * with delta = beta_j' - beta_j and m_i = expm1(delta * x_ij),
//       l(beta') - l(beta) = delta * (X^T y)_j - sum_i log(1 + m_i sigma_i),
//     which is exact algebra (softplus(eta + d) - softplus(eta) =
//     log1p(expm1(d) sigma)) and needs ONE transcendental (lg2) per subject;
//   * on acceptance sigma_i <- sigma_i (1 + m_i) / (1 + m_i sigma_i);
//   * integer-coded columns take only 3 values, so m_i is one of 3 per-
//     coordinate constants selected from two genotype bit planes;
//   * eta/sigma and the log-likelihood are re-materialised from beta at the
//     start of every call, so float32 drift cannot accumulate across steps.
// Proposal randomness: per-particle Philox stream keyed exactly like the
// reference (seed, tag, t, i0 + k); sweep s uses block index s*q + j, i.e.
// Philox counter s*q + j + 1 (normal from words 0,1 by Box-Muller, uniform
// from word 2).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "../../include/spa_b200.h"
#include "common.cuh"
#include "philox.cuh"

namespace spa {

struct MwgParams {
  spa_design d;
  float* beta;
  int64_t m;
  int ldb;
  double a, c, sd;
  int de;
  int cycles;
  uint64_t seed;
  int tag;
  int64_t t, i0, sweep0;
  double* ll;
  double* lp;
  unsigned long long* accepted;
  int per_particle;  // accepted[row] instead of one total
  // chain-slot mode (initialisation): slots > 0 runs `slots` blocks of
  // `cycles` sweeps and stores the state after each block in slot
  // row * slots + s of slot_beta ([.][ldb]), slot_ll and slot_lp
  int slots;
  float* slot_beta;
  double* slot_ll;
  double* slot_lp;
  // coded designs: the pair tables of all q coordinates are built with the
  // sweep's slots (shared memory permitting) instead of per round in the ring
  int full_tables;
};

__device__ __forceinline__ double mwg_gt(double b, const MwgParams& P) {
  const double x = fabs(b);
  if (P.de) return -log(2.0 * P.c) - x / P.c;
  return -log(2.0 * P.c) - (P.a + 1.0) * log1p(x / (P.a * P.c));
}

// Per-coordinate proposal data for one sweep (computed once per sweep:
// within a sweep coordinate j is visited once, so beta_j at its visit is
// its value at sweep start).
struct CoordSlot {
  double delta;   // beta_j' - beta_j (exact, float64)
  double dsy;     // delta * (X^T y)_j (formed with the slot: off the per-coordinate critical path)
  double dlp;     // prior difference
  double logu;    // log of the MH uniform
  float m0, m1, m2;  // expm1(delta * x) for codes 0, 1, 2 (16-byte aligned: one vector load)
  float newv;        // beta_j' (float32 state)
};

// Genotype code from the two bit planes: (0,0)->0, (1,0)->1, (0,1)->2.  A
// padding subject (1,1) gets m2: harmless, because its sigma is exactly 0 and
// the m are kept finite (so 1 + m sigma = 1 and sigma stays 0 on acceptance).
// Two predicate tests and two selects per subject.
__device__ __forceinline__ float sel_m(uint32_t b1, uint32_t b2, const CoordSlot& cs) {
  const float a = (b1 & 1) ? cs.m1 : cs.m0;
  return (b2 & 1) ? cs.m2 : a;
}

// expm1 kept finite (|delta x| > 88 would need a ~40-sigma proposal)
__device__ __forceinline__ float finite_expm1(float v) { return fminf(expm1f(v), 3.0e38f); }

template <int S>
__device__ __forceinline__ void load_bits(const spa_design& d, int j, int tid, uint32_t& p1, uint32_t& p2) {
  static_assert(S == 8 || S == 16 || S == 32, "subjects per thread");
  const int bit0 = tid * S;
  const uint2 a = reinterpret_cast<const uint2*>(d.planes)[(size_t)j * d.n_words + (bit0 >> 5)];
  const int sh = bit0 & 31;
  p1 = a.x >> sh;
  p2 = a.y >> sh;
}

// eta_i = sum_j x_ij beta_j for this thread's S subjects (float32), then
// l = sum_j beta_j (X^T y)_j - sum_i softplus(eta_i) (block-reduced, float64,
// identical in every thread); optionally returns sigma_i = logistic(eta_i).
template <int S, bool CODED>
__device__ double materialise_ll(const MwgParams& P, const float* bsh, int tid, int nthr, int lane, int wid, int nw,
                                 double* red, float* sig_out) {
  const int q = P.d.q;
  float eta[S];
#pragma unroll
  for (int s = 0; s < S; ++s) eta[s] = 0.0f;
  const int sub0 = tid * S;
  uint32_t nb1 = 0, nb2 = 0;
  if (CODED) load_bits<S>(P.d, 0, tid, nb1, nb2);
  for (int j = 0; j < q; ++j) {
    const float bj = bsh[j];
    if (CODED) {
      const float4 lv = reinterpret_cast<const float4*>(P.d.xlev)[j];
      const float v0 = lv.x * bj, v1 = lv.y * bj, v2 = lv.z * bj;
      const uint32_t p1 = nb1, p2 = nb2;
      if (j + 1 < q) load_bits<S>(P.d, j + 1, tid, nb1, nb2);
#pragma unroll
      for (int s = 0; s < S; ++s) eta[s] += ((p2 >> s) & 1) ? v2 : (((p1 >> s) & 1) ? v1 : v0);
    } else {
      const float* xc = P.d.xcols + (size_t)j * P.d.n_words * 32 + sub0;
#pragma unroll
      for (int s = 0; s < S; ++s) eta[s] = fmaf(xc[s], bj, eta[s]);
    }
  }
  float sp_part = 0.0f;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const bool valid = (sub0 + s) < P.d.n;
    if (sig_out) sig_out[s] = valid ? 1.0f / (1.0f + expf(-eta[s])) : 0.0f;
    if (valid) sp_part += fmaxf(eta[s], 0.0f) + log1pf(expf(-fabsf(eta[s])));
  }
  double yl = 0.0;
  for (int j = tid; j < q; j += nthr) yl += (double)bsh[j] * P.d.sy[j];
  double v0 = (double)sp_part, v1 = yl;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  if (lane == 0) {
    red[wid] = v0;
    red[32 + wid] = v1;
  }
  __syncthreads();
  double sp = 0.0, ylt = 0.0;
  for (int w = 0; w < nw; ++w) {
    sp += red[w];
    ylt += red[32 + w];
  }
  __syncthreads();
  return ylt - sp;
}

// sum_s log2(1 + m_s sigma_s) for one coordinate over this thread's S
// subjects, as log2 of 8-term products (two independent 4-term chains): one
// MUFU per 8 subjects and fewer rounding errors; a product outside
// [1e-30, 1e30] (extreme proposals only) falls back to per-term logs.
template <int S, bool CODED>
__device__ __forceinline__ float coord_log2_sum(const float (&sig)[S], uint32_t p1, uint32_t p2, const CoordSlot& cs,
                                                const float* xc, float df) {
  float part = 0.0f;
#pragma unroll
  for (int c8 = 0; c8 < S / 8; ++c8) {
    float fac[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int s = 8 * c8 + k;
      const float mm = CODED ? sel_m(p1 >> s, p2 >> s, cs) : expm1f(df * xc[s]);
      fac[k] = fmaf(mm, sig[s], 1.0f);
    }
    const float prod = ((fac[0] * fac[1]) * (fac[2] * fac[3])) * ((fac[4] * fac[5]) * (fac[6] * fac[7]));
    if (prod >= 1e-30f && prod <= 1e30f) {
      part += fast_lg2(prod);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) part += fast_lg2(fmaxf(fac[k], 1e-37f));
    }
  }
  return part;
}

// sigma_s <- sigma_s (1 + m_s) / (1 + m_s sigma_s) after an accepted move
template <int S, bool CODED>
__device__ __forceinline__ void coord_accept(float (&sig)[S], uint32_t p1, uint32_t p2, const CoordSlot& cs,
                                             const float* xc, float df) {
  // opaque copies: otherwise the compiler keeps the 2 S code predicates of
  // coord_log2_sum alive (in predicate and general registers) for this path
  asm volatile("mov.b32 %0, %0;" : "+r"(p1));
  asm volatile("mov.b32 %0, %0;" : "+r"(p2));
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const float mm = CODED ? sel_m(p1 >> s, p2 >> s, cs) : expm1f(df * xc[s]);
    sig[s] = __fdividef(sig[s] * (1.0f + mm), fmaf(mm, sig[s], 1.0f));
  }
}

// Pair-table form of coord_log2_sum / coord_accept (coded designs): cw holds
// this thread's 2-bit genotype codes, subjects 2k and 2k+1 in nibble k (code
// 3 = padding); tbl[nibble] = (m of the first subject, m of the second).
// The factors, products and logs are those of coord_log2_sum (same values,
// same order), so the sums are bit-identical to the bit-plane form.
template <int S>
__device__ __forceinline__ float coord_log2_sum_tbl(const float (&sig)[S], const uint32_t (&cw)[S >= 16 ? S / 16 : 1],
                                                    const float2* tbl) {
  float part = 0.0f;
#pragma unroll
  for (int c8 = 0; c8 < S / 8; ++c8) {
    float fac[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int pk = 4 * c8 + k;  // subject pair
      const float2 mm = tbl[(cw[pk >> 3] >> (4 * (pk & 7))) & 15u];
      fac[2 * k] = fmaf(mm.x, sig[2 * pk], 1.0f);
      fac[2 * k + 1] = fmaf(mm.y, sig[2 * pk + 1], 1.0f);
    }
    const float prod = ((fac[0] * fac[1]) * (fac[2] * fac[3])) * ((fac[4] * fac[5]) * (fac[6] * fac[7]));
    if (prod >= 1e-30f && prod <= 1e30f) {
      part += fast_lg2(prod);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) part += fast_lg2(fmaxf(fac[k], 1e-37f));
    }
  }
  return part;
}

template <int S>
__device__ __forceinline__ void coord_accept_tbl(float (&sig)[S], const uint32_t (&cw)[S >= 16 ? S / 16 : 1],
                                                 const float2* tbl) {
#pragma unroll
  for (int pk = 0; pk < S / 2; ++pk) {
    const float2 mm = tbl[(cw[pk >> 3] >> (4 * (pk & 7))) & 15u];
    sig[2 * pk] = __fdividef(sig[2 * pk] * (1.0f + mm.x), fmaf(mm.x, sig[2 * pk], 1.0f));
    sig[2 * pk + 1] = __fdividef(sig[2 * pk + 1] * (1.0f + mm.y), fmaf(mm.y, sig[2 * pk + 1], 1.0f));
  }
}

// Blocked coordinate rounds (coded designs).  A coordinate's sum
// sum_i log(1 + m_i sigma_i) depends on the state only through sigma, which
// changes only when a coordinate is accepted (~8-30% of proposals).  A round
// therefore evaluates the sums of the next D coordinates against the current
// sigma, reduces all D in ONE block reduction (one barrier instead of D),
// then decides them in order: the decisions up to and including the first
// acceptance are exactly the sequential ones (same sigma, same per-thread
// partials, same reduction tree), the sums after it are discarded and the
// next round starts at the coordinate after it.  States are bit-identical to
// D = 1.  The genotype codes and pair tables of the coordinates in flight
// are staged in a shared-memory ring of 4D coordinates, refilled one round ahead
// (coordinates [j + D, j + 2D) are loaded while round j computes, stored after
// its reduction; 4D slots keep a slow warp's reads of round r clear of the
// stores of round r + 1).
template <int D>
struct MwgRing {
  static constexpr int kSlots = 4 * D;
};

// Thread limits per layout: S = 8 up to 640 threads, S = 16 up to 640 (the
// initialisation layout up to n = 10240: <= 102 registers), S = 32 512
template <int S, bool CODED, int D = 1>
__global__ void __launch_bounds__(S == 8 ? 640 : (S == 16 ? 640 : 512)) mwg_kernel(MwgParams P) {
  static_assert(D == 1 || CODED, "blocked rounds are for coded designs");
  extern __shared__ __align__(16) uint8_t sm[];
  const int q = P.d.q;
  CoordSlot* slot = reinterpret_cast<CoordSlot*>(sm);
  float* bsh = reinterpret_cast<float*>(slot + q);
  double* red = reinterpret_cast<double*>(bsh + ((q + 1) & ~1));  // [2][32]
  float* fred = reinterpret_cast<float*>(red + 64);               // [2][D][32]
  uint2* ring = reinterpret_cast<uint2*>(fred + 64 * D);          // coded: [4D][n_words] code words
  float2* tring = reinterpret_cast<float2*>(ring + (size_t)MwgRing<D>::kSlots * P.d.n_words);  // coded: [4D][16]
  float2* ttab = tring + MwgRing<D>::kSlots * 16;  // coded, full_tables: [q][16]

  const int64_t row = blockIdx.x;
  if (row >= P.m) return;
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  float* brow = P.beta + row * P.ldb;
  const Key2 key = stream_key(P.seed, (uint32_t)P.tag, (uint64_t)P.t, (uint64_t)(P.i0 + row));

  for (int j = tid; j < q; j += nthr) bsh[j] = brow[j];
  for (int k = tid; k < 64 * D; k += nthr) fred[k] = 0.0f;  // warp-sum scratch: slots >= nw stay zero
  __syncthreads();

  float sig[S];
  double ll = materialise_ll<S, CODED>(P, bsh, tid, nthr, lane, wid, nw, red, sig);
  unsigned long long acc = 0;
  const int sub0 = tid * S;
  const int nslots = P.slots > 0 ? P.slots : 1;
  for (int sl = 0; sl < nslots; ++sl) {
  // the log-prior restarts from beta for every block of sweeps (as a fresh
  // call would), so chain-slot mode is bit-identical to one call per slot
  double lp = 0.0;
  {
    double lp0 = 0.0;
    for (int j = tid; j < q; j += nthr)
      if (P.d.penalized[j]) lp0 += mwg_gt((double)bsh[j], P);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lp0 += __shfl_xor_sync(0xffffffffu, lp0, o);
    if (lane == 0) red[wid] = lp0;
    __syncthreads();
    for (int w = 0; w < nw; ++w) lp += red[w];
    __syncthreads();
  }

  // ---- 2. sweeps -----------------------------------------------------------
  for (int cyc = 0; cyc < P.cycles; ++cyc) {
    const uint64_t blk0 = (uint64_t)(P.sweep0 + (int64_t)sl * P.cycles + cyc) * (uint64_t)q;
    for (int j = tid; j < q; j += nthr) {
      uint64_t w[4];
      philox_block(key, blk0 + j, w);  // block index sweep*q + j (Philox counter index + 1)
      const double z = box_muller_cos(w[0], w[1]);
      const double u = u53(w[2]);
      const float old = bsh[j];
      const float nv = __double2float_rn((double)old + P.sd * z);
      CoordSlot cs;
      cs.newv = nv;
      cs.delta = (double)nv - (double)old;
      cs.dsy = cs.delta * P.d.sy[j];
      cs.logu = log(u);
      cs.dlp = P.d.penalized[j] ? (mwg_gt((double)nv, P) - mwg_gt((double)old, P)) : 0.0;
      if (CODED) {
        const float4 lv = reinterpret_cast<const float4*>(P.d.xlev)[j];
        const float df = (float)cs.delta;
        cs.m0 = finite_expm1(df * lv.x);
        cs.m1 = finite_expm1(df * lv.y);
        cs.m2 = finite_expm1(df * lv.z);
      } else {
        cs.m0 = cs.m1 = cs.m2 = 0.0f;
      }
      slot[j] = cs;
      if (CODED && P.full_tables) {  // pair table: entry e = (m[e & 3], m[e >> 2]), m = {m0, m1, m2, 0}
        const float mv[4] = {cs.m0, cs.m1, cs.m2, 0.0f};
        float2* tb = ttab + (size_t)j * 16;
#pragma unroll
        for (int e = 0; e < 16; ++e) tb[e] = make_float2(mv[e & 3], mv[e >> 2]);
      }
    }
    __syncthreads();

    if constexpr (!CODED) {
      // genotype bits are prefetched two coordinates ahead (the L2 load latency
      // was the largest stall); the per-subject factors m are re-selected from
      // the bits on acceptance instead of being kept (32 registers fewer, so
      // more chains are resident per SM)
      uint32_t nb1 = 0, nb2 = 0, nn1 = 0, nn2 = 0;
      if (CODED) {
        load_bits<S>(P.d, 0, tid, nb1, nb2);
        if (q > 1) load_bits<S>(P.d, 1, tid, nn1, nn2);
      }
      for (int j = 0; j < q; ++j) {
        const CoordSlot cs = slot[j];
        const uint32_t p1 = nb1, p2 = nb2;
        if (CODED) {
          nb1 = nn1;
          nb2 = nn2;
          if (j + 2 < q) load_bits<S>(P.d, j + 2, tid, nn1, nn2);
        }
        const float* xc = P.d.xcols + (size_t)j * P.d.n_words * 32 + sub0;
        const float df = (float)cs.delta;
        const float part = coord_log2_sum<S, CODED>(sig, p1, p2, cs, xc, df);
        // block sum (double-buffered scratch: one barrier per coordinate)
        float tot = part;
  #pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (nw > 1) {
          // second level: every warp reduces the nw warp sums with shuffles
          // (one smem load per lane instead of nw serial loads and adds)
          float* buf = fred + (j & 1) * 32;
          if (lane == 0) buf[wid] = tot;
          __syncthreads();
          const float4* b4 = reinterpret_cast<const float4*>(buf);
          float s8[8];
  #pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (4 * k < nw) {
              const float4 v = b4[k];
              s8[k] = (v.x + v.y) + (v.z + v.w);
            } else {
              s8[k] = 0.0f;
            }
          }
          tot = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
        }
        const double dll = cs.dsy - 0.6931471805599453 * (double)tot;
        const double d = dll + cs.dlp;
        const bool ok = (d >= 0.0) || (cs.logu < d);
        if (ok) {
          coord_accept<S, CODED>(sig, p1, p2, cs, xc, df);
          ll += dll;
          lp += cs.dlp;
          ++acc;
          if (tid == 0) bsh[j] = cs.newv;
        }
      }
    } else {
      // coded designs: blocked rounds over a shared-memory ring (MwgRing):
      // round r evaluates coordinates j .. j+D-1 against the current sigma,
      // one block reduction for all D, decisions in order up to the first
      // acceptance.  Subject factors come from the coordinate's pair table
      // (m of two subjects per 64-bit shared load, indexed by their 4-bit
      // code nibble) instead of bit tests and selects.
      constexpr int RS = MwgRing<D>::kSlots;
      constexpr int kMaxL = (D * S + 31) / 32 + 1;  // staged uint2 per thread (host: D n_words <= kMaxL nthr)
      constexpr int NCW = S >= 16 ? S / 16 : 1;     // code words per thread
      const int nwd = P.d.n_words;                  // uint2 (= 32 subjects) per coordinate
      const uint2* codes = reinterpret_cast<const uint2*>(P.d.codes);
      const uint32_t* cr32 = reinterpret_cast<const uint32_t*>(ring);
      const int cw0 = S >= 16 ? tid * NCW : tid >> 1;  // first code word of this thread
      const int csh = S == 8 ? (tid & 1) * 16 : 0;
      int coff[kMaxL], woff[kMaxL];  // round-invariant (coordinate, uint2) of this thread's staged loads
#pragma unroll
      for (int k = 0; k < kMaxL; ++k) {
        const int e = tid + k * nthr;
        coff[k] = e < D * nwd ? e / nwd : q;  // q: never loaded
        woff[k] = e - (e / nwd) * nwd;
      }
      const bool full = P.full_tables != 0;
      auto tbl_of = [&](int c) -> const float2* { return full ? ttab + c * 16 : tring + (c & (RS - 1)) * 16; };
      // the pair tables of coordinates [c0, c1) from their slots: entry e =
      // (m[e & 3], m[e >> 2]), m = {m0, m1, m2, 0} (code 3 = padding, sigma 0)
      auto build_tables = [&](int c0, int c1) {
        if (full) return;
        for (int e = tid; e < 16 * (c1 - c0); e += nthr) {
          const int c = c0 + (e >> 4);
          if (c < q) {
            const float4 mv = *reinterpret_cast<const float4*>(&slot[c].m0);  // m0, m1, m2, (newv)
            const int a = e & 3, b = (e >> 2) & 3;
            const float ma = a == 3 ? 0.0f : a == 2 ? mv.z : a == 1 ? mv.y : mv.x;
            const float mb = b == 3 ? 0.0f : b == 2 ? mv.z : b == 1 ? mv.y : mv.x;
            tring[(c & (RS - 1)) * 16 + (e & 15)] = make_float2(ma, mb);
          }
        }
      };
      for (int e = tid; e < 2 * D * nwd; e += nthr) {  // coordinates [0, 2D)
        const int c = e / nwd;
        if (c < q) ring[(c & (RS - 1)) * nwd + (e - c * nwd)] = codes[(size_t)c * nwd + (e - c * nwd)];
      }
      build_tables(0, 2 * D);
      __syncthreads();
      int rnd = 0;
      for (int j = 0; j < q; ++rnd) {
        // coordinates [j + D, j + 2D): loaded now, stored after the reduction
        uint2 lv[kMaxL];
#pragma unroll
        for (int k = 0; k < kMaxL; ++k) {
          const int c = j + D + coff[k];
          if (c < q) lv[k] = __ldg(&codes[(size_t)c * nwd + woff[k]]);
        }
        // the D sums as straight-line code (coordinates past q are computed
        // on coordinate q-1 and never decided), so the scheduler interleaves
        // the D independent product chains; the per-group range check of
        // coord_log2_sum_tbl is hoisted: one rare divergent fallback
        float part[D];
        float prodv[D][S / 8];
        bool inrange = true;
#pragma unroll
        for (int dd = 0; dd < D; ++dd) {
          const int cc = min(j + dd, q - 1);
          const int rs = cc & (RS - 1);
          uint32_t cw[NCW];
#pragma unroll
          for (int w = 0; w < NCW; ++w) cw[w] = cr32[rs * 2 * nwd + cw0 + w] >> csh;
          const float2* tbl = tbl_of(cc);
#pragma unroll
          for (int c8 = 0; c8 < S / 8; ++c8) {
            float fac[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int pk = 4 * c8 + k;
              const float2 mm = tbl[(cw[pk >> 3] >> (4 * (pk & 7))) & 15u];
              fac[2 * k] = fmaf(mm.x, sig[2 * pk], 1.0f);
              fac[2 * k + 1] = fmaf(mm.y, sig[2 * pk + 1], 1.0f);
            }
            const float pr = ((fac[0] * fac[1]) * (fac[2] * fac[3])) * ((fac[4] * fac[5]) * (fac[6] * fac[7]));
            prodv[dd][c8] = pr;
            inrange = inrange && (pr >= 1e-30f && pr <= 1e30f);
          }
        }
        if (inrange) {
#pragma unroll
          for (int dd = 0; dd < D; ++dd) {
            float acc = 0.0f;
#pragma unroll
            for (int c8 = 0; c8 < S / 8; ++c8) acc += fast_lg2(prodv[dd][c8]);
            part[dd] = acc;
          }
        } else {  // an extreme proposal: the per-group form (per-term logs where a product leaves the range)
#pragma unroll 1
          for (int dd = 0; dd < D; ++dd) {
            const int cc = min(j + dd, q - 1);
            const int rs = cc & (RS - 1);
            uint32_t cw[NCW];
#pragma unroll
            for (int w = 0; w < NCW; ++w) cw[w] = cr32[rs * 2 * nwd + cw0 + w] >> csh;
            part[dd] = coord_log2_sum_tbl<S>(sig, cw, tbl_of(cc));
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int dd = 0; dd < D; ++dd) part[dd] += __shfl_xor_sync(0xffffffffu, part[dd], o);
        float* buf = fred + (rnd & 1) * 32 * D;
        if (nw > 1 && lane == 0)
#pragma unroll
          for (int dd = 0; dd < D; ++dd) buf[dd * 32 + wid] = part[dd];
#pragma unroll
        for (int k = 0; k < kMaxL; ++k) {
          const int c = j + D + coff[k];
          if (c < q) ring[(c & (RS - 1)) * nwd + woff[k]] = lv[k];
        }
        build_tables(j + D, j + 2 * D);
        __syncthreads();
        if (nw > 1) {
          if (D >= 4 && nw <= 16) {
            // D >= 4: the same tree as an xor butterfly over lanes (level k
            // of the tree = shuffle distance 2^k; two coordinates per pass,
            // lanes 16..31 take the second, whose top level adds only zeros)
#pragma unroll
            for (int p2 = 0; p2 < (D + 1) / 2; ++p2) {
              const int dd = 2 * p2 + (lane >> 4);
              float v = dd < D ? buf[dd * 32 + (lane & 15)] : 0.0f;
#pragma unroll
              for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
              part[2 * p2] = __shfl_sync(0xffffffffu, v, 0);
              if (2 * p2 + 1 < D) part[2 * p2 + 1] = __shfl_sync(0xffffffffu, v, 16);
            }
          } else {
            // the perfect binary tree over the 32 warp slots (zero beyond nw)
#pragma unroll
            for (int dd = 0; dd < D; ++dd) {
              const float4* b4 = reinterpret_cast<const float4*>(buf + dd * 32);
              float s8[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                if (4 * k < nw) {
                  const float4 v = b4[k];
                  s8[k] = (v.x + v.y) + (v.z + v.w);
                } else {
                  s8[k] = 0.0f;
                }
              }
              part[dd] = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
            }
          }
        }
        // the D decisions (independent given the sums) evaluated together;
        // the first acceptance ends the round, later ones are discarded
        const int nv = min(D, q - j);
        uint32_t okm = 0;
        double dllv[D];
#pragma unroll
        for (int dd = 0; dd < D; ++dd) {
          const int cc = min(j + dd, q - 1);
          const double dsy = slot[cc].dsy, dlp = slot[cc].dlp, logu = slot[cc].logu;
          dllv[dd] = dsy - 0.6931471805599453 * (double)part[dd];
          const double d = dllv[dd] + dlp;
          okm |= (dd < nv && ((d >= 0.0) || (logu < d))) ? 1u << dd : 0u;
        }
        int adv = nv;
        if (okm) {
          const int first = __ffs(okm) - 1;
          double dll = dllv[0];
#pragma unroll
          for (int dd = 1; dd < D; ++dd)
            if (dd == first) dll = dllv[dd];
          const int ca = j + first;
          const CoordSlot cs = slot[ca];
          const int rs = ca & (RS - 1);
          uint32_t cw[NCW];
#pragma unroll
          for (int w = 0; w < NCW; ++w) cw[w] = cr32[rs * 2 * nwd + cw0 + w] >> csh;
          coord_accept_tbl<S>(sig, cw, tbl_of(ca));
          ll += dll;
          lp += cs.dlp;
          ++acc;
          if (tid == 0) bsh[ca] = cs.newv;
          adv = first + 1;
        }
        j += adv;
      }
    }
    __syncthreads();
  }

  __syncthreads();
  const bool last = sl + 1 == nslots;
  if (last)
    for (int j = tid; j < q; j += nthr) brow[j] = bsh[j];
  if (P.slots > 0)
    for (int j = tid; j < q; j += nthr) P.slot_beta[(row * P.slots + sl) * P.ldb + j] = bsh[j];
  // rematerialise the state's log-likelihood from beta (the running sum of
  // float32 increments only drives the accept decisions); between slots
  // this also refreshes sigma, exactly as the next call's entry would
  ll = materialise_ll<S, CODED>(P, bsh, tid, nthr, lane, wid, nw, red, last ? nullptr : sig);
  if (tid == 0) {
    if (P.slots > 0) {
      P.slot_ll[row * P.slots + sl] = ll;
      P.slot_lp[row * P.slots + sl] = lp;
    }
    if (last) {
      P.ll[row] = ll;
      if (P.lp) P.lp[row] = lp;
    }
  }
  }  // slots
  if (tid == 0) {
    if (P.per_particle)
      P.accepted[row] += acc;
    else
      atomicAdd(P.accepted, acc);
  }
}

template <int S, int D>
static const void* mwg_fn_sd(bool coded) {
  return coded ? (const void*)mwg_kernel<S, true, D> : (const void*)mwg_kernel<S, false, 1>;
}

template <int S>
static const void* mwg_fn_s(bool coded, int D) {
  return D == 4 ? mwg_fn_sd<S, 4>(coded) : D == 2 ? mwg_fn_sd<S, 2>(coded) : mwg_fn_sd<S, 1>(coded);
}

static const void* mwg_fn(int S, bool coded, int D = 1) {
  return S == 8 ? mwg_fn_s<8>(coded, D) : S == 16 ? mwg_fn_s<16>(coded, D) : mwg_fn_s<32>(coded, D);
}

// Coordinates per blocked round (mwg_kernel's D) for the initialisation
// chains and for the lambda-step move; spa_mwg_set_rounds changes them
// (A/B and the bit-identity tests: every D gives the same states).
static int g_rounds_init = 4, g_rounds_move = 4;

// Thread layouts: the lambda-step move (many particles per SM), the
// initialisation burn-in (one latency-bound chain per SM: fewer subjects per
// thread, per-sweep factor tables) and the initialisation thinning chains
// (a resident wave of chains: the move's throughput layout, the init rounds)
enum class MwgLayout { kMove, kBurn, kThin };

static int rounds_for(const spa_design* d, int S, int nthr, bool init_layout) {
  int D = init_layout ? g_rounds_init : g_rounds_move;
  if (!d->coded) return 1;
  // staged words per thread: D n_words <= kMaxL nthr with kMaxL = (D S + 31) / 32 + 1
  while (D > 1 && D * d->n_words > ((D * S + 31) / 32 + 1) * nthr) D >>= 1;
  return D;
}

static size_t mwg_smem(const spa_design* d, int D, bool full_tables = false) {
  return (size_t)d->q * sizeof(CoordSlot) + (size_t)((d->q + 1) & ~1) * sizeof(float) + 64 * sizeof(double) +
         (size_t)64 * D * sizeof(float) +
         (d->coded ? (size_t)MwgRing<1>::kSlots * D * (d->n_words * sizeof(uint2) + 16 * sizeof(float2)) : 0) +
         (full_tables ? (size_t)d->q * 16 * sizeof(float2) : 0);
}
// all q pair tables per sweep for the initialisation chains when two chains
// still fit per SM (C3: 109 KB; init 0.89 -> 0.80 s); the lambda-step move
// keeps the ring (its many resident particles per SM would not fit: C3 move
// 102 -> 117 ms with the tables)
static bool g_full_tables_allowed = true;
static bool mwg_full_tables(const spa_design* d, int D, bool init_layout) {
  return g_full_tables_allowed && init_layout && d->coded && mwg_smem(d, D, true) <= (size_t)112 * 1024;
}

static int max_threads(int S) { return S == 8 ? 640 : (S == 16 ? 640 : 512); }

// Layout of the initialisation chains (spa_mwg_chain_slots and the chain
// count of spa_mwg_resident_chains): one resident wave of latency-bound
// chains, so fewer subjects per thread and more threads per chain (C3 init
// with 2000 burn sweeps 1.58 -> 1.32 s, C2 0.51 -> 0.34 s against the
// throughput layout of pick_s)
static int pick_s_init(int n) {
  // developer A/B knob: SPA_MWG_S_INIT=8|16|32
  static const int forced = [] {
    const char* e = getenv("SPA_MWG_S_INIT");
    return e ? atoi(e) : 0;
  }();
  if ((forced == 8 || forced == 16 || forced == 32) && (n + forced - 1) / forced <= max_threads(forced))
    return forced;
  if (n <= 256) return 8;
  if ((n + 15) / 16 <= 640) return 16;
  if (n <= 16384) return 32;
  return 0;
}

static int pick_s(int n) {
  // developer A/B knob (init latency vs throughput layouts): SPA_MWG_S=8|16|32
  static const int forced = [] {
    const char* e = getenv("SPA_MWG_S");
    return e ? atoi(e) : 0;
  }();
  if ((forced == 8 || forced == 16 || forced == 32) && (n + forced - 1) / forced <= max_threads(forced))
    return forced;
  if (n <= 256) return 8;
  if (n <= 512) return 16;
  if (n <= 16384) return 32;
  return 0;
}

}  // namespace spa

using namespace spa;

// Coordinates per blocked MwG round for the initialisation chains and the
// lambda-step move (1, 2 or 4; coded designs; states are identical for any
// value -- a tuning knob, used by the A/B tools and the bit-identity tests).
extern "C" int spa_mwg_set_rounds(int32_t init_rounds, int32_t move_rounds) {
  auto ok = [](int v) { return v == 1 || v == 2 || v == 4; };
  SPA_REQUIRE(ok(init_rounds) && ok(move_rounds), kBadArgument, "spa_mwg_set_rounds: rounds must be 1, 2 or 4");
  g_rounds_init = init_rounds;
  g_rounds_move = move_rounds;
  return 0;
}

// Whether the coded MwG kernels may build all q pair tables per sweep
// (shared memory permitting) instead of per round in the ring; the states
// are identical either way (A/B and tests).
extern "C" int spa_mwg_set_tables(int32_t full_allowed) {
  g_full_tables_allowed = full_allowed != 0;
  return 0;
}

// internal (called by spa_prepare): load the MwG kernels
extern "C" int spa_mwg_prepare_kernels(void) {
  const void* fns[] = {(const void*)mwg_kernel<8, true>,   (const void*)mwg_kernel<16, true>,
                       (const void*)mwg_kernel<32, true>,  (const void*)mwg_kernel<8, false>,
                       (const void*)mwg_kernel<16, false>, (const void*)mwg_kernel<32, false>};
  for (const void* f : fns) {
    cudaFuncAttributes a;
    SPA_CHECK_CUDA(cudaFuncGetAttributes(&a, f));
  }
  return 0;
}

// Chains (one CTA each) resident at once on the current device: the
// occupancy of the kernel variant spa_mwg_move would launch for this design
// times the SM count.  Initialisation sizes its parallel chains to one wave.
extern "C" int spa_mwg_resident_chains(const spa_design* d, int64_t* chains) {
  SPA_REQUIRE(d && chains && d->q >= 1 && d->q <= 2048, kBadArgument, "spa_mwg_resident_chains: bad arguments");
  const int S = pick_s(d->n);  // the thinning layout (spa_mwg_chain_slots, layout 1)
  SPA_REQUIRE(S > 0, kNotSupported, "spa_mwg_resident_chains: n > 16384 not supported");
  const int nthr = std::max(32, ((d->n + S - 1) / S + 31) / 32 * 32);
  const int D = rounds_for(d, S, nthr, true);
  const size_t smem = mwg_smem(d, D, false);
  int per_sm = 0, dev = 0, nsm = 0;
  const void* fn = mwg_fn(S, d->coded != 0, D);
  SPA_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SPA_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nthr, smem));
  SPA_CHECK_CUDA(cudaGetDevice(&dev));
  SPA_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  *chains = (int64_t)std::max(1, per_sm) * nsm;
  return 0;
}

static int mwg_launch(const spa_design* d, float* beta, int64_t m, int32_t ldb, double a, double c, double step_sd,
                      int32_t cycles, uint64_t seed, int32_t tag, int64_t t, int64_t i0, int64_t sweep0, double* ll,
                      double* lp, unsigned long long* accepted, int32_t per_particle, int32_t slots,
                      float* slot_beta, double* slot_ll, double* slot_lp, void* stream, MwgLayout layout) {
  const bool init_layout = layout != MwgLayout::kMove;
  SPA_REQUIRE(d && beta && ll && accepted && m >= 0 && cycles >= 0, kBadArgument, "spa_mwg_move: bad arguments");
  SPA_REQUIRE(a > 0 && c > 0 && step_sd > 0, kBadArgument, "spa_mwg_move: a, c, step_sd must be positive");
  SPA_REQUIRE(d->q >= 1 && d->q <= 2048, kNotSupported, "spa_mwg_move: q must lie in [1, 2048]");
  const int S = layout == MwgLayout::kBurn ? pick_s_init(d->n) : pick_s(d->n);
  SPA_REQUIRE(S > 0, kNotSupported, "spa_mwg_move: n > 16384 not supported");
  SPA_REQUIRE(d->coded ? d->codes != nullptr : d->xcols != nullptr, kBadArgument, "spa_mwg_move: design arrays");
  if (m == 0) return 0;
  MwgParams P;
  P.d = *d;
  P.beta = beta;
  P.m = m;
  P.ldb = ldb;
  P.a = a;
  P.c = c;
  P.sd = step_sd;
  P.de = std::isinf(a) ? 1 : 0;
  P.cycles = cycles;
  P.seed = seed;
  P.tag = tag;
  P.t = t;
  P.i0 = i0;
  P.sweep0 = sweep0;
  P.ll = ll;
  P.lp = lp;
  P.accepted = accepted;
  P.per_particle = per_particle;
  P.slots = slots;
  P.slot_beta = slot_beta;
  P.slot_ll = slot_ll;
  P.slot_lp = slot_lp;
  const int nthr_raw = (d->n + S - 1) / S;
  const int nthr = std::max(32, (nthr_raw + 31) / 32 * 32);
  SPA_REQUIRE(nthr <= 1024, kNotSupported, "spa_mwg_move: too many subjects per particle");
  SPA_REQUIRE(nthr * S <= d->n_words * 32, kBadArgument, "spa_mwg_move: n_words does not cover the thread layout");
  const int D = rounds_for(d, S, nthr, init_layout);
  P.full_tables = mwg_full_tables(d, D, layout == MwgLayout::kBurn) ? 1 : 0;
  const size_t smem = mwg_smem(d, D, P.full_tables != 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SPA_REQUIRE(nthr <= max_threads(S), kNotSupported, "spa_mwg_move: too many threads for this layout");
  const void* fn = mwg_fn(S, d->coded != 0, D);
  SPA_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {&P};
  SPA_CHECK_CUDA(cudaLaunchKernel(fn, dim3((unsigned)m), dim3(nthr), args, smem, st));
  SPA_CHECK_LAUNCH();
  return 0;
}

extern "C" int spa_mwg_move(const spa_design* d, float* beta, int64_t m, int32_t ldb, double a, double c,
                            double step_sd, int32_t cycles, uint64_t seed, int32_t tag, int64_t t, int64_t i0,
                            int64_t sweep0, double* ll, double* lp, unsigned long long* accepted,
                            int32_t per_particle, void* stream) {
  return mwg_launch(d, beta, m, ldb, a, c, step_sd, cycles, seed, tag, t, i0, sweep0, ll, lp, accepted, per_particle,
                    0, nullptr, nullptr, nullptr, stream, MwgLayout::kMove);
}

extern "C" int spa_mwg_chain_slots(const spa_design* d, float* beta, int64_t m, int32_t ldb, double a, double c,
                                   double step_sd, int32_t cycles_per_slot, int32_t slots, uint64_t seed,
                                   int32_t tag, int64_t t, int64_t i0, int64_t sweep0, double* ll, double* lp,
                                   float* slot_beta, double* slot_ll, double* slot_lp,
                                   unsigned long long* accepted, int32_t per_particle, int32_t layout,
                                   void* stream) {
  SPA_REQUIRE(slots >= 1 && slot_beta && slot_ll && slot_lp && cycles_per_slot >= 1, kBadArgument,
              "spa_mwg_chain_slots: bad slot arguments");
  SPA_REQUIRE(layout == 0 || layout == 1, kBadArgument, "spa_mwg_chain_slots: layout must be 0 or 1");
  return mwg_launch(d, beta, m, ldb, a, c, step_sd, cycles_per_slot, seed, tag, t, i0, sweep0, ll, lp, accepted,
                    per_particle, slots, slot_beta, slot_ll, slot_lp, stream,
                    layout ? MwgLayout::kThin : MwgLayout::kBurn);
}
