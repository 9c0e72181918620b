// K4: bit-exact systematic resampling, parallel (reference smc.py:273-281).
//
// The reference normalises by np.cumsum(W): s_i = fl(s_{i-1} + w_i), a
// strictly sequential float64 chain, so a tree-ordered parallel scan rounds
// differently.  This file reproduces the sequential bits in parallel
// (hard part 3, "binade-segmented" scan):
//
// * While the running sum stays in one binade [2^E, 2^(E+1)) it is
//   s = k * u with u = 2^(E-52) and an integer mantissa k in [2^52, 2^53),
//   and fl(s + w) = round_half_even(k + w/u) * u: with x = w/u = I + f
//   (I = floor x), the increment is I (f < 1/2), I + 1 (f > 1/2), or on a
//   tie whichever of the two makes the result even -- it depends on the
//   parity of k only.  So an element is a map on the mantissa, given by the
//   pair (increment if k is even, increment if k is odd), and these maps
//   compose associatively: (f then g)(p) = f(p) + g((p + f(p)) mod 2).
//   Inside a binade the sequential chain is an integer scan of such pairs.
// * Where the binade changes the element is added with one plain float64
//   add -- exactly the reference's operation.  Binade changes are predicted
//   from an exact fixed-point prefix sum P (w scaled by 2^100, unsigned
//   128-bit, associative, so every block agrees on every prefix); elements
//   whose predicted binade differs from their predecessor's, and positive
//   weights whose prefix lies within the float64 chain's rounding window of
//   a power of two ("ambiguous"), are "heads".
// * The prediction is speculative and verified: the sequential chain over
//   the heads (one thread, float64 adds at the heads, integer maps between)
//   checks that every unambiguous head lands in its predicted binade, that an
//   ambiguous head that lands elsewhere is followed only by zero weights up
//   to the next head, and that no mantissa passes 2^53 before the next head
//   (mantissas only grow, so each segment's end suffices).  Any violation --
//   or input the fast path does not cover (weights >= 2^16, NaN, a positive
//   prefix below 2^-100, more than kHMax heads in a tile) -- falls back to
//   the sequential scan, run by one block of the same launch.  The result is
//   np.cumsum's either way.
//
// Three kernels per scan, each one block per 2048-element tile:
//   A  tile fixed-point sums; the last block to finish scans them (tile offsets)
//   B  binades, heads and per-segment pair compositions of each tile; the last
//      block runs the head chain (or the sequential fallback)
//   C  every element's value from its segment's head (or the tile's incoming
//      state) and its in-segment prefix pair; also cum / cum[N-1]
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "resample.cuh"

namespace spa {
namespace {

typedef unsigned long long u64;
typedef unsigned __int128 u128;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = 8;
constexpr int kTile = kThreads * kPer;  // 2048 weights per block
constexpr int kHMax = 64;               // heads per tile on the fast path
constexpr int kChainMax = 896;          // heads in the whole array on the fast path
constexpr int kFB = 100;                // fraction bits of the fixed-point prefix
constexpr int kZero = -100000;          // "binade" of an exactly-zero prefix
constexpr u64 kSat = 1ull << 62;        // saturation of mantissa increments
// A mantissa may end a segment at exactly 2^53: the map rounded an exact sum
// below 2^(E+1) up to 2^(E+1) (both binades agree), or it rounded down a sum
// in [2^(E+1), 2^(E+1) + u) -- which the next binade's spacing 2u also rounds
// to 2^(E+1); later zero increments agree too (w < u/2), any other one
// pushes the mantissa past 2^53 and fails the check.
constexpr u64 kTwo53 = 1ull << 53;
constexpr unsigned FULL = 0xffffffffu;

struct Pair {
  u64 d0, d1;  // mantissa increment when the running mantissa is even / odd
};
__device__ __forceinline__ u64 sat_add(u64 a, u64 b) {
  const u64 s = a + b;
  return s > kSat ? kSat : s;
}
// f then g
__device__ __forceinline__ Pair compose(Pair f, Pair g) {
  Pair r;
  r.d0 = sat_add(f.d0, (f.d0 & 1) ? g.d1 : g.d0);
  r.d1 = sat_add(f.d1, (f.d1 & 1) ? g.d0 : g.d1);
  return r;
}
__device__ __forceinline__ u64 apply(Pair p, u64 k) { return sat_add(k, (k & 1) ? p.d1 : p.d0); }

// The segmented-scan monoid: heads so far, and since the last head the
// composition of the element maps plus whether any weight was nonzero.
struct Agg {
  int c;
  unsigned nz;
  Pair p;
};
__device__ __forceinline__ Agg agg_op(Agg a, Agg b) {
  Agg r;
  r.c = a.c + b.c;
  r.nz = b.c > 0 ? b.nz : (a.nz | b.nz);
  r.p = b.c > 0 ? b.p : compose(a.p, b.p);
  return r;
}
__device__ __forceinline__ Agg agg_ident() { return Agg{0, 0u, Pair{0, 0}}; }

__device__ __forceinline__ double ld_w(const WSrc& w, int64_t i) {
  if (w.nparts == 1) return __ldg(w.p[0] + i);
  return w.p[i / w.len][i % w.len];
}

// floor(w * 2^kFB) for 0 <= w < 2^16 (a tile sum stays below 2^127; the
// running total is checked against 2^126); anything else turns the fast path off
__device__ __forceinline__ u128 to_fix(double w, bool& bad) {
  if (!(w >= 0.0 && w < 65536.0)) {
    bad = true;
    return 0;
  }
  const u64 b = (u64)__double_as_longlong(w);
  const int ex = (int)(b >> 52);  // sign bit is 0 here
  if (ex == 0) return 0;          // subnormal: below 2^-1022, far under 2^-kFB
  const u64 mant = (b & ((1ull << 52) - 1)) | (1ull << 52);  // w = mant 2^(ex - 1075)
  const int sh = ex - 1075 + kFB;
  if (sh >= 0) return (u128)mant << sh;
  if (sh <= -64) return 0;
  return (u128)(mant >> (-sh));
}

// 2^e as a double (-1022 <= e <= 1023), and the exponent of a positive normal double
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ int exponent_of(double x) {
  return (int)(((u64)__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
}

__device__ __forceinline__ int msb128(u128 P) {
  const u64 hi = (u64)(P >> 64), lo = (u64)P;
  return hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
}
// binade of P * 2^-kFB (floor log2), kZero for P = 0
__device__ __forceinline__ int binade(u128 P) { return P == 0 ? kZero : msb128(P) - kFB; }

// Is the prefix through element idx so close to a power of two that the
// float64 chain may lie on the other side of it?  |fl_i - S_i| <= (i+1) 2^-53
// S_i for a sequential sum of nonnegatives, |P_i 2^-kFB - S_i| <= (i+1) 2^-kFB;
// the window is twice that.
__device__ __forceinline__ bool ambiguous(u128 P, int64_t idx) {
  if (P == 0) return false;
  const int m = msb128(P);  // 2^m <= P < 2^(m+1), m <= 126
  const u128 lo = (u128)1 << m;
  const u128 dlo = P - lo, dhi = (lo << 1) - P;
  const int sh = m + 1 - 52;
  const u128 n = (u128)(idx + 2);
  const u128 tol = (sh >= 0 ? (n << sh) : (n >> (-sh))) + n;
  return dlo <= tol || dhi <= tol;
}

// the mantissa map of adding w inside binade E
__device__ __forceinline__ Pair elem_pair(double w, int E) {
  const double x = w * pow2(52 - E);  // exact power-of-two scaling (52 - E in [36, 152])
  if (!(x < 18014398509481984.0)) return Pair{kSat, kSat};  // >= 2^54: cannot stay in the binade
  const double fl = floor(x);
  const u64 I = (u64)fl;
  const double f = x - fl;
  if (f < 0.5) return Pair{I, I};
  if (f > 0.5) return Pair{I + 1, I + 1};
  return Pair{I + (I & 1), I + ((I + 1) & 1)};  // tie: round half to even
}

__device__ __forceinline__ u128 shfl_up(u128 v, int d) {
  const u64 lo = __shfl_up_sync(FULL, (u64)v, d);
  const u64 hi = __shfl_up_sync(FULL, (u64)(v >> 64), d);
  return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ Agg shfl_up(Agg v, int d) {
  Agg r;
  r.c = __shfl_up_sync(FULL, v.c, d);
  r.nz = __shfl_up_sync(FULL, v.nz, d);
  r.p.d0 = __shfl_up_sync(FULL, v.p.d0, d);
  r.p.d1 = __shfl_up_sync(FULL, v.p.d1, d);
  return r;
}
__device__ __forceinline__ int shfl_up(int v, int d) { return __shfl_up_sync(FULL, v, d); }
__device__ __forceinline__ u128 op_add(u128 a, u128 b) { return a + b; }
__device__ __forceinline__ int op_addi(int a, int b) { return a + b; }

// Block-wide exclusive scan (kThreads threads, op associative: op(a, b) =
// a then b).  *total = the op over all threads.  wsum: kWarps smem slots.
template <class T, class Op>
__device__ __forceinline__ T block_excl_scan(T v, T ident, Op op, T* wsum, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T o = shfl_up(inc, d);
    if (lane >= d) inc = op(o, inc);
  }
  T ex = shfl_up(inc, 1);
  if (lane == 0) ex = ident;
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T x = lane < kWarps ? wsum[lane] : ident;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
      const T o = shfl_up(x, d);
      if (lane >= d) x = op(o, x);
    }
    if (lane < kWarps) wsum[lane] = x;
  }
  __syncthreads();
  const T res = warp ? op(wsum[warp - 1], ex) : ex;
  if (total) *total = wsum[kWarps - 1];
  __syncthreads();
  return res;
}

// Workspace layout (byte offsets from ws; cum [N] float64 first).
struct Layout {
  int64_t ntiles;
  size_t cumn, tsum, toff, tpre, tprenz, tnh, tinE, tink, cinc, cinp, cinnz, htl, hpos, hE, hamb, hw, hseg, hsegnz, hk,
      gE, gk, tot, ctrl, total;
};
__host__ __device__ inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
__host__ __device__ inline Layout layout(int64_t N) {
  Layout L;
  L.ntiles = (N + kTile - 1) / kTile;
  const size_t T = (size_t)L.ntiles, H = T * kHMax;
  size_t o = al256((size_t)N * 8);
  L.cumn = o; o = al256(o + (size_t)N * 8);
  L.tsum = o; o = al256(o + T * 16);
  L.toff = o; o = al256(o + T * 16);
  L.tpre = o; o = al256(o + T * 16);
  L.tprenz = o; o = al256(o + T * 4);
  L.tnh = o; o = al256(o + T * 4);
  L.tinE = o; o = al256(o + T * 4);
  L.tink = o; o = al256(o + T * 8);
  L.cinc = o; o = al256(o + T * 4);
  L.cinp = o; o = al256(o + T * 16);
  L.cinnz = o; o = al256(o + T * 4);
  L.htl = o; o = al256(o + T * 4);
  L.hpos = o; o = al256(o + H * 8);
  L.hE = o; o = al256(o + H * 4);
  L.hamb = o; o = al256(o + H * 4);
  L.hw = o; o = al256(o + H * 8);
  L.hseg = o; o = al256(o + H * 16);
  L.hsegnz = o; o = al256(o + H * 4);
  L.hk = o; o = al256(o + H * 8);
  L.gE = o; o = al256(o + H * 4);
  L.gk = o; o = al256(o + H * 8);
  L.tot = o; o = al256(o + 8);
  L.ctrl = o; o = al256(o + 16);
  L.total = o;
  return L;
}
template <class T>
__host__ __device__ inline T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + off);
}
template <class T>
__host__ __device__ inline const T* at(const void* ws, size_t off) {
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(ws) + off);
}
__device__ __forceinline__ Pair ldcg_pair(const Pair* p) {
  Pair r;
  r.d0 = __ldcg(&p->d0);
  r.d1 = __ldcg(&p->d1);
  return r;
}
__device__ __forceinline__ u128 ldcg_u128(const u128* p) {
  const u64* q = reinterpret_cast<const u64*>(p);
  return (u128)__ldcg(q) | ((u128)__ldcg(q + 1) << 64);
}

__device__ __forceinline__ bool gated_off(const double* gate) { return gate != nullptr && !(gate[0] != 0.0); }

// Per-tile preamble shared by kernels B and C: this thread's 8 weights, the
// predicted binade of each, head / ambiguity flags.
struct TileView {
  double w[kPer];
  int E[kPer];
  unsigned head;  // bit i: element i is a head
  unsigned amb;   // bit i: element i is an ambiguous head
  int nvalid;     // valid elements of this thread
  bool bad;
};

__device__ __forceinline__ void tile_view(const WSrc& src, int64_t N, int64_t t, u128 toff_t, TileView& v,
                                          u128* wsum128) {
  const int64_t i0 = t * kTile + (int64_t)threadIdx.x * kPer;
  bool bad = false;
  const int64_t rem = N - i0;
  const int nvalid = rem <= 0 ? 0 : (rem >= kPer ? kPer : (int)rem);
  u128 F[kPer];
  u128 tsum = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    v.w[i] = i < nvalid ? ld_w(src, i0 + i) : 0.0;
    F[i] = to_fix(v.w[i], bad);
    tsum += F[i];
  }
  u128 total;
  u128 P = toff_t + block_excl_scan<u128>(tsum, (u128)0, op_add, wsum128, &total);
  int Eprev = binade(P);
  unsigned head = 0, amb = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    P += F[i];
    v.E[i] = binade(P);
    if (i < nvalid) {
      const bool a = v.w[i] != 0.0 && ambiguous(P, i0 + i);
      if (v.E[i] != Eprev || a) head |= 1u << i;
      if (a) amb |= 1u << i;
      if (v.E[i] == kZero && v.w[i] != 0.0) bad = true;  // positive weight under a 2^-100 prefix
    }
    Eprev = v.E[i];
  }
  v.head = head;
  v.amb = amb;
  v.nvalid = nvalid;
  v.bad = bad;
}

__device__ __forceinline__ Pair elem_map(const TileView& v, int i) {
  return (v.E[i] == kZero || i >= v.nvalid) ? Pair{0, 0} : elem_pair(v.w[i], v.E[i]);
}

// the thread's aggregate over its elements
__device__ __forceinline__ Agg thread_agg(const TileView& v) {
  Agg a = agg_ident();
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (v.head >> i & 1u) {
      a.c += 1;
      a.nz = 0u;
      a.p = Pair{0, 0};
    } else if (i < v.nvalid) {
      a.p = compose(a.p, elem_map(v, i));
      a.nz |= v.w[i] != 0.0 ? 1u : 0u;
    }
  }
  return a;
}

// Kernel A: tile sums of the fixed-point weights; the last block scans them.
__global__ void __launch_bounds__(kThreads) scan_tile_sums_kernel(const __grid_constant__ WSrc src, int64_t N, void* ws,
                                                                  const double* gate) {
  __shared__ u128 wsum[kWarps];
  __shared__ bool last;
  if (gated_off(gate)) return;
  const Layout L = layout(N);
  unsigned* ctrl = at<unsigned>(ws, L.ctrl);
  const int64_t t = blockIdx.x;
  const int64_t i0 = t * kTile + (int64_t)threadIdx.x * kPer;
  bool bad = false;
  u128 s = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (i0 + i < N) s += to_fix(ld_w(src, i0 + i), bad);
  u128 total;
  (void)block_excl_scan<u128>(s, (u128)0, op_add, wsum, &total);
  bad = __syncthreads_or(bad) || (total >> 118) != 0;  // keeps every 256-tile scan chunk below 2^126
  if (threadIdx.x == 0) {
    at<u128>(ws, L.tsum)[t] = total;
    if (bad) atomicOr(ctrl + 2, 1u);
    __threadfence();
    last = atomicAdd(ctrl + 0, 1u) == (unsigned)(L.ntiles - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // exclusive scan of the tile sums, kThreads tiles at a time
  const u128* ts = at<u128>(ws, L.tsum);
  u128* to = at<u128>(ws, L.toff);
  u128 carry = 0;
  for (int64_t b = 0; b < L.ntiles; b += kThreads) {
    const int64_t k = b + threadIdx.x;
    const u128 v = k < L.ntiles ? ldcg_u128(ts + k) : (u128)0;
    u128 tot;
    const u128 ex = block_excl_scan<u128>(v, (u128)0, op_add, wsum, &tot);
    if (k < L.ntiles) to[k] = carry + ex;
    carry += tot;
    if ((carry >> 126) != 0) {  // total >= 2^26: off the fast path (uniform across the block)
      if (threadIdx.x == 0) atomicOr(ctrl + 2, 1u);
      break;
    }
  }
}

// The reference's sequential float64 chain, one thread summing while warp 1
// stages the next 2048 weights in shared memory (the fallback path).
__device__ void serial_cumsum(const WSrc& src, int64_t N, double* cum, double (*tile)[2048]) {
  const int64_t ntiles = (N + 2047) / 2048;
  if (threadIdx.x >= 32 && threadIdx.x < 64)
    for (int i = threadIdx.x - 32; i < 2048; i += 32) tile[0][i] = (i < N) ? ld_w(src, i) : 0.0;
  __syncthreads();
  double s = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int cur = (int)(t & 1);
    if (threadIdx.x == 0) {
      const int64_t base = t * 2048;
      const int cnt = (int)(N - base < 2048 ? N - base : 2048);
      const double* tl = tile[cur];
      for (int i = 0; i < cnt; ++i) {
        s = s + tl[i];  // np.cumsum's association
        cum[base + i] = s;
      }
    } else if (threadIdx.x >= 32 && threadIdx.x < 64 && t + 1 < ntiles) {
      const int64_t base = (t + 1) * 2048;
      for (int i = threadIdx.x - 32; i < 2048; i += 32) tile[cur ^ 1][i] = (base + i < N) ? ld_w(src, base + i) : 0.0;
    }
    __syncthreads();
  }
}

// cumn = cum / cum[N-1] with cumn[N-1] = 1 (smc.py:277-278), block-strided.
__device__ void normalise_block(const double* cum, double* cumn, int64_t N) {
  const double total = cum[N - 1];
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) cumn[i] = (i == N - 1) ? 1.0 : cum[i] / total;
}

// The last block of kernel B.
// (1) Carry-in of every tile: a segmented scan over the tiles' aggregates,
//     and the list of tiles holding heads.
// (2) Every head's inputs (the map since the previous head, whether a weight
//     in between was nonzero, its weight and predicted binade) are gathered
//     into shared memory in parallel; then one thread walks the heads: the
//     value before a head is the previous head's mantissa through that map,
//     the head is the reference's float64 add, checked as described at the
//     top of the file.
// (3) Each tile's incoming state, in parallel.
// Any failed check: the sequential scan (and its normalisation) instead.
struct ChainSmem {
  Pair comp[kChainMax];
  double w[kChainMax];
  int epred[kChainMax];
  int slot[kChainMax];
  unsigned flags[kChainMax];  // bit 0: ambiguous head, bit 1: a nonzero weight since the previous head
};
static_assert(sizeof(ChainSmem) <= 2 * 2048 * sizeof(double), "chain staging must fit the fallback's tile buffer");

__device__ void chain_block(const WSrc& src, int64_t N, void* ws, const Layout& L, double (*stage)[2048],
                            Agg* wsumA) {
  __shared__ int wsumI[kWarps];
  __shared__ unsigned ok_s;
  __shared__ int nheads_s;
  ChainSmem& cs = *reinterpret_cast<ChainSmem*>(&stage[0][0]);
  unsigned* ctrl = at<unsigned>(ws, L.ctrl);
  const Pair* tpre = at<const Pair>(ws, L.tpre);
  const unsigned* tprenz = at<const unsigned>(ws, L.tprenz);
  const int* tnh = at<const int>(ws, L.tnh);
  const Pair* hs = at<const Pair>(ws, L.hseg);
  const unsigned* hsnz = at<const unsigned>(ws, L.hsegnz);
  int* cinc = at<int>(ws, L.cinc);
  Pair* cinp = at<Pair>(ws, L.cinp);
  unsigned* cinnz = at<unsigned>(ws, L.cinnz);
  int* htl = at<int>(ws, L.htl);
  const int64_t T = L.ntiles;
  bool bad = false;
  Agg carry = agg_ident();
  int hcarry = 0;
  // (1)
  for (int64_t b = 0; b < T; b += kThreads) {
    const int64_t t = b + threadIdx.x;
    Agg a = agg_ident();
    int ht = 0;
    if (t < T) {
      const int nh = __ldcg(tnh + t);
      if (nh > kHMax) bad = true;
      const int nc = nh > kHMax ? kHMax : nh;
      a.c = nh;
      if (nc) {
        a.p = ldcg_pair(hs + t * kHMax + nc - 1);
        a.nz = __ldcg(hsnz + t * kHMax + nc - 1);
      } else {
        a.p = ldcg_pair(tpre + t);
        a.nz = __ldcg(tprenz + t);
      }
      ht = nh > 0;
    }
    Agg tot;
    const Agg ex = block_excl_scan<Agg>(a, agg_ident(), agg_op, wsumA, &tot);
    int htot;
    const int hex = block_excl_scan<int>(ht, 0, op_addi, wsumI, &htot);
    if (t < T) {
      const Agg c = agg_op(carry, ex);
      cinc[t] = c.c;
      cinp[t] = c.p;
      cinnz[t] = c.nz;
      if (ht) htl[hcarry + hex] = (int)t;
    }
    carry = agg_op(carry, tot);
    hcarry += htot;
  }
  bad = __syncthreads_or(bad || carry.c > kChainMax);
  // (2) gather the heads' inputs (this block wrote cinc / cinp / htl: visible after the barrier)
  if (!bad) {
    const int* hE = at<const int>(ws, L.hE);
    const int* hamb = at<const int>(ws, L.hamb);
    const double* hw = at<const double>(ws, L.hw);
    for (int i = threadIdx.x; i < hcarry; i += kThreads) {
      const int t = htl[i];
      const int nh = __ldcg(tnh + t);
      const int g0 = cinc[t];
      for (int j = 0; j < nh; ++j) {
        const size_t h = (size_t)t * kHMax + j;
        const int g = g0 + j;
        if (j == 0) {
          cs.comp[g] = compose(cinp[t], ldcg_pair(tpre + t));
          cs.flags[g] = (unsigned)__ldcg(hamb + h) | ((cinnz[t] | __ldcg(tprenz + t)) ? 2u : 0u);
        } else {
          cs.comp[g] = ldcg_pair(hs + h - 1);
          cs.flags[g] = (unsigned)__ldcg(hamb + h) | (__ldcg(hsnz + h - 1) ? 2u : 0u);
        }
        cs.w[g] = __ldcg(hw + h);
        cs.epred[g] = __ldcg(hE + h);
        cs.slot[g] = (int)h;
      }
    }
  }
  if (threadIdx.x == 0) nheads_s = carry.c;
  __syncthreads();
  if (threadIdx.x == 0) {
    // why == 0: fast path; else the first failed check (reported as the mode)
    unsigned why = bad ? 2u : (__ldcg(ctrl + 2) != 0u ? 1u : 0u);
    bool ok = why == 0u;
    int* hE = at<int>(ws, L.hE);
    u64* hk = at<u64>(ws, L.hk);
    int* gE = at<int>(ws, L.gE);
    u64* gk = at<u64>(ws, L.gk);
    int E = kZero;
    u64 k = 0;
    bool moved = false;  // the previous head's actual binade differs from its segment's prediction
    const int nheads = nheads_s;
    for (int g = 0; g < nheads && ok; ++g) {
      const unsigned fl = cs.flags[g];
      if (moved && (fl & 2u)) {  // nonzero weights mapped in the predicted binade: invalid
        ok = false;
        why = 6u;
        break;
      }
      double sprev = 0.0;
      if (E != kZero) {
        const u64 kp = moved ? k : apply(cs.comp[g], k);  // the mantissa just before this head
        if (kp > kTwo53) {
          ok = false;
          why = 3u;
          break;
        }
        sprev = (double)kp * pow2(E - 52);
      }
      const double sh = sprev + cs.w[g];  // the reference's float64 add
      if (!(sh >= 2.2250738585072014e-308)) {  // a positive normal double
        ok = false;
        why = 4u;
        break;
      }
      const int Ea = exponent_of(sh), Ep = cs.epred[g];
      if (Ea != Ep && !(fl & 1u)) {  // an unambiguous head must land where predicted
        ok = false;
        why = 5u;
        break;
      }
      moved = Ea != Ep;
      k = (u64)(sh * pow2(52 - Ea));
      E = Ea;
      hE[cs.slot[g]] = Ea;  // the actual binade (kernel C)
      hk[cs.slot[g]] = k;
      gE[g] = Ea;
      gk[g] = k;
    }
    double total = 0.0;
    if (ok && E != kZero) {
      const u64 ke = moved ? k : apply(carry.p, k);  // after the last head, to the end
      if ((moved && carry.nz) || ke > kTwo53) {
        ok = false;
        why = 7u;
      } else {
        total = (double)ke * pow2(E - 52);
      }
    }
    *at<double>(ws, L.tot) = total;
    ok_s = ok ? 1u : 0u;
    ctrl[3] = ok ? 0u : (why ? why : 8u);  // mode: > 0 = the sequential fallback wrote cum
    ctrl[2] = 0u;
  }
  __syncthreads();
  if (ok_s) {
    // (3)
    const int* gE = at<const int>(ws, L.gE);
    const u64* gk = at<const u64>(ws, L.gk);
    int* tinE = at<int>(ws, L.tinE);
    u64* tink = at<u64>(ws, L.tink);
    for (int64_t t = threadIdx.x; t < T; t += kThreads) {
      const int c = cinc[t];
      if (c == 0) {
        tinE[t] = kZero;
        tink[t] = 0;
      } else {
        // (after a moved head the segment holds zero weights only: identity maps)
        tinE[t] = __ldcg(gE + c - 1);
        tink[t] = apply(cinp[t], __ldcg(gk + c - 1));
      }
    }
  } else {
    double* cum = reinterpret_cast<double*>(ws);
    serial_cumsum(src, N, cum, stage);
    __syncthreads();
    normalise_block(cum, at<double>(ws, L.cumn), N);
  }
}

// Kernel B: heads and segment maps per tile; the last block runs the chain.
__global__ void __launch_bounds__(kThreads) scan_segments_kernel(const __grid_constant__ WSrc src, int64_t N, void* ws, const double* gate) {
  __shared__ u128 wsum128[kWarps];
  __shared__ Agg wsumA[kWarps];
  __shared__ unsigned first_head[kThreads];
  __shared__ bool last;
  __shared__ __align__(16) double stage[2][2048];
  if (gated_off(gate)) return;
  const Layout L = layout(N);
  unsigned* ctrl = at<unsigned>(ws, L.ctrl);
  const int64_t t = blockIdx.x;
  const u128 toff_t = ldcg_u128(at<const u128>(ws, L.toff) + t);
  TileView v;
  tile_view(src, N, t, toff_t, v, wsum128);
  const Agg a = thread_agg(v);
  first_head[threadIdx.x] = v.nvalid > 0 ? (v.head & 1u) : 1u;  // past the end: a segment boundary
  Agg tot;
  Agg run = block_excl_scan<Agg>(a, agg_ident(), agg_op, wsumA, &tot);  // (its barriers publish first_head)
  const int64_t i0 = t * kTile + (int64_t)threadIdx.x * kPer;
  bool bad = v.bad;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (i < v.nvalid) {
      if (v.head >> i & 1u) {
        run.c += 1;
        run.nz = 0u;
        run.p = Pair{0, 0};
        const int h = run.c - 1;
        if (h < kHMax) {
          const size_t hh = (size_t)t * kHMax + h;
          at<int64_t>(ws, L.hpos)[hh] = i0 + i;
          at<int>(ws, L.hE)[hh] = v.E[i];
          at<int>(ws, L.hamb)[hh] = (int)(v.amb >> i & 1u);
          at<double>(ws, L.hw)[hh] = v.w[i];
        } else {
          bad = true;
        }
      } else {
        run.p = compose(run.p, elem_map(v, i));
        run.nz |= v.w[i] != 0.0 ? 1u : 0u;
      }
      const bool next_head = (i + 1 < kPer) ? (i + 1 >= v.nvalid || (v.head >> (i + 1) & 1u))
                                            : (threadIdx.x + 1 == kThreads || first_head[threadIdx.x + 1] != 0u);
      if (next_head) {  // the last element of its segment inside this tile
        if (run.c == 0) {
          at<Pair>(ws, L.tpre)[t] = run.p;
          at<unsigned>(ws, L.tprenz)[t] = run.nz;
        } else if (run.c - 1 < kHMax) {
          at<Pair>(ws, L.hseg)[(size_t)t * kHMax + run.c - 1] = run.p;
          at<unsigned>(ws, L.hsegnz)[(size_t)t * kHMax + run.c - 1] = run.nz;
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    if (v.head & 1u) {  // empty pre-head region
      at<Pair>(ws, L.tpre)[t] = Pair{0, 0};
      at<unsigned>(ws, L.tprenz)[t] = 0u;
    }
    at<int>(ws, L.tnh)[t] = tot.c;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    if (bad) atomicOr(ctrl + 2, 1u);
    __threadfence();
    last = atomicAdd(ctrl + 1, 1u) == (unsigned)(L.ntiles - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  chain_block(src, N, ws, L, stage, wsumA);
}

// Kernel C: every element's float64 prefix value, and cum / cum[N-1].
__global__ void __launch_bounds__(kThreads) scan_values_kernel(const __grid_constant__ WSrc src, int64_t N, void* ws, const double* gate) {
  __shared__ u128 wsum128[kWarps];
  __shared__ Agg wsumA[kWarps];
  if (gated_off(gate)) return;
  const Layout L = layout(N);
  if (__ldcg(at<unsigned>(ws, L.ctrl) + 3) != 0u) return;  // the fallback already wrote cum / cumn
  const int64_t t = blockIdx.x;
  // tile-level state, loaded before the block scans
  const u128 toff_t = ldcg_u128(at<const u128>(ws, L.toff) + t);
  const int tin_E = __ldcg(at<const int>(ws, L.tinE) + t);
  const u64 tin_k = __ldcg(at<const u64>(ws, L.tink) + t);
  const double total = __ldcg(at<const double>(ws, L.tot));
  TileView v;
  tile_view(src, N, t, toff_t, v, wsum128);
  Agg run = block_excl_scan<Agg>(thread_agg(v), agg_ident(), agg_op, wsumA, nullptr);
  // the state this thread's first segment continues from
  const int* hE = at<const int>(ws, L.hE);
  const u64* hk = at<const u64>(ws, L.hk);
  int E = tin_E;
  u64 k0 = tin_k;
  if (run.c > 0) {
    const size_t h = (size_t)t * kHMax + run.c - 1;
    E = __ldcg(hE + h);
    k0 = __ldcg(hk + h);
  }
  double* cum = reinterpret_cast<double*>(ws);
  double* cumn = at<double>(ws, L.cumn);
  const int64_t i0 = t * kTile + (int64_t)threadIdx.x * kPer;
  double out[kPer], nrm[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (v.head >> i & 1u) {
      run.c += 1;
      run.p = Pair{0, 0};
      const size_t h = (size_t)t * kHMax + run.c - 1;
      E = __ldcg(hE + h);
      k0 = __ldcg(hk + h);
    } else if (i < v.nvalid) {
      run.p = compose(run.p, elem_map(v, i));
    }
    out[i] = (E == kZero) ? 0.0 : (double)apply(run.p, k0) * pow2(E - 52);
    // normalised copy for the ancestor search (smc.py:277-278, the same IEEE division)
    nrm[i] = (i0 + i == N - 1) ? 1.0 : out[i] / total;
  }
  if (v.nvalid == kPer) {
#pragma unroll
    for (int i = 0; i < kPer; i += 2) {
      *reinterpret_cast<double2*>(cum + i0 + i) = make_double2(out[i], out[i + 1]);
      *reinterpret_cast<double2*>(cumn + i0 + i) = make_double2(nrm[i], nrm[i + 1]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (i < v.nvalid) {
        cum[i0 + i] = out[i];
        cumn[i0 + i] = nrm[i];
      }
  }
}

}  // namespace

size_t exact_cumsum_ws_bytes(int64_t N) { return layout(N).total; }
size_t exact_cumsum_norm_offset(int64_t N) { return layout(N).cumn; }

int exact_cumsum_mode(int64_t N, const void* ws, int32_t* mode, cudaStream_t st) {
  SPA_CHECK_CUDA(cudaMemcpyAsync(mode, reinterpret_cast<const char*>(ws) + layout(N).ctrl + 12, sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, st));
  return 0;
}

int exact_cumsum(const WSrc& w, int64_t N, void* ws, const double* gate, cudaStream_t st) {
  SPA_REQUIRE(N > 0 && ws && w.nparts >= 1 && w.nparts <= 8, kBadArgument, "exact_cumsum: bad arguments");
  const Layout L = layout(N);
  SPA_CHECK_CUDA(cudaMemsetAsync(at<char>(ws, L.ctrl), 0, 16, st));
  const unsigned grid = (unsigned)L.ntiles;
  scan_tile_sums_kernel<<<grid, kThreads, 0, st>>>(w, N, ws, gate);
  SPA_CHECK_LAUNCH();
  scan_segments_kernel<<<grid, kThreads, 0, st>>>(w, N, ws, gate);
  SPA_CHECK_LAUNCH();
  scan_values_kernel<<<grid, kThreads, 0, st>>>(w, N, ws, gate);
  SPA_CHECK_LAUNCH();
  return 0;
}

}  // namespace spa
