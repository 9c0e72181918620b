// libspa_b200: C-ABI entry points and the bandwidth-bound SMC kernels
// (pack, prior/reweight, log-sum-exp/ESS, systematic resampling, gather,
// RW-cov moments/factor/propose/accept) plus the tcgen05 likelihood launcher.
//
// Reference functions replaced are cited on each entry point (see also
// include/spa_b200.h).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cooperative_groups.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>
#include <thread>
#include <cstring>
#include <string>

#include "../../include/spa_b200.h"
#include "common.cuh"
#include "philox.cuh"
#include "resample.cuh"
#include "tc_gemm.cuh"
#include "tc_k1_i8.cuh"
#include "tc_lz_pair.cuh"

namespace spa {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// TMA descriptor construction via the driver entry point (no -lcuda link).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_memGetAddressRange mem_range_fn() {
  static PFN_memGetAddressRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_memGetAddressRange>(p);
  });
  return fn;
}

// cuTensorMapEncodeTiled through a small per-thread cache: a map depends only
// on its arguments, and the sampler re-encodes the same few maps (the same
// buffers) for every launch -- ~2 us of host time each in a launch-bound step.
struct TmapKey {
  int dev, dtype, rank, swizzle, l2;
  const void* ptr;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3];
};
static int encode_tmap_cached(CUtensorMap* map, CUtensorMapDataType dt, int rank, const void* ptr,
                              const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                              CUtensorMapSwizzle sw, CUtensorMapL2promotion l2) {
  struct Entry {
    TmapKey key;
    CUtensorMap map;
    bool used;
  };
  static thread_local Entry cache[64];
  static thread_local int next = 0;
  TmapKey k;
  std::memset(&k, 0, sizeof(k));
  SPA_CHECK_CUDA(cudaGetDevice(&k.dev));
  k.dtype = (int)dt;
  k.rank = rank;
  k.swizzle = (int)sw;
  k.l2 = (int)l2;
  k.ptr = ptr;
  for (int i = 0; i < rank; ++i) {
    k.dims[i] = dims[i];
    k.box[i] = box[i];
    if (i + 1 < rank) k.strides[i] = strides[i];
  }
  for (auto& e : cache)
    if (e.used && std::memcmp(&e.key, &k, sizeof(k)) == 0) {
      *map = e.map;
      return 0;
    }
  auto enc = tmap_encoder();
  if (!enc) return fail(kDriverEntryPoint, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, dt, (cuuint32_t)rank, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(kDriverEntryPoint, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  Entry& e = cache[next];
  next = (next + 1) % 64;
  e.key = k;
  e.map = *map;
  e.used = true;
  return 0;
}

// 16-bit (bf16 / fp16) matrix [rows][cols] row-major; box = 64 columns x
// box_rows rows, 128B swizzle.
static int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t cols, uint64_t rows, uint32_t box_rows,
                          bool f16 = false) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  return encode_tmap_cached(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims,
                            strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

// byte matrix [rows][cols] row-major (the int8 K1 planes); box = 64 columns
// x 128 rows, 64B swizzle (one swizzle atom per row of the box)
static int make_tmap_u8(CUtensorMap* map, const void* ptr, uint64_t cols, uint64_t rows, uint32_t box_rows = 128) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {(cuuint32_t)kI8BK, box_rows};
  return encode_tmap_cached(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ptr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

// Output map for EpiStoreT: [units][rows][cols] (OutT = float / bf16), row
// stride ld, unit stride unit_stride elements; box 32 x 32 x 1 with the
// swizzle matching the epilogue's staging layout (SW128 fp32, SW64 bf16).
template <class OutT>
static int make_tmap_out(CUtensorMap* map, void* ptr, uint64_t cols, uint64_t rows, uint64_t units, uint64_t ld,
                         uint64_t unit_stride) {
  constexpr bool f32 = sizeof(OutT) == 4;
  if ((ld * sizeof(OutT)) % 16 || (unit_stride * sizeof(OutT)) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15))
    return fail(kBadArgument, "TMA store: output rows must be 16-byte aligned");
  cuuint64_t dims[3] = {cols, rows, units};
  cuuint64_t strides[2] = {ld * sizeof(OutT), unit_stride * sizeof(OutT)};
  cuuint32_t box[3] = {32, 32, 1};
  return encode_tmap_cached(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ptr, dims,
                            strides, box, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE);
}

template <int TA, int TB, int BN, class Epi, int TM = 1, bool F16 = false>
static int launch_tc(const void* A, uint64_t a_cols, const void* B, uint64_t b_cols, uint64_t b_rows, TcArgs args,
                     int units, const Epi& epi, cudaStream_t st) {
  constexpr int kSmem = tc_smem_bytes<TA, TB, BN, Epi, TM>();
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, A, a_cols, (uint64_t)args.m, kTcBM, F16);
  if (rc) return rc;
  rc = make_tmap_bf16(&tb, B, b_cols, b_rows, BN, F16);
  if (rc) return rc;
  auto kern = tc_gemm_kernel<TA, TB, BN, Epi, TM, F16>;
  static bool attr_done = false;  // per template instantiation
  if (!attr_done) {
    SPA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_done = true;
  }
  args.units = units;
  // persistent: one CTA per SM (the ring uses ~200 KB of smem) over all items
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    SPA_CHECK_CUDA(cudaGetDevice(&dev));
    SPA_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int grid = std::min((args.m_tiles + TM - 1) / TM * units, sms);
  kern<<<grid, kTcThreads, kSmem, st>>>(ta, tb, args, epi);
  SPA_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Generalised-t prior pieces (reference model.py:78-88)
struct PriorConst {
  double a, c, c_prev;
  double lc;  // -log(2c)
  double lr;  // log(c_prev / c)
  int de;     // a = +inf: double exponential
  double k, k_prev;  // 1 / (a c), 1 / (a c_prev) (0 for de); the same IEEE division as on the device
};

__device__ __forceinline__ double gt_logpdf(double b, const PriorConst& p) {
  const double x = fabs(b);
  if (p.de) return p.lc - x / p.c;
  return p.lc - (p.a + 1.0) * log1p(x / (p.a * p.c));
}

// gt(b; c) - gt(b; c_prev) without cancellation:
//   log(c_prev/c) - (a+1) log1p( (x/a)(1/c - 1/c_prev) / (1 + x/(a c_prev)) )
__device__ __forceinline__ double gt_logratio(double b, const PriorConst& p) {
  const double x = fabs(b);
  const double lr = p.lr;
  if (p.de) return lr - x * (1.0 / p.c - 1.0 / p.c_prev);
  const double num = (x / p.a) * (1.0 / p.c - 1.0 / p.c_prev);
  return lr - (p.a + 1.0) * log1p(num / (1.0 + x / (p.a * p.c_prev)));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 2^-48 fixed point for the order-independent moment sums
constexpr double kFix = 281474976710656.0;  // 2^48

__device__ __forceinline__ unsigned long long to_fix(double v) { return (unsigned long long)llrint(v * kFix); }
__device__ __forceinline__ double from_fix(unsigned long long v) { return (double)(long long)v / kFix; }

// Per-lane log-prior accumulator shared by pack_kernel, pack_eps_kernel and
// prior_kernel mode 2 (same lane->column mapping and multiplication order, so
// all three produce identical bits):
//   sum_j gt(p_j) = npen*(-log 2c) - (a+1) * log prod_j (1 + |p_j|/(a c))
// Columns arrive in groups of 4 with 0/1 penalty flags; the group factor is
// formed branch-free (an unpenalised column contributes exactly 1) and the
// float64 running product is flushed into the log sum, once per group,
// before it could overflow (a = inf: the linear double-exponential form).
struct LpAcc {
  double logsum = 0.0, prod = 1.0, lin = 0.0;
  float npen = 0.f;
  __device__ __forceinline__ void add4(const float (&p)[4], const float (&pen)[4], double K, int de) {
    npen += (pen[0] + pen[1]) + (pen[2] + pen[3]);
    // an unpenalised column enters as x = 0 (factor exactly 1): a float32
    // select instead of a float64 multiply by the 0/1 flag
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (double)(pen[i] != 0.f ? fabsf(p[i]) : 0.f);
    if (de) {
      lin += (x[0] + x[1]) + (x[2] + x[3]);
      return;
    }
    const double g = fma(x[0], K, 1.0) * fma(x[1], K, 1.0) * (fma(x[2], K, 1.0) * fma(x[3], K, 1.0));
    if (prod < 1e200 && g < 1e100) {
      prod *= g;
    } else {
      logsum += log(prod) + log(g);
      prod = 1.0;
    }
  }
  __device__ __forceinline__ double value(const PriorConst& pc) const {
    return pc.de ? (double)npen * pc.lc - lin / pc.c : (double)npen * pc.lc - (pc.a + 1.0) * (logsum + log(prod));
  }
};

// ---------------------------------------------------------------------------
// K1 operand element: fp16 hi/lo split.  hi = fp16(x), lo = fp16(x - hi)
// carries 22 significant bits (bf16 hi/lo: 16, which left 1e-5-relative
// log-likelihood errors on diffuse particles: tests/test_gpu_bench_shapes.py);
// the MMA rate of kind::f16 is the same for fp16 and bf16.  fp16 has a finite
// range: a row with |alpha_j beta_j| >= 65504 (|beta| ~ 4e4) cannot be packed
// and gets a NaN linear term (its log-likelihood is NaN: an MH proposal with
// NaN log-ratio is rejected; the reference's value there is ~ -1e4 * n).
constexpr float kOpMax = 65504.f;
__device__ __forceinline__ void split_op(float x, __half& h, __half& l, float& flag_into) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
  if (!(fabsf(x) < kOpMax)) flag_into = __int_as_float(0x7fc00000);
}

// Integer-coded designs feed K1 on the int8 tensor cores (tc_k1_i8.cuh): the
// row is a 22-bit fixed-point vector relative to its largest |alpha_j beta_j|,
// Q = rint(alpha_j beta_j / s) with |Q| <= 2^21 - 1, stored as three byte
// planes [hi | mid | lo] (Q = hi 2^14 + mid 2^6 + lo, hi signed), followed
// after the m rows by {s, o} per row (o = sum_j gamma_j beta_j).  A row
// whose maximum is not finite gets s = 0 and a NaN linear term.
constexpr float kQMax = 2097151.0f;  // 2^21 - 1
__device__ __forceinline__ uint32_t pack_low_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ void emit_i8_4(uint8_t* __restrict__ row8, int kp, int j0, const float (&bs)[4],
                                          float inv) {
  // rint(bs * inv) through the 1.5 * 2^23 magic constant: the float's low 22
  // bits are Q mod 2^22 (|bs * inv| <= 2^21 - 1 + 1/4 for a finite row, so no
  // clamp: a non-finite row has inv = 0 and s = 0, its bytes are never used).
  // r << 2 puts Q's bits 6..13 in byte 1 and bits 14..21 (hi, two's
  // complement) in byte 2; lo = the low 6 bits of byte 0.
  uint32_t r[4], r4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[i] = __float_as_uint(fmaf(bs[i], inv, 12582912.0f));
    r4[i] = r[i] << 2;
  }
  const uint32_t p01 = __byte_perm(r4[0], r4[1], 0x6521);  // {mid0, hi0, mid1, hi1}
  const uint32_t p23 = __byte_perm(r4[2], r4[3], 0x6521);
  const uint32_t hi = __byte_perm(p01, p23, 0x7531);
  const uint32_t mid = __byte_perm(p01, p23, 0x6420);
  const uint32_t lo = pack_low_bytes(r[0], r[1], r[2], r[3]) & 0x3F3F3F3Fu;
  __stcs(reinterpret_cast<uint32_t*>(row8 + j0), hi);
  __stcs(reinterpret_cast<uint32_t*>(row8 + kp + j0), mid);
  __stcs(reinterpret_cast<uint32_t*>(row8 + 2 * kp + j0), lo);
}
__device__ __forceinline__ void emit_f16_4(__half* __restrict__ row16, int kp, int j0, const float (&bs)[4]) {
  __align__(8) __half h[4], l[4];
  float unused = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) split_op(bs[i], h[i], l[i], unused);
  __stcs(reinterpret_cast<uint2*>(row16 + j0), *reinterpret_cast<const uint2*>(h));
  __stcs(reinterpret_cast<uint2*>(row16 + kp + j0), *reinterpret_cast<const uint2*>(l));
}
// {s, o} of the coded rows, after the m rows of byte planes
__host__ __device__ inline float2* k1_rowc(void* A, int64_t m, int kp) {
  return reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(A) + (size_t)m * 3 * kp);
}
// (1/2) sum_i eta_ki = (1/2) prop_k . X^T 1 of the coded rows, after {s, o}:
// K1 sums the symmetric part |eta|/2 + log(1 + e^-|eta|) of softplus(eta)
// (one instruction per element fewer than max(eta, 0) + log(1 + e^-|eta|))
// and adds this linear half in its row reduction
__host__ __device__ inline double* k1_half(void* A, int64_t m, int kp) {
  return reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(k1_rowc(A, m, kp)) + (size_t)m * sizeof(float2));
}
__device__ __forceinline__ void emit_row_constants(void* A, int64_t m, int kp, int64_t row, float amax, double off,
                                                   double hx, double* ylin_row) {
  const bool ok = amax < INFINITY;  // false for inf / NaN
  k1_rowc(A, m, kp)[row] = make_float2(ok ? amax / kQMax : 0.f, (float)off);
  k1_half(A, m, kp)[row] = 0.5 * hx;
  if (!ok || !(fabs(off) < 3.0e38)) *ylin_row = __longlong_as_double(0x7ff8000000000000ll);
}
// max that propagates NaN (PTX max.NaN): the row maximum flags a NaN / inf row by itself
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float i8_inv(float amax) { return (amax > 0.f && amax < INFINITY) ? kQMax / amax : 0.f; }

// ---------------------------------------------------------------------------
// Pack particle rows into the K1 A operand [m][2*kp] fp16 = [hi | lo] of the
// scaled coefficients; coded designs carry the centring offset
// o = sum_j gamma_j beta_j in three fp16 columns q..q+2 of the hi block (the
// B operand holds 1 there), so the MMA yields eta directly.
// One warp per particle row; lanes take 4 consecutive columns (float4).
// prop = beta (+ eps); A = [hi | lo] of alpha*prop; ylin = prop . X^T y;
// off (coded) into the offset columns; lp = sum gt(prop) (float32 terms,
// float64 accumulation).
__global__ void pack_kernel(spa_design d, const float* __restrict__ beta, const __nv_bfloat16* __restrict__ eps, int64_t m,
                            int ldb, void* __restrict__ A, double* __restrict__ ylin, PriorConst pc,
                            double* __restrict__ lp) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const float* b = beta + row * ldb;
  const __nv_bfloat16* e = eps ? eps + row * ldb : nullptr;
  double yl = 0.0, off = 0.0, hx = 0.0;
  LpAcc la;
  const double K = pc.de ? 0.0 : 1.0 / (pc.a * pc.c);
  const bool vec = (ldb & 3) == 0;
  auto load_p = [&](int j0, float (&p)[4]) {
    p[0] = p[1] = p[2] = p[3] = 0.f;
    if (vec && j0 + 4 <= d.q) {
      const float4 x = *reinterpret_cast<const float4*>(b + j0);
      p[0] = x.x;
      p[1] = x.y;
      p[2] = x.z;
      p[3] = x.w;
      if (e) {
        const uint2 yv = *reinterpret_cast<const uint2*>(e + j0);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&yv);
        const float2 ya = __bfloat1622float2(y2[0]), yb = __bfloat1622float2(y2[1]);
        p[0] += ya.x;
        p[1] += ya.y;
        p[2] += yb.x;
        p[3] += yb.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (j0 + i < d.q) p[i] = b[j0 + i] + (e ? __bfloat162float(e[j0 + i]) : 0.f);
    }
  };
  // pass 1: linear term, offset, log-prior and the row maximum of |alpha p|
  float amax = 0.f;
  bool bad = false;
  for (int j0 = lane * 4; j0 < d.kp; j0 += 128) {
    float p[4];
    load_p(j0, p);
    float fy = 0.f, fo = 0.f, fx = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = j0 + i;
      if (j < d.q) {
        const float bs = (float)d.alpha[j] * p[i];
        amax = fmaxf(amax, fabsf(bs));
        bad |= !(fabsf(bs) < INFINITY);
        fy = fmaf(p[i], (float)d.sy[j], fy);
        fo = fmaf(p[i], d.coded ? (float)d.gamma[j] : 0.f, fo);
        fx = fmaf(p[i], d.coded ? (float)d.sx[j] : 0.f, fx);
        if (!d.coded && !(fabsf(bs) < kOpMax)) fy = __int_as_float(0x7fc00000);
      }
    }
    hx += fx;
    if (lp != nullptr) {
      float pen[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pen[i] = (j0 + i < d.q && d.penalized[j0 + i]) ? 1.f : 0.f;
      la.add4(p, pen, K, pc.de);
    }
    yl += fy;
    off += fo;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (__any_sync(0xffffffffu, bad)) amax = INFINITY;  // NaN / inf in the row
  // pass 2: the K1 operand (int8 planes for coded designs, fp16 hi/lo otherwise)
  const float inv = i8_inv(amax);
  for (int j0 = lane * 4; j0 < d.kp; j0 += 128) {
    float p[4], bs[4];
    load_p(j0, p);
#pragma unroll
    for (int i = 0; i < 4; ++i) bs[i] = j0 + i < d.q ? (float)d.alpha[j0 + i] * p[i] : 0.f;
    if (d.coded)
      emit_i8_4(reinterpret_cast<uint8_t*>(A) + row * 3 * (int64_t)d.kp, d.kp, j0, bs, inv);
    else
      emit_f16_4(reinterpret_cast<__half*>(A) + row * 2 * (int64_t)d.kp, d.kp, j0, bs);
  }
  yl = warp_sum(yl);
  off = warp_sum(off);
  hx = warp_sum(hx);
  double lps = 0.0;
  if (lp != nullptr) lps = warp_sum(la.value(pc));
  if (lane == 0) {
    ylin[row] = yl;
    if (lp != nullptr) lp[row] = lps;
    // eta = sum_j g_ij alpha_j beta_j + sum_j gamma_j beta_j: the offset rides in the row constants
    if (d.coded) emit_row_constants(A, m, d.kp, row, amax, off, hx, ylin + row);
  }
}

// Proposal pack (spa_rw_propose): same arithmetic as pack_kernel.  Each block
// stages the per-column constants (alpha, X^T y, gamma as float32, the
// penalty flag) in shared memory once; each warp then walks its rows through
// a 2-slot shared-memory ring filled by 1-D bulk copies (beta row | eps row),
// so the next row streams in while the current one is packed and no load
// data lives in registers.  IT = kp/128 groups of 4 columns per lane.
constexpr int kPackWarps = 8;
constexpr int kPackSlots = 2;  // rows in flight per warp (current + 1 ahead; 3 blocks per SM)

// prop = beta + eps for 4 columns of a staged (shared-memory) row
__device__ __forceinline__ void ring_prop4(const float* b, const __nv_bfloat16* e, int j0, int q, bool full,
                                           float (&p)[4]) {
  p[0] = p[1] = p[2] = p[3] = 0.f;
  if (full && j0 + 4 <= q) {
    const float4 xv = *reinterpret_cast<const float4*>(b + j0);
    const uint2 ev = *reinterpret_cast<const uint2*>(e + j0);
    const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&ev);
    const float2 ya = __bfloat1622float2(y2[0]), yb = __bfloat1622float2(y2[1]);
    p[0] = xv.x + ya.x;
    p[1] = xv.y + ya.y;
    p[2] = xv.z + yb.x;
    p[3] = xv.w + yb.y;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (j0 + i < q) p[i] = b[j0 + i] + __bfloat162float(e[j0 + i]);
  }
}

__host__ __device__ inline size_t pack_eps_smem_bytes(int kp, int ldb) {
  return (size_t)20 * kp + (size_t)kPackWarps * kPackSlots * ((size_t)ldb * 6);
}

template <int IT, bool CODED>
__global__ void __launch_bounds__(32 * kPackWarps, 3) pack_eps_kernel(spa_design d, const float* __restrict__ beta,
                                                                const __nv_bfloat16* __restrict__ eps, int64_t m,
                                                                int ldb, void* __restrict__ A,
                                                                double* __restrict__ ylin, PriorConst pc,
                                                                double* __restrict__ lp) {
  extern __shared__ float4 csm[];  // [kp] x {alpha, sy, gamma, pen}, then the row rings
  __shared__ uint64_t bars[kPackWarps][kPackSlots];
  float* ca = reinterpret_cast<float*>(csm);
  float* cs = ca + d.kp;
  float* cg = cs + d.kp;
  float* cp = cg + d.kp;
  float* cx = cp + d.kp;  // X^T 1 (coded: the linear half of softplus)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rowB = (uint32_t)ldb * 4, slotB = (uint32_t)ldb * 6;
  uint8_t* ring = reinterpret_cast<uint8_t*>(cx + d.kp) + (size_t)warp * kPackSlots * slotB;
  for (int j = threadIdx.x; j < d.kp; j += blockDim.x) {
    const bool v = j < d.q;
    ca[j] = v ? (float)d.alpha[j] : 0.f;
    cs[j] = v ? (float)d.sy[j] : 0.f;
    cg[j] = (v && CODED) ? (float)d.gamma[j] : 0.f;
    cp[j] = (v && d.penalized[j]) ? 1.f : 0.f;
    cx[j] = (v && CODED) ? (float)d.sx[j] : 0.f;
  }
  if (lane == 0) {
    for (int sl = 0; sl < kPackSlots; ++sl) mbar_init(&bars[warp][sl], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t warp0 = (int64_t)blockIdx.x * kPackWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kPackWarps;
  auto issue = [&](int64_t row, int s) {
    if (row < m) {
      mbar_arrive_expect_tx(&bars[warp][s], slotB);
      bulk_g2s(ring + s * slotB, beta + row * ldb, rowB, &bars[warp][s]);
      bulk_g2s(ring + s * slotB + rowB, eps + row * ldb, slotB - rowB, &bars[warp][s]);
    }
  };
  if (lane == 0)
    for (int sl = 0; sl < kPackSlots; ++sl) issue(warp0 + sl * nwarps, sl);
  const double K = pc.de ? 0.0 : 1.0 / (pc.a * pc.c);
  const bool full = (d.q % 4 == 0);  // every 4-column group is either all-valid or all-padding
  uint32_t phase = 0;                // bit s = parity of slot s
  int s = 0;
  for (int64_t row = warp0; row < m; row += nwarps, s = (s + 1 == kPackSlots) ? 0 : s + 1) {
    mbar_wait(&bars[warp][s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const float* b = reinterpret_cast<const float*>(ring + s * slotB);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(ring + s * slotB + rowB);
    double yl = 0.0, off = 0.0, hx = 0.0;  // same grouping as pack_kernel => identical sums
    float amax = 0.f;  // NaN-propagating: a NaN / inf row ends non-finite
    float bsr[IT][4];  // alpha * prop, kept for the operand pass
    // log-prior: the LpAcc product order without its per-chunk overflow
    // branch (factors are >= 1, so the running product can only overflow
    // upwards; one check per lane below), the flag applied as a multiply
    double prod = 1.0, lin = 0.0;
    float npen = 0.f;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int j0 = it * 128 + lane * 4;
      if (j0 >= d.kp) break;
      float fy = 0.f, fo = 0.f, fx = 0.f;
      float p[4];
      ring_prop4(b, e, j0, d.q, full, p);
      const float4 va = *reinterpret_cast<const float4*>(ca + j0);
      const float4 vs = *reinterpret_cast<const float4*>(cs + j0);
      const float4 vg = *reinterpret_cast<const float4*>(cg + j0);
      const float4 vp = *reinterpret_cast<const float4*>(cp + j0);
      const float4 vx = *reinterpret_cast<const float4*>(cx + j0);
      const float a4[4] = {va.x, va.y, va.z, va.w}, s4[4] = {vs.x, vs.y, vs.z, vs.w};
      const float g4[4] = {vg.x, vg.y, vg.z, vg.w}, p4[4] = {vp.x, vp.y, vp.z, vp.w};
      const float x4[4] = {vx.x, vx.y, vx.z, vx.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float bs = a4[i] * p[i];
        bsr[it][i] = bs;
        fy = fmaf(p[i], s4[i], fy);
        fo = fmaf(p[i], g4[i], fo);
        if (CODED) fx = fmaf(p[i], x4[i], fx);
        if (CODED) {
          amax = fmax_nan(amax, fabsf(bs));
        } else if (!(fabsf(bs) < kOpMax)) {
          fy = __int_as_float(0x7fc00000);
        }
      }
      {
        npen += (p4[0] + p4[1]) + (p4[2] + p4[3]);
        const double x0 = (double)(fabsf(p[0]) * p4[0]), x1 = (double)(fabsf(p[1]) * p4[1]);
        const double x2 = (double)(fabsf(p[2]) * p4[2]), x3 = (double)(fabsf(p[3]) * p4[3]);
        if (pc.de)
          lin += (x0 + x1) + (x2 + x3);
        else
          prod *= fma(x0, K, 1.0) * fma(x1, K, 1.0) * (fma(x2, K, 1.0) * fma(x3, K, 1.0));
      }
      yl += fy;
      off += fo;
      hx += fx;
    }
    if (CODED) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (!(amax < INFINITY)) amax = INFINITY;  // NaN / inf in the row
    }
    double lpl;
    if (pc.de) {
      lpl = (double)npen * pc.lc - lin / pc.c;
    } else {
      double lsum;
      if (prod < 1e200) {
        lsum = log(prod);
      } else {  // a huge |beta + eps|: the same factors as a sum of logs
        lsum = 0.0;
#pragma unroll 1
        for (int j = lane * 4; j < d.q; j += 128)
#pragma unroll 1
          for (int i = j; i < j + 4 && i < d.q; ++i) {
            const double x = (double)(fabsf(b[i] + __bfloat162float(e[i])) * cp[i]);
            lsum += log(fma(x, K, 1.0));
          }
      }
      lpl = (double)npen * pc.lc - (pc.a + 1.0) * lsum;
    }
    __syncwarp();  // every lane is done with slot s: refill it
    if (lane == 0) {
      fence_proxy_async_smem();
      issue(row + kPackSlots * nwarps, s);
    }
    {  // the K1 operand from the registers
      const float inv = i8_inv(amax);
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int j0 = it * 128 + lane * 4;
        if (j0 >= d.kp) break;
        if (CODED)
          emit_i8_4(reinterpret_cast<uint8_t*>(A) + row * 3 * (int64_t)d.kp, d.kp, j0, bsr[it], inv);
        else
          emit_f16_4(reinterpret_cast<__half*>(A) + row * 2 * (int64_t)d.kp, d.kp, j0, bsr[it]);
      }
    }
    yl = warp_sum(yl);
    off = warp_sum(off);
    if (CODED) hx = warp_sum(hx);
    const double lps = warp_sum(lpl);
    if (lane == 0) {
      ylin[row] = yl;
      if (lp != nullptr) lp[row] = lps;
      if (CODED) emit_row_constants(A, m, d.kp, row, amax, off, hx, ylin + row);
    }
  }
}

// pack_eps with R = 32 / LPR particle rows per warp iteration (LPR lanes per
// row, lane l of a row takes columns 4 (it LPR + l) .. +3): the per-row
// overhead -- the ring wait, three reductions, the log, the row's scalar
// stores -- is shared by R rows, which halves it at LPR = 16.  A hi/lo are
// the same bits as pack_eps_kernel; ylin / lp / the offset are summed in a
// different order (float64 rounding).
template <int IT, int LPR, bool CODED>
__global__ void __launch_bounds__(32 * kPackWarps, 2) pack_eps_rows_kernel(
    spa_design d, const float* __restrict__ beta, const __nv_bfloat16* __restrict__ eps, int64_t m, int ldb,
    void* __restrict__ A, double* __restrict__ ylin, PriorConst pc, double* __restrict__ lp) {
  constexpr int R = 32 / LPR;
  extern __shared__ float4 csm[];  // [kp] x {alpha, sy, gamma, pen}, then the row rings
  __shared__ uint64_t bars[kPackWarps][kPackSlots];
  float* ca = reinterpret_cast<float*>(csm);
  float* cs = ca + d.kp;
  float* cg = cs + d.kp;
  float* cp = cg + d.kp;
  float* cx = cp + d.kp;  // X^T 1 (coded: the linear half of softplus)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane % LPR, rsub = lane / LPR;
  const uint32_t rowB = (uint32_t)ldb * 4, slotB = (uint32_t)ldb * 6, groupB = slotB * R;
  uint8_t* ring = reinterpret_cast<uint8_t*>(cx + d.kp) + (size_t)warp * kPackSlots * groupB;
  for (int j = threadIdx.x; j < d.kp; j += blockDim.x) {
    const bool v = j < d.q;
    ca[j] = v ? (float)d.alpha[j] : 0.f;
    cs[j] = v ? (float)d.sy[j] : 0.f;
    cg[j] = (v && CODED) ? (float)d.gamma[j] : 0.f;
    cp[j] = (v && d.penalized[j]) ? 1.f : 0.f;
    cx[j] = (v && CODED) ? (float)d.sx[j] : 0.f;
  }
  if (lane == 0) {
    for (int sl = 0; sl < kPackSlots; ++sl) mbar_init(&bars[warp][sl], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t ngroups = (m + R - 1) / R;
  const int64_t warp0 = (int64_t)blockIdx.x * kPackWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kPackWarps;
  auto issue = [&](int64_t g, int s) {
    if (g < ngroups) {
      const int nr = (m - g * R) < R ? (int)(m - g * R) : R;
      mbar_arrive_expect_tx(&bars[warp][s], slotB * nr);
      for (int r = 0; r < nr; ++r) {
        const int64_t row = g * R + r;
        uint8_t* dst = ring + s * groupB + r * slotB;
        bulk_g2s(dst, beta + row * ldb, rowB, &bars[warp][s]);
        bulk_g2s(dst + rowB, eps + row * ldb, slotB - rowB, &bars[warp][s]);
      }
    }
  };
  if (lane == 0)
    for (int sl = 0; sl < kPackSlots; ++sl) issue(warp0 + sl * nwarps, sl);
  const double K = pc.de ? 0.0 : 1.0 / (pc.a * pc.c);
  const bool full = (d.q % 4 == 0);  // every 4-column group is either all-valid or all-padding
  uint32_t phase = 0;                // bit s = parity of slot s
  int s = 0;
  for (int64_t g = warp0; g < ngroups; g += nwarps, s = (s + 1 == kPackSlots) ? 0 : s + 1) {
    mbar_wait(&bars[warp][s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const int64_t row = g * R + rsub;
    const bool live = row < m;
    const float* b = reinterpret_cast<const float*>(ring + s * groupB + rsub * slotB);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(ring + s * groupB + rsub * slotB + rowB);
    double yl = 0.0, off = 0.0, hx = 0.0, prod = 1.0, lin = 0.0;
    float npen = 0.f, amax = 0.f;  // amax: NaN-propagating, so a NaN / inf row ends non-finite
    float bsr[IT][4];  // alpha * prop, kept for the operand pass
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      if (it * LPR * 4 >= d.kp) break;  // kp % (4 LPR) == 0 (host-checked): warp-uniform
      const int j0 = (it * LPR + sub) * 4;
      float fy = 0.f, fo = 0.f, fx = 0.f;
      float p[4] = {0.f, 0.f, 0.f, 0.f};
      if (full) {  // q % 4 == 0: the 4 columns are all valid or all padding; selects, no branch
        const bool v = live && j0 < d.q;
        const int jj = v ? j0 : 0;
        const float4 xv = *reinterpret_cast<const float4*>(b + jj);
        const uint2 ev = *reinterpret_cast<const uint2*>(e + jj);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&ev);
        const float2 ya = __bfloat1622float2(y2[0]), yb = __bfloat1622float2(y2[1]);
        p[0] = v ? xv.x + ya.x : 0.f;
        p[1] = v ? xv.y + ya.y : 0.f;
        p[2] = v ? xv.z + yb.x : 0.f;
        p[3] = v ? xv.w + yb.y : 0.f;
      } else if (live) {
        ring_prop4(b, e, j0, d.q, false, p);
      }
      const float4 va = *reinterpret_cast<const float4*>(ca + j0);
      const float4 vs = *reinterpret_cast<const float4*>(cs + j0);
      const float4 vg = *reinterpret_cast<const float4*>(cg + j0);
      const float4 vp = *reinterpret_cast<const float4*>(cp + j0);
      const float4 vx = *reinterpret_cast<const float4*>(cx + j0);
      const float a4[4] = {va.x, va.y, va.z, va.w}, s4[4] = {vs.x, vs.y, vs.z, vs.w};
      const float g4[4] = {vg.x, vg.y, vg.z, vg.w}, p4[4] = {vp.x, vp.y, vp.z, vp.w};
      const float x4[4] = {vx.x, vx.y, vx.z, vx.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float bs = a4[i] * p[i];
        bsr[it][i] = bs;
        fy = fmaf(p[i], s4[i], fy);
        fo = fmaf(p[i], g4[i], fo);
        if (CODED) fx = fmaf(p[i], x4[i], fx);
        if (CODED) {
          amax = fmax_nan(amax, fabsf(bs));
        } else if (!(fabsf(bs) < kOpMax)) {
          fy = __int_as_float(0x7fc00000);
        }
      }
      npen += (p4[0] + p4[1]) + (p4[2] + p4[3]);
      const double x0 = (double)(fabsf(p[0]) * p4[0]), x1 = (double)(fabsf(p[1]) * p4[1]);
      const double x2 = (double)(fabsf(p[2]) * p4[2]), x3 = (double)(fabsf(p[3]) * p4[3]);
      if (pc.de)
        lin += (x0 + x1) + (x2 + x3);
      else
        prod *= fma(x0, K, 1.0) * fma(x1, K, 1.0) * (fma(x2, K, 1.0) * fma(x3, K, 1.0));
      yl += fy;
      off += fo;
      hx += fx;
    }
    // row maximum over the row's LPR lanes (aligned groups of the warp)
    if (CODED) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (!(amax < INFINITY)) amax = INFINITY;  // NaN / inf in the row
    }
    double lpl;
    if (pc.de) {
      lpl = (double)npen * pc.lc - lin / pc.c;
    } else {
      double lsum;
      if (prod < 1e200) {
        lsum = log(prod);
      } else {  // a huge |beta + eps|: the same factors as a sum of logs
        lsum = 0.0;
#pragma unroll 1
        for (int j = sub * 4; j < d.q; j += LPR * 4)
#pragma unroll 1
          for (int i = j; i < j + 4 && i < d.q; ++i) {
            const double x = (double)(fabsf(b[i] + __bfloat162float(e[i])) * cp[i]);
            lsum += log(fma(x, K, 1.0));
          }
      }
      lpl = (double)npen * pc.lc - (pc.a + 1.0) * lsum;
    }
    __syncwarp();  // every lane is done with slot s: refill it
    if (lane == 0) {
      fence_proxy_async_smem();
      issue(g + kPackSlots * nwarps, s);
    }
    if (live) {  // the K1 operand from the registers
      const float inv = i8_inv(amax);
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        if (it * LPR * 4 >= d.kp) break;
        const int j0 = (it * LPR + sub) * 4;
        if (CODED)
          emit_i8_4(reinterpret_cast<uint8_t*>(A) + row * 3 * (int64_t)d.kp, d.kp, j0, bsr[it], inv);
        else
          emit_f16_4(reinterpret_cast<__half*>(A) + row * 2 * (int64_t)d.kp, d.kp, j0, bsr[it]);
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
      yl += __shfl_xor_sync(0xffffffffu, yl, o);
      off += __shfl_xor_sync(0xffffffffu, off, o);
      lpl += __shfl_xor_sync(0xffffffffu, lpl, o);
      if (CODED) hx += __shfl_xor_sync(0xffffffffu, hx, o);
    }
    if (live && sub == 0) {
      ylin[row] = yl;
      if (lp != nullptr) lp[row] = lpl;
      if (CODED) emit_row_constants(A, m, d.kp, row, amax, off, hx, ylin + row);
    }
  }
}

__global__ void prior_kernel(spa_design d, const float* __restrict__ beta, int64_t m, int ldb, PriorConst pc,
                             int mode, double* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const float* b = beta + row * ldb;
  double s = 0.0;
  if (mode == 2) {  // identical arithmetic (and lane->column mapping) to the pack kernels' lp
    LpAcc la;
    const double K = pc.de ? 0.0 : 1.0 / (pc.a * pc.c);
    for (int j0 = lane * 4; j0 < d.kp; j0 += 128) {
      float x[4], pen[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool v = j0 + i < d.q;
        x[i] = v ? b[j0 + i] : 0.f;
        pen[i] = (v && d.penalized[j0 + i]) ? 1.f : 0.f;
      }
      la.add4(x, pen, K, pc.de);
    }
    s = la.value(pc);
  } else if (pc.de) {
    for (int j = lane; j < d.q; j += 32) {
      if (!d.penalized[j]) continue;
      const double bj = (double)b[j];
      s += mode == 0 ? gt_logpdf(bj, pc) : gt_logratio(bj, pc);
    }
  } else {
    // float64 without per-element transcendentals or divisions:
    //   mode 0: sum_j gt = npen*(-log 2c) - (a+1) log prod_j (1 + x_j/(a c))
    //   mode 1: 1 + u_j = (1 + x_j/(a c)) / (1 + x_j/(a c_prev)), so
    //           lw = npen*log(c_prev/c) - (a+1) [log prod (1 + x K) - log prod (1 + x K')]
    // Lanes own 4 consecutive columns (float4 loads); each lane's product is
    // flushed into a log every 8 factors.  Relative error ~1e-14.
    const double K1 = 1.0 / (pc.a * pc.c), K2 = 1.0 / (pc.a * pc.c_prev);
    double la = 0.0, lb = 0.0, pa = 1.0, pb = 1.0;
    int cnt = 0, npen = 0;
    const bool vec = (d.q % 4 == 0) && (ldb % 4 == 0);
    for (int j0 = lane * 4; j0 < d.q; j0 += 128) {
      float xv[4];
      if (vec) {
        const float4 x = __ldcs(reinterpret_cast<const float4*>(b + j0));
        xv[0] = x.x;
        xv[1] = x.y;
        xv[2] = x.z;
        xv[3] = x.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[i] = (j0 + i < d.q) ? b[j0 + i] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (j0 + i >= d.q || !d.penalized[j0 + i]) continue;
        const double x = fabs((double)xv[i]);
        pa *= fma(x, K1, 1.0);
        if (mode == 1) pb *= fma(x, K2, 1.0);
        ++npen;
        ++cnt;
      }
      if (cnt >= 8 || !(pa < 1e250 && pb < 1e250)) {
        la += log(pa);
        if (mode == 1) lb += log(pb);
        pa = pb = 1.0;
        cnt = 0;
      }
    }
    la += log(pa);
    if (mode == 1) lb += log(pb);
    s = mode == 0 ? (double)npen * pc.lc - (pc.a + 1.0) * la : (double)npen * pc.lr - (pc.a + 1.0) * (la - lb);
  }
  s = warp_sum(s);
  if (lane == 0) out[row] = s;
}

// Reweight pass fused with the log-prior at the new scale: one read of the
// particles gives both the incremental weights lw = sum_j gt(c) - gt(c_prev)
// and lp = sum_j gt(c) in the LpAcc arithmetic of prior mode 2 / the pack
// kernels (bit-identical to them), which the move kernels need next.
template <int IT>
__global__ void __launch_bounds__(256) prior_reweight_kernel(spa_design d, const float* __restrict__ beta, int64_t m,
                                                             int ldb, PriorConst pc, double* __restrict__ lw,
                                                             double* __restrict__ lp) {
  __shared__ __align__(16) float pen_s[IT * 128];  // 0/1 penalty flags, padding columns 0
  for (int j = threadIdx.x; j < IT * 128; j += blockDim.x) pen_s[j] = (j < d.q && d.penalized[j]) ? 1.f : 0.f;
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const float* b = beta + row * ldb;
  const double K1 = pc.de ? 0.0 : 1.0 / (pc.a * pc.c), K2 = pc.de ? 0.0 : 1.0 / (pc.a * pc.c_prev);
  const bool full = (d.q % 4 == 0) && (ldb % 4 == 0);
  float4 xv[IT];  // all of the row's loads in flight before any arithmetic
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j0 = it * 128 + lane * 4;
    if (full && j0 + 4 <= d.q) xv[it] = __ldcs(reinterpret_cast<const float4*>(b + j0));
  }
  LpAcc la, lb;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j0 = it * 128 + lane * 4;
    if (j0 >= d.kp) break;
    float x[4], pen[4];
    if (full && j0 + 4 <= d.q) {
      x[0] = xv[it].x;
      x[1] = xv[it].y;
      x[2] = xv[it].z;
      x[3] = xv[it].w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = j0 + i < d.q ? b[j0 + i] : 0.f;
    }
    const float4 pv = *reinterpret_cast<const float4*>(pen_s + j0);
    pen[0] = pv.x;
    pen[1] = pv.y;
    pen[2] = pv.z;
    pen[3] = pv.w;
    la.add4(x, pen, K1, pc.de);
    if (!pc.de) lb.add4(x, pen, K2, 0);
  }
  const double lpv = la.value(pc);
  const double lwv = pc.de ? (double)la.npen * pc.lr - la.lin * (1.0 / pc.c - 1.0 / pc.c_prev)
                           : (double)la.npen * pc.lr -
                                 (pc.a + 1.0) * ((la.logsum + log(la.prod)) - (lb.logsum + log(lb.prod)));
  const double s_lp = warp_sum(lpv), s_lw = warp_sum(lwv);
  if (lane == 0) {
    lw[row] = s_lw;
    lp[row] = s_lp;
  }
}

// Same pass with LPR lanes per particle row (32/LPR rows per warp): lane l
// takes columns 4 (it LPR + l) .. +3, it < IT, all loads in flight first.
// Fewer lanes per row amortise the two float64 logs and the shuffle
// reduction of the per-lane products over 4 IT columns instead of 16.
template <int LPR, int IT>
__global__ void __launch_bounds__(256, 4) prior_reweight_rows_kernel(spa_design d, const float* __restrict__ beta,
                                                                  int64_t m, int ldb, PriorConst pc,
                                                                  double* __restrict__ lw, double* __restrict__ lp) {
  __shared__ __align__(16) float pen_s[LPR * IT * 4];  // 0/1 penalty flags, padding columns 0
  for (int j = threadIdx.x; j < LPR * IT * 4; j += blockDim.x) pen_s[j] = (j < d.q && d.penalized[j]) ? 1.f : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane % LPR;
  const int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / LPR) + lane / LPR;
  const bool live = row < m;
  const float* b = beta + (live ? row : 0) * ldb;
  const double K1 = pc.de ? 0.0 : 1.0 / (pc.a * pc.c), K2 = pc.de ? 0.0 : 1.0 / (pc.a * pc.c_prev);
  const bool full = (d.q % 4 == 0) && (ldb % 4 == 0);
  float4 xv[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j0 = (it * LPR + sub) * 4;
    if (live && full && j0 + 4 <= d.q) xv[it] = __ldcs(reinterpret_cast<const float4*>(b + j0));
  }
  LpAcc la, lb;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j0 = (it * LPR + sub) * 4;
    float x[4], pen[4];
    if (full && j0 + 4 <= d.q) {
      x[0] = xv[it].x;
      x[1] = xv[it].y;
      x[2] = xv[it].z;
      x[3] = xv[it].w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = (live && j0 + i < d.q) ? b[j0 + i] : 0.f;
    }
    const float4 pv = *reinterpret_cast<const float4*>(pen_s + j0);
    pen[0] = pv.x;
    pen[1] = pv.y;
    pen[2] = pv.z;
    pen[3] = pv.w;
    la.add4(x, pen, K1, pc.de);
    if (!pc.de) lb.add4(x, pen, K2, 0);
  }
  double lpv = la.value(pc);
  double lwv = pc.de ? (double)la.npen * pc.lr - la.lin * (1.0 / pc.c - 1.0 / pc.c_prev)
                     : (double)la.npen * pc.lr -
                           (pc.a + 1.0) * ((la.logsum + log(la.prod)) - (lb.logsum + log(lb.prod)));
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    lpv += __shfl_xor_sync(0xffffffffu, lpv, o);
    lwv += __shfl_xor_sync(0xffffffffu, lwv, o);
  }
  if (live && sub == 0) {
    lw[row] = lwv;
    lp[row] = lpv;
  }
}

// The rows kernel for the vector layout (q % 4 == 0, ldb % 4 == 0, a
// 4-byte aligned penalty mask), lean: no per-chunk overflow branch (the
// float64 running product of a lane's factors 1 + |x| K >= 1 can only
// overflow to +inf, which one check per lane at the end catches and
// recomputes as a sum of logs), and no block preamble -- each lane reads the
// 0/1 penalty bytes of its 4 columns as one word (a byte-replicated mask
// zeroes unpenalised columns; popc counts the penalised ones) and the scale
// reciprocals come from the host.  Same lane -> column map and product order
// as the rows kernel: bit-identical to it whenever its overflow branch does
// not fire (every product below 1e200).
template <int LPR, int IT>
__global__ void __launch_bounds__(256, IT >= 16 ? 3 : 4) prior_reweight_lean_kernel(spa_design d, const float* __restrict__ beta,
                                                                  int64_t m, int ldb, PriorConst pc,
                                                                  double* __restrict__ lw, double* __restrict__ lp) {
  const int lane = threadIdx.x & 31, sub = lane % LPR;
  const int64_t row = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / LPR) + lane / LPR;
  const bool live = row < m;
  const float* b = beta + (live ? row : 0) * ldb;
  // the mask words are loaded with the row when registers allow (IT <= 8),
  // else next to their use (L1 hits after the first warps)
  constexpr bool kEager = IT <= 8;
  float4 xv[IT];
  uint32_t pw[kEager ? IT : 1];
  auto mask_word = [&](int it) -> uint32_t {
    const int j0 = (it * LPR + sub) * 4;
    return j0 < d.q ? __ldg(reinterpret_cast<const uint32_t*>(d.penalized + j0)) : 0u;
  };
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j0 = (it * LPR + sub) * 4;
    const bool v = live && j0 < d.q;
    xv[it] = v ? __ldcs(reinterpret_cast<const float4*>(b + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (kEager) pw[kEager ? it : 0] = mask_word(it);
  }
  const double K1 = pc.k, K2 = pc.k_prev;
  int npen = 0;
  double lpv, lwv;
  auto masked = [&](const float4& x, uint32_t w, double (&o)[4]) {
    const uint32_t mk = (w * 0xffu);  // 0x01 -> 0xff per byte (flags are 0/1: no carries)
    o[0] = (double)__uint_as_float(__float_as_uint(fabsf(x.x)) & __byte_perm(mk, 0, 0x8888));
    o[1] = (double)__uint_as_float(__float_as_uint(fabsf(x.y)) & __byte_perm(mk, 0, 0x9999));
    o[2] = (double)__uint_as_float(__float_as_uint(fabsf(x.z)) & __byte_perm(mk, 0, 0xaaaa));
    o[3] = (double)__uint_as_float(__float_as_uint(fabsf(x.w)) & __byte_perm(mk, 0, 0xbbbb));
  };
  if (pc.de) {
    double lin = 0.0;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      double x[4];
      const uint32_t w = kEager ? pw[kEager ? it : 0] : mask_word(it);
      masked(xv[it], w, x);
      npen += __popc(w);
      lin += (x[0] + x[1]) + (x[2] + x[3]);
    }
    lpv = (double)npen * pc.lc - lin / pc.c;
    lwv = (double)npen * pc.lr - lin * (1.0 / pc.c - 1.0 / pc.c_prev);
  } else {
    double pa = 1.0, pb = 1.0;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      double x[4];
      const uint32_t w = kEager ? pw[kEager ? it : 0] : mask_word(it);
      masked(xv[it], w, x);
      npen += __popc(w);
      pa *= fma(x[0], K1, 1.0) * fma(x[1], K1, 1.0) * (fma(x[2], K1, 1.0) * fma(x[3], K1, 1.0));
      pb *= fma(x[0], K2, 1.0) * fma(x[1], K2, 1.0) * (fma(x[2], K2, 1.0) * fma(x[3], K2, 1.0));
    }
    double la, lb;
    if (pa < 1e200 && pb < 1e200) {
      la = log(pa);
      lb = log(pb);
    } else {  // a huge |beta|: the same factors as a sum of logs (row re-read)
      la = lb = 0.0;
#pragma unroll 1
      for (int it = 0; it < IT; ++it) {
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          const int j = (it * LPR + sub) * 4 + i;
          const double x = (j < d.q && d.penalized[j]) ? (double)fabsf(b[j]) : 0.0;
          la += log(fma(x, K1, 1.0));
          lb += log(fma(x, K2, 1.0));
        }
      }
    }
    lpv = (double)npen * pc.lc - (pc.a + 1.0) * la;
    lwv = (double)npen * pc.lr - (pc.a + 1.0) * (la - lb);
  }
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) {
    lpv += __shfl_xor_sync(0xffffffffu, lpv, o);
    lwv += __shfl_xor_sync(0xffffffffu, lwv, o);
  }
  if (live && sub == 0) {
    lw[row] = lwv;
    lp[row] = lpv;
  }
}

// ---------------------------------------------------------------------------
// f1: per-step weighted marginal summaries (reference summary.py:36-61) on
// the device -- weighted mean, weighted quantiles ("smallest value whose
// cumulative weight reaches q") and concentration V(delta) per coordinate.
// Weights are 2^-62 fixed point and every sum is an exact integer sum, so
// results do not depend on the schedule or the number of GPUs (histograms
// all-reduce exactly).  Quantiles by 4-pass radix select on order-preserving
// 32-bit keys of the float32 particles: pass p histograms the p-th key byte
// of the rows whose higher bytes match the level's prefix, a select step
// picks the byte where the cumulative weight reaches q * total.
constexpr int kSumMaxLev = 4, kSumMaxDelta = 4, kSumCols = 8, kSumRows = 2048, kSumTile = 256;
constexpr double kWFix = 4611686018427387904.0;  // 2^62

struct SumParams {
  int nlev, ndelta;
  double level[kSumMaxLev];
  float delta[kSumMaxDelta];
};

__device__ __forceinline__ uint32_t sum_key(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float sum_unkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ unsigned long long sum_wfix(double w) {
  return w > 0.0 ? (unsigned long long)llrint(w * kWFix) : 0ull;
}

// Shared-memory 64-bit bin counters as two native 32-bit atomics (a 64-bit
// shared atomicAdd compiles to a CAS spin loop): the low-word add returns the
// old value, so each adder knows its own carry exactly.
__device__ __forceinline__ void sum_add64(uint32_t* h2, unsigned long long v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(h2, lo);
  const uint32_t carry = (old + lo < old) ? 1u : 0u;
  if (hi + carry) atomicAdd(h2 + 1, hi + carry);
}

// Warp-wide histogram add of (bin, v) for the lanes with `hit` (called by
// all 32 lanes): up to kAgg distinct bins are summed in registers first
// (ballot + __reduce_add_sync over 21-bit limbs) -- pass 0 keys (sign and
// exponent) concentrate in few bins, which would otherwise serialise on one
// counter -- the rest add directly (later passes: spread digits, kAgg = 0).
template <int kAgg>
__device__ __forceinline__ void sum_warp_add(uint32_t* h2, bool hit, uint32_t bin, unsigned long long v) {
  const int lane = threadIdx.x & 31;
  unsigned pending = __ballot_sync(0xffffffffu, hit);
#pragma unroll 1
  for (int it = 0; it < kAgg && pending; ++it) {
    const int leader = __ffs(pending) - 1;
    const uint32_t b = __shfl_sync(0xffffffffu, bin, leader);
    const bool mine = hit && bin == b && ((pending >> lane) & 1u);
    const unsigned grp = __ballot_sync(0xffffffffu, mine);
    const uint32_t l0 = mine ? (uint32_t)(v & 0x1FFFFFull) : 0u;
    const uint32_t l1 = mine ? (uint32_t)((v >> 21) & 0x1FFFFFull) : 0u;
    const uint32_t l2 = mine ? (uint32_t)(v >> 42) : 0u;
    const unsigned long long s = (unsigned long long)__reduce_add_sync(0xffffffffu, l0) +
                                 ((unsigned long long)__reduce_add_sync(0xffffffffu, l1) << 21) +
                                 ((unsigned long long)__reduce_add_sync(0xffffffffu, l2) << 42);
    if (lane == leader) sum_add64(h2 + 2 * b, s);
    pending &= ~grp;
  }
  if ((pending >> lane) & 1u) sum_add64(h2 + 2 * bin, v);
}

// Pass p over a block of kSumCols columns x kSumRows particles, staged per
// kSumTile-row tile in shared memory; warp c owns column c0 + c.  Pass 0 also
// accumulates the weighted mean (2^-48 fixed point), the mass inside
// (-delta, delta) per delta and the total weight (2^-62 fixed point).
__global__ void __launch_bounds__(256) summary_hist_kernel(const float* __restrict__ beta, int64_t m, int ldb, int q,
                                                           const double* __restrict__ w, SumParams sp, int pass,
                                                           const uint32_t* __restrict__ prefix,
                                                           unsigned long long* __restrict__ hist,
                                                           unsigned long long* __restrict__ acc_mean,
                                                           unsigned long long* __restrict__ acc_in,
                                                           unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t sh[];  // [nh][kSumCols][256] x {lo, hi} words
  __shared__ float xs[kSumTile][kSumCols + 1];
  __shared__ unsigned long long wf[kSumTile];
  __shared__ double wd[kSumTile];
  const int nh = pass == 0 ? 1 : sp.nlev;
  for (int e = threadIdx.x; e < nh * kSumCols * 256 * 2; e += blockDim.x) sh[e] = 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * kSumCols, col = c0 + warp;
  const int64_t r0 = (int64_t)blockIdx.y * kSumRows;
  uint32_t pre[kSumMaxLev];
#pragma unroll
  // levels past nlev get a prefix no key can have (tops are at most 24 bits)
  for (int l = 0; l < kSumMaxLev; ++l) pre[l] = (pass > 0 && l < sp.nlev && col < q) ? prefix[l * q + col] : ~0u;
  double smean = 0.0;
  unsigned long long sin[kSumMaxDelta] = {0ull, 0ull, 0ull, 0ull}, stot = 0ull;
  // the next tile's particles and weights are loaded into registers while
  // the current tile is histogrammed (the one-tile-at-a-time form spent
  // most of its time waiting on the loads)
  constexpr int kPer = kSumTile * kSumCols / 256;  // elements per thread (blockDim 256)
  static_assert(kSumTile == 256, "one weight per thread");
  const int64_t r1 = min(m, r0 + kSumRows);
  float px[kPer];
  double pw = 0.0;
  auto load_tile = [&](int64_t t0) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * 256, rr = e / kSumCols, cc = e % kSumCols;
      const int64_t row = t0 + rr;
      px[k] = (row < m && c0 + cc < q) ? __ldcs(beta + row * ldb + c0 + cc) : 0.f;
    }
    pw = (t0 + threadIdx.x < m) ? w[t0 + threadIdx.x] : 0.0;
  };
  load_tile(r0);
  for (int64_t t0 = r0; t0 < r1; t0 += kSumTile) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = threadIdx.x + k * 256;
      xs[e / kSumCols][e % kSumCols] = px[k];
    }
    wd[threadIdx.x] = pw;
    wf[threadIdx.x] = sum_wfix(pw);
    __syncthreads();
    if (t0 + kSumTile < r1) load_tile(t0 + kSumTile);
    if (col >= q) continue;
    // rows past m carry weight 0 (wd = wf = 0): no liveness tests needed
    if (pass == 0) {
#pragma unroll 2
      for (int rr = lane; rr < kSumTile; rr += 32) {
        const float x = xs[rr][warp];
        const unsigned long long v = wf[rr];
        smean = fma(wd[rr], (double)x, smean);
#pragma unroll
        for (int dd = 0; dd < kSumMaxDelta; ++dd)
          if (dd < sp.ndelta && fabsf(x) < sp.delta[dd]) sin[dd] += v;
        stot += v;
        sum_warp_add<2>(sh + warp * 512, v != 0ull, sum_key(x) >> 24, v);
      }
    } else {
      const int shift = 32 - 8 * pass;
#pragma unroll 4
      for (int rr = lane; rr < kSumTile; rr += 32) {
        const uint32_t key = sum_key(xs[rr][warp]);
        const uint32_t top = key >> shift;
        const bool any = (top == pre[0]) | (top == pre[1]) | (top == pre[2]) | (top == pre[3]);
        if (__ballot_sync(0xffffffffu, any) == 0u) continue;  // most rows match no level's prefix
        const unsigned long long v = any ? wf[rr] : 0ull;
        const uint32_t dig = (key >> (shift - 8)) & 255u;
#pragma unroll
        for (int l = 0; l < kSumMaxLev; ++l) {
          if (l >= sp.nlev) break;
          sum_warp_add<0>(sh + (l * kSumCols + warp) * 512, v != 0ull && top == pre[l], dig, v);
        }
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nh * kSumCols * 256; e += blockDim.x) {
    const int l = e / (kSumCols * 256), cc = (e / 256) % kSumCols, bin = e % 256;
    const unsigned long long v = (unsigned long long)sh[2 * e] | ((unsigned long long)sh[2 * e + 1] << 32);
    if (v != 0ull && c0 + cc < q) atomicAdd(&hist[((size_t)l * q + c0 + cc) * 256 + bin], v);
  }
  if (pass == 0 && col < q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smean += __shfl_xor_sync(0xffffffffu, smean, o);
#pragma unroll
    for (int dd = 0; dd < kSumMaxDelta; ++dd) {
      unsigned long long v = sin[dd];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && dd < sp.ndelta && v) atomicAdd(&acc_in[(size_t)dd * q + col], v);
    }
    if (lane == 0) atomicAdd(&acc_mean[col], to_fix(smean));
    if (warp == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) stot += __shfl_xor_sync(0xffffffffu, stot, o);
      if (lane == 0 && blockIdx.x == 0) atomicAdd(total, stot);
    }
  }
}

// One warp per (level, column): lanes own 8 bins each; a shuffle scan of the
// lane sums finds the byte whose cumulative weight reaches level * total,
// then the prefix is extended and the weight below it carried.
__global__ void summary_select_kernel(const unsigned long long* __restrict__ hist, int q, SumParams sp, int pass,
                                      const unsigned long long* __restrict__ total, uint32_t* __restrict__ prefix,
                                      unsigned long long* __restrict__ below) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= sp.nlev * q) return;  // warp-uniform
  const int l = i / q, col = i % q;
  const unsigned long long* h = hist + ((size_t)(pass == 0 ? 0 : l) * q + col) * 256 + lane * 8;
  // target = ceil(level * total) in exact integer arithmetic (level as 2^-64 fixed point)
  const unsigned long long qf = (unsigned long long)(sp.level[l] * 18446744073709551616.0);
  const unsigned long long T = *total;
  const unsigned long long target = __umul64hi(qf, T) + ((qf * T) != 0ull ? 1ull : 0ull);
  const unsigned long long base = pass == 0 ? 0ull : below[i];
  unsigned long long hv[8], ls = 0ull;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    hv[k] = h[k];
    ls += hv[k];
  }
  unsigned long long incl = ls;  // inclusive scan over lanes
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const unsigned long long excl = incl - ls;
  const unsigned reach = __ballot_sync(0xffffffffu, base + incl >= target);
  const unsigned nz = __ballot_sync(0xffffffffu, ls != 0ull);
  int pick_lane, pick = -1;
  unsigned long long acc = 0ull;
  if (reach) {
    pick_lane = __ffs(reach) - 1;
    if (lane == pick_lane) {
      acc = base + excl;
      for (int k = 0; k < 8; ++k) {
        if (hv[k] == 0ull) continue;
        if (acc + hv[k] >= target) {
          pick = lane * 8 + k;
          break;
        }
        acc += hv[k];
      }
    }
  } else {  // rounding left the target above the total: the largest value
    pick_lane = 31 - __clz(nz);
    if (lane == pick_lane) {
      int kk = 7;
      while (kk > 0 && hv[kk] == 0ull) --kk;
      pick = lane * 8 + kk;
      acc = base + incl - hv[kk];
    }
  }
  if (lane == pick_lane) {
    below[i] = acc;
    prefix[i] = (pass == 0 ? 0u : prefix[i] << 8) | (uint32_t)pick;
  }
}

__global__ void summary_finish_kernel(int q, SumParams sp, const uint32_t* __restrict__ prefix,
                                      const unsigned long long* __restrict__ acc_mean,
                                      const unsigned long long* __restrict__ acc_in,
                                      const unsigned long long* __restrict__ total, double* __restrict__ out_mean,
                                      double* __restrict__ out_quant, double* __restrict__ out_conc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= q) return;
  const double W = (double)*total / kWFix;
  out_mean[j] = from_fix(acc_mean[j]) / W;
  for (int l = 0; l < sp.nlev; ++l) out_quant[(size_t)l * q + j] = (double)sum_unkey(prefix[(size_t)l * q + j]);
  for (int d = 0; d < sp.ndelta; ++d)
    out_conc[(size_t)d * q + j] = 1.0 - (double)acc_in[(size_t)d * q + j] / (double)*total;
}

// ---------------------------------------------------------------------------
// K3: fixed-chunk log-sum-exp statistics
constexpr int kChunk = 4096;

// One 1024-thread block per fixed 4096-particle chunk; each thread keeps its
// 4 values in registers across the max and sum passes.  The reduction tree is
// fixed (shuffles, then one warp over the 32 warp results), so the chunk
// statistics do not depend on how particles are sharded.
constexpr int kLseThreads = 1024;

__device__ __forceinline__ double block_reduce_1024(double v, double* red, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = red[threadIdx.x & 31];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  __syncthreads();  // red reusable
  return v;
}

__device__ __forceinline__ void lse_chunk_stats(const double* __restrict__ logw, const double* __restrict__ lw,
                                                int64_t m, double* __restrict__ stats, int64_t chunk, double* red) {
  constexpr int kPer = kChunk / kLseThreads;
  const int64_t c0 = chunk * kChunk;
  double x[kPer];
  double mx = -INFINITY;
  bool nan = false;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t k = c0 + threadIdx.x + i * kLseThreads;
    x[i] = k < m ? logw[k] + (lw ? lw[k] : 0.0) : -INFINITY;
    if (x[i] != x[i]) nan = true;
    mx = fmax(mx, x[i]);
  }
  nan = __syncthreads_or(nan);
  mx = block_reduce_1024(mx, red, true);
  double s1 = 0.0, s2 = 0.0;
  if (mx > -INFINITY) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const double e = exp(x[i] - mx);
      s1 += e;
      s2 += e * e;
    }
  }
  s1 = block_reduce_1024(s1, red, false);
  s2 = block_reduce_1024(s2, red, false);
  if (threadIdx.x == 0) {
    stats[3 * chunk + 0] = nan ? NAN : mx;
    stats[3 * chunk + 1] = s1;
    stats[3 * chunk + 2] = s2;
  }
}

__global__ void __launch_bounds__(kLseThreads) lse_stats_kernel(const double* __restrict__ logw,
                                                                const double* __restrict__ lw, int64_t m,
                                                                double* __restrict__ stats) {
  __shared__ double red[32];
  lse_chunk_stats(logw, lw, m, stats, blockIdx.x, red);
}

// one thread: the fixed-order combine of the chunk statistics (L2 loads: in
// reweight_finish_kernel other blocks wrote them, and L1 is not coherent)
// The chunk statistics' combine, one warp: lanes load and exponentiate the
// chunks in parallel; lane 0 then accumulates s1, s2 in chunk order with the
// sequential loop's exact arithmetic (fma(a, f, s1), fma(b f, f, s2)).  A
// single thread doing the loads and exp()s one chunk after another spent
// ~0.5 us per chunk on L2 latency (C3: 16 chunks, twice per lambda step).
__device__ __forceinline__ void lse_combine_warp(const double* __restrict__ stats, int64_t nchunks,
                                                 double* __restrict__ res) {
  const int lane = threadIdx.x & 31;
  double M = -INFINITY;
  bool nan = false;
  for (int64_t c = lane; c < nchunks; c += 32) {
    const double v = __ldcg(&stats[3 * c]);
    if (v != v) nan = true;
    M = fmax(M, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
  nan = __any_sync(0xffffffffu, nan);
  double s1 = 0.0, s2 = 0.0;
  if (M > -INFINITY && !nan) {
    for (int64_t base = 0; base < nchunks; base += 32) {
      const int64_t c = base + lane;
      double av = 0.0, bv = 0.0, f = 0.0;
      int live = 0;
      if (c < nchunks) {
        const double mc = __ldcg(&stats[3 * c]);
        if (mc != -INFINITY) {
          live = 1;
          f = exp(mc - M);
          av = __ldcg(&stats[3 * c + 1]);
          bv = __ldcg(&stats[3 * c + 2]);
        }
      }
      const int cnt = nchunks - base < 32 ? (int)(nchunks - base) : 32;
      for (int l = 0; l < cnt; ++l) {
        const double al = __shfl_sync(0xffffffffu, av, l), bl = __shfl_sync(0xffffffffu, bv, l);
        const double fl = __shfl_sync(0xffffffffu, f, l);
        if (__shfl_sync(0xffffffffu, live, l)) {
          s1 = fma(al, fl, s1);
          s2 = fma(bl * fl, fl, s2);
        }
      }
    }
  }
  if (lane == 0) {
    res[0] = nan ? NAN : (M > -INFINITY ? M + log(s1) : -INFINITY);
    res[1] = nan ? NAN : s1 * s1 / s2;
    res[2] = M;
  }
}

__global__ void lse_combine_kernel(const double* __restrict__ stats, int64_t nchunks, double* __restrict__ res) {
  if (threadIdx.x >= 32) return;
  lse_combine_warp(stats, nchunks, res);
}

__global__ void logw_apply_kernel(double* __restrict__ logw, const double* __restrict__ lw, int64_t m,
                                  const double* __restrict__ res, double* __restrict__ w) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  if (lw) {
    const double v = logw[k] + lw[k] - res[0];
    logw[k] = v;
    if (w) w[k] = exp(v);
  } else if (w) {
    w[k] = exp(logw[k] - res[0]);  // normalised weights, logw untouched
  }
}

// ---------------------------------------------------------------------------
// K4: systematic resampling, bit-exact with the reference (smc.py:273-281).
// The reference cumsum is a strictly sequential float64 accumulation; it is
// reproduced by the parallel binade-segmented scan of resample.cu.  Ancestor
// search is parallel (one thread per slot, binary search on cum / cum[N-1]).
// gate: optional device flag (a step record's "resampled" field); kernels of
// the device-decided resampling path return at once when it is 0.
__device__ __forceinline__ bool gated_off(const double* gate) { return gate != nullptr && !(gate[0] != 0.0); }

// cumn = cum / cum[N-1] with cumn[N-1] = 1 (written by the exact scan):
// anc = searchsorted(cumn, u + k/N, side='right') for slots k0.. (smc.py:279-281)
__global__ void ancestors_kernel(const double* __restrict__ cumn, int64_t N, double u, int64_t k0, int64_t count,
                                 int64_t* __restrict__ anc, const double* __restrict__ gate) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count || gated_off(gate)) return;
  const int64_t k = k0 + i;
  const double pos = u + (double)k / (double)N;
  // first index j with cumn[j] > pos
  int64_t lo = 0, hi = N;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(cumn + mid) > pos)
      hi = mid;
    else
      lo = mid + 1;
  }
  anc[i] = lo;
}

// One warp copies one float32 row of q values (16-byte aligned rows): all of
// a lane's float4 loads are issued before its stores (4 in flight per lane
// for q <= 512), so a warp-per-row copy keeps enough bytes in flight to run
// at HBM speed.
__device__ __forceinline__ void warp_copy_row(float* __restrict__ o, const float* __restrict__ a, int q, int lane) {
  const int q4 = q >> 2;
  for (int base = 0; base < q4; base += 128) {
    float4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = base + u * 32 + lane;
      if (c < q4) r[u] = __ldcs(reinterpret_cast<const float4*>(a) + c);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = base + u * 32 + lane;
      if (c < q4) reinterpret_cast<float4*>(o)[c] = r[u];
    }
  }
  for (int c = 4 * q4 + lane; c < q; c += 32) o[c] = a[c];
}

// K5: row gather (+ up to two per-particle float64 vectors)
__global__ void gather_kernel(const float* __restrict__ src, int ld_src, float* __restrict__ dst, int ld_dst, int q,
                              const int64_t* __restrict__ idx, int64_t base, int64_t m, const double* __restrict__ v0,
                              double* __restrict__ v0o, const double* __restrict__ v1, double* __restrict__ v1o,
                              const double* __restrict__ gate) {
  // grid-stride over rows with a capped grid: a gated-off launch (most
  // steps) retires a few hundred blocks instead of one per 8 rows
  if (gated_off(gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m; row += stride) {
  const int64_t s = idx[row] - base;  // (callers pass ancestors < N; see peer_gather_kernel for j = N)
  const float* a = src + s * ld_src;
  float* o = dst + row * ld_dst;
  if ((ld_src & 3) == 0 && (ld_dst & 3) == 0) {
    warp_copy_row(o, a, q, lane);
  } else {
    for (int j = lane; j < q; j += 32) o[j] = a[j];
  }
  if (lane == 0) {
    if (v0) v0o[row] = v0[s];
    if (v1) v1o[row] = v1[s];
  }
  }
}

// Step record (device-decided resampling): rec[t] = {inc, ESS, resampled,
// log Z_t/Z_1}, the running log-evidence accumulated in step order (the same
// float64 additions as the host loop).
__device__ __forceinline__ void step_record_body(const double* __restrict__ res, double* __restrict__ rec, int64_t t,
                                                 double ess_threshold) {
  const double inc = res[0], e = res[1];
  rec[4 * t + 0] = inc;
  rec[4 * t + 1] = e;
  rec[4 * t + 2] = (e < ess_threshold) ? 1.0 : 0.0;
  rec[4 * t + 3] = rec[4 * (t - 1) + 3] + inc;
}

__global__ void step_record_kernel(const double* __restrict__ res, double* __restrict__ rec, int64_t t,
                                   double ess_threshold) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  step_record_body(res, rec, t, ess_threshold);
}

// The whole weight update of an unsharded lambda step in one cooperative
// launch (one 1024-thread block per 4096-particle chunk): the chunk
// statistics of logw + lw, their combine (log Z_t / Z_t-1, ESS) and the step
// record, logw <- logw + lw - lse, the statistics of the new logw, their
// combine and the normalised weights w = exp(logw - lse) -- the arithmetic of
// lse_stats / lse_combine / logw_apply / step_record / logw_apply(w), in the
// same order (bit-identical).  Every block runs the (deterministic) combine
// itself, so two grid barriers suffice (one per set of chunk statistics);
// the second set goes to stats[nchunks..2 nchunks) and each block copies its
// own entry down at the end (stats ends as after the last combine).
__global__ void __launch_bounds__(kLseThreads) reweight_finish_kernel(double* logw, const double* __restrict__ lw,
                                                                      int64_t m, double* stats, int64_t nchunks,
                                                                      double* res, double* rec, int64_t t,
                                                                      double ess_threshold, double* __restrict__ w) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  __shared__ double rs[3];
  const int64_t c = blockIdx.x;
  double* stats2 = stats + 3 * nchunks;
  lse_chunk_stats(logw, lw, m, stats, c, red);
  grid.sync();
  if (threadIdx.x < 32) {
    lse_combine_warp(stats, nchunks, rs);
    if (c == 0 && threadIdx.x == 0) {
      res[0] = rs[0];
      res[1] = rs[1];
      res[2] = rs[2];
      step_record_body(rs, rec, t, ess_threshold);
    }
  }
  __syncthreads();
  constexpr int kPer = kChunk / kLseThreads;
  const double r0 = rs[0];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t k = c * kChunk + threadIdx.x + i * kLseThreads;
    if (k < m) logw[k] = logw[k] + lw[k] - r0;
  }
  __syncthreads();
  lse_chunk_stats(logw, nullptr, m, stats2, c, red);  // this block's own updated chunk
  grid.sync();
  if (threadIdx.x < 32) lse_combine_warp(stats2, nchunks, rs);
  __syncthreads();
  const double r1 = rs[0];
  if (c == 0 && threadIdx.x < 3) res[threadIdx.x] = rs[threadIdx.x];
  if (threadIdx.x < 3) stats[3 * c + threadIdx.x] = __ldcg(&stats2[3 * c + threadIdx.x]);
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t k = c * kChunk + threadIdx.x + i * kLseThreads;
    if (k < m) w[k] = exp(logw[k] - r1);
  }
}

// Gated copy-back of the gathered rows (alt -> main) and log-weight reset to
// -log N: what the host-decided path does with a buffer swap and a fill.
__global__ void resample_commit_kernel(const float* __restrict__ beta_alt, float* __restrict__ beta, int ldb, int q,
                                       const double* __restrict__ ll_alt, double* __restrict__ ll,
                                       const double* __restrict__ lp_alt, double* __restrict__ lp,
                                       double* __restrict__ logw, double logw0, int64_t m,
                                       const double* __restrict__ gate) {
  if (gated_off(gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m; row += stride) {
  const float* a = beta_alt + row * ldb;
  float* o = beta + row * ldb;
  if ((ldb & 3) == 0) {
    warp_copy_row(o, a, q, lane);
  } else {
    for (int j = lane; j < q; j += 32) o[j] = a[j];
  }
  if (lane == 0) {
    ll[row] = ll_alt[row];
    lp[row] = lp_alt[row];
    logw[row] = logw0;
  }
  }
}

// Sharded resampling (K5 over NVLink): slot row i of this rank takes global
// ancestor j = anc[i], owned by rank j / M at row j % M, read straight from
// the owner's particle buffers through CUDA-IPC peer pointers (P2P loads).
// j = N (a position that rounded to 1.0: the reference's searchsorted
// returns N and its gather raises) reads the last row instead of out of
// bounds.
struct PeerRows {
  const float* beta[8];
  const double* ll[8];
  const double* lp[8];
};
__global__ void peer_gather_kernel(const __grid_constant__ PeerRows src, int64_t M, int64_t N, int ldb, int q,
                                   const int64_t* __restrict__ anc, float* __restrict__ beta_alt,
                                   double* __restrict__ ll_alt, double* __restrict__ lp_alt,
                                   const double* __restrict__ gate) {
  if (gated_off(gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < M; row += stride) {
    const int64_t j = min(anc[row], N - 1);
    const int r = (int)(j / M);
    const int64_t off = j - (int64_t)r * M;
    const float* a = src.beta[r] + off * ldb;
    float* o = beta_alt + row * ldb;
    warp_copy_row(o, a, q, lane);  // ldb % 4 == 0 (checked by the caller)
    if (lane == 0) {
      ll_alt[row] = src.ll[r][off];
      lp_alt[row] = src.lp[r][off];
    }
  }
}

__global__ void philox_blocks_kernel(Key2 k, uint64_t first, int64_t count, uint64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t w[4];
  philox_block(k, first + (uint64_t)i, w);
  for (int j = 0; j < 4; ++j) out[4 * i + j] = w[j];
}

// hh (coded K1): the linear half (1/2) sum_i eta_ki added to the symmetric sums
__global__ void reduce_units_kernel(const double* __restrict__ partial, int units, int64_t m,
                                    const double* __restrict__ ylin, double* __restrict__ out,
                                    const double* __restrict__ hh = nullptr) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double s = 0.0;
  for (int u = 0; u < units; ++u) s += partial[(size_t)u * m + k];
  if (hh) s += hh[k];
  out[k] = ylin ? ylin[k] - s : s;
}

// ---------------------------------------------------------------------------
// K8: population random-walk moves.
//
// Moments: mu = sum_k w_k beta_k, then S = sum_k w_k (beta_k-mu)(beta_k-mu)^T,
// each accumulated in float32 over fixed particle chunks / 64x64 tiles and
// converted to 2^-48 fixed point before 64-bit integer atomics: integer sums
// are associative, so the moments are bit-identical for any CTA order or GPU
// count (the same property the reference guarantees for `threads`).

// Weighted mean sum_k w_k beta_kj over a 128-particle block: row-major,
// coalesced reads (warp w takes rows w, w+NW, ..; lane l columns 4 (l + 32 it)
// .. +3), float64 per-lane column sums, a fixed-order reduction over the NW
// warps in shared memory, then one fixed-point atomic per
// (column, block) -- order-independent, so deterministic for any schedule
// and, for shards that are multiples of 128 particles, any number of GPUs.
constexpr int kMeanRows = 128;  // particles per block (one fixed-point atomic per column per block)

template <int IT, int NW = (IT <= 4 ? 8 : 4)>
__global__ void __launch_bounds__(256) rw_mean_kernel(const float* __restrict__ beta, int64_t m, int ldb, int q,
                                                      const double* __restrict__ w,
                                                      unsigned long long* __restrict__ acc) {
  __shared__ double part[NW][IT * 128];  // NW warps per block (static smem <= 32 KB)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * kMeanRows;
  const int64_t k1 = min(m, k0 + kMeanRows);
  const bool vec = (q % 4 == 0) && (ldb % 4 == 0);
  double s[IT][4];
#pragma unroll
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[it][i] = 0.0;
  for (int64_t k = k0 + warp; k < k1; k += NW) {
    const float* b = beta + k * ldb;
    const double wk = w[k];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int j0 = (lane + 32 * it) * 4;
      float x[4] = {0.f, 0.f, 0.f, 0.f};
      if (vec && j0 + 4 <= q) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(b + j0));
        x[0] = v.x;
        x[1] = v.y;
        x[2] = v.z;
        x[3] = v.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = j0 + i < q ? b[j0 + i] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s[it][i] = fma(wk, (double)x[i], s[it][i]);
    }
  }
#pragma unroll
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) part[warp][(lane + 32 * it) * 4 + i] = s[it][i];
  __syncthreads();
  for (int j = threadIdx.x; j < q; j += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) t += part[ww][j];
    atomicAdd(&acc[j], to_fix(t));
  }
}


// Blocked right-looking Cholesky of S = M2c + jitter*I in float32.  L only
// parameterises the symmetric random-walk increment L z (any fixed L keeps the
// Metropolis ratio exact), so float32 suffices; a non-positive pivot is
// clamped (reported through *info) and still yields a valid proposal.
//   rw_cov_kernel        : S (lower, float32) from the fixed-point moments
//   rw_chol_panel_kernel : per 32-column panel, one launch: the diagonal block
//                          factor + inverse (one warp per CTA), then L21 rows
//                          and A22 -= L21 L21^T on 32x32 tiles (one per CTA)
// The q/32 dependent launches are recorded once into a CUDA graph per
// (workspace, q) and replayed every step.
//   rw_emit_kernel       : scale, write float32 L and the bf16 operand [q][kq]
constexpr int kPanel = 32;

// Fixed point -> float32 covariance with the trace-scaled jitter; one block
// per row i (coalesced row writes).  Every block computes the trace with the
// same warp-shuffle order, so all rows see the same jitter bits.
// S = M - delta delta^T with M = sum_k w_k (beta_k - c)(beta_k - c)^T and
// delta = sum_k w_k (beta_k - c) = mu - c (weights sum to 1), i.e. the
// weighted covariance for any centring point c.  Block i also moves the
// centre to the mean (center[i] += delta_i) for the next call.
__global__ void __launch_bounds__(256) rw_cov_kernel(const unsigned long long* __restrict__ acc, int q,
                                                     double jitter, float* __restrict__ S,
                                                     float* __restrict__ center) {
  __shared__ double s_add;
  const int i = blockIdx.x;
  if (threadIdx.x < 32) {
    double tr = 0.0;
    for (int d = threadIdx.x; d < q; d += 32) {
      const double dd = from_fix(acc[d]);
      tr += from_fix(acc[q + (size_t)d * q + d]) - dd * dd;
    }
    tr = warp_sum(tr);
    if (threadIdx.x == 0) {
      const double t = tr / q;
      s_add = jitter * (t > 0 ? t : 1.0) + 1e-30;
    }
  }
  __syncthreads();
  const double add = s_add, di = from_fix(acc[i]);
  const unsigned long long* row = acc + q + (size_t)i * q;
  float* out = S + (size_t)i * q;
  for (int j = threadIdx.x; j < q; j += blockDim.x)
    out[j] = (j > i) ? 0.f : (float)(from_fix(row[j]) - di * from_fix(acc[j]) + (i == j ? add : 0.0));
  if (center && threadIdx.x == 0) center[i] = (float)((double)center[i] + di);
}

// Factor one 32 x 32 diagonal block with one warp (lane = row, a[k] =
// A[lane][k] for k <= lane; identity rows past nb) and form its inverse: on
// return a[] holds the row of L11 and x[k] = (L11^-1)[k][lane].  Column j of
// L is published once to shared memory (col) and read back as broadcast
// float4s, the rows of L11 likewise (Ls) for the forward substitutions --
// instead of one warp shuffle per element (the factor's critical path).
// The substitution's dot products use 4 partial sums.  info records the first
// non-positive pivot (1-based, offset jb).
__device__ __forceinline__ void chol_block32(float (&a)[kPanel], float (&x)[kPanel], int lane, int nb, int jb,
                                             int* info, float* col, float (*Ls)[kPanel + 4]) {
#pragma unroll
  for (int j = 0; j < kPanel; ++j) {
    float djj = __shfl_sync(0xffffffffu, a[j], j);
    if (!(djj > 0.f)) {
      if (lane == 0 && info && j < nb && *info == 0) *info = jb + j + 1;
      djj = 1e-30f;
    }
    const float rd = rsqrtf(djj);
    a[j] = (lane == j) ? djj * rd : (lane > j ? a[j] * rd : a[j]);
    if (j + 1 < kPanel) {
      col[lane] = a[j];  // column j of L (rows > j)
      __syncwarp();
#pragma unroll
      for (int c4 = ((j + 1) / 4) * 4; c4 < kPanel; c4 += 4) {
        const float4 v = *reinterpret_cast<const float4*>(col + c4);
        const float lv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = c4 + u;
          // no lane >= k test: entries above the diagonal (lane < k) are
          // never read back, so they may absorb the update unconditionally
          if (k > j) a[k] = fmaf(-a[j], lv[u], a[k]);
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int k = 0; k < kPanel; k += 4)
    *reinterpret_cast<float4*>(&Ls[lane][k]) = make_float4(a[k], a[k + 1], a[k + 2], a[k + 3]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kPanel; ++i) {
    float v[4] = {(i == lane) ? 1.f : 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k4 = 0; k4 < i; k4 += 4) {
      const float4 r = *reinterpret_cast<const float4*>(&Ls[i][k4]);
      const float rv[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k4 + u < i) v[u] = fmaf(-rv[u], x[k4 + u], v[u]);
    }
    x[i] = (i >= lane) ? __fdividef((v[0] + v[1]) + (v[2] + v[3]), Ls[i][i]) : 0.f;
  }
}



// One launch per panel: every CTA's warp 0 factors the 32 x 32 diagonal
// block and its inverse (chol_block32, redundantly per CTA, in parallel)
// into shared memory; CTA 0 stores L11 and records pivot failures; then each
// CTA owns one lower-triangle trailing tile (bi, bj), bi >= bj: the L21 rows
// it needs are recomputed from A21 and L11^-1, diagonal tiles store theirs
// transposed in the unused upper triangle (other CTAs still read A21 from
// the lower one), and S -= L21_bi L21_bj^T.
__global__ void __launch_bounds__(256) rw_chol_panel_kernel(float* __restrict__ S, int q, int jb, int* info) {
  __shared__ float iv[kPanel][kPanel + 1];
  __shared__ float li[32][kPanel + 1];
  __shared__ float lj[32][kPanel + 1];
  __shared__ __align__(16) float colb[kPanel];
  __shared__ __align__(16) float Ls[kPanel][kPanel + 4];
  const int tid = threadIdx.x;
  const int j0 = jb + kPanel;
  const int rest = q - j0;
  int bi = 0, bj = 0, r0 = 0, c0 = 0;
  if (rest > 0) {
    int t = blockIdx.x;
    while (t > bi) {
      t -= bi + 1;
      ++bi;
    }
    bj = t;
    r0 = j0 + bi * 32;
    c0 = j0 + bj * 32;
    // the tile's A21 rows (read before CTA 0 overwrites the diagonal block:
    // disjoint locations, so order does not matter)
    for (int e = tid; e < 32 * kPanel; e += blockDim.x) {
      const int r = e / kPanel, k = e % kPanel;
      li[r][k] = (r0 + r < q) ? S[(size_t)(r0 + r) * q + jb + k] : 0.f;
      lj[r][k] = (c0 + r < q) ? S[(size_t)(c0 + r) * q + jb + k] : 0.f;
    }
  }
  if (tid < 32) {
    const int lane = tid;
    const int nb = min(kPanel, q - jb);
    float a[kPanel], x[kPanel];
#pragma unroll
    for (int k = 0; k < kPanel; ++k)
      a[k] = (lane < nb && k <= lane) ? S[(size_t)(jb + lane) * q + jb + k] : (k == lane ? 1.f : 0.f);
    __syncwarp();
    chol_block32(a, x, lane, nb, jb, blockIdx.x == 0 ? info : nullptr, colb, Ls);
#pragma unroll
    for (int k = 0; k < kPanel; ++k) iv[k][lane] = x[k];
    if (blockIdx.x == 0) {
      // L11 must not overwrite A11 in place: the other CTAs of this launch
      // may not have read it yet (they are not co-scheduled when the device
      // is shared with other streams).  Its strict lower part goes transposed
      // into the block's unused upper triangle, its diagonal to S + q*q.
      float dv = 0.f;
#pragma unroll
      for (int k = 0; k < kPanel; ++k) {
        if (lane < nb && k < lane) S[(size_t)(jb + k) * q + jb + lane] = a[k];
        if (k == lane) dv = a[k];
      }
      if (lane < nb) S[(size_t)q * q + jb + lane] = dv;
    }
  }
  if (rest <= 0) return;
  __syncthreads();
  {
    const int r = tid >> 3, cb = (tid & 7) * 4;
    float xi[4], xj[4];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      float si = 0.f, sj = 0.f;
#pragma unroll 8
      for (int k = 0; k < kPanel; ++k) {
        si = fmaf(li[r][k], iv[cb + cc][k], si);
        sj = fmaf(lj[r][k], iv[cb + cc][k], sj);
      }
      xi[cc] = si;
      xj[cc] = sj;
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      li[r][cb + cc] = xi[cc];
      lj[r][cb + cc] = xj[cc];
    }
  }
  __syncthreads();
  if (bi == bj) {
    for (int e = tid; e < 32 * kPanel; e += blockDim.x) {
      const int k = e / 32, r = e % 32;
      if (r0 + r < q) S[(size_t)(jb + k) * q + r0 + r] = li[r][k];
    }
  }
  const int ty = tid >> 3, tx = (tid & 7) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int k = 0; k < kPanel; ++k) {
    const float av = li[ty][k];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) acc[cc] = fmaf(av, lj[tx + cc][k], acc[cc]);
  }
  const int i = r0 + ty;
  if (i < q) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int j = c0 + tx + cc;
      if (j < q && j <= i) S[(size_t)i * q + j] -= acc[cc];
    }
  }
}


__global__ void rw_emit_kernel(const float* __restrict__ S, int q, int kq, float f, float* __restrict__ L,
                               __nv_bfloat16* __restrict__ Lb) {
  const int64_t total = (int64_t)q * kq;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / kq), j = (int)(e % kq);
    // the factor's strict lower part was stored transposed in the upper
    // triangle, its diagonal at S + q*q (rw_chol_panel_kernel)
    float v = 0.f;
    if (j < q && j <= i) v = (i == j ? S[(size_t)q * q + i] : S[(size_t)j * q + i]) * f;
    if (j < q) L[(size_t)i * q + j] = v;
    Lb[e] = __float2bfloat16(v);
  }
}

// Proposal normals: Z[k][j] (bf16, [m][kq]).  Counter-based Philox4x32-10
// keyed by the seed, counter (j/8, particle i0+k, t, move | tag 3 << 24);
// every 32-bit output word carries one Box-Muller pair: two 15-bit uniforms
// (radius, angle) and two sign bits, so one Philox call gives 8 normals.
// Each normal is |r cos(pi/2 u)| (resp. sin) with an independent random sign,
// so the law is exactly symmetric whatever the rounding of the fast
// intrinsics (the RW increment must be symmetric for the plain Metropolis
// ratio; its exact shape is immaterial -- the radius tail stops at 4.56 sd).
__device__ __forceinline__ void rw_normals8(uint64_t seed, int64_t t, int64_t k, int move, uint32_t blk, float z[8]) {
  uint32_t w[4] = {blk, (uint32_t)k, (uint32_t)t, (uint32_t)move | (3u << 24)};
  philox4x32_10(w, (uint32_t)seed, (uint32_t)(seed >> 32));
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const uint32_t a = w[h];
    // 15-bit uniforms without int -> float conversions (those issue on the
    // XU pipe beside the log / sqrt / sincos): the bits become the top of a
    // float mantissa in [1, 2); subtracting 1 is exact
    const float u2 = __uint_as_float(0x3F800000u | ((a >> 17) & 0x7FFFu) << 8) - 1.0f;       // [0, 1)
    const float u1 = (__uint_as_float(0x3F800000u | ((a >> 1) & 0x7FFFu) << 8) - 1.0f) + 0x1.0p-15f;  // (0, 1]
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-2.0f * __logf(u1)));
    float sn, cs;
    __sincosf(1.5707963267948966f * u2, &sn, &cs);
    const float m0 = fabsf(r * cs), m1 = fabsf(r * sn);
    z[2 * h] = (a & 1u) ? -m0 : m0;
    z[2 * h + 1] = (a & 0x10000u) ? -m1 : m1;
  }
}

__global__ void __launch_bounds__(256) rw_normals_kernel(int64_t m, int q, int kq, uint64_t seed, int64_t t,
                                                          int64_t i0, int move, __nv_bfloat16* __restrict__ Z) {
  // warp-stride over particle rows, lanes over 8-column groups (16-byte
  // stores, 512 B per warp)
  const int kq8 = kq / 8;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < m; k += nw) {
    __nv_bfloat16* zr = Z + (size_t)k * kq;
    for (int jb = lane; jb < kq8; jb += 32) {
      float zz[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (8 * jb < q) rw_normals8(seed, t, i0 + k, move, (uint32_t)jb, zz);
      uint4 u;
      uint32_t* up = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(8 * jb + 2 * i < q ? zz[2 * i] : 0.0f,
                                                        8 * jb + 2 * i + 1 < q ? zz[2 * i + 1] : 0.0f);
        up[i] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(zr + 8 * jb) = u;
    }
  }
}

// Centre (around c, the previous population mean), weight and transpose
// the particles for the tensor-core SYRK -- Dt[j][k] = bf16(sqrt(w_k)
// (beta_kj - c_j)), rows of ldk particles -- and accumulate the mean offset
// delta_j = sum_k w_k (beta_kj - c_j) (one fixed-point atomic per column and
// block).  One pass over the particles: the exact covariance is
// M - delta delta^T (rw_cov_kernel).  bf16 is ample here: the factor only
// scales a symmetric proposal.
// Transposed in registers: lane (cq, pg) of warp w holds columns 4 cq .. +3
// of the 8 particles 16 w + 8 pg .. +7, so loads are 256-byte row segments
// and each column's 8 particles leave as one 16-byte store (a warp writes
// 16 full 32-byte sectors).  Block: 64 columns x 128 particles.
constexpr int kCtrRows = 128, kCtrCols = 64;
__global__ void __launch_bounds__(256) rw_center_kernel(const float* __restrict__ beta, int64_t m, int ldb, int q,
                                                        const double* __restrict__ w,
                                                        const float* __restrict__ center,
                                                        unsigned long long* __restrict__ acc,
                                                        __nv_bfloat16* __restrict__ Dt, int64_t ldk) {
  __shared__ float red[8][kCtrCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cq = lane & 15, pg = lane >> 4;
  const int j = blockIdx.y * kCtrCols + 4 * cq;
  const int64_t kb = (int64_t)blockIdx.x * kCtrRows + 16 * warp + 8 * pg;
  const bool vec = (q % 4 == 0) && (ldb % 4 == 0);
  float x[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t k = kb + r;
    if (vec) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < m && j < q) v = __ldcs(reinterpret_cast<const float4*>(beta + k * ldb + j));
      x[r][0] = v.x;
      x[r][1] = v.y;
      x[r][2] = v.z;
      x[r][3] = v.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) x[r][i] = (k < m && j + i < q) ? beta[k * ldb + j + i] : 0.f;
    }
  }
  float c[4], d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (j + i < q) ? center[j + i] : 0.f;
  // lane cq < 8 of each half-warp forms the weight scalars of particle kb + cq
  // once (the float64 sqrt is the costly part); shuffles hand them to the
  // 16 lanes of the half-warp
  float wf_own = 0.f, sf_own = 0.f;
  if (cq < 8) {
    const double wd = (kb + cq < m) ? w[kb + cq] : 0.0;
    wf_own = (float)wd;
    sf_own = (float)sqrt(wd);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const float wf = __shfl_sync(0xffffffffu, wf_own, 16 * pg + r);
    const float sf = __shfl_sync(0xffffffffu, sf_own, 16 * pg + r);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float v = x[r][i] - c[i];
      d[i] = fmaf(wf, v, d[i]);
      x[r][i] = sf * v;  // exactly 0 for padding particles and columns
    }
  }
  if (kb < ldk) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (j + i >= q) break;
      uint4 u;
      uint32_t* up = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(x[2 * h][i], x[2 * h + 1][i]);
        up[h] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(Dt + (size_t)(j + i) * ldk + kb) = u;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] += __shfl_xor_sync(0xffffffffu, d[i], 16);
  if (pg == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red[warp][4 * cq + i] = d[i];
  }
  __syncthreads();
  if (threadIdx.x < kCtrCols) {
    const int jj = blockIdx.y * kCtrCols + threadIdx.x;
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) s += (double)red[ww][threadIdx.x];
    if (jj < q) atomicAdd(&acc[jj], to_fix(s));
  }
}

constexpr int kAcceptThreads = 128;  // 4 warps x 32 particles: all blocks resident in one wave

struct SpArray {  // the softplus sums as an array (spa_loglik_softplus)
  const double* sp;
  __device__ __forceinline__ double softplus_sum(int64_t k) const { return sp[k]; }
};

template <int kR, class SP>
__global__ void __launch_bounds__(kAcceptThreads) rw_accept_kernel(float* __restrict__ beta, int ldb,
                                                         const __nv_bfloat16* __restrict__ eps, int q, int64_t m,
                                                         const double* __restrict__ ylin_p, const SP sp,
                                                         const double* __restrict__ lp_p, double* __restrict__ ll,
                                                         double* __restrict__ lp, uint64_t seed, int64_t t, int64_t i0,
                                                         int move, unsigned long long* accepted) {
  // one warp per 32 consecutive particles: lane l decides particle base + l
  // (coalesced loads, Philox and the float64 log in parallel), then the warp
  // walks the ballot of accepted rows applying beta += eps with vector
  // accesses; one counter atomic per warp
  const int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  const int lane = threadIdx.x & 31;
  if (base >= m) return;
  const int64_t row = base + lane;
  bool ok = false;
  if (row < m) {
    uint32_t w[4] = {0xFFFFFFFFu, (uint32_t)(i0 + row), (uint32_t)t, (uint32_t)move | (3u << 24)};
    philox4x32_10(w, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double u = (double)(((uint64_t)w[0] << 21) | (w[1] >> 11)) * 0x1.0p-53;
    const double llp = ylin_p[row] - sp.softplus_sum(row);
    const double lpp = lp_p[row];
    const double d = (llp + lpp) - (ll[row] + lp[row]);
    ok = (d >= 0.0) || (log(u) < d);
    if (ok) {
      ll[row] = llp;
      lp[row] = lpp;
    }
  }
  unsigned mask = __ballot_sync(0xffffffffu, ok);
  if (lane == 0 && mask) atomicAdd(accepted, (unsigned long long)__popc(mask));
  if ((q % 4 == 0) && (ldb % 4 == 0) && q <= 512) {
    // beta' = beta + eps (the same float32 sum the pack used), accepted rows
    // taken kR at a time with all their loads in flight before any store
    constexpr int kV = 4;  // float4 per lane per row (q <= 512)
    while (mask) {
      int rows[kR];
#pragma unroll
      for (int b = 0; b < kR; ++b) {
        rows[b] = mask ? __ffs(mask) - 1 : -1;
        if (mask) mask &= mask - 1;
      }
      float4 x[kR][kV];
      uint2 y[kR][kV];
#pragma unroll
      for (int b = 0; b < kR; ++b)
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const int j = (v * 32 + lane) * 4;
          if (rows[b] >= 0 && j < q) {
            x[b][v] = *reinterpret_cast<const float4*>(beta + (base + rows[b]) * ldb + j);
            y[b][v] = *reinterpret_cast<const uint2*>(eps + (base + rows[b]) * ldb + j);
          }
        }
#pragma unroll
      for (int b = 0; b < kR; ++b)
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          const int j = (v * 32 + lane) * 4;
          if (rows[b] >= 0 && j < q) {
            const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y[b][v]);
            const float2 ya = __bfloat1622float2(y2[0]), yb = __bfloat1622float2(y2[1]);
            float4 o = x[b][v];
            o.x += ya.x;
            o.y += ya.y;
            o.z += yb.x;
            o.w += yb.y;
            *reinterpret_cast<float4*>(beta + (base + rows[b]) * ldb + j) = o;
          }
        }
    }
  } else {
    while (mask) {
      const int r = __ffs(mask) - 1;
      mask &= mask - 1;
      float* o = beta + (base + r) * ldb;
      const __nv_bfloat16* e = eps + (base + r) * ldb;
      for (int j = lane; j < q; j += 32) o[j] = o[j] + __bfloat162float(e[j]);
    }
  }
}

// Record the panel loop of the Cholesky once per (S, q, inv, info) and replay it.
struct CholGraphKey {
  float* S;
  int q;
  float* inv;
  int* info;
  bool operator==(const CholGraphKey& o) const { return S == o.S && q == o.q && inv == o.inv && info == o.info; }
};

static cudaError_t chol_record(float* S, int q, float* inv, int* info, cudaStream_t st) {
  (void)inv;
  for (int jb = 0; jb < q; jb += 32) {
    const int rest = q - jb - 32;
    const int nt = rest > 0 ? (rest + 31) / 32 : 0;
    rw_chol_panel_kernel<<<nt > 0 ? nt * (nt + 1) / 2 : 1, 256, 0, st>>>(S, q, jb, info);
  }
  return cudaGetLastError();
}

static cudaError_t chol_graph_launch(float* S, int q, float* inv, int* info, cudaStream_t st) {
  static std::mutex mu;
  static std::vector<std::pair<CholGraphKey, cudaGraphExec_t>> cache;
  const CholGraphKey key{S, q, inv, info};
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : cache)
      if (kv.first == key) exec = kv.second;
  }
  if (exec == nullptr) {
    cudaStream_t cap;
    cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    cudaGraph_t g = nullptr;
    e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      cudaError_t er = chol_record(S, q, inv, info, cap);
      e = cudaStreamEndCapture(cap, &g);
      if (er != cudaSuccess) e = er;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 16) {  // bounded: drop the oldest
      cudaGraphExecDestroy(cache.front().second);
      cache.erase(cache.begin());
    }
    cache.push_back({key, exec});
  }
  return cudaGraphLaunch(exec, st);
}

static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Likelihood work split: units of BN tiles so the grid covers several waves.
static void loglik_split(int64_t m, int n, int& m_tiles, int& n_tiles, int& tpu, int& units, int bn = 256,
                         double item_cost = 0.1, int bm = kTcBM, int kSms = 148) {
  // persistent kernel: items = (particle tile, group of tpu subject tiles),
  // CTA b takes items b, b + 148, ...  The group size minimises the makespan
  // in subject-tile times, ceil(items / 148) * tpu, plus a small per-item
  // cost (epilogue drain, partial-sum write, pipeline ramp) -- e.g. C3
  // (512 x 20 tiles): tpu = 10, 7 rounds of 10 (the 4-tile groups of round 1
  // took 18 rounds of 4: 72 vs 70 tile times)
  m_tiles = (int)((m + bm - 1) / bm);
  n_tiles = (n + bn - 1) / bn;
  double best = 1e300;
  tpu = 1;
  for (int g = 1; g <= n_tiles; ++g) {
    const int u = (n_tiles + g - 1) / g;
    if (g > 1 && (u - 1) * g >= n_tiles) continue;  // same units as a smaller group
    const int64_t items = (int64_t)m_tiles * u;
    const int64_t rounds = (items + kSms - 1) / kSms;
    const double cost = (double)rounds * g + item_cost * (double)rounds;
    if (cost < best - 1e-9) {
      best = cost;
      tpu = g;
    }
  }
  units = (n_tiles + tpu - 1) / tpu;
}

}  // namespace spa

using namespace spa;

// ===========================================================================
// C ABI
extern "C" {

const char* spa_last_error(void) { return g_last_error.c_str(); }
int spa_version(void) { return 1; }

int spa_philox_blocks(uint64_t k0, uint64_t k1, uint64_t first_block, int64_t count, uint64_t* out, void* stream) {
  SPA_REQUIRE(count >= 0 && out, kBadArgument, "spa_philox_blocks: bad arguments");
  if (count == 0) return 0;
  philox_blocks_kernel<<<cdiv(count, 256), 256, 0, as_stream(stream)>>>(Key2{k0, k1}, first_block, count, out);
  SPA_CHECK_LAUNCH();
  return 0;
}

size_t spa_k1_operand_bytes(const spa_design* d, int64_t m) {
  if (!d || m < 0) return 0;
  return d->coded ? (size_t)m * (3 * (size_t)d->kp + sizeof(float2) + sizeof(double)) : (size_t)m * 4 * (size_t)d->kp;
}

size_t spa_loglik_workspace_bytes(int64_t m, int32_t n) {
  int mt, nt, tpu, units, units8r, units8s;
  loglik_split(m, n, mt, nt, tpu, units);  // fp16 path (general designs)
  // int8 paths (coded designs): kI8EpiGroups partial rows per segment slot
  loglik_split(m, n, mt, nt, tpu, units8r, kI8BN, 0.3, 256, 74);
  loglik_split(m, n, mt, nt, tpu, units8s, kI8BN, 0.1, 256, 74);
  return (size_t)std::max({units, kI8EpiGroups * k1_i8_max_slots(m, n), kI8EpiGroups * units8r,
                           kI8EpiGroups * units8s}) * (size_t)m * sizeof(double);
}

// K1 for coded designs on the int8 tensor cores (tc_k1_i8.cuh): CTA-pair
// kernels -- resident particle tiles for kp <= 512, streamed above.  The
// (particle tile, subject tile) units are cut into equal contiguous ranges,
// one per pair (K1Seg).
static bool k1_i8_resident(int kp) { return kp <= kI8MaxKb * kI8BK && k1_i8_pair_stages(kp) >= 2; }

// Per-row partial sums of the segments covering the row's particle tile
// (k1_slots_of), summed in slot order, then ylin - sum.
__global__ void reduce_k1_slots_kernel(const double* __restrict__ partial, int64_t m, int n_tiles, int U,
                                       int nclus, const double* __restrict__ ylin, double* __restrict__ out,
                                       const double* __restrict__ hh) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int units = kI8EpiGroups * k1_slots_of((int)(k >> 8), n_tiles, U, nclus);
  double s = 0.0;
  for (int u = 0; u < units; ++u) s += partial[(size_t)u * m + k];
  s += hh[k];
  out[k] = ylin ? ylin[k] - s : s;
}

// How the int8 K1 launch for (design, m) lays out its partial row sums: the
// schedule, and the (slot) count per row the reductions add up in fixed order.
struct K1Plan {
  K1I8Args args;
  bool res;
  int sched, U, nclus;
};

static int k1_i8_plan(const spa_design* d, const void* A, int64_t m, void* ws, K1Plan& pl) {
  pl.res = k1_i8_resident(d->kp);
  K1I8Args& args = pl.args;
  args.m_tiles = (int)((m + 255) / 256);
  args.n_tiles = (d->n + kI8BN - 1) / kI8BN;
  args.m = (int)m;
  args.n = d->n;
  args.kp = d->kp;
  args.stages = pl.res ? k1_i8_pair_stages(d->kp) : kI8PairStreamStages;
  args.rowc = k1_rowc(const_cast<void*>(A), m, d->kp);
  args.partial = reinterpret_cast<double*>(ws);
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    SPA_CHECK_CUDA(cudaGetDevice(&dev));
    SPA_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // contiguous unit ranges for the resident kernel (its operand reloads then
  // fall at different times per pair: C3 289 -> 283 us); the streamed kernel
  // (kp > 512) re-reads each particle tile's operand per subject tile, so it
  // keeps round-robin items, whose concurrently live particle tiles stay in
  // L2 (contiguous ranges: C5 1.49 -> 1.72 ms).  SPA_K1_SCHED=0|1|2 overrides
  // (developer A/B knob, K1Seg)
  static const int forced = [] {
    const char* e = getenv("SPA_K1_SCHED");
    return e ? atoi(e) : -1;
  }();
  pl.sched = (forced >= 0 && forced <= 2) ? forced : (pl.res ? 0 : 1);
  args.sched = pl.sched;
  loglik_split(m, d->n, args.m_tiles, args.n_tiles, args.tpu, args.units, kI8BN, pl.res ? 0.3 : 0.1, 256, 74);
  pl.U = args.m_tiles * (pl.sched == 0 ? args.n_tiles : args.units);  // < 2^31: m < 2^31, n_tiles <= 128
  pl.nclus = std::min(pl.U, std::min(kI8MaxPairs, sms / 2));
  return 0;
}

// the K1 kernel alone: partial row sums in ws (see K1Plan)
static int k1_i8_launch(const spa_design* d, const void* A, int64_t m, const K1Plan& pl, cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_tmap_u8(&ta, A, 3ull * d->kp, (uint64_t)m);
  if (rc) return rc;
  rc = make_tmap_u8(&tb, d->gemm_b, 2ull * d->kp, (uint64_t)d->n, kI8PairB);
  if (rc) return rc;
  const int grid = 2 * pl.nclus;
  if (pl.res) {
    const int smem = k1_i8_pair_smem(d->kp);
    static int attr = 0;  // largest size set so far
    if (smem > attr) {
      SPA_CHECK_CUDA(cudaFuncSetAttribute(k1_i8_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = smem;
    }
    k1_i8_pair_kernel<true><<<grid, kI8Threads, smem, st>>>(ta, tb, pl.args);
  } else {
    static bool attr_done = false;
    if (!attr_done) {
      SPA_CHECK_CUDA(cudaFuncSetAttribute(k1_i8_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kI8PairStreamSmem));
      attr_done = true;
    }
    k1_i8_pair_kernel<false><<<grid, kI8Threads, kI8PairStreamSmem, st>>>(ta, tb, pl.args);
  }
  SPA_CHECK_LAUNCH();
  return 0;
}

// The row reduction of a K1Plan's partial sums (the order of the reduction
// kernels below), for kernels that consume the log-likelihood directly.
struct K1Reduce {
  const double* partial;
  const double* hh;
  int64_t m;
  int sched, n_tiles, U, nclus, units;
  __device__ __forceinline__ double softplus_sum(int64_t k) const {
    const int n = kI8EpiGroups * (sched == 0 ? k1_slots_of((int)(k >> 8), n_tiles, U, nclus) : units);
    double s = 0.0;
    for (int u = 0; u < n; ++u) s += partial[(size_t)u * m + k];
    return s + hh[k];
  }
};
static K1Reduce k1_reduce_of(const spa_design* d, const void* A, int64_t m, const void* ws, const K1Plan& pl) {
  K1Reduce r;
  r.partial = reinterpret_cast<const double*>(ws);
  r.hh = k1_half(const_cast<void*>(A), m, d->kp);
  r.m = m;
  r.sched = pl.sched;
  r.n_tiles = pl.args.n_tiles;
  r.U = pl.U;
  r.nclus = pl.nclus;
  r.units = pl.args.units;
  return r;
}

static int loglik_i8(const spa_design* d, const void* A, int64_t m, const double* ylin, double* out, void* ws,
                     cudaStream_t st) {
  K1Plan pl;
  int rc = k1_i8_plan(d, A, m, ws, pl);
  if (rc) return rc;
  rc = k1_i8_launch(d, A, m, pl, st);
  if (rc) return rc;
  if (pl.sched == 0)
    reduce_k1_slots_kernel<<<cdiv(m, 256), 256, 0, st>>>(reinterpret_cast<double*>(ws), m, pl.args.n_tiles, pl.U,
                                                         pl.nclus, ylin, out, k1_half(const_cast<void*>(A), m, d->kp));
  else
    reduce_units_kernel<<<cdiv(m, 256), 256, 0, st>>>(reinterpret_cast<double*>(ws), kI8EpiGroups * pl.args.units, m,
                                                      ylin, out, k1_half(const_cast<void*>(A), m, d->kp));
  SPA_CHECK_LAUNCH();
  return 0;
}

static int loglik_impl(const spa_design* d, const void* A, int64_t m, const double* ylin, double* out, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  SPA_REQUIRE(d && A && out && ws, kBadArgument, "spa_loglik: null argument");
  SPA_REQUIRE(d->kp % 64 == 0 && d->kp > 0, kBadArgument, "spa_loglik: kp must be a positive multiple of 64");
  SPA_REQUIRE(m > 0 && m < (1ll << 31), kBadArgument, "spa_loglik: m out of range");
  SPA_REQUIRE(ws_bytes >= spa_loglik_workspace_bytes(m, d->n), kWorkspaceTooSmall, "spa_loglik: workspace too small");
  SPA_REQUIRE(d->terms == 1 || d->terms == 2, kBadArgument, "spa_loglik: terms must be 1 or 2");
  if (d->coded) {
    SPA_REQUIRE(d->kp <= 1024, kNotSupported, "spa_loglik: coded designs with q > 1024 not supported");
    return loglik_i8(d, A, m, ylin, out, ws, st);
  }
  TcArgs args;
  int units;
  loglik_split(m, d->n, args.m_tiles, args.n_tiles, args.tiles_per_unit, units);
  args.m = (int)m;
  args.ncols = d->n;
  args.kp = d->kp;
  args.kb_per_unit = 0;
  EpiSoftplusRowSum epi{reinterpret_cast<double*>(ws)};
  int rc;
  if (d->terms == 1)
    rc = launch_tc<2, 1, 256, EpiSoftplusRowSum, 1, true>(A, 2ull * d->kp, d->gemm_b, (uint64_t)d->kp,
                                                          (uint64_t)d->n, args, units, epi, st);
  else
    rc = launch_tc<2, 2, 256, EpiSoftplusRowSum, 1, true>(A, 2ull * d->kp, d->gemm_b, 2ull * d->kp,
                                                          (uint64_t)d->n, args, units, epi, st);
  if (rc) return rc;
  reduce_units_kernel<<<cdiv(m, 256), 256, 0, st>>>(reinterpret_cast<double*>(ws), units, m, ylin, out);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_loglik_softplus(const spa_design* d, const void* A, int64_t m, double* out_sp, void* ws, size_t ws_bytes,
                        void* stream) {
  return loglik_impl(d, A, m, nullptr, out_sp, ws, ws_bytes, as_stream(stream));
}

static PriorConst make_prior(double a, double c, double c_prev) {
  PriorConst p;
  p.a = a;
  p.c = c;
  p.c_prev = c_prev;
  p.lc = -std::log(2.0 * c);
  p.lr = std::log(c_prev / c);
  p.de = std::isinf(a) ? 1 : 0;
  p.k = p.de ? 0.0 : 1.0 / (a * c);
  p.k_prev = p.de ? 0.0 : 1.0 / (a * c_prev);
  return p;
}

int spa_pack_particles(const spa_design* d, const float* beta, int64_t m, int32_t ldb, void* A, double* ylin,
                       double a, double c, double* lp, void* stream) {
  SPA_REQUIRE(d && beta && A && ylin && m >= 0, kBadArgument, "spa_pack_particles: bad arguments");
  SPA_REQUIRE(d->kp >= d->q && d->kp % 64 == 0, kBadArgument, "spa_pack_particles: kp must be >= q, a multiple of 64");
  if (m == 0) return 0;
  pack_kernel<<<cdiv(m, 8), 256, 0, as_stream(stream)>>>(*d, beta, (const __nv_bfloat16*)nullptr, m, ldb, A, ylin,
                                                        make_prior(a, c, c), lp);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_loglik_rows(const spa_design* d, const float* beta, int64_t m, int32_t ldb, void* A_ws, double* ylin_ws,
                    double* out_ll, void* ws, size_t ws_bytes, void* stream) {
  int rc = spa_pack_particles(d, beta, m, ldb, A_ws, ylin_ws, 1.0, 1.0, nullptr, stream);
  if (rc) return rc;
  return loglik_impl(d, A_ws, m, ylin_ws, out_ll, ws, ws_bytes, as_stream(stream));
}

int spa_prior_rows(const spa_design* d, const float* beta, int64_t m, int32_t ldb, double a, double c,
                   double c_prev, int32_t mode, double* out, void* stream) {
  SPA_REQUIRE(d && beta && out && m >= 0 && mode >= 0 && mode <= 2, kBadArgument, "spa_prior_rows: bad arguments");
  SPA_REQUIRE(a > 0 && c > 0 && c_prev > 0, kBadArgument, "spa_prior_rows: a, c must be positive");
  if (m == 0) return 0;
  prior_kernel<<<cdiv(m, 8), 256, 0, as_stream(stream)>>>(*d, beta, m, ldb, make_prior(a, c, c_prev), mode, out);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_prior_reweight(const spa_design* d, const float* beta, int64_t m, int32_t ldb, double a, double c,
                       double c_prev, double* lw, double* lp, void* stream) {
  SPA_REQUIRE(d && beta && lw && lp && m >= 0, kBadArgument, "spa_prior_reweight: bad arguments");
  SPA_REQUIRE(a > 0 && c > 0 && c_prev > 0, kBadArgument, "spa_prior_reweight: a, c must be positive");
  SPA_REQUIRE(d->kp <= 32 * 128, kNotSupported, "spa_prior_reweight: q > 4093 not supported");
  if (m == 0) return 0;
  const PriorConst pc = make_prior(a, c, c_prev);
  cudaStream_t st = as_stream(stream);
  const unsigned grid = (unsigned)cdiv(m, 8);
  if (d->q % 4 == 0 && ldb % 4 == 0 && d->kp <= 1024 && ((uintptr_t)d->penalized & 3) == 0) {
    if (d->kp <= 128)
      prior_reweight_lean_kernel<8, 4><<<(unsigned)cdiv(m, 32), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
    else if (d->kp <= 256)
      prior_reweight_lean_kernel<8, 8><<<(unsigned)cdiv(m, 32), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
    else if (d->kp <= 512)
      prior_reweight_lean_kernel<16, 8><<<(unsigned)cdiv(m, 16), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
    else
      prior_reweight_lean_kernel<16, 16><<<(unsigned)cdiv(m, 16), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  } else if (d->kp <= 128)
    prior_reweight_rows_kernel<8, 4><<<(unsigned)cdiv(m, 32), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  else if (d->kp <= 256)
    prior_reweight_rows_kernel<8, 8><<<(unsigned)cdiv(m, 32), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  else if (d->kp <= 512)
    prior_reweight_rows_kernel<16, 8><<<(unsigned)cdiv(m, 16), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  else if (d->kp <= 1024)
    prior_reweight_rows_kernel<16, 16><<<(unsigned)cdiv(m, 16), 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  else if (d->kp <= 2048)
    prior_reweight_rows_kernel<32, 16><<<grid, 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  else
    prior_reweight_kernel<32><<<grid, 256, 0, st>>>(*d, beta, m, ldb, pc, lw, lp);
  SPA_CHECK_LAUNCH();
  return 0;
}

static int sum_params(int32_t nlev, const double* levels, int32_t ndelta, const double* deltas, SumParams* sp) {
  SPA_REQUIRE(nlev >= 0 && nlev <= kSumMaxLev && ndelta >= 0 && ndelta <= kSumMaxDelta, kBadArgument,
              "spa_summary: at most 4 levels and 4 deltas");
  sp->nlev = nlev;
  sp->ndelta = ndelta;
  for (int i = 0; i < kSumMaxLev; ++i) sp->level[i] = i < nlev ? levels[i] : 0.5;
  // float32 threshold t = the smallest float >= delta, so that for float32
  // particles |x| < t  <=>  |x| < delta in float64 (summary.py:54-61)
  for (int i = 0; i < kSumMaxDelta; ++i) {
    float t = i < ndelta ? (float)deltas[i] : 0.f;
    if (i < ndelta && (double)t < deltas[i]) t = std::nextafter(t, INFINITY);
    sp->delta[i] = t;
  }
  for (int i = 0; i < nlev; ++i) SPA_REQUIRE(levels[i] > 0.0 && levels[i] < 1.0, kBadArgument, "spa_summary: level");
  for (int i = 0; i < ndelta; ++i) SPA_REQUIRE(deltas[i] > 0.0, kBadArgument, "spa_summary: delta");
  return 0;
}

int spa_summary_pass(const float* beta, int64_t m, int32_t ldb, int32_t q, const double* w, int32_t nlev,
                     const double* levels, int32_t ndelta, const double* deltas, int32_t pass, const uint32_t* prefix,
                     unsigned long long* hist, unsigned long long* acc_mean, unsigned long long* acc_in,
                     unsigned long long* total, void* stream) {
  SPA_REQUIRE(beta && w && hist && m >= 0 && q > 0 && pass >= 0 && pass < 4, kBadArgument,
              "spa_summary_pass: bad arguments");
  SPA_REQUIRE(pass == 0 ? (acc_mean && total && (ndelta == 0 || acc_in)) : prefix != nullptr, kBadArgument,
              "spa_summary_pass: missing accumulators");
  SumParams sp;
  int rc = sum_params(nlev, levels, ndelta, deltas, &sp);
  if (rc) return rc;
  if (m == 0) return 0;
  const int nh = pass == 0 ? 1 : nlev;
  if (nh == 0) return 0;
  const size_t smem = (size_t)nh * kSumCols * 256 * 2 * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    SPA_CHECK_CUDA(cudaFuncSetAttribute(summary_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(kSumMaxLev * kSumCols * 256 * sizeof(unsigned long long))));
    attr = true;
  }
  dim3 grid((unsigned)cdiv(q, kSumCols), (unsigned)cdiv(m, kSumRows));
  summary_hist_kernel<<<grid, 256, smem, as_stream(stream)>>>(beta, m, ldb, q, w, sp, pass, prefix, hist, acc_mean,
                                                              acc_in, total);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_summary_select(const unsigned long long* hist, int32_t q, int32_t nlev, const double* levels, int32_t pass,
                       const unsigned long long* total, uint32_t* prefix, unsigned long long* below, void* stream) {
  SPA_REQUIRE(hist && total && prefix && below && q > 0 && pass >= 0 && pass < 4, kBadArgument,
              "spa_summary_select: bad arguments");
  SumParams sp;
  int rc = sum_params(nlev, levels, 0, nullptr, &sp);
  if (rc) return rc;
  if (nlev == 0) return 0;
  summary_select_kernel<<<cdiv((int64_t)nlev * q * 32, 256), 256, 0, as_stream(stream)>>>(hist, q, sp, pass, total,
                                                                                            prefix, below);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_summary_finish(int32_t q, int32_t nlev, int32_t ndelta, const uint32_t* prefix,
                       const unsigned long long* acc_mean, const unsigned long long* acc_in,
                       const unsigned long long* total, double* out_mean, double* out_quant, double* out_conc,
                       void* stream) {
  SPA_REQUIRE(acc_mean && total && out_mean && q > 0, kBadArgument, "spa_summary_finish: bad arguments");
  SPA_REQUIRE((nlev == 0 || (prefix && out_quant)) && (ndelta == 0 || (acc_in && out_conc)), kBadArgument,
              "spa_summary_finish: missing outputs");
  SumParams sp;
  double lv[kSumMaxLev] = {0.5, 0.5, 0.5, 0.5}, dl[kSumMaxDelta] = {1.0, 1.0, 1.0, 1.0};
  int rc = sum_params(nlev, lv, ndelta, dl, &sp);
  if (rc) return rc;
  summary_finish_kernel<<<cdiv(q, 128), 128, 0, as_stream(stream)>>>(q, sp, prefix, acc_mean, acc_in, total, out_mean,
                                                                     out_quant, out_conc);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_lse_chunk_stats(const double* logw, const double* lw, int64_t m, double* stats, void* stream) {
  SPA_REQUIRE(logw && stats && m > 0, kBadArgument, "spa_lse_chunk_stats: bad arguments");
  lse_stats_kernel<<<cdiv(m, kChunk), kLseThreads, 0, as_stream(stream)>>>(logw, lw, m, stats);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_lse_combine(const double* stats, int64_t nchunks, double* res, void* stream) {
  SPA_REQUIRE(stats && res && nchunks > 0, kBadArgument, "spa_lse_combine: bad arguments");
  lse_combine_kernel<<<1, 32, 0, as_stream(stream)>>>(stats, nchunks, res);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_logw_apply(double* logw, const double* lw, int64_t m, const double* res, double* w, void* stream) {
  SPA_REQUIRE(logw && res && m > 0, kBadArgument, "spa_logw_apply: bad arguments");
  logw_apply_kernel<<<cdiv(m, 256), 256, 0, as_stream(stream)>>>(logw, lw, m, res, w);
  SPA_CHECK_LAUNCH();
  return 0;
}

size_t spa_resample_workspace_bytes(int64_t N) { return exact_cumsum_ws_bytes(N); }

int spa_systematic_ancestors(const double* w, int64_t N, double u, int64_t k0, int64_t count, int64_t* anc,
                             void* ws, size_t ws_bytes, void* stream) {
  SPA_REQUIRE(w && anc && ws && N > 0 && k0 >= 0 && count >= 0 && k0 + count <= N, kBadArgument,
              "spa_systematic_ancestors: bad arguments");
  SPA_REQUIRE(ws_bytes >= spa_resample_workspace_bytes(N), kWorkspaceTooSmall,
              "spa_systematic_ancestors: workspace too small");
  cudaStream_t st = as_stream(stream);
  const double* cumn = reinterpret_cast<const double*>(reinterpret_cast<char*>(ws) + exact_cumsum_norm_offset(N));
  WSrc src{};
  src.p[0] = w;
  src.len = N;
  src.nparts = 1;
  int rc = exact_cumsum(src, N, ws, nullptr, st);
  if (rc) return rc;
  if (count == 0) return 0;
  ancestors_kernel<<<cdiv(count, 256), 256, 0, st>>>(cumn, N, u, k0, count, anc, nullptr);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_exact_cumsum(const double* w, int64_t N, double* cum, int32_t* mode, void* ws, size_t ws_bytes,
                     void* stream) {
  SPA_REQUIRE(w && cum && ws && N > 0, kBadArgument, "spa_exact_cumsum: bad arguments");
  SPA_REQUIRE(ws_bytes >= spa_resample_workspace_bytes(N), kWorkspaceTooSmall, "spa_exact_cumsum: workspace too small");
  cudaStream_t st = as_stream(stream);
  WSrc src{};
  src.p[0] = w;
  src.len = N;
  src.nparts = 1;
  int rc = exact_cumsum(src, N, ws, nullptr, st);
  if (rc) return rc;
  SPA_CHECK_CUDA(cudaMemcpyAsync(cum, ws, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (mode) return exact_cumsum_mode(N, ws, mode, st);
  return 0;
}

int spa_gather_rows(const float* src, int32_t ld_src, float* dst, int32_t ld_dst, int32_t q, const int64_t* idx,
                    int64_t base, int64_t m, const double* v0, double* v0_out, const double* v1, double* v1_out,
                    void* stream) {
  SPA_REQUIRE(src && dst && idx && m >= 0 && q > 0, kBadArgument, "spa_gather_rows: bad arguments");
  if (m == 0) return 0;
  gather_kernel<<<std::min<unsigned>(cdiv(m, 8), 8 * 148), 256, 0, as_stream(stream)>>>(src, ld_src, dst, ld_dst, q, idx, base, m, v0, v0_out, v1,
                                                          v1_out, nullptr);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_reweight_finish(double* logw, const double* lw, int64_t m, double* stats, double* res, double* rec, int64_t t,
                        double ess_threshold, double* w, void* stream) {
  SPA_REQUIRE(logw && lw && stats && res && rec && w && m > 0 && t >= 1, kBadArgument,
              "spa_reweight_finish: bad arguments");
  const int64_t nchunks = cdiv(m, kChunk);
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int dev = 0, nsm = 0, per_sm = 0;
    SPA_CHECK_CUDA(cudaGetDevice(&dev));
    SPA_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SPA_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reweight_finish_kernel, kLseThreads, 0));
    max_blocks = std::max(1, per_sm * nsm);
  }
  SPA_REQUIRE(nchunks <= max_blocks, kNotSupported, "spa_reweight_finish: more chunks than co-resident blocks");
  void* args[] = {&logw, (void*)&lw, &m, &stats, (void*)&nchunks, &res, &rec, &t, &ess_threshold, &w};
  SPA_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)reweight_finish_kernel, dim3((unsigned)nchunks),
                                             dim3(kLseThreads), args, 0, as_stream(stream)));
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_reweight_finish_max_particles(void) {
  int dev = 0, nsm = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reweight_finish_kernel, kLseThreads, 0) != cudaSuccess)
    return 0;
  return per_sm * nsm * kChunk;
}

int spa_step_record(const double* res, double* rec, int64_t t, double ess_threshold, void* stream) {
  SPA_REQUIRE(res && rec && t >= 1, kBadArgument, "spa_step_record: bad arguments");
  step_record_kernel<<<1, 32, 0, as_stream(stream)>>>(res, rec, t, ess_threshold);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_resample_gated(const double* gate, const double* w, int64_t N, double u, float* beta, float* beta_alt,
                       int32_t ldb, int32_t q, double* ll, double* ll_alt, double* lp, double* lp_alt, double* logw,
                       int64_t* anc, void* ws, size_t ws_bytes, void* stream) {
  SPA_REQUIRE(gate && w && N > 0 && beta && beta_alt && ll && ll_alt && lp && lp_alt && logw && anc && ws && q > 0 &&
                  (ldb & 3) == 0,
              kBadArgument, "spa_resample_gated: bad arguments");
  SPA_REQUIRE(ws_bytes >= spa_resample_workspace_bytes(N), kWorkspaceTooSmall,
              "spa_resample_gated: workspace too small");
  cudaStream_t st = as_stream(stream);
  const double* cumn = reinterpret_cast<const double*>(reinterpret_cast<char*>(ws) + exact_cumsum_norm_offset(N));
  WSrc src{};
  src.p[0] = w;
  src.len = N;
  src.nparts = 1;
  int rc = exact_cumsum(src, N, ws, gate, st);
  if (rc) return rc;
  ancestors_kernel<<<cdiv(N, 256), 256, 0, st>>>(cumn, N, u, 0, N, anc, gate);
  SPA_CHECK_LAUNCH();
  PeerRows rows{};  // one part: the local buffers (clamps an ancestor index N like the sharded path)
  rows.beta[0] = beta;
  rows.ll[0] = ll;
  rows.lp[0] = lp;
  peer_gather_kernel<<<std::min<unsigned>(cdiv(N, 8), 8 * 148), 256, 0, st>>>(rows, N, N, ldb, q, anc, beta_alt,
                                                                             ll_alt, lp_alt, gate);
  SPA_CHECK_LAUNCH();
  resample_commit_kernel<<<std::min<unsigned>(cdiv(N, 8), 8 * 148), 256, 0, st>>>(beta_alt, beta, ldb, q, ll_alt, ll, lp_alt, lp, logw,
                                                      -std::log((double)N), N, gate);
  SPA_CHECK_LAUNCH();
  return 0;
}

static void syrk_split(int64_t m, int q, int& m_tiles, int& kb_per_unit, int& units) {
  const int64_t ldk = (m + 63) / 64 * 64;
  const int kblocks = (int)(ldk / kTcBK);
  m_tiles = (q + kTcBM - 1) / kTcBM;
  // one wave of work items (m_tiles x units ~ 148): fewer split partials to
  // write and reduce than two waves, same tensor work per CTA
  units = std::max(1, std::min(kblocks, 148 / m_tiles));
  kb_per_unit = (kblocks + units - 1) / units;
  units = (kblocks + kb_per_unit - 1) / kb_per_unit;
}

size_t spa_rw_moments_workspace_bytes(int64_t m, int32_t q) {
  const int64_t ldk = (m + 63) / 64 * 64;
  int mt, kbpu, units;
  syrk_split(m, q, mt, kbpu, units);
  const size_t dt = (((size_t)q * ldk * sizeof(__nv_bfloat16)) + 255) & ~size_t(255);
  const size_t qp = (q + 3) / 4 * 4;  // 16-byte partial rows (TMA store)
  return dt + (size_t)units * q * qp * sizeof(float);
}

// Sum the per-split float32 SYRK tiles in fixed split order (float64) and
// store the lower triangle as 2^-48 fixed point.
__global__ void syrk_reduce_kernel(const float* __restrict__ part, int units, int q, int qp,
                                   unsigned long long* __restrict__ acc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)q * q) return;
  const int i = (int)(e / q), j = (int)(e % q);
  if (j > i) return;
  double s = 0.0;
  for (int u = 0; u < units; ++u) s += (double)part[((size_t)u * q + i) * qp + j];
  acc[q + e] += to_fix(s);
}

int spa_rw_moments(const float* beta, int64_t m, int32_t ldb, int32_t q, const double* w, const float* center,
                   int32_t phase, int64_t* partial, void* ws, size_t ws_bytes, void* stream) {
  SPA_REQUIRE(beta && w && partial && m > 0 && q > 0 && phase >= 0 && phase <= 3, kBadArgument,
              "spa_rw_moments: bad arguments");
  cudaStream_t st = as_stream(stream);
  auto* acc = reinterpret_cast<unsigned long long*>(partial);
  if (phase == 0) {
    const unsigned grid = (unsigned)cdiv(m, kMeanRows);
    const int kq = (q + 127) / 128 * 128;
    if (kq <= 128)
      rw_mean_kernel<1><<<grid, 256, 0, st>>>(beta, m, ldb, q, w, acc);
    else if (kq <= 256)
      rw_mean_kernel<2><<<grid, 256, 0, st>>>(beta, m, ldb, q, w, acc);
    else if (kq <= 512)
      rw_mean_kernel<4><<<grid, 256, 0, st>>>(beta, m, ldb, q, w, acc);
    else if (kq <= 1024)
      rw_mean_kernel<8><<<grid, 128, 0, st>>>(beta, m, ldb, q, w, acc);
    else
      return fail(kNotSupported, "spa_rw_moments: q > 1024 not supported");
    SPA_CHECK_LAUNCH();
    return 0;
  }
  // phase 1 = 2 then 3: centre/weight/transpose (the one read of beta, also
  // accumulating delta), then M = Dt Dt^T on tcgen05 (split-K over
  // particles) + fixed-order reduce
  SPA_REQUIRE(ws && ws_bytes >= spa_rw_moments_workspace_bytes(m, q), kWorkspaceTooSmall,
              "spa_rw_moments: workspace too small");
  const int64_t ldk = (m + 63) / 64 * 64;
  __nv_bfloat16* Dt = reinterpret_cast<__nv_bfloat16*>(ws);  // [q][ldk]
  if (phase != 3) {
    SPA_REQUIRE(center, kBadArgument, "spa_rw_moments: phases 1 and 2 need the centring point");
    dim3 grid(cdiv(ldk, kCtrRows), cdiv(q, kCtrCols));
    rw_center_kernel<<<grid, 256, 0, st>>>(beta, m, ldb, q, w, center, acc, Dt, ldk);
    SPA_CHECK_LAUNCH();
    if (phase == 2) return 0;
  }
  TcArgs args;
  int units;
  syrk_split(m, q, args.m_tiles, args.kb_per_unit, units);
  args.m = q;
  args.ncols = q;
  args.kp = (int)ldk;
  args.n_tiles = (q + 255) / 256;
  args.tiles_per_unit = args.n_tiles;
  float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                         ((((size_t)q * ldk * sizeof(__nv_bfloat16)) + 255) & ~size_t(255)));
  const int qp = (q + 3) / 4 * 4;
  EpiStoreT<float> epi{};
  int rc = make_tmap_out<float>(&epi.tmc, part, (uint64_t)q, (uint64_t)q, (uint64_t)units, (uint64_t)qp,
                                (uint64_t)q * qp);
  if (rc) return rc;
  epi.m = q;
  rc = launch_tc<1, 1, 256>(Dt, (uint64_t)ldk, Dt, (uint64_t)ldk, (uint64_t)q, args, units, epi, st);
  if (rc) return rc;
  syrk_reduce_kernel<<<cdiv((int64_t)q * q, 256), 256, 0, st>>>(part, units, q, qp, acc);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_rw_factor(const int64_t* partial, int32_t q, double scale, double jitter, float* L, double* ws, int* info,
                  float* center, void* stream) {
  SPA_REQUIRE(partial && L && ws && q > 0 && q <= 8192, kBadArgument, "spa_rw_factor: bad arguments");
  cudaStream_t st = as_stream(stream);
  const int kq = (q + 63) / 64 * 64;
  float* S = reinterpret_cast<float*>(ws);
  char* base = reinterpret_cast<char*>(ws);
  __nv_bfloat16* Lb = reinterpret_cast<__nv_bfloat16*>(base + (((size_t)8 * q * q + 255) & ~size_t(255)));
  float* inv = reinterpret_cast<float*>(base + (((size_t)8 * q * q + 255) & ~size_t(255)) +
                                        (((size_t)2 * q * kq + 255) & ~size_t(255)));
  if (info) SPA_CHECK_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  rw_cov_kernel<<<q, 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(partial), q, jitter, S, center);
  SPA_CHECK_LAUNCH();
  SPA_CHECK_CUDA(chol_graph_launch(S, q, inv, info, st));
  rw_emit_kernel<<<std::min<unsigned>(cdiv((int64_t)q * kq, 256), 1184), 256, 0, st>>>(
      S, q, kq, (float)(scale / std::sqrt((double)q)), L, Lb);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_rw_normals(int64_t m, int32_t q, uint64_t seed, int64_t t, int64_t i0, int32_t move, void* zbuf,
                   void* stream) {
  SPA_REQUIRE(zbuf && m > 0 && q > 0, kBadArgument, "spa_rw_normals: bad arguments");
  const int kq = (q + 63) / 64 * 64;
  // one particle row per warp, no grid cap: the blocks are short, so the
  // high-priority sampler stream's kernels get SMs as soon as a few retire
  // (a persistent 4-blocks-per-SM grid held them: C3 2.184 -> 2.169 ms/step)
  static const unsigned max_grid = [] {
    const char* e = getenv("SPA_NORMALS_GRID");  // developer A/B knob
    return e ? (unsigned)atoi(e) : 0xFFFFFFFFu;
  }();
  const unsigned grid = std::min<unsigned>(cdiv(m, 8), max_grid);
  rw_normals_kernel<<<grid, 256, 0, as_stream(stream)>>>(m, q, kq, seed, t, i0, move,
                                                          reinterpret_cast<__nv_bfloat16*>(zbuf));
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_rw_increments(int64_t m, int32_t q, int32_t ldb, const void* Lb, const void* zbuf, void* eps,
                      void* stream) {
  SPA_REQUIRE(Lb && zbuf && eps && m > 0 && q > 0 && ldb >= q, kBadArgument, "spa_rw_increments: bad arguments");
  SPA_REQUIRE(m < (1ll << 31), kNotSupported, "spa_rw_increments: m >= 2^31 rows");
  cudaStream_t st = as_stream(stream);
  const int kq = (q + 63) / 64 * 64;
  const __nv_bfloat16* Z = reinterpret_cast<const __nv_bfloat16*>(zbuf);
  TcArgs args;
  args.m = (int)m;
  args.ncols = q;
  args.kp = kq;
  args.m_tiles = (int)((m + kTcBM - 1) / kTcBM);
  // (two 128-particle tiles per item sharing each L tile, resident L, and one
  // column tile per item were measured no faster: DESIGN.md section 9)
  constexpr int kPropBN = 256;
  args.n_tiles = (q + kPropBN - 1) / kPropBN;
  // q <= 512: the two column tiles (4 and 8 k-blocks under the triangle) are
  // separate work items, alternating between rounds per CTA (tc_gemm.cuh
  // item_range): 1024 items balance over 148 CTAs better than 512 whole
  // m-tiles (3 or 4 per CTA); propose 103.4 -> 101.2 us at C3
  static const int lz_units = [] {
    const char* e = getenv("SPA_LZ_UNITS");  // developer A/B knob
    return e ? atoi(e) : 2;
  }();
  const int units = (lz_units == 2 && args.n_tiles == 2) ? 2 : 1;
  args.tiles_per_unit = units == 1 ? args.n_tiles : 1;
  args.kb_per_unit = 0;
  args.tri_b = 1;  // L is lower triangular: column tile nt needs k < (nt + 1) BN only
  auto* epsb = reinterpret_cast<__nv_bfloat16*>(eps);
  EpiStoreT<__nv_bfloat16> epi{};
  int rc = make_tmap_out<__nv_bfloat16>(&epi.tmc, epsb, (uint64_t)q, (uint64_t)m, 1, (uint64_t)ldb,
                                        (uint64_t)m * ldb);
  if (rc) return rc;
  epi.m = (int)m;
  epi.slabs = 0;
  static const bool pair = [] {
    const char* e = getenv("SPA_LZ_PAIR");  // developer A/B knob: 0 = the single-CTA engine
    return !(e && atoi(e) == 0);
  }();
  if (pair) {  // CTA pairs (tc_lz_pair.cuh)
    CUtensorMap tz, tl;
    rc = make_tmap_bf16(&tz, Z, (uint64_t)kq, (uint64_t)m, 128);
    if (rc) return rc;
    rc = make_tmap_bf16(&tl, Lb, (uint64_t)kq, (uint64_t)q, 128);
    if (rc) return rc;
    static int nsm = 0;
    if (nsm == 0) {
      int dev = 0;
      SPA_CHECK_CUDA(cudaGetDevice(&dev));
      SPA_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      SPA_CHECK_CUDA(cudaFuncSetAttribute(lz_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLzSmem));
    }
    LzArgs la;
    la.m = (int)m;
    la.kq = kq;
    la.mtp = (int)((m + 255) / 256);
    la.n_tiles = (q + kLzBN - 1) / kLzBN;
    const int nclus = std::min(la.mtp * la.n_tiles, nsm / 2);
    lz_pair_kernel<<<2 * nclus, kLzThreads, kLzSmem, st>>>(tz, tl, la, epi);
    SPA_CHECK_LAUNCH();
    return 0;
  }
  return launch_tc<1, 1, kPropBN, EpiStoreT<__nv_bfloat16>>(Z, (uint64_t)kq, Lb, (uint64_t)kq, (uint64_t)q, args,
                                                            units, epi, st);
}

int spa_rw_pack(const spa_design* d, const float* beta, int64_t m, int32_t ldb, const void* eps, void* A,
                double* ylin, double a, double c, double* lp, void* stream) {
  SPA_REQUIRE(d && beta && eps && A && ylin && m > 0, kBadArgument, "spa_rw_pack: bad arguments");
  SPA_REQUIRE((ldb & 3) == 0 && (const void*)beta != eps, kBadArgument, "spa_rw_pack: ldb % 4 != 0 or beta aliases eps");
  SPA_REQUIRE(d->kp >= d->q && d->kp % 64 == 0, kBadArgument, "spa_rw_pack: kp must be >= q, a multiple of 64");
  cudaStream_t st = as_stream(stream);
  const __nv_bfloat16* epsb = reinterpret_cast<const __nv_bfloat16*>(eps);
  void* Ab = A;
  const PriorConst pc = make_prior(a, c, c);
  const size_t sm = pack_eps_smem_bytes(d->kp, ldb);
  auto run = [&](auto kern) -> int {
    SPA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 0, dev = 0, nsm = 0;
    SPA_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kPackWarps, sm));
    SPA_CHECK_CUDA(cudaGetDevice(&dev));
    SPA_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SPA_REQUIRE(per_sm > 0, kNotSupported, "spa_rw_propose: pack ring does not fit in shared memory");
    const unsigned grid = std::min<unsigned>(cdiv(m, kPackWarps), (unsigned)(per_sm * nsm));
    kern<<<grid, 32 * kPackWarps, sm, st>>>(*d, beta, epsb, m, ldb, Ab, ylin, pc, lp);
    SPA_CHECK_LAUNCH();
    return 0;
  };
  // 2 rows per warp iteration where the doubled ring still fits 2 blocks per SM
  if (d->kp > 128 && d->kp <= 512) {
    const size_t sm2 = (size_t)20 * d->kp + (size_t)kPackWarps * kPackSlots * 2 * ((size_t)ldb * 6);
    auto kern = d->coded ? (d->kp <= 256 ? pack_eps_rows_kernel<4, 16, true> : pack_eps_rows_kernel<8, 16, true>)
                         : (d->kp <= 256 ? pack_eps_rows_kernel<4, 16, false> : pack_eps_rows_kernel<8, 16, false>);
    // the attribute / occupancy queries once per (kernel, smem size): the
    // move loop calls this 5 times per step
    struct Geo {
      const void* k;
      size_t sm;
      int per_sm, nsm;
    };
    static thread_local Geo geo[4] = {};
    Geo* g = nullptr;
    for (auto& e : geo)
      if (e.k == (const void*)kern && e.sm == sm2) g = &e;
    if (!g) {
      int per_sm = 0, dev = 0, nsm = 0;
      SPA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
      SPA_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kPackWarps, sm2));
      SPA_CHECK_CUDA(cudaGetDevice(&dev));
      SPA_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      for (auto& e : geo)
        if (e.k == nullptr) {
          e = Geo{(const void*)kern, sm2, per_sm, nsm};
          g = &e;
          break;
        }
      if (!g) g = &geo[0];
      *g = Geo{(const void*)kern, sm2, per_sm, nsm};
    }
    const int per_sm = g->per_sm, nsm = g->nsm;
    if (per_sm > 0) {
      const unsigned grid = std::min<unsigned>(cdiv(cdiv(m, 2), kPackWarps), (unsigned)(per_sm * nsm));
      kern<<<grid, 32 * kPackWarps, sm2, st>>>(*d, beta, epsb, m, ldb, Ab, ylin, pc, lp);
      SPA_CHECK_LAUNCH();
      return 0;
    }
  }
  if (d->coded) {
    if (d->kp <= 128) return run(pack_eps_kernel<1, true>);
    if (d->kp <= 256) return run(pack_eps_kernel<2, true>);
    if (d->kp <= 512) return run(pack_eps_kernel<4, true>);
    if (d->kp <= 1024 && sm <= 200 * 1024) return run(pack_eps_kernel<8, true>);
  } else {
    if (d->kp <= 128) return run(pack_eps_kernel<1, false>);
    if (d->kp <= 256) return run(pack_eps_kernel<2, false>);
    if (d->kp <= 512) return run(pack_eps_kernel<4, false>);
    if (d->kp <= 1024 && sm <= 200 * 1024) return run(pack_eps_kernel<8, false>);
  }
  pack_kernel<<<cdiv(m, 8), 256, 0, st>>>(*d, beta, epsb, m, ldb, Ab, ylin, pc, lp);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_rw_propose(const spa_design* d, const float* beta, int64_t m, int32_t ldb, const void* Lb, uint64_t seed,
                   int64_t t, int64_t i0, int32_t move, void* zbuf, void* eps, void* A, double* ylin, double a,
                   double c, double* lp, void* stream) {
  SPA_REQUIRE(d && beta && Lb && zbuf && eps && A && ylin && m > 0, kBadArgument, "spa_rw_propose: bad arguments");
  SPA_REQUIRE((ldb & 3) == 0 && (const void*)beta != eps, kBadArgument, "spa_rw_propose: ldb % 4 != 0 or beta aliases eps");
  SPA_REQUIRE(d->kp >= d->q && d->kp % 64 == 0, kBadArgument, "spa_rw_propose: kp must be >= q, a multiple of 64");
  (void)seed;
  (void)t;
  (void)i0;
  (void)move;
  const int rc = spa_rw_increments(m, d->q, ldb, Lb, zbuf, eps, stream);
  if (rc) return rc;
  return spa_rw_pack(d, beta, m, ldb, eps, A, ylin, a, c, lp, stream);
}

extern "C" int spa_mwg_prepare_kernels(void);  // mwg.cu

// Load every hot-path kernel now (CUDA lazy module loading would otherwise
// load each on its first launch inside the first lambda step) and apply the
// shared-memory attributes; callable while other work runs on the device.
int spa_prepare(void) {
  const void* fns[] = {
      (const void*)tc_gemm_kernel<2, 1, 256, EpiSoftplusRowSum, 1, true>,
      (const void*)tc_gemm_kernel<2, 2, 256, EpiSoftplusRowSum, 1, true>,
      (const void*)tc_gemm_kernel<1, 1, 256, EpiStoreT<__nv_bfloat16>>,
      (const void*)tc_gemm_kernel<2, 2, 256, EpiStoreT<float>>,
      (const void*)pack_kernel, (const void*)pack_eps_kernel<1, true>, (const void*)pack_eps_kernel<2, true>,
      (const void*)pack_eps_kernel<4, true>, (const void*)pack_eps_kernel<8, true>,
      (const void*)pack_eps_kernel<1, false>, (const void*)pack_eps_kernel<2, false>,
      (const void*)pack_eps_kernel<4, false>, (const void*)pack_eps_kernel<8, false>,
      (const void*)pack_eps_rows_kernel<4, 16, true>, (const void*)pack_eps_rows_kernel<8, 16, true>,
      (const void*)pack_eps_rows_kernel<4, 16, false>, (const void*)pack_eps_rows_kernel<8, 16, false>,
      (const void*)k1_i8_pair_kernel<true>, (const void*)k1_i8_pair_kernel<false>, (const void*)lz_pair_kernel, (const void*)prior_kernel,
      (const void*)prior_reweight_rows_kernel<8, 4>, (const void*)prior_reweight_rows_kernel<8, 8>,
      (const void*)prior_reweight_rows_kernel<16, 8>, (const void*)prior_reweight_rows_kernel<16, 16>,
      (const void*)prior_reweight_rows_kernel<32, 16>, (const void*)prior_reweight_kernel<32>, (const void*)lse_stats_kernel, (const void*)lse_combine_kernel,
      (const void*)logw_apply_kernel, (const void*)ancestors_kernel,
      (const void*)gather_kernel, (const void*)step_record_kernel, (const void*)resample_commit_kernel,
      (const void*)peer_gather_kernel,
      (const void*)reduce_units_kernel, (const void*)rw_mean_kernel<4>, (const void*)rw_cov_kernel,
      (const void*)rw_chol_panel_kernel, (const void*)rw_emit_kernel,
      (const void*)rw_normals_kernel, (const void*)rw_center_kernel, (const void*)rw_accept_kernel<2, SpArray>, (const void*)rw_accept_kernel<2, K1Reduce>,
      (const void*)syrk_reduce_kernel, (const void*)summary_hist_kernel, (const void*)summary_select_kernel,
      (const void*)summary_finish_kernel};
  for (const void* f : fns) {
    cudaFuncAttributes a;
    SPA_CHECK_CUDA(cudaFuncGetAttributes(&a, f));
  }
  return spa_mwg_prepare_kernels();
}

// ---------------------------------------------------------------------------
// f2: run-directory writer fast path (host code).  Formats particle-file rows
// "i,weight,p_0,...,p_{q-1}\n" exactly as smc.py:532-549 (f"{v:.17g}": glibc's
// correctly rounded %.17g is byte-identical to Python's format for every
// double), with the rows split over host threads.
int spa_format_particle_rows(const double* weights, const double* particles, int64_t n, int32_t q, int64_t index0,
                             char* buf, size_t cap, size_t* used, int32_t threads) {
  SPA_REQUIRE(weights && particles && buf && used && n >= 0 && q >= 0, kBadArgument,
              "spa_format_particle_rows: bad arguments");
  const int nt = std::max<int>(1, std::min<int64_t>(threads > 0 ? threads : 1, std::max<int64_t>(1, n / 256)));
  std::vector<std::string> parts((size_t)nt);
  auto work = [&](int k) {
    const int64_t r0 = n * k / nt, r1 = n * (k + 1) / nt;
    std::string& out = parts[(size_t)k];
    out.reserve((size_t)(r1 - r0) * (size_t)(q + 2) * 24);
    char tmp[40];
    for (int64_t i = r0; i < r1; ++i) {
      int len = snprintf(tmp, sizeof(tmp), "%lld,", (long long)(index0 + i));
      out.append(tmp, (size_t)len);
      len = snprintf(tmp, sizeof(tmp), "%.17g", weights[i]);
      out.append(tmp, (size_t)len);
      const double* row = particles + (size_t)i * (size_t)q;
      for (int32_t j = 0; j < q; ++j) {
        tmp[0] = ',';
        len = snprintf(tmp + 1, sizeof(tmp) - 1, "%.17g", row[j]);
        out.append(tmp, (size_t)len + 1);
      }
      out.push_back('\n');
    }
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < nt; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (const auto& p : parts) total += p.size();
  *used = total;
  SPA_REQUIRE(total <= cap, kWorkspaceTooSmall, "spa_format_particle_rows: buffer too small");
  size_t off = 0;
  for (const auto& p : parts) {
    memcpy(buf + off, p.data(), p.size());
    off += p.size();
  }
  return 0;
}

int spa_tc_gemm_f32(const void* A, int64_t m, int32_t terms_a, const void* B, int32_t rows_b, int32_t kp, float* C,
                    int32_t ldc, void* stream) {
  SPA_REQUIRE(A && B && C && m > 0 && rows_b > 0 && kp % 64 == 0 && (terms_a == 1 || terms_a == 2), kBadArgument,
              "spa_tc_gemm_f32: bad arguments");
  TcArgs args;
  args.m = (int)m;
  args.ncols = rows_b;
  args.kp = kp;
  args.m_tiles = (int)((m + kTcBM - 1) / kTcBM);
  args.n_tiles = (rows_b + 255) / 256;
  args.tiles_per_unit = args.n_tiles;
  args.kb_per_unit = 0;
  EpiStoreT<float> epi{};
  int rc = make_tmap_out<float>(&epi.tmc, C, (uint64_t)rows_b, (uint64_t)m, 1, (uint64_t)ldc, (uint64_t)m * ldc);
  if (rc) return rc;
  epi.m = (int)m;
  if (terms_a == 1)
    return launch_tc<1, 1, 256>(A, (uint64_t)kp, B, (uint64_t)kp, (uint64_t)rows_b, args, 1, epi, as_stream(stream));
  return launch_tc<2, 1, 256>(A, 2ull * kp, B, (uint64_t)kp, (uint64_t)rows_b, args, 1, epi, as_stream(stream));
}

int spa_rw_accept(float* beta, int32_t ldb, const void* eps, int32_t q, int64_t m, const double* ylin_p,
                  const double* sp_p, const double* lp_p, double* ll, double* lp, uint64_t seed, int64_t t,
                  int64_t i0, int32_t move, unsigned long long* accepted, void* stream) {
  SPA_REQUIRE(beta && eps && ylin_p && sp_p && lp_p && ll && lp && accepted && m > 0, kBadArgument,
              "spa_rw_accept: bad arguments");
  rw_accept_kernel<2, SpArray><<<cdiv(m, kAcceptThreads), kAcceptThreads, 0, as_stream(stream)>>>(
      beta, ldb, reinterpret_cast<const __nv_bfloat16*>(eps), q, m, ylin_p, SpArray{sp_p}, lp_p, ll, lp, seed, t, i0,
      move, accepted);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_loglik_partials(const spa_design* d, const void* A, int64_t m, void* ws, size_t ws_bytes, void* stream) {
  SPA_REQUIRE(d && A && ws && m > 0 && m < (1ll << 31), kBadArgument, "spa_loglik_partials: bad arguments");
  SPA_REQUIRE(d->coded && d->kp <= 1024, kNotSupported, "spa_loglik_partials: integer-coded designs only");
  SPA_REQUIRE(ws_bytes >= spa_loglik_workspace_bytes(m, d->n), kWorkspaceTooSmall,
              "spa_loglik_partials: workspace too small");
  K1Plan pl;
  int rc = k1_i8_plan(d, A, m, ws, pl);
  if (rc) return rc;
  return k1_i8_launch(d, A, m, pl, as_stream(stream));
}

int spa_rw_accept_k1(float* beta, int32_t ldb, const void* eps, int32_t q, int64_t m, const spa_design* d,
                     const void* A, const double* ylin_p, const void* ws, const double* lp_p, double* ll, double* lp,
                     uint64_t seed, int64_t t, int64_t i0, int32_t move, unsigned long long* accepted, void* stream) {
  SPA_REQUIRE(beta && eps && d && A && ylin_p && ws && lp_p && ll && lp && accepted && m > 0, kBadArgument,
              "spa_rw_accept_k1: bad arguments");
  SPA_REQUIRE(d->coded && d->kp <= 1024, kNotSupported, "spa_rw_accept_k1: integer-coded designs only");
  K1Plan pl;
  int rc = k1_i8_plan(d, A, m, const_cast<void*>(ws), pl);
  if (rc) return rc;
  const K1Reduce red = k1_reduce_of(d, A, m, ws, pl);
  rw_accept_kernel<2, K1Reduce><<<cdiv(m, kAcceptThreads), kAcceptThreads, 0, as_stream(stream)>>>(
      beta, ldb, reinterpret_cast<const __nv_bfloat16*>(eps), q, m, ylin_p, red, lp_p, ll, lp, seed, t, i0, move,
      accepted);
  SPA_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Peer memory for the sharded sampler (one process per GPU).  A rank exports
// CUDA-IPC handles of its particle buffers; every other rank opens them once
// and the gated resampling kernels read remote rows directly (P2P loads over
// NVLink / NVSwitch), so no host round trip decides or sizes the exchange.
int spa_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  SPA_REQUIRE(ptr && handle && offset, kBadArgument, "spa_ipc_export: bad arguments");
  auto range = mem_range_fn();
  SPA_REQUIRE(range != nullptr, kDriverEntryPoint, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = range(&base, &size, (CUdeviceptr)ptr);
  SPA_REQUIRE(r == CUDA_SUCCESS, kBadArgument, "spa_ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  SPA_CHECK_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)ptr - base);
  return 0;
}

int spa_ipc_open(const void* handle, void** base) {
  SPA_REQUIRE(handle && base, kBadArgument, "spa_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SPA_CHECK_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int spa_ipc_close(void* base) {
  SPA_REQUIRE(base, kBadArgument, "spa_ipc_close: bad arguments");
  SPA_CHECK_CUDA(cudaIpcCloseMemHandle(base));
  return 0;
}

int spa_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  SPA_REQUIRE(dst && src, kBadArgument, "spa_copy_async: bad arguments");
  if (bytes) SPA_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return 0;
}

int spa_resample_sharded(const double* gate, const double* const* w_parts, int32_t nparts, int64_t M, double u,
                         int32_t rank, const float* const* beta_parts, const double* const* ll_parts,
                         const double* const* lp_parts, int32_t ldb, int32_t q, float* beta_alt, double* ll_alt,
                         double* lp_alt, int64_t* anc, void* ws, size_t ws_bytes, void* stream) {
  SPA_REQUIRE(gate && w_parts && beta_parts && ll_parts && lp_parts && beta_alt && ll_alt && lp_alt && anc && ws,
              kBadArgument, "spa_resample_sharded: null argument");
  SPA_REQUIRE(nparts >= 1 && nparts <= 8 && rank >= 0 && rank < nparts && M > 0 && q > 0 && (ldb & 3) == 0,
              kBadArgument, "spa_resample_sharded: bad shape");
  const int64_t N = (int64_t)nparts * M;
  SPA_REQUIRE(ws_bytes >= spa_resample_workspace_bytes(N), kWorkspaceTooSmall,
              "spa_resample_sharded: workspace too small");
  cudaStream_t st = as_stream(stream);
  WSrc src{};
  PeerRows rows{};
  for (int r = 0; r < nparts; ++r) {
    SPA_REQUIRE(w_parts[r] && beta_parts[r] && ll_parts[r] && lp_parts[r], kBadArgument,
                "spa_resample_sharded: null peer pointer");
    src.p[r] = w_parts[r];
    rows.beta[r] = beta_parts[r];
    rows.ll[r] = ll_parts[r];
    rows.lp[r] = lp_parts[r];
  }
  src.len = M;
  src.nparts = nparts;
  // every rank scans the global weights (read over the peer pointers) with
  // the exact scan, then searches only its own slots
  int rc = exact_cumsum(src, N, ws, gate, st);
  if (rc) return rc;
  const double* cumn = reinterpret_cast<const double*>(reinterpret_cast<char*>(ws) + exact_cumsum_norm_offset(N));
  ancestors_kernel<<<cdiv(M, 256), 256, 0, st>>>(cumn, N, u, (int64_t)rank * M, M, anc, gate);
  SPA_CHECK_LAUNCH();
  peer_gather_kernel<<<std::min<unsigned>(cdiv(M, 8), 8 * 148), 256, 0, st>>>(rows, M, N, ldb, q, anc, beta_alt,
                                                                             ll_alt, lp_alt, gate);
  SPA_CHECK_LAUNCH();
  return 0;
}

int spa_resample_commit(const double* gate, float* beta, const float* beta_alt, int32_t ldb, int32_t q, double* ll,
                        const double* ll_alt, double* lp, const double* lp_alt, double* logw, double logw0, int64_t M,
                        void* stream) {
  SPA_REQUIRE(gate && beta && beta_alt && ll && ll_alt && lp && lp_alt && logw && M > 0 && q > 0, kBadArgument,
              "spa_resample_commit: bad arguments");
  resample_commit_kernel<<<std::min<unsigned>(cdiv(M, 8), 8 * 148), 256, 0, as_stream(stream)>>>(
      beta_alt, beta, ldb, q, ll_alt, ll, lp_alt, lp, logw, logw0, M, gate);
  SPA_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
