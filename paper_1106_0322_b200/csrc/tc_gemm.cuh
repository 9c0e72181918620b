// Warp-specialised tcgen05 GEMM engine for sm_100a with fused epilogues.
//
//   D[128 x BN] = sum_terms A_t[128 x K] * B_t[BN x K]^T   (bf16 in, fp32 TMEM accumulate)
//
// One CTA owns one 128-row A tile (particles) and walks a contiguous range of
// BN-column tiles (subjects for the likelihood, coordinates for the proposal).
// Roles (192 threads):
//   warp 0      TMA producer   (one elected lane): A_t / B_t k-blocks -> smem ring
//   warp 1      MMA issuer     (one elected lane): tcgen05.mma into a 2-deep TMEM ring
//   warps 2..5  epilogue       (128 threads = 128 TMEM lanes = 128 A rows):
//                              tcgen05.ld -> fused epilogue functor
// Split-precision products ride along the K loop of one accumulator:
//   TA = 2 (A = [hi | lo]),  TB = 1:  hi*B0 + lo*B0             (integer-coded X)
//   TA = 2,                 TB = 2:  hi*B0 + lo*B0 + hi*B1     (general X = B0 + B1)
//   TA = 1,                 TB = 1:  plain bf16 GEMM            (proposal L z)
// The B k-block is loaded once per stage and reused by both A terms.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace spa {

constexpr int kTcThreads = 192;
constexpr int kTcBM = 128;
constexpr int kTcBK = 64;  // bf16 elements per 128-byte swizzled row

template <int TA, int TB, int BN>
struct TcShape {
  static constexpr int kABytes = kTcBM * kTcBK * 2;  // 16 KB per A term
  static constexpr int kBBytes = BN * kTcBK * 2;     // per B term
  static constexpr int kStageBytes = TA * kABytes + TB * kBBytes;
  static constexpr int kBudget = 196 * 1024;
  static constexpr int kStagesRaw = kBudget / kStageBytes;
  static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  static constexpr int kScratchPerWarp = 32 * 33 * 4;  // epilogue transpose tile
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + 4 * kScratchPerWarp;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static_assert(kStages >= 2, "tile too large");
  static_assert(kTmemCols <= 512 && (kTmemCols & (kTmemCols - 1)) == 0, "TMEM columns must be a power of 2");
};

struct TcArgs {
  int m;               // valid A rows
  int ncols;           // valid output columns (subjects / coordinates)
  int kp;              // K per term (multiple of 64)
  int m_tiles;         // ceil(m / 128)
  int n_tiles;         // ceil(ncols / BN)
  int tiles_per_unit;  // BN tiles per CTA (column split), or
  int kb_per_unit;     // > 0: split-K -- a CTA covers all BN tiles over this many k-blocks
  int units;           // column (or K) units per A tile; work items = m_tiles * units
};

// Epilogue contract:
//   begin_unit(row, unit)                       once per CTA (per thread)
//   consume(row, col0, float v[32], ncols, scratch)
//                                               32 consecutive columns of one row; scratch is a
//                                               per-warp 32x33 float smem tile
//   end_tile(row)                               after every BN tile
//   end_unit(row, unit, m)                      once per CTA
template <int TA, int TB, int BN, class Epi>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, TcArgs args,
                   Epi epi) {
  using S = TcShape<TA, TB, BN>;
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (keeps the shared
  // address space visible to the compiler: LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kStages * S::kStageBytes);
  uint64_t* empty = full + S::kStages;
  uint64_t* tfull = empty + S::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Persistent: CTA b processes work items b, b + gridDim.x, ... where item
  // w = (mt = w / units, unit = w % units); consecutive items share the A
  // tile, and CTAs running concurrently hold consecutive items, so each A
  // tile is read from DRAM once and re-used from L2.  The smem and TMEM
  // pipelines (stage / accumulator phases) run on across items.
  const int units = args.units;
  const int items = args.m_tiles * units;
  auto item_range = [&](int w, int& mt, int& unit, int& nt0, int& nt1, int& kb0, int& kb1) {
    mt = w / units;
    unit = w % units;
    if (args.kb_per_unit > 0) {
      nt0 = 0;
      nt1 = args.n_tiles;
      kb0 = unit * args.kb_per_unit;
      kb1 = min(args.kp / kTcBK, kb0 + args.kb_per_unit);
    } else {
      nt0 = unit * args.tiles_per_unit;
      nt1 = min(args.n_tiles, nt0 + args.tiles_per_unit);
      kb0 = 0;
      kb1 = args.kp / kTcBK;
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      prefetch_tmap(&tma);
      prefetch_tmap(&tmb);
      int s = 0;
      uint32_t ph = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
      int mt, unit, nt0, nt1, kb0, kb1;
      item_range(w, mt, unit, nt0, nt1, kb0, kb1);
      for (int nt = nt0; nt < nt1; ++nt) {
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * S::kStageBytes;
          mbar_arrive_expect_tx(&full[s], S::kStageBytes);
#pragma unroll
          for (int t = 0; t < TA; ++t)
            tma_load_2d(st + t * S::kABytes, &tma, &full[s], t * args.kp + kb * kTcBK, mt * kTcBM);
#pragma unroll
          for (int t = 0; t < TB; ++t)
            tma_load_2d(st + TA * S::kABytes + t * S::kBBytes, &tmb, &full[s], t * args.kp + kb * kTcBK,
                        nt * BN);
          if (++s == S::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = idesc_bf16_f32(kTcBM, BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
      int mt, unit, nt0, nt1, kb0, kb1;
      item_range(w, mt, unit, nt0, nt1, kb0, kb1);
      for (int nt = nt0; nt < nt1; ++nt, ++it) {
        const int buf = it & 1;
        const uint32_t bph = (it >> 1) & 1;
        mbar_wait(&tempty[buf], bph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * S::kStageBytes);
          const uint64_t a0 = umma_desc_sw128(st);
          const uint64_t a1 = umma_desc_sw128(st + S::kABytes);
          const uint64_t b0 = umma_desc_sw128(st + TA * S::kABytes);
          const uint64_t b1 = umma_desc_sw128(st + TA * S::kABytes + S::kBBytes);
#pragma unroll
          for (int k = 0; k < kTcBK / 16; ++k) {
            const uint64_t adv = (uint64_t)(k * 2);  // 16 bf16 = 32 B = 2 x 16 B
            tc_mma_f16(d, a0 + adv, b0 + adv, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            if (TA == 2) tc_mma_f16(d, a1 + adv, b0 + adv, idesc, 1u);
            if (TB == 2) tc_mma_f16(d, a0 + adv, b1 + adv, idesc, 1u);
          }
          tc_commit(&empty[s]);  // frees the smem stage once these MMAs retire
          if (++s == S::kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[buf]);  // accumulator ready for the epilogue
      }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    float* scratch = reinterpret_cast<float*>(smem + S::kStages * S::kStageBytes + 256) + (warp - 2) * 32 * 33;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
    int mt, unit, nt0, nt1, kb0, kb1;
    item_range(w, mt, unit, nt0, nt1, kb0, kb1);
    (void)kb0;
    (void)kb1;
    const int row = mt * kTcBM + quarter * 32 + lane;
    epi.begin_unit(row, unit);
    for (int nt = nt0; nt < nt1; ++nt, ++it) {
      const int buf = it & 1;
      const uint32_t bph = (it >> 1) & 1;
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        epi.consume(row, nt * BN + c * 32, v, args.ncols, scratch);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      epi.end_tile(row);
    }
    epi.end_unit(row, unit, args.m);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S::kTmemCols);
  }
}

// ---- epilogues ------------------------------------------------------------

// Likelihood: per row sum over valid columns of softplus(eta); eta never
// leaves the SM.  Partial sums per unit are written to ws[unit][m] (float64)
// and reduced in fixed unit order by a second kernel (deterministic).
struct EpiSoftplusRowSum {
  double* partial;
  float tile_acc;
  double acc;
  __device__ __forceinline__ void begin_unit(int, int) {
    acc = 0.0;
    tile_acc = 0.0f;
  }
  __device__ __forceinline__ void consume(int, int col0, const float (&v)[32], int ncols, float*) {
    if (col0 + 32 <= ncols) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        s0 += softplus_f32(v[i]);
        s1 += softplus_f32(v[i + 1]);
      }
      tile_acc += s0 + s1;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < ncols) tile_acc += softplus_f32(v[i]);
    }
  }
  __device__ __forceinline__ void end_tile(int) {
    acc += (double)tile_acc;
    tile_acc = 0.0f;
  }
  __device__ __forceinline__ void end_unit(int row, int unit, int m) {
    if (row < m) partial[(size_t)unit * m + row] = acc;
  }
};

// Proposal: out[row][col] = base[row][col] + v for valid rows / columns.
struct EpiStoreAdd {
  const float* base;
  float* out;
  int ld;
  int m;
  __device__ __forceinline__ void begin_unit(int, int) {}
  __device__ __forceinline__ void consume(int row, int col0, const float (&v)[32], int ncols, float*) {
    if (row >= m) return;
    const float* b = base + (size_t)row * ld + col0;
    float* o = out + (size_t)row * ld + col0;
    if (col0 + 32 <= ncols && (ld & 3) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 x = *reinterpret_cast<const float4*>(b + i);
        *reinterpret_cast<float4*>(o + i) = make_float4(x.x + v[i], x.y + v[i + 1], x.z + v[i + 2], x.w + v[i + 3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < ncols) o[i] = b[i] + v[i];
    }
  }
  __device__ __forceinline__ void end_tile(int) {}
  __device__ __forceinline__ void end_unit(int, int, int) {}
};

// Split-K accumulation into a 2^-48 fixed-point int64 matrix with integer
// atomics (order-independent => bit-deterministic for any schedule).
struct EpiFixAtomic {
  unsigned long long* acc;  // [m][ld]
  int ld;
  int m;
  int lower_only;
  __device__ __forceinline__ void begin_unit(int, int) {}
  __device__ __forceinline__ void consume(int row, int col0, const float (&v)[32], int ncols, float*) {
    if (row >= m) return;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int c = col0 + i;
      if (c < ncols && (!lower_only || c <= row))
        atomicAdd(&acc[(size_t)row * ld + c], (unsigned long long)llrint((double)v[i] * 281474976710656.0));
    }
  }
  __device__ __forceinline__ void end_tile(int) {}
  __device__ __forceinline__ void end_unit(int, int, int) {}
};

// Raw accumulator store: each thread owns one row and writes its 32
// consecutive columns straight from registers with 16-byte stores (64 B of
// bf16 / 128 B of fp32 per thread per chunk; a warp's 32 rows fill whole
// sectors).  out[unit*unit_stride + row*ld + col] = D for valid entries
// (OutT = float or __nv_bfloat16; ld * sizeof(OutT) must be a multiple of 16
// for the vector path, otherwise element stores are used).
template <class OutT>
struct EpiStoreT {
  OutT* out;
  int ld;
  int m;
  size_t unit_stride;
  OutT* base_;
  __device__ __forceinline__ void begin_unit(int, int unit) { base_ = out + (size_t)unit * unit_stride; }
  __device__ __forceinline__ void consume(int row, int col0, const float (&v)[32], int ncols, float*) {
    if (row >= m) return;
    OutT* p = base_ + (size_t)row * ld + col0;
    const bool vec = col0 + 32 <= ncols && ((ld * sizeof(OutT)) & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(base_) & 15) == 0);
    if (vec) {
      if constexpr (sizeof(OutT) == 2) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          __nv_bfloat162 h0 = __floats2bfloat162_rn(v[i], v[i + 1]), h1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]), h3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
          u.x = *reinterpret_cast<uint32_t*>(&h0);
          u.y = *reinterpret_cast<uint32_t*>(&h1);
          u.z = *reinterpret_cast<uint32_t*>(&h2);
          u.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(p + i) = u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < ncols) p[i] = (OutT)v[i];
    }
  }
  __device__ __forceinline__ void end_tile(int) {}
  __device__ __forceinline__ void end_unit(int, int, int) {}
};

}  // namespace spa
