// Warp-specialised tcgen05 GEMM engine for sm_100a with fused epilogues.
//
//   D[128 x BN] = sum_terms A_t[128 x K] * B_t[BN x K]^T   (bf16 or fp16 in, fp32 TMEM accumulate)
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

constexpr int kTcSmemLimit = 232448;  // 227 KB dynamic shared memory per CTA

// EpiBytes: shared memory the epilogue needs (its staging / tables); the
// stage ring gets what remains (at most 6 stages).
template <int TA, int TB, int BN, int TM = 1, int EpiBytes = 0>
struct TcShape {
  static constexpr int kABytes = kTcBM * kTcBK * 2;  // 16 KB per A term and m-tile
  static constexpr int kBBytes = BN * kTcBK * 2;     // per B term
  static constexpr int kStageBytes = TM * TA * kABytes + TB * kBBytes;
  static constexpr int kBudget = kTcSmemLimit - 1024 /*align*/ - 256 /*barriers*/ - EpiBytes;
  static constexpr int kStagesRaw = kBudget / kStageBytes;
  static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  static constexpr int kRingBytes = kStages * kStageBytes;
  static constexpr int kTmemCols = 2 * TM * BN;  // double-buffered accumulator(s)
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
  int tri_b = 0;       // 1: B[n][k] is lower triangular (k <= n), so column tile nt stops at
                       // k-block ceil((nt + 1) BN / BK) -- the zero upper part is never loaded
};

// (the epilogue contract is documented with the epilogues below)
// Dynamic shared memory: [stage ring][epilogue region (Epi::kSmemBytes)]
// [barriers], 1024-aligned (SW128 operands, swizzled staging).
template <int TA, int TB, int BN, class Epi, int TM = 1>
constexpr int tc_smem_bytes() {
  return TcShape<TA, TB, BN, TM, Epi::kSmemBytes>::kRingBytes + Epi::kSmemBytes + 1024 /*align*/ +
         256 /*barriers*/;
}

// The epilogue object is a __grid_constant__ parameter: its tensor maps stay
// addressable in parameter space for TMA; per-thread mutable state lives in
// Epi::State.
// F16: operands are fp16 (the K1 likelihood's hi/lo split), else bf16.
template <int TA, int TB, int BN, class Epi, int TM = 1, bool F16 = false>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, TcArgs args,
                   const __grid_constant__ Epi epi) {
  using S = TcShape<TA, TB, BN, TM, Epi::kSmemBytes>;
  static_assert(tc_smem_bytes<TA, TB, BN, Epi, TM>() <= kTcSmemLimit, "shared memory budget exceeded");
  static_assert(TM == 1 || !Epi::kRowState, "TM > 1 interleaves rows: stateless epilogues only");
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (keeps the shared
  // address space visible to the compiler: LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + S::kRingBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + Epi::kSmemBytes);
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
  // TM > 1: an item covers TM consecutive m-tiles that share every B tile
  // loaded into shared memory (B traffic from L2 / TM).
  const int units = args.units;
  const int items = (args.m_tiles + TM - 1) / TM * units;
  auto item_range = [&](int w, int& mt, int& unit, int& nt0, int& nt1, int& kb0, int& kb1) {
    mt = w / units * TM;
    unit = w % units;
    // triangular B with two column units: unit 1 costs twice unit 0 (8 vs 4
    // k-blocks at q = 512), and with an even grid CTA b would always draw the
    // same unit (odd CTAs twice the work: SMs 26% idle in the L z GEMM), so
    // the unit alternates between rounds (a bijection: an m-tile's two items
    // never straddle a round when the grid is even)
    if (args.tri_b && units == 2 && (gridDim.x & 1) == 0) unit ^= (w / gridDim.x) & 1;
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
        const int kbe = args.tri_b ? min(kb1, ((nt + 1) * BN + kTcBK - 1) / kTcBK) : kb1;
        for (int kb = kb0; kb < kbe; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * S::kStageBytes;
          mbar_arrive_expect_tx(&full[s], S::kStageBytes);
#pragma unroll
          for (int tm = 0; tm < TM; ++tm)
#pragma unroll
            for (int t = 0; t < TA; ++t)
              tma_load_2d(st + (tm * TA + t) * S::kABytes, &tma, &full[s], t * args.kp + kb * kTcBK,
                          (mt + tm) * kTcBM);
#pragma unroll
          for (int t = 0; t < TB; ++t)
            tma_load_2d(st + TM * TA * S::kABytes + t * S::kBBytes, &tmb, &full[s], t * args.kp + kb * kTcBK,
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
      constexpr uint32_t idesc = F16 ? idesc_f16_f32(kTcBM, BN) : idesc_bf16_f32(kTcBM, BN);
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
        const int kbe = args.tri_b ? min(kb1, ((nt + 1) * BN + kTcBK - 1) / kTcBK) : kb1;
        for (int kb = kb0; kb < kbe; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * S::kStageBytes);
          const uint64_t b0 = umma_desc_sw128(st + TM * TA * S::kABytes);
          const uint64_t b1 = umma_desc_sw128(st + TM * TA * S::kABytes + S::kBBytes);
#pragma unroll
          for (int tm = 0; tm < TM; ++tm) {
            const uint32_t d = tmem_base + (buf * TM + tm) * BN;
            const uint64_t a0 = umma_desc_sw128(st + tm * TA * S::kABytes);
            const uint64_t a1 = umma_desc_sw128(st + (tm * TA + 1) * S::kABytes);
#pragma unroll
            for (int k = 0; k < kTcBK / 16; ++k) {
              const uint64_t adv = (uint64_t)(k * 2);  // 16 bf16 = 32 B = 2 x 16 B
              tc_mma_f16(d, a0 + adv, b0 + adv, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
              if (TA == 2) tc_mma_f16(d, a1 + adv, b0 + adv, idesc, 1u);
              if (TB == 2) tc_mma_f16(d, a0 + adv, b1 + adv, idesc, 1u);
            }
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
    typename Epi::State st;
    epi.init(st, staging, warp - 2, args);
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
    int mt, unit, nt0, nt1, kb0, kb1;
    item_range(w, mt, unit, nt0, nt1, kb0, kb1);
    (void)kb0;
    (void)kb1;
    const int row = mt * kTcBM + quarter * 32 + lane;
    epi.begin_unit(st, row, unit, nt0 * BN, nt1 * BN);
    for (int nt = nt0; nt < nt1; ++nt, ++it) {
      const int buf = it & 1;
      const uint32_t bph = (it >> 1) & 1;
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
#pragma unroll 1
      for (int tm = 0; tm < TM; ++tm) {
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (buf * TM + tm) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          epi.consume(st, row + tm * kTcBM, nt * BN + c * 32, v, args.ncols);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      epi.end_tile(st, row);
    }
    epi.end_unit(st, row, unit, args.m);
    }
    epi.finish(st);
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S::kTmemCols);
  }
}

// ---- epilogues ------------------------------------------------------------
// Contract (the epilogue object is read-only; per-thread state in State; a
// warp's 32 threads hold 32 consecutive rows = one TMEM lane quarter):
//   kRowState   true if State carries per-row sums across tiles
//   kSmemBytes  shared memory of the epilogue region (1024-aligned base)
//   init(st, smem, ew, args)               once per epilogue thread (ew = 0..3)
//   begin_unit(st, row, unit, c0, c1)      per work item (columns [c0, c1))
//   consume(st, row, col0, v[32], ncols)   32 consecutive columns of one row
//   end_tile(st, row) / end_unit(st, row, unit, m) / finish(st)

// Likelihood: per row sum over valid columns of softplus(eta); eta never
// leaves the SM.  Partial sums per unit are written to ws[unit][m] (float64)
// and reduced in fixed unit order by a second kernel (deterministic).
struct EpiSoftplusRowSum {
  static constexpr bool kRowState = true;
  static constexpr int kSmemBytes = 0;
  double* partial;
  struct State {
    float tile_acc;
    double acc;
  };
  __device__ __forceinline__ void init(State&, uint8_t*, int, const TcArgs&) const {}
  __device__ __forceinline__ void begin_unit(State& s, int, int, int, int) const {
    s.acc = 0.0;
    s.tile_acc = 0.0f;
  }
  __device__ __forceinline__ void consume(State& s, int, int col0, const float (&v)[32], int ncols) const {
    if (col0 + 32 <= ncols) {
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        s0 += softplus_f32(v[i]);
        s1 += softplus_f32(v[i + 1]);
      }
      s.tile_acc += s0 + s1;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < ncols) s.tile_acc += softplus_f32(v[i]);
    }
  }
  __device__ __forceinline__ void end_tile(State& s, int) const {
    s.acc += (double)s.tile_acc;
    s.tile_acc = 0.0f;
  }
  __device__ __forceinline__ void end_unit(State& s, int row, int unit, int m) const {
    if (row < m) partial[(size_t)unit * m + row] = s.acc;
  }
  __device__ __forceinline__ void finish(State&) const {}
};

// Raw accumulator store through TMA: each thread writes its row's 32 columns
// (64 B bf16 / 128 B fp32) into a per-warp swizzled staging tile (SW64 /
// SW128: conflict-free 16-byte shared stores), then one lane issues a 3-D
// bulk tensor store of the 32 x 32 box at (col0, row0, unit).  The tensor map
// tmc (built by the launcher) clips columns >= ncols, rows >= m and keeps
// split-K units apart.  Two staging buffers per warp alternate; a buffer is
// rewritten only after its previous store has finished reading it.
template <class OutT>
struct EpiStoreT {
  static constexpr bool kRowState = false;
  static constexpr int kBoxBytes = 32 * 32 * (int)sizeof(OutT);
  static constexpr int kSmemBytes = 4 * 2 * kBoxBytes;
  CUtensorMap tmc;
  int m;
  int slabs = 1;  // 1: unit u stores into slab u (split-K partials); 0: column units share one output
  struct State {
    uint8_t* scratch;
    int unit;
    int nbuf;
  };
  __device__ __forceinline__ void init(State& s, uint8_t* smem, int ew, const TcArgs&) const {
    s.scratch = smem + ew * 2 * kBoxBytes;
    s.unit = 0;
    s.nbuf = 0;
    if ((threadIdx.x & 31) == 0) prefetch_tmap(&tmc);
  }
  __device__ __forceinline__ void begin_unit(State& s, int, int unit, int, int) const { s.unit = slabs ? unit : 0; }
  __device__ __forceinline__ void consume(State& s, int row, int col0, const float (&v)[32], int) const {
    const int lane = threadIdx.x & 31;
    const int row0 = row - lane;  // warp-uniform
    if (row0 >= m) return;
    uint8_t* buf = s.scratch + (s.nbuf & 1) * kBoxBytes;
    ++s.nbuf;
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    if constexpr (sizeof(OutT) == 2) {
      // 64-byte rows, SWIZZLE_64B: 16-byte chunk i of row r sits at chunk i ^ ((r >> 1) & 3)
      const int sw = (lane >> 1) & 3;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * i], v[8 * i + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * i + 2], v[8 * i + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * i + 4], v[8 * i + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * i + 6], v[8 * i + 7]);
        uint4 u;
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(buf + lane * 64 + ((i ^ sw) << 4)) = u;
      }
    } else {
      // 128-byte rows, SWIZZLE_128B: chunk i of row r sits at chunk i ^ (r & 7)
      const int sw = lane & 7;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(buf + lane * 128 + ((i ^ sw) << 4)) =
            make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&tmc, buf, col0, row0, s.unit);
      bulk_commit();
    }
  }
  __device__ __forceinline__ void end_tile(State&, int) const {}
  __device__ __forceinline__ void end_unit(State&, int, int, int) const {}
  __device__ __forceinline__ void finish(State&) const {
    if ((threadIdx.x & 31) == 0) bulk_wait<0>();
  }
};

}  // namespace spa
