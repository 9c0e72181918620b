// K1 on the int8 tensor cores (tcgen05.mma.kind::i8, twice the fp16 rate)
// for integer-coded designs (x_ij = alpha_j g_ij + gamma_j, g in {0,1,2}).
//
// Operands.  Each particle row k is a 22-bit fixed-point vector relative to
// its own largest |alpha_j beta_j|: Q_kj = rint(alpha_j beta_j / s_k) with
// |Q| <= 2^21 - 1, split exactly as Q = hi * 2^14 + mid * 2^6 + lo with
// hi = floor(Q / 2^14) in [-128, 127] (s8), mid in [0, 255] and lo in [0, 63]
// (u8) -- three byte planes per row [hi | mid | lo], each kp bytes, followed
// after the m rows by one {s_k, o_k} float pair per row (o_k = sum_j gamma_j
// beta_j, the centring offset).  The design gives two u8 planes [G | 64 G].
// Per 64-byte k-block the MMA issuer runs, for each 32-element half,
//     acc1 += hi * G        (s8 x u8)
//     acc2 += mid * (64 G)  (u8 x u8)
//     acc2 += lo * G        (u8 x u8)
// into two int32 TMEM accumulators, so sum_j g_ij Q_kj = 2^14 acc1 + acc2
// exactly (|acc1| < 2^19, 0 <= acc2 < 2^25 for kp <= 1024) and
//     eta_ki = s_k (2^14 acc1 + acc2) + o_k.
// Precision: 22 significant bits of the row maximum (float64 emulation at
// sigma = 0.3: 1.8e-6 relative log-likelihood error, tools/k1_precision.py;
// the bar is 1e-5).  Three i8 products cost 1.5 bf16-equivalents against
// the fp16 hi/lo pair's 2.
//
// Kernel: CTA pairs (cta_group::2), MMA M = 256 (128 particle rows per CTA),
// N = 128 subjects (64 B rows per CTA), K = 32; SWIZZLE_64B operands, 64-byte
// k-blocks; the two accumulators double-buffered in TMEM (2 x 2 x 128 = 512
// columns per CTA).  Warp 0 produces (TMA); warp 1 of the leader CTA issues
// the MMAs -- the whole warp runs the loop so the descriptors stay in uniform
// registers and one elected lane issues (an MMA is 64 tensor cycles, so the
// issue path must be a handful of instructions); warps 2..17 drain the
// accumulators (two sets of eight on alternate TMEM buffers).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "tc_gemm.cuh"

namespace spa {

constexpr int kI8EpiGroups = 4;                      // partial row sums per (CTA, work item): 2 sets x 2 groups
constexpr int kI8Threads = 64 + 128 * kI8EpiGroups;  // 2 + 16 warps
constexpr int kI8BN = 128;                           // subjects per tile (the pair's MMA N)
constexpr int kI8BK = 64;                            // bytes (= int8 elements) per k-block
constexpr int kI8Tile = 128 * kI8BK;                 // 8 KB: one 128-row operand tile
constexpr int kI8PairB = 64;                         // subject rows per CTA of a 128-subject tile
constexpr int kI8HalfTile = kI8PairB * kI8BK;        // 4 KB
constexpr int kI8MaxStages = 8;
constexpr int kI8MaxKb = 8;                          // resident particle tiles: kp <= 512
constexpr int kI8Extra = 1024 + 512;                 // alignment + barriers
constexpr int kI8SmemLimit = 232448;
// kp <= 512: each CTA keeps its 128 particle rows x 3 planes x kp resident for
// a whole work item; a stage is its half of the B k-block (2 x 4 KB)
__host__ __device__ constexpr int k1_i8_pair_stages(int kp) {
  return (kI8SmemLimit - kI8Extra - (kp / kI8BK) * 3 * kI8Tile) / (2 * kI8HalfTile) > kI8MaxStages
             ? kI8MaxStages
             : (kI8SmemLimit - kI8Extra - (kp / kI8BK) * 3 * kI8Tile) / (2 * kI8HalfTile);
}
__host__ __device__ constexpr int k1_i8_pair_smem(int kp) {
  return (kp / kI8BK) * 3 * kI8Tile + k1_i8_pair_stages(kp) * 2 * kI8HalfTile + kI8Extra;
}
// kp > 512: a stage carries the CTA's A k-block (3 x 8 KB) and its half of
// the B k-block (2 x 4 KB)
constexpr int kI8PairStreamStage = 3 * kI8Tile + 2 * kI8HalfTile;
constexpr int kI8PairStreamStages =
    (kI8SmemLimit - kI8Extra) / kI8PairStreamStage > kI8MaxStages ? kI8MaxStages
                                                                  : (kI8SmemLimit - kI8Extra) / kI8PairStreamStage;
constexpr int kI8PairStreamSmem = kI8PairStreamStages * kI8PairStreamStage + kI8Extra;

__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;            // SWIZZLE_64B
  return d;
}

// kind::i8 instruction descriptor: s32 accumulate, A s8 / u8, B u8, K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed) {
  return (2u << 4)                          // D format s32
         | ((a_signed ? 1u : 0u) << 7)      // A: 1 = s8, 0 = u8
         | (0u << 10)                       // B: u8
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Symmetric softplus sum of one 32-column accumulator chunk of a row, in log2
// units (softplus(eta) = eta / 2 + S(eta), the linear half added from the
// pack's row constant (1/2) prop . X^T 1 by the row reduction):
//   sum_i S(eta_i) = ln 2 * [ sum_i |y_i| / 2 + log2 prod_i (1 + 2^-|y_i|) ],  y = eta log2 e
// with the product over four interleaved groups of eight factors in [1, 2]
// (one lg2 per group: the XU pipe does one exp2 per element and 1/8 lg2).
// The accumulators combine into the integer T in one shift-add:
//   WIDE = false (kp <= 512): T = 2^14 acc1 + acc2 = sum_j g_j Q_j exactly
//     (|sum_j g_j Q_j| <= 2 * 512 * (2^21 - 1) < 2^31; the int32 arithmetic
//     is modular, so the exact in-range value comes out);
//   WIDE = true (kp <= 1024): T = 2^12 acc1 + floor(acc2 / 4) (|T| < 2^31),
//     the dropped fraction's mean (3/8) carried by the caller's offset;
// then y = sl * float(T) + ol (sl = s log2 e, ol = o log2 e, per row).
// float(T) rounds to 24 bits: relative 6e-8 of eta's linear part.
// Returns the chunk's sum of softplus / ln 2.  Columns >= nval (ragged last
// subject tile) contribute nothing (y = -inf).
template <bool WIDE, bool RAGGED>
__device__ __forceinline__ float k1_i8_chunk_sum(const uint32_t (&r1)[32], const uint32_t (&r2)[32], float sl,
                                                 float ol, int nval) {
  float P[4] = {1.f, 1.f, 1.f, 1.f}, R[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int T = WIDE ? (int)((r1[i] << 12) + (r2[i] >> 2)) : (int)((r1[i] << 14) + r2[i]);
    float y = fmaf(sl, __int2float_rn(T), ol);
    if (RAGGED && i >= nval) y = -INFINITY;  // only the last subject tile's chunks
#if defined(K1_EPI_MODE) && K1_EPI_MODE == 2
    const float e = fmaf(fmaf(y, y * 0.1f, 0.5f), -fabsf(y), 1.0f);  // timing experiment only (no MUFU)
#else
    const float e = fast_ex2(-fabsf(y));
#endif
    P[i & 3] = fmaf(P[i & 3], e, P[i & 3]);
    R[i & 1] += RAGGED && i >= nval ? 0.0f : fabsf(y);
  }
  const float lg = (fast_lg2(P[0]) + fast_lg2(P[1])) + (fast_lg2(P[2]) + fast_lg2(P[3]));
#if defined(K1_EPI_MODE) && K1_EPI_MODE == 1
  return __int_as_float(r1[0] ^ r2[31]);  // timing experiment only (TMEM loads, no softplus)
#endif
  return 0.5f * (R[0] + R[1]) + lg;
}

struct K1I8Args {
  int m;         // valid particle rows
  int n;         // valid subjects
  int kp;        // K (bytes per plane), multiple of 64
  int m_tiles;   // ceil(m / 256): particle tiles of a CTA pair
  int n_tiles;   // ceil(n / 128)
  int stages;    // stage ring depth
  int sched;     // 0: contiguous unit ranges; 1: items (tpu tiles) round-robin; 2: items in contiguous blocks
  int tpu;       // sched 1/2: subject tiles per item
  int units;     // sched 1/2: items per particle tile
  const float2* rowc;  // [m] {s_k, o_k}
  double* partial;     // [kI8EpiGroups * slots][m] per-group, per-segment softplus sums
};

// Work schedule: the m_tiles x n_tiles (particle tile, subject tile) units in
// row-major order are cut into nclus contiguous ranges of equal length (+-1:
// the first U % nclus ranges are one longer), one per CTA pair.  A pair walks
// its range as segments -- maximal runs of one particle tile -- keeping the
// tile's operand resident over a segment, so every pair does the same number
// of tile products (no rounding to whole items) and the pairs reach their
// segment boundaries (operand reloads) at different times instead of all at
// once.  Particle tile mt is covered by pairs k1_pair_of(mt n_tiles) ..
// k1_pair_of((mt + 1) n_tiles - 1); pair c writes its segment's partial sums
// to slot c - k1_pair_of(mt n_tiles).  32-bit arithmetic throughout: the MMA
// issuer's loop must stay in uniform registers (a 64-bit division is a
// subroutine call whose results are not uniform, and the descriptor math then
// moves to vector registers, ~10 instructions per MMA).
__host__ __device__ __forceinline__ int k1_range_start(int c, int U, int nclus) {
  const int base = U / nclus, rem = U % nclus;
  return c * base + min(c, rem);
}
__host__ __device__ __forceinline__ int k1_pair_of(int u, int U, int nclus) {  // pair owning unit u
  const int base = U / nclus, rem = U % nclus;
  return u < rem * (base + 1) ? u / (base + 1) : rem + (u - rem * (base + 1)) / base;
}
__host__ __device__ __forceinline__ int k1_slots_of(int mt, int n_tiles, int U, int nclus) {
  const int u0 = mt * n_tiles;
  return k1_pair_of(u0 + n_tiles - 1, U, nclus) - k1_pair_of(u0, U, nclus) + 1;
}
// CTA pairs of the K1 launch (148 SMs on B200); the workspace bound below
// holds for any pair count up to this
constexpr int kI8MaxPairs = 74;
// most segment slots of any particle tile for m particles and n subjects
inline int k1_i8_max_slots(int64_t m, int n) {
  const int64_t m_tiles = (m + 255) / 256, n_tiles = (n + kI8BN - 1) / kI8BN, U = m_tiles * n_tiles;
  const int64_t L = std::max<int64_t>(1, U / std::min<int64_t>(U, kI8MaxPairs));  // shortest range
  return (int)((n_tiles + L - 1) / L + 1);
}
// the segments of pair cid: (particle tile, subject tiles [nt0, nt1), slot)
struct K1Seg {
  int u, uend, U;
  int n_tiles, nclus, cid, sched, tpu, units;
  __device__ __forceinline__ K1Seg(const K1I8Args& a, int cid_, int nclus_)
      : n_tiles(a.n_tiles), nclus(nclus_), cid(cid_), sched(a.sched), tpu(a.tpu), units(a.units) {
    if (sched == 0) {
      U = a.m_tiles * n_tiles;
      u = k1_range_start(cid, U, nclus);
      uend = k1_range_start(cid + 1, U, nclus);
    } else {
      U = a.m_tiles * units;  // items
      u = sched == 1 ? cid : k1_range_start(cid, U, nclus);
      uend = sched == 1 ? U : k1_range_start(cid + 1, U, nclus);
    }
  }
  // odd pairs walk their range backwards, so the two pairs sharing a
  // particle tile at a range boundary work on it at the same time (both at
  // the start or both at the end of their walks: one DRAM read of its operand)
  __device__ __forceinline__ bool next(int& mt, int& nt0, int& nt1, int& slot) {
    if (u >= uend) return false;
    if (sched != 0) {
      mt = u / units;
      slot = u - mt * units;
      nt0 = slot * tpu;
      nt1 = min(n_tiles, nt0 + tpu);
      u += sched == 1 ? nclus : 1;
      return true;
    }
    if (cid & 1) {
      mt = (uend - 1) / n_tiles;
      const int lo = max(u, mt * n_tiles);
      nt0 = lo - mt * n_tiles;
      nt1 = uend - mt * n_tiles;
      uend = lo;
    } else {
      mt = u / n_tiles;
      nt0 = u - mt * n_tiles;
      nt1 = min(n_tiles, nt0 + (uend - u));
      u += nt1 - nt0;
    }
    slot = cid - k1_pair_of(mt * n_tiles, U, nclus);
    return true;
  }
};

// ---------------------------------------------------------------------------
// CTA-pair kernel (cta_group::2).  Cluster of 2 CTAs on one TPC; the pair
// owns a 256-particle tile (rank r: rows 128 r ..), each CTA holds its 128
// rows x 3 planes x kp resident in shared memory for the whole work item and
// streams 64 of the 128 subject rows of each B tile (the MMA reads the other
// half from the peer).  Per SM and 128 x 128 tile the operand stream is
// 2 planes x 64 rows x kp = 64 KB at kp = 512 instead of 320 KB, so the
// MMAs, not TMA delivery, set the pace.  The leader (rank 0) issues every
// MMA (M = 256, N = 128, K = 32) and owns the full / A-full / TMEM-empty
// barriers; both CTAs' TMA loads complete on the leader's barriers
// (.cta_group::2), MMA completion is multicast to both CTAs' empty /
// A-empty / TMEM-full barriers, and the peer's epilogue releases the leader's
// TMEM-empty barrier remotely.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {  // this smem object in CTA rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(0u));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  // default .release.cta semantics (as CUTLASS's ClusterBarrier::arrive): the
  // TMEM reads are ordered by tcgen05.wait::ld + fence::before_thread_sync;
  // .release.cluster would add a GPU-scope MEMBAR per arrive
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t bar_caddr, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_caddr), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs once the issued MMAs complete
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t"
      ".reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t"
      "}\n" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <bool kResA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kI8Threads, 1)
    k1_i8_pair_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                      K1I8Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int kblocks = args.kp / kI8BK;
  const int nst = args.stages;
  // resident: stage = B planes G / 64 G (64 rows each); else A k-block + B half
  constexpr uint32_t st_bytes = kResA ? 2 * kI8HalfTile : kI8PairStreamStage;
  constexpr uint32_t b_off = kResA ? 0 : 3 * kI8Tile;  // B half tiles inside a stage
  uint8_t* ring = smem + (kResA ? (uint32_t)kblocks * 3 * kI8Tile : 0u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + nst * st_bytes);
  uint64_t* empty = full + kI8MaxStages;
  uint64_t* afull = empty + kI8MaxStages;
  uint64_t* aempty = afull + kI8MaxKb;
  uint64_t* tfull = aempty + kI8MaxKb;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, nclus = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int kb = 0; kb < kblocks; ++kb) {
      mbar_init(&afull[kb], 1);
      mbar_init(&aempty[kb], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * 8);  // the buffer's set of eight warps, in both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      prefetch_tmap(&tma);
      prefetch_tmap(&tmb);
      int s = 0;
      uint32_t ph = 0, ic = 0;
      K1Seg seg(args, cid, nclus);
      for (int mt, nt0, nt1, slot; seg.next(mt, nt0, nt1, slot); ++ic) {
        const int arow = mt * 256 + (int)rank * 128;
        for (int nt = nt0; nt < nt1; ++nt) {
          for (int kb = 0; kb < kblocks; ++kb) {
            if (kResA && nt == nt0) {  // the item's A k-block, once the previous item is done with it
              mbar_wait(&aempty[kb], (ic & 1) ^ 1);
              if (rank == 0) mbar_arrive_expect_tx(&afull[kb], 2 * 3 * kI8Tile);
              const uint32_t bar = leader_addr(&afull[kb]);
#pragma unroll
              for (int t = 0; t < 3; ++t)
                tma_load_2d_pair(smem + (kb * 3 + t) * kI8Tile, &tma, bar, t * args.kp + kb * kI8BK, arow);
            }
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = ring + s * st_bytes;
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * st_bytes);
            const uint32_t bar = leader_addr(&full[s]);
            if (!kResA) {
#pragma unroll
              for (int t = 0; t < 3; ++t)  // A planes hi / mid / lo of this CTA's 128 particles
                tma_load_2d_pair(st + t * kI8Tile, &tma, bar, t * args.kp + kb * kI8BK, arow);
            }
#pragma unroll
            for (int t = 0; t < 2; ++t)  // B planes G / 64 G: this CTA's 64 of the tile's 128 subjects
              tma_load_2d_pair(st + b_off + t * kI8HalfTile, &tmb, bar, t * args.kp + kb * kI8BK,
                               nt * kI8BN + (int)rank * kI8PairB);
            if (++s == nst) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA, whole warp) ----------------
      constexpr uint32_t id_s = idesc_i8(256, kI8BN, true);
      constexpr uint32_t id_u = idesc_i8(256, kI8BN, false);
      constexpr uint64_t kT = kI8Tile >> 4, kH = kI8HalfTile >> 4;
      const uint64_t d0 = umma_desc_sw64(smem_u32(smem));
      const uint64_t dr = umma_desc_sw64(smem_u32(ring));
      int s = 0;
      uint32_t ph = 0, ic = 0;
      int it = 0;
      K1Seg seg(args, cid, nclus);
      for (int mt, nt0, nt1, slot; seg.next(mt, nt0, nt1, slot); ++ic) {
        for (int nt = nt0; nt < nt1; ++nt, ++it) {
          const int buf = it & 1;
          const uint32_t bph = (it >> 1) & 1;
          mbar_wait(&tempty[buf], bph ^ 1);
          tc_fence_after();
          const uint32_t d1 = tmem_base + buf * 256, d2 = d1 + 128;
          for (int kb = 0; kb < kblocks; ++kb) {
            if (kResA && nt == nt0) mbar_wait(&afull[kb], ic & 1);
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint64_t dst = dr + (uint64_t)(s * (st_bytes >> 4));
            const uint64_t da = kResA ? d0 + (uint64_t)(kb * 3) * kT : dst;
            const uint64_t db = dst + (b_off >> 4);
#pragma unroll
            for (int k = 0; k < kI8BK / 32; ++k) {
              const uint64_t a = da + 2 * k, b = db + 2 * k;
              const uint32_t acc = (kb != 0 || k != 0) ? 1u : 0u;
              tc_mma_i8_pair(d1, a, b, id_s, acc);            // hi x G
              tc_mma_i8_pair(d2, a + kT, b + kH, id_u, acc);  // mid x 64 G
              tc_mma_i8_pair(d2, a + 2 * kT, b, id_u, 1u);    // lo x G
            }
            tc_commit_pair(&empty[s]);
            if (kResA && nt == nt1 - 1) tc_commit_pair(&aempty[kb]);
            if (++s == nst) {
              s = 0;
              ph ^= 1;
            }
          }
          tc_commit_pair(&tfull[buf]);
        }
      }
    }
  } else {
    // ---------------- epilogue (both CTAs, warps 2..17) ----------------
    // Two sets of eight warps take alternate tiles (set = TMEM buffer), so
    // one set's softplus work overlaps the other's accumulator wait; in a
    // set, two groups of four warps (one per TMEM lane quarter) take 64
    // columns each, in two 32-column chunks.  The buffer is released after
    // the second chunk is in registers.
    // eta = s (2^14 acc1 + acc2) + o (k1_i8_chunk_sum; the streamed kp > 512
    // variant drops acc2's two low bits -- an absolute error below 1.5 s,
    // under the 22-bit quantisation's own; tests: 1e-5 relative).
    const int quarter = warp & 3;
    const int set = (warp - 2) >> 3;
    const int grp = ((warp - 2) >> 2) & 1;
    const uint32_t tempty_c = leader_addr(&tempty[set]);
    int it = 0;
    K1Seg seg(args, cid, nclus);
    for (int mt, nt0, nt1, slot; seg.next(mt, nt0, nt1, slot);) {
      const int row = mt * 256 + (int)rank * 128 + quarter * 32 + lane;
      float2 rc = make_float2(0.f, 0.f);
      if (row < args.m) rc = args.rowc[row];
      // log2-unit row constants (see k1_i8_chunk_sum)
      constexpr float kLog2e = 1.4426950408889634f;
      const float sl = kResA ? rc.x * kLog2e : rc.x * (4.0f * kLog2e);
      const float ol = kResA ? rc.y * kLog2e : fmaf(rc.x, 1.5f, rc.y) * kLog2e;
      double acc = 0.0;
      for (int nt = nt0; nt < nt1; ++nt, ++it) {
        if ((it & 1) != set) continue;
        const uint32_t bph = (it >> 1) & 1;
        mbar_wait(&tfull[set], bph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + set * 256 + grp * 64;
        float tile = 0.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r1[32], r2[32];
          tmem_ld_32x32b_x32(taddr + c * 32, r1);
          tmem_ld_32x32b_x32(taddr + 128 + c * 32, r2);
          tmem_ld_wait();
          if (c == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_c);  // the leader's barrier
          }
          const int nval = args.n - (nt * kI8BN + grp * 64 + c * 32);  // warp-uniform
          tile += nval >= 32 ? k1_i8_chunk_sum<!kResA, false>(r1, r2, sl, ol, 32)
                             : k1_i8_chunk_sum<!kResA, true>(r1, r2, sl, ol, nval);
        }
        acc += (double)tile;
      }
      if (row < args.m)
        args.partial[(size_t)(kI8EpiGroups * slot + set * 2 + grp) * args.m + row] = acc * 0.6931471805599453;
    }
  }

  tc_fence_before();
  cluster_sync_all();  // every MMA consumed and both epilogues done with TMEM
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

}  // namespace spa
