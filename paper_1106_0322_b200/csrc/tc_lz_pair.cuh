// Proposal increments eps = z L^T on CTA pairs (cta_group::2), bf16 in, fp32
// TMEM accumulate, bf16 out by TMA store.
//
// The single-CTA engine (tc_gemm.cuh, 128 x 256 tiles) streams 48 KB of
// operands per 64-wide k-block from L2 for 128 x 256 outputs.  Here a cluster
// of two CTAs computes 256 particles x 256 coordinates per MMA (M = 256,
// N = 256, K = 16): each CTA loads its own 128 particle rows of z and HALF of
// the L tile (128 coordinates), 32 KB per k-block for the same 128 x 256
// outputs per SM, and the smaller stage leaves room for 6 stages.  L is lower
// triangular: column tile nt stops at k-block 4 (nt + 1) (256 / 64).
//
// Roles (192 threads per CTA): warp 0 TMA producer (both CTAs; the loads
// complete on the leader's barriers), warp 1 of the leader MMA issuer (whole
// warp, elect.sync), warps 2..5 epilogue (both CTAs: TMEM lane quarter ->
// 32-column chunks -> EpiStoreT's swizzled staging -> TMA store).  MMA
// completion is multicast to both CTAs' stage-empty and TMEM-full barriers;
// both CTAs' epilogue warps release the leader's TMEM-empty barrier.
#pragma once

#include "tc_gemm.cuh"
#include "tc_k1_i8.cuh"

namespace spa {

constexpr int kLzThreads = 192;
constexpr int kLzBN = 256;                          // coordinates per pair tile (MMA N)
constexpr int kLzStageBytes = 2 * 128 * kTcBK * 2;  // z k-block (16 KB) + L half k-block (16 KB)
constexpr int kLzStages = 6;
constexpr int kLzSmem = kLzStages * kLzStageBytes + EpiStoreT<__nv_bfloat16>::kSmemBytes + 1024 + 256;

struct LzArgs {
  int m;        // particles
  int kq;       // K (multiple of 64)
  int mtp;      // particle pair tiles: ceil(m / 256)
  int n_tiles;  // coordinate tiles of 256
};

__device__ __forceinline__ void tc_mma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// work item w of a cluster walk -> (pair tile, column tile).  With two column
// tiles (8 vs 4 k-blocks under the triangle) and an even number of clusters,
// cluster c would always draw the same column tile; it alternates per round.
__device__ __forceinline__ void lz_item(const LzArgs& a, int w, int nclus, int& mp, int& nt) {
  mp = w / a.n_tiles;
  nt = w % a.n_tiles;
  if (a.n_tiles == 2 && (nclus & 1) == 0) nt ^= (w / nclus) & 1;
}
__device__ __forceinline__ int lz_kblocks(const LzArgs& a, int nt) {
  return min(a.kq / kTcBK, ((nt + 1) * kLzBN + kTcBK - 1) / kTcBK);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLzThreads, 1)
    lz_pair_kernel(const __grid_constant__ CUtensorMap tmz, const __grid_constant__ CUtensorMap tml, LzArgs args,
                   const __grid_constant__ EpiStoreT<__nv_bfloat16> epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + kLzStages * kLzStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + EpiStoreT<__nv_bfloat16>::kSmemBytes);
  uint64_t* empty = full + kLzStages;
  uint64_t* tfull = empty + kLzStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, nclus = gridDim.x >> 1;
  const int items = args.mtp * args.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * 4);  // the four epilogue warps of both CTAs
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      prefetch_tmap(&tmz);
      prefetch_tmap(&tml);
      int s = 0;
      uint32_t ph = 0;
      for (int w = cid; w < items; w += nclus) {
        int mp, nt;
        lz_item(args, w, nclus, mp, nt);
        const int kbe = lz_kblocks(args, nt);
        for (int kb = 0; kb < kbe; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * kLzStageBytes;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kLzStageBytes);
          const uint32_t bar = leader_addr(&full[s]);
          tma_load_2d_pair(st, &tmz, bar, kb * kTcBK, mp * 256 + (int)rank * 128);
          tma_load_2d_pair(st + kLzStageBytes / 2, &tml, bar, kb * kTcBK, nt * kLzBN + (int)rank * 128);
          if (++s == kLzStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA, whole warp) ----------------
      constexpr uint32_t idesc = idesc_bf16_f32(256, kLzBN);
      const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int w = cid; w < items; w += nclus, ++it) {
        int mp, nt;
        lz_item(args, w, nclus, mp, nt);
        const int kbe = lz_kblocks(args, nt);
        const int buf = it & 1;
        mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * kLzBN;
        for (int kb = 0; kb < kbe; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t da = d0 + (uint64_t)(s * (kLzStageBytes >> 4));
          const uint64_t db = da + (uint64_t)((kLzStageBytes / 2) >> 4);
#pragma unroll
          for (int k = 0; k < kTcBK / 16; ++k)  // 16 bf16 = 32 B = 2 x 16 B per K step
            tc_mma_f16_pair(d, da + 2 * k, db + 2 * k, idesc, (kb != 0 || k != 0) ? 1u : 0u);
          tc_commit_pair(&empty[s]);
          if (++s == kLzStages) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit_pair(&tfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue (both CTAs, warps 2..5) ----------------
    const int quarter = warp & 3;
    const uint32_t tempty_c = leader_addr(&tempty[0]);
    typename EpiStoreT<__nv_bfloat16>::State st;
    TcArgs unused{};
    epi.init(st, staging, warp - 2, unused);
    epi.begin_unit(st, 0, 0, 0, 0);
    int it = 0;
    for (int w = cid; w < items; w += nclus, ++it) {
      int mp, nt;
      lz_item(args, w, nclus, mp, nt);
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      tc_fence_after();
      const int row = mp * 256 + (int)rank * 128 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * kLzBN;
#pragma unroll 1
      for (int c = 0; c < kLzBN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        if (c == kLzBN / 32 - 1) {  // the whole accumulator is in registers or stored: release it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_c + buf * 8);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        epi.consume(st, row, nt * kLzBN + c * 32, v, 0);
      }
    }
    epi.finish(st);
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

}  // namespace spa
