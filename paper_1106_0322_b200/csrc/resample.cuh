// Exact parallel prefix sum for systematic resampling (K4).
//
// The reference's ancestors come from np.cumsum(W), a strictly sequential
// float64 accumulation s_i = fl(s_{i-1} + w_i) (smc.py:273-281).  The
// kernels in resample.cu reproduce those bits with a parallel scan; see the
// algorithm notes there.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spa {

// Weight source: one contiguous array, or up to 8 equal parts (one per rank
// of a sharded particle set, read through peer pointers): element i lives
// at p[i / len][i % len].
struct WSrc {
  const double* p[8];
  int64_t len;
  int nparts;
};

// Workspace bytes of exact_cumsum for N weights (cum [N] first, then the
// per-tile scan state and control words).
size_t exact_cumsum_ws_bytes(int64_t N);
// Byte offset in ws of cumn [N] = cum / cum[N-1] with cumn[N-1] = 1
// (smc.py:277-278), written by the same launches.
size_t exact_cumsum_norm_offset(int64_t N);

// cum[i] = np.cumsum(w)[i] bit for bit (cum is the first N doubles of ws).
// Gated (gate != nullptr and *gate == 0): every kernel returns at once.
// Launches 3 kernels (+ a 16-byte memset); a speculative-binade failure
// falls back to the sequential scan inside the second kernel.
int exact_cumsum(const WSrc& w, int64_t N, void* ws, const double* gate, cudaStream_t st);
// Copy the path flag of the last exact_cumsum on ws (0 fast, 1 fallback).
int exact_cumsum_mode(int64_t N, const void* ws, int32_t* mode, cudaStream_t st);

}  // namespace spa
