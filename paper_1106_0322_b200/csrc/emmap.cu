// f3: batched EM MAP (reference emmap.py:117-165, used by summary.py:173-211).
//
// One CTA per problem (seed, prior).  EM alternates closed-form adaptive L1
// weights w_j = (a+1)/(a c + |beta_j|) (emmap.py:48-56) with a weighted-L1
// logistic solve by cyclic coordinate descent on the quadratic majorisation
// (curvature 0.25 sum_i x_ij^2) with soft thresholding (emmap.py:69-108),
// until the largest KKT violation is below inner_tol; EM stops when no
// coordinate moves more than tol.  Everything is float64 as in the
// reference (the 1e-8 KKT tolerance needs it).  The subjects' eta_i and
// mu_i = expit(eta_i) live in shared memory; thread t owns subjects
// t + blockDim * k, so a warp reads each genotype bit-plane word once.  The
// gradient reuses X^T y: g_j = (X^T y)_j - sum_i x_ij mu_i.  Genotype-coded
// designs only (x_ij = alpha_j g_ij + gamma_j, exact in float64).
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/spa_b200.h"
#include "common.cuh"

namespace spa {

constexpr int kEmThreads = 512;

struct EmParams {
  spa_design d;
  int problems;
  const double* seeds;  // [P][q]
  const double* a;      // [P]
  const double* c;      // [P]
  const double* curv;   // [q]  0.25 sum_i x_ij^2
  double tol, inner_tol;
  int max_iter, inner_max_sweeps;
  double* beta_out;  // [P][q]
  double* log_post;  // [P]
  int* info;         // [P]: bit 0 EM converged, bit 1 every inner solve converged
  int* iters;        // [P]: EM iterations
};

// deterministic block sum (fixed shuffle tree, then one warp over the warp sums)
__device__ __forceinline__ double em_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double s = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double em_block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double s = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

// x_ij for subject i (0 for padding subjects, code (1,1))
__device__ __forceinline__ double em_x(const spa_design& d, int j, int i, bool& valid) {
  const uint2 wv = reinterpret_cast<const uint2*>(d.planes)[(size_t)j * d.n_words + (i >> 5)];
  const uint32_t b1 = (wv.x >> (i & 31)) & 1u, b2 = (wv.y >> (i & 31)) & 1u;
  valid = !(b1 && b2);
  return valid ? fma(d.alpha[j], (double)(b1 + 2u * b2), d.gamma[j]) : 0.0;
}

__device__ __forceinline__ double em_expit(double x) { return 1.0 / (1.0 + exp(-x)); }

__global__ void __launch_bounds__(kEmThreads) em_map_kernel(EmParams P) {
  extern __shared__ double esm[];
  const spa_design& d = P.d;
  const int q = d.q, npad = d.n_words * 32, prob = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  double* eta = esm;
  double* mu = eta + npad;
  double* beta = mu + npad;
  double* w = beta + q;
  double* bold = w + q;
  double* red = bold + q;  // 33 doubles
  const double a = P.a[prob], c = P.c[prob];
  for (int j = tid; j < q; j += nt) {
    beta[j] = P.seeds[(size_t)prob * q + j];
    bold[j] = beta[j];
  }
  __syncthreads();
  // eta = X beta, mu = expit(eta)
  for (int i = tid; i < npad; i += nt) {
    double e = 0.0;
    for (int j = 0; j < q; ++j) {
      bool v;
      const double x = em_x(d, j, i, v);
      e = fma(x, beta[j], e);
    }
    eta[i] = e;
    mu[i] = em_expit(e);
  }
  for (int j = tid; j < q; j += nt) w[j] = d.penalized[j] ? (a + 1.0) / (a * c + fabs(beta[j])) : 0.0;
  __syncthreads();
  bool converged = false, inner_ok = true;
  int it = 0;
  for (it = 1; it <= P.max_iter; ++it) {
    // ---- weighted-L1 logistic by cyclic coordinate descent (emmap.py:69-108)
    bool inner_conv = false;
    for (int sweep = 1; sweep <= P.inner_max_sweeps; ++sweep) {
      for (int j = 0; j < q; ++j) {
        double s = 0.0;
        for (int i = tid; i < npad; i += nt) {
          bool v;
          const double x = em_x(d, j, i, v);
          s = fma(x, mu[i], s);
        }
        const double g = d.sy[j] - em_block_sum(s, red);
        const double cj = P.curv[j];
        const double z = beta[j] + g / cj;
        const double thr = fabs(z) - w[j] / cj;
        const double nw = thr > 0.0 ? copysign(thr, z) : 0.0;
        if (nw != beta[j]) {  // identical in every thread
          const double delta = nw - beta[j];
          for (int i = tid; i < npad; i += nt) {
            bool v;
            const double x = em_x(d, j, i, v);
            if (v) {
              const double e = fma(x, delta, eta[i]);
              eta[i] = e;
              mu[i] = em_expit(e);
            }
          }
          __syncthreads();
          if (tid == 0) beta[j] = nw;
          __syncthreads();
        }
      }
      // KKT residual of X^T (y - expit(eta)) (emmap.py:59-66)
      double viol = 0.0;
      for (int j = 0; j < q; ++j) {
        double s = 0.0;
        for (int i = tid; i < npad; i += nt) {
          bool v;
          const double x = em_x(d, j, i, v);
          s = fma(x, mu[i], s);
        }
        const double g = d.sy[j] - em_block_sum(s, red);
        const double vj = beta[j] == 0.0 ? fmax(fabs(g) - w[j], 0.0) : fabs(g - copysign(w[j], beta[j]));
        viol = fmax(viol, vj);
      }
      if (viol < P.inner_tol) {
        inner_conv = true;
        break;
      }
    }
    inner_ok = inner_ok && inner_conv;
    // ---- EM step: move, new weights (emmap.py:145-163)
    double mv = 0.0;
    for (int j = tid; j < q; j += nt) mv = fmax(mv, fabs(beta[j] - bold[j]));
    mv = em_block_max(mv, red);
    for (int j = tid; j < q; j += nt) {
      w[j] = d.penalized[j] ? (a + 1.0) / (a * c + fabs(beta[j])) : 0.0;
      bold[j] = beta[j];
    }
    __syncthreads();
    if (mv < P.tol) {
      converged = true;
      break;
    }
  }
  // log posterior: sum_j beta_j (X^T y)_j - sum_i softplus(eta_i) + sum_pen gt(beta_j)
  double sp = 0.0;
  for (int i = tid; i < d.n; i += nt) sp += fmax(eta[i], 0.0) + log1p(exp(-fabs(eta[i])));
  double lin = 0.0, lpr = 0.0;
  for (int j = tid; j < q; j += nt) {
    lin += beta[j] * d.sy[j];
    if (d.penalized[j]) lpr += -log(2.0 * c) - (a + 1.0) * log1p(fabs(beta[j]) / (a * c));
  }
  const double tot = em_block_sum(lin - sp + lpr, red);
  for (int j = tid; j < q; j += nt) P.beta_out[(size_t)prob * q + j] = beta[j];
  if (tid == 0) {
    P.log_post[prob] = tot;
    P.info[prob] = (converged ? 1 : 0) | (inner_ok ? 2 : 0);
    P.iters[prob] = converged ? it : P.max_iter;
  }
}

}  // namespace spa

using namespace spa;

extern "C" int spa_em_map(const spa_design* d, int32_t problems, const double* seeds, const double* a,
                          const double* c, const double* curv, double tol, int32_t max_iter, double inner_tol,
                          int32_t inner_max_sweeps, double* beta_out, double* log_post, int32_t* info,
                          int32_t* iters, void* stream) {
  SPA_REQUIRE(d && seeds && a && c && curv && beta_out && log_post && info && iters && problems >= 0, kBadArgument,
              "spa_em_map: bad arguments");
  SPA_REQUIRE(d->coded && d->planes && d->alpha && d->gamma && d->sy && d->penalized, kNotSupported,
              "spa_em_map: genotype-coded designs only");
  SPA_REQUIRE(max_iter >= 1 && inner_max_sweeps >= 1 && tol > 0 && inner_tol > 0, kBadArgument,
              "spa_em_map: iteration limits and tolerances must be positive");
  if (problems == 0) return 0;
  const size_t smem = sizeof(double) * ((size_t)2 * d->n_words * 32 + 3 * (size_t)d->q + 40);
  SPA_REQUIRE(smem <= 227 * 1024, kNotSupported, "spa_em_map: too many subjects for the shared-memory state");
  SPA_CHECK_CUDA(cudaFuncSetAttribute(em_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  EmParams P;
  P.d = *d;
  P.problems = problems;
  P.seeds = seeds;
  P.a = a;
  P.c = c;
  P.curv = curv;
  P.tol = tol;
  P.inner_tol = inner_tol;
  P.max_iter = max_iter;
  P.inner_max_sweeps = inner_max_sweeps;
  P.beta_out = beta_out;
  P.log_post = log_post;
  P.info = info;
  P.iters = iters;
  em_map_kernel<<<problems, kEmThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(P);
  SPA_CHECK_LAUNCH();
  return 0;
}
