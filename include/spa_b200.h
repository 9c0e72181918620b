/*
 * libspa_b200 -- C ABI of the B200-native SMC lambda-path sampler.
 *
 * The reference (`spa` 0.1.0) is pure Python/NumPy and has no FFI of its
 * own.  Each entry point below replaces one reference
 * function on the hot path (cited as reference file:line); the Python host
 * package `paper_1106_0322_b200` binds them with ctypes and keeps the
 * reference's public surface (`run_sampler`, `reweight`, `ess`,
 * `systematic_resample_indices`, `smc_step`, ...).
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer owned by the caller (no allocation
 *     inside the library); `stream` is a cudaStream_t passed as void*;
 *   - calls are stream-ordered and reentrant; the only process-global state
 *     is one-time kernel attribute setup;
 *   - return 0 on success, a cudaError_t value or an SPA_E* code otherwise;
 *     spa_last_error() returns the calling thread's last message.
 *   - particles are float32 rows with leading dimension `ldb` (elements).
 */
#ifndef SPA_B200_H_
#define SPA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPA_E_BAD_ARGUMENT 1001
#define SPA_E_NOT_SUPPORTED 1002
#define SPA_E_WORKSPACE 1003
#define SPA_E_DRIVER 1004

/* Design matrix in the layouts the kernels read (built once per dataset by
 * the host from Dataset.X / Dataset.y; reference smc.py:106-123 make_design,
 * including the optional unpenalised intercept column). */
typedef struct spa_design {
  int32_t n;          /* subjects */
  int32_t q;          /* coordinates (p, +1 with intercept) */
  int32_t coded;      /* 1: every column is x = alpha*g + gamma, g in {0,1,2} */
  int32_t n_words;    /* 32-subject words per column in the bit planes */
  const uint32_t* planes;   /* coded: [q][n_words][2] bit planes (g==1, g==2)  */
  const float* xcols;       /* general: [q][n_words*32] float32 columns, 0-padded */
  const float* xlev;        /* [q][4]  x value of code 0,1,2 (coded designs)   */
  const double* sy;         /* [q]     X^T y                                    */
  const double* alpha;      /* [q]     coded: x = alpha*g + gamma; general: the
                               power-of-two column scale of gemm_b (X = alpha*Xs) */
  const double* gamma;      /* [q]                                              */
  const uint8_t* penalized; /* [q]     1 = prior applies (smc.py:266-270)      */
  /* tensor-core operand of the batched likelihood (K1) */
  const void* gemm_b;       /* B operand: coded -> uint8 [n][2*kp] = [G | 64 G]
                               (int8 K1); general -> fp16 [Xshi | Xslo]
                               [n][2*kp], Xs = X/alpha                        */
  int32_t kp;               /* K per plane, multiple of 64, >= q (<= 1024 coded) */
  int32_t terms;            /* general designs: 2 B terms; coded: 1 (unused) */
  const uint32_t* codes;    /* coded: [q][2*n_words] genotype codes for the MwG
                               kernel, 16 subjects per word, subject s of the
                               word in bits 2s..2s+1 (0,1,2; 3 = padding)    */
  const double* sx;         /* [q]     X^T 1 (coded K1: softplus(eta) =
                               eta/2 + (|eta|/2 + log(1 + e^-|eta|)), the
                               linear half summed by the pack)              */
} spa_design;

/* Prior description: a > 0 (generalised t, model.py:78-81) or a = +inf
 * (double-exponential limit, model.py:84-88). */

const char* spa_last_error(void);
int spa_version(void);

/* ---- K6: Philox4x64-10 streams (smc.py:40-43) -------------------------- */
/* Raw blocks first_block..first_block+count-1 of stream key (k0, k1):
 * out[4*count] uint64 (device). Test hook for bit parity with NumPy. */
int spa_philox_blocks(uint64_t k0, uint64_t k1, uint64_t first_block, int64_t count, uint64_t* out,
                      void* stream);

/* ---- K1: batched log-likelihood on tcgen05 tensor cores -----------------
 * Replaces model.py:131-145 log_likelihood evaluated for many particles
 * (batched as summary.py:154-170).  A = packed particles (spa_pack_particles),
 * spa_k1_operand_bytes(d, m) bytes:
 *   coded designs  -- int8 tensor cores: three byte planes [hi | mid | lo]
 *                     [m][3*kp] of the 22-bit per-row fixed point of
 *                     alpha*beta, then {scale, offset} float2 [m], then
 *                     (1/2) sum_i eta_ki = (1/2) beta_k . X^T 1 float64 [m];
 *   general        -- fp16 [m][2*kp] = [hi | lo] (22 significant bits).
 * out_sp[m] = sum_i softplus(eta_ki) (float64).
 * ws: workspace of spa_loglik_workspace_bytes(m, n) bytes. */
size_t spa_k1_operand_bytes(const spa_design* d, int64_t m);
size_t spa_loglik_workspace_bytes(int64_t m, int32_t n);
int spa_loglik_softplus(const spa_design* d, const void* A, int64_t m, double* out_sp, void* ws, size_t ws_bytes,
                        void* stream);

/* Pack particle rows into the K1 A-operand and emit the exact linear term
 * y.eta = beta . X^T y (float64).  Optionally (lp != NULL) also the log-prior
 * sum at scale c (model.py:78-81 summed over penalised coordinates). */
int spa_pack_particles(const spa_design* d, const float* beta, int64_t m, int32_t ldb, void* A, double* ylin,
                       double a, double c, double* lp, void* stream);

/* Full per-particle log-likelihood l_k = ylin_k - sp_k (float64): pack + K1.
 * Convenience used by the parity tests and by the host between moves. */
int spa_loglik_rows(const spa_design* d, const float* beta, int64_t m, int32_t ldb, void* A_ws, double* ylin_ws,
                    double* out_ll, void* ws, size_t ws_bytes, void* stream);

/* ---- K2: generalised-t log-prior / incremental weights -----------------
 * mode 0: out[k] = sum_j gt(beta_kj; a, c)             (model.py:78-81)
 * mode 1: out[k] = sum_j gt(beta_kj; a, c) - gt(beta_kj; a, c_prev)
 *         (smc.py:248-257 reweight increments, cancellation-free form);
 * mode 2: as mode 0 in the arithmetic of the RW proposal pack (float64
 *         products of (1 + |beta|/(a c)) per lane, one log each), so the MH
 *         ratio compares bit-identical quantities. */
int spa_prior_rows(const spa_design* d, const float* beta, int64_t m, int32_t ldb, double a, double c,
                   double c_prev, int32_t mode, double* out, void* stream);

/* Fused reweight pass (smc.py:248-257 increments + model.py:78-81 at the new
 * scale): lw[k] = sum_j gt(beta_kj; a, c) - gt(beta_kj; a, c_prev) and
 * lp[k] = sum_j gt(beta_kj; a, c), lp bit-identical to mode 2 above. */
int spa_prior_reweight(const spa_design* d, const float* beta, int64_t m, int32_t ldb, double a, double c,
                       double c_prev, double* lw, double* lp, void* stream);

/* ---- K3: log-sum-exp / ESS (smc.py:151-157, 171-174, 258-262) ----------
 * Fixed 4096-particle chunks -> per-chunk (max, sum e^(x-max), sum e^(2(x-max)))
 * of x = logw + lw; deterministic for any particle sharding. */
int spa_lse_chunk_stats(const double* logw, const double* lw, int64_t m, double* stats /*[ceil(m/4096)][3]*/,
                        void* stream);
/* Combine chunk stats in fixed order: res[0] = log sum e^x, res[1] = ESS,
 * res[2] = max.  Device pointer res[3]. */
int spa_lse_combine(const double* stats, int64_t nchunks, double* res, void* stream);
/* lw != NULL: logw <- logw + lw - res[0] and (w != NULL) w <- exp(logw)
 *             (smc.py:258-262 renormalisation);
 * lw == NULL: w <- exp(logw - res[0]), logw untouched (smc.py:151-154). */
int spa_logw_apply(double* logw, const double* lw, int64_t m, const double* res, double* w, void* stream);

/* ---- K4/K5: systematic resampling (smc.py:273-295) ----------------------
 * Bit-exact with systematic_resample_indices(w, u): sequential float64
 * cumsum, division by the last entry, cum[-1] = 1, positions u + k/N,
 * searchsorted(side='right').  anc[k] for k in [k0, k0+count) of the N slots.
 * The cumsum is np.cumsum's strictly sequential chain reproduced by a
 * parallel binade-segmented scan (csrc/resample.cu; speculative, verified,
 * sequential fallback inside the same launches).
 * ws: spa_resample_workspace_bytes(N). */
size_t spa_resample_workspace_bytes(int64_t N);
/* Test hook: cum[i] = np.cumsum(w)[i] bit for bit (smc.py:276) into the
 * device array cum (N doubles); *mode (device int32) = 0 if the parallel
 * fast path produced it, else the sequential fallback did (the value is the
 * first failed check, csrc/resample.cu chain_block). */
int spa_exact_cumsum(const double* w, int64_t N, double* cum, int32_t* mode, void* ws, size_t ws_bytes,
                     void* stream);
int spa_systematic_ancestors(const double* w, int64_t N, double u, int64_t k0, int64_t count, int64_t* anc,
                             void* ws, size_t ws_bytes, void* stream);
/* dst_rows[k] = src_rows[idx[k] - base] (float32 rows) and the per-particle
 * float64 vectors (each may be NULL). */
int spa_gather_rows(const float* src, int32_t ld_src, float* dst, int32_t ld_dst, int32_t q, const int64_t* idx,
                    int64_t base, int64_t m, const double* v0, double* v0_out, const double* v1, double* v1_out,
                    void* stream);

/* ---- device-decided resampling (no host sync inside a lambda step) -------
 * smc.py:258-263 / 397-424: the ESS test and its consequences without a
 * host round trip.  spa_step_record stores rec[t] = {log(Z_t/Z_t-1) = res[0],
 * ESS = res[1], resampled = ESS < ess_threshold, log(Z_t/Z_1)} (running sum
 * in step order) from a spa_lse_combine result; spa_resample_gated then runs
 * the bit-exact systematic resampling (spa_systematic_ancestors) and gather
 * for all N rows, commits them in place and resets logw to -log N -- every
 * kernel returning immediately when *gate (rec[t][2]) is 0.  w = normalised
 * weights, u = the step's uniform / N. */
int spa_step_record(const double* res, double* rec, int64_t t, double ess_threshold, void* stream);
/* The weight update of an unsharded device-decided lambda step in one
 * cooperative launch: spa_lse_chunk_stats(logw, lw) -> spa_lse_combine ->
 * spa_step_record(t) -> spa_logw_apply(logw, lw) -> the statistics and
 * combine of the new logw -> w = exp(logw - lse) (stats / res end as after
 * that last combine); bit-identical to those calls (reference smc.py:151-157,
 * 171-174, 248-262).  m <= spa_reweight_finish_max_particles().  stats holds
 * 6 ceil(m / 4096) doubles: the first half ends as the chunk statistics of the
 * new logw, the second half is scratch. */
int spa_reweight_finish(double* logw, const double* lw, int64_t m, double* stats, double* res, double* rec, int64_t t,
                        double ess_threshold, double* w, void* stream);
int spa_reweight_finish_max_particles(void);
int spa_resample_gated(const double* gate, const double* w, int64_t N, double u, float* beta, float* beta_alt,
                       int32_t ldb, int32_t q, double* ll, double* ll_alt, double* lp, double* lp_alt, double* logw,
                       int64_t* anc, void* ws, size_t ws_bytes, void* stream);

/* ---- sharded particles: peer memory and the exchange --------------------
 * One process per GPU; rank r owns global particles [r M, (r+1) M) (the
 * reference's partition-invariant particle blocks, smc.py:335-359).
 * spa_ipc_export: CUDA-IPC handle (64 bytes) of the allocation holding ptr
 * and ptr's byte offset in it; spa_ipc_open / spa_ipc_close map a peer's
 * allocation into this process (its base pointer).
 * spa_resample_sharded: the device-decided systematic resampling of the
 * global particle set (smc.py:273-295) for this rank's M slots -- every rank
 * scans the global normalised weights through the peer pointers w_parts[r]
 * (exact scan, bit-identical to np.cumsum on the concatenation), searches
 * its own slots and gathers the ancestor rows (beta, ll, lp) straight from
 * their owners' buffers into the *_alt buffers (P2P loads); all kernels
 * return at once when *gate == 0.  The caller fences the ranks before (all
 * weights / rows written) and after (all reads done, before the owners'
 * spa_resample_commit overwrites them).  ws: spa_resample_workspace_bytes(nparts*M).
 * spa_resample_commit: gated copy *_alt -> live buffers and logw = logw0. */
int spa_ipc_export(const void* ptr, void* handle, uint64_t* offset);
int spa_ipc_open(const void* handle, void** base);
int spa_ipc_close(void* base);
int spa_copy_async(void* dst, const void* src, size_t bytes, void* stream);
int spa_resample_sharded(const double* gate, const double* const* w_parts, int32_t nparts, int64_t M, double u,
                         int32_t rank, const float* const* beta_parts, const double* const* ll_parts,
                         const double* const* lp_parts, int32_t ldb, int32_t q, float* beta_alt, double* ll_alt,
                         double* lp_alt, int64_t* anc, void* ws, size_t ws_bytes, void* stream);
int spa_resample_commit(const double* gate, float* beta, const float* beta_alt, int32_t ldb, int32_t q, double* ll,
                        const double* ll_alt, double* lp, const double* lp_alt, double* logw, double logw0, int64_t M,
                        void* stream);

/* ---- K7/K9: Metropolis-within-Gibbs coordinate moves --------------------
 * smc.py:298-332 (_move_block) / smc.py:177-199 (mwg_sweep): `cycles` sweeps
 * of single-coordinate random-walk updates with per-particle Philox streams
 * keyed (seed, tag, t, i0+k); sweep s draws from block index s*q + j
 * (Philox counter index + 1, the NumPy convention).
 * Writes ll (log-likelihood) and lp (log-prior at c) of the final state,
 * and adds the number of accepted updates to *accepted (device u64), or,
 * with per_particle != 0, particle k's count to accepted[k]. */
/* Chains (CTAs) of spa_mwg_chain_slots (layout 1, the thinning chains)
 * resident at once on the current device for this design (occupancy x SMs);
 * init_particles sizes its parallel chains to one such wave (the
 * reference's single init chain, smc.py:202-245, is replaced by parallel
 * chains). */
int spa_mwg_resident_chains(const spa_design* d, int64_t* chains);

int spa_mwg_move(const spa_design* d, float* beta, int64_t m, int32_t ldb, double a, double c, double step_sd,
                 int32_t cycles, uint64_t seed, int32_t tag, int64_t t, int64_t i0, int64_t sweep0, double* ll,
                 double* lp, unsigned long long* accepted, int32_t per_particle, void* stream);
/* Initialisation chains in one launch: `slots` blocks of cycles_per_slot
 * sweeps (sweep indices sweep0 ..), the state after block s stored in slot
 * row*slots + s of slot_beta ([m*slots][ldb] float32), slot_ll and slot_lp;
 * beta/ll/lp end at the last slot's state.  Bit-identical to `slots` calls
 * of spa_mwg_chain_slots with slots = 1 and sweep0 advanced by
 * cycles_per_slot (one materialisation of the subject cache per slot
 * instead of two, one launch instead of `slots`).  layout 0 (burn-in):
 * the latency layout (fewer subjects per thread, more threads per chain,
 * the factor tables of a whole sweep: one long chain per SM); layout 1
 * (thinning): the throughput layout of spa_mwg_move (a resident wave of
 * chains, several per SM).  Layouts differ in float32 summation order. */
int spa_mwg_chain_slots(const spa_design* d, float* beta, int64_t m, int32_t ldb, double a, double c,
                        double step_sd, int32_t cycles_per_slot, int32_t slots, uint64_t seed, int32_t tag,
                        int64_t t, int64_t i0, int64_t sweep0, double* ll, double* lp, float* slot_beta,
                        double* slot_ll, double* slot_lp, unsigned long long* accepted, int32_t per_particle,
                        int32_t layout, void* stream);

/* Coordinates per blocked MwG round (1, 2 or 4) for spa_mwg_chain_slots
 * (init_rounds) and spa_mwg_move (move_rounds), coded designs: a round
 * evaluates the next `rounds` coordinates' log-likelihood differences
 * against the current subject cache in one block reduction and decides them
 * in order up to the first acceptance.  The chain states are bit-identical
 * for every value (the same sums, reduction order and decisions as one
 * coordinate at a time, reference smc.py:177-199); it trades reductions and
 * barriers for discarded work after an acceptance.  Defaults: 4 / 4. */
int spa_mwg_set_rounds(int32_t init_rounds, int32_t move_rounds);
/* Whether the coded MwG kernels may keep the per-coordinate factor tables of
 * a whole sweep in shared memory (when two chains per SM still fit; else they
 * are built a round ahead in a ring).  Identical states either way; default 1. */
int spa_mwg_set_tables(int32_t full_allowed);

/* ---- K8: population random-walk moves (north-star kernel) --------------
 * Weighted moments into an int64 fixed-point (2^-48) accumulator
 * partial[q + q*q] zeroed by the caller:
 *   phase 0: partial[0:q] += sum_k w_k beta_k (the weighted mean; seeds the
 *            centring point on the first call)
 *   phase 2: one pass over beta: Dt = bf16(sqrt(w_k) (beta_k - c)) into ws
 *            and partial[0:q] += sum_k w_k (beta_k - c) = mu - c, for the
 *            caller's centring point c = center[q] (float32; normally the
 *            previous population mean)
 *   phase 3: partial[q:] (lower) += Dt Dt^T = sum_k w_k (beta_k-c)(beta_k-c)^T
 *            as a split-K tcgen05 SYRK; per-split float32 tiles summed in
 *            fixed order (ws: spa_rw_moments_workspace_bytes)
 *   phase 1: 2 then 3.  The particles may be modified once phase 2 has
 *            completed.
 * Integer sums are order-independent, so the moments are bit-identical for any
 * CTA schedule or particle sharding (multi-GPU: all-reduce `partial`). */
size_t spa_rw_moments_workspace_bytes(int64_t m, int32_t q);
int spa_rw_moments(const float* beta, int64_t m, int32_t ldb, int32_t q, const double* w, const float* center,
                   int32_t phase, int64_t* partial, void* ws, size_t ws_bytes, void* stream);
/* Covariance from the phase 1 moments: S = M - delta delta^T (delta =
 * partial[0:q], M = partial[q:]) = the weighted covariance for any centring
 * point, plus trace-scaled jitter; blocked float32 Cholesky (L only
 * parameterises a symmetric proposal, so float32 suffices);
 * L = s*chol(S) as float32 [q][q] row-major lower (s = scale/sqrt(q)) and as
 * the bf16 proposal operand [q][kq] at byte offset roundup(8*q*q, 256) of ws
 * (kq = roundup(q, 64)); ws >= roundup(8*q*q, 256) + roundup(2*q*kq, 256) + 8192
 * bytes (the last 8 KB hold the 32x32 panel inverse);
 * *info = 0 or the failing column + 1.  center (optional, the point phase 2
 * used) is moved to the mean: center += delta. */
int spa_rw_factor(const int64_t* partial, int32_t q, double scale, double jitter, float* L, double* ws, int* info,
                  float* center, void* stream);
/* Proposal normals Z (bf16 [m][kq], kq = roundup(q, 64), zero padded) from
 * Philox4x32-10 keyed by seed with counter (j/8, i0+k, t, move | 3<<24): each
 * 32-bit word gives one sign-symmetric Box-Muller pair from two 15-bit
 * uniforms, 8 normals per block (csrc/spa_core.cu rw_normals8).
 * Independent of the particle state, so all moves of a step can be drawn
 * ahead, e.g. on a side stream while the covariance is factored. */
int spa_rw_normals(int64_t m, int32_t q, uint64_t seed, int64_t t, int64_t i0, int32_t move, void* zbuf,
                   void* stream);
/* prop = beta + L z for the normals in zbuf (spa_rw_normals of this move): L z
 * on tcgen05, stored as eps (bf16 [m][ldb] -- rounding keeps the increment law
 * exactly symmetric --, coalesced through an smem transpose); then one
 * vectorised pass packs prop = beta + eps into the K1 operand A and emits
 * ylin and lp at c.  `Lb` is the bf16 operand written by spa_rw_factor
 * (lower triangular with zeros above the diagonal, as that call writes it: K blocks
 * wholly above a 256-column output tile are skipped);
 * seed/t/i0/move are unused (kept for ABI stability). */
int spa_rw_propose(const spa_design* d, const float* beta, int64_t m, int32_t ldb, const void* Lb, uint64_t seed,
                   int64_t t, int64_t i0, int32_t move, void* zbuf, void* eps, void* A, double* ylin, double a,
                   double c, double* lp, void* stream);
/* The two halves of spa_rw_propose.  spa_rw_increments: eps = L z for m rows
 * (the tcgen05 GEMM; zbuf bf16 [m][roundup(q,64)], eps bf16 [m][ldb], q
 * columns written) -- the increments do not depend on beta, so the sampler
 * computes all moves of a lambda step in one call (m = moves x N) beside the
 * step's reweighting.  spa_rw_pack: prop = beta + eps packed into the K1
 * operand, ylin and the log-prior at c, as spa_rw_propose. */
int spa_rw_increments(int64_t m, int32_t q, int32_t ldb, const void* Lb, const void* zbuf, void* eps,
                      void* stream);
int spa_rw_pack(const spa_design* d, const float* beta, int64_t m, int32_t ldb, const void* eps, void* A,
                double* ylin, double a, double c, double* lp, void* stream);
/* Metropolis accept: d = (ylin' - sp' + lp') - (ll + lp); u (53 bits) from
 * Philox4x32 counter (0xFFFFFFFF, i0+k, t, move | 3<<24); on accept beta <- beta + eps (the
 * proposal) and ll, lp are updated; adds the accepted count to *accepted. */
int spa_rw_accept(float* beta, int32_t ldb, const void* eps, int32_t q, int64_t m, const double* ylin_p,
                  const double* sp_p, const double* lp_p, double* ll, double* lp, uint64_t seed, int64_t t,
                  int64_t i0, int32_t move, unsigned long long* accepted, void* stream);
/* Integer-coded designs: K1 without its row reduction (spa_loglik_partials
 * leaves the partial row sums in ws), and the accept that reduces them itself
 * (spa_rw_accept_k1: sp = the same fixed-order sum spa_loglik_softplus forms,
 * so the decisions and states are bit-identical to spa_loglik_softplus +
 * spa_rw_accept, one launch fewer per move).  ws and A as passed to
 * spa_loglik_partials for the same design and m. */
int spa_loglik_partials(const spa_design* d, const void* A, int64_t m, void* ws, size_t ws_bytes, void* stream);
int spa_rw_accept_k1(float* beta, int32_t ldb, const void* eps, int32_t q, int64_t m, const spa_design* d,
                     const void* A, const double* ylin_p, const void* ws, const double* lp_p, double* ll, double* lp,
                     uint64_t seed, int64_t t, int64_t i0, int32_t move, unsigned long long* accepted, void* stream);

/* ---- f1: per-step weighted marginal summaries (summary.py:36-61) --------
 * Weighted mean, weighted quantiles at nlev <= 4 levels ("smallest value whose
 * cumulative weight reaches q", summary.py:36-45) and concentration
 * V(delta) = mass outside (-delta, delta) for ndelta <= 4 deltas, per
 * coordinate of beta [m][ldb] (q columns) with normalised weights w [m].
 * All sums are exact integers (weights as 2^-62 fixed point), so the
 * accumulators of shards may be added (all-reduce) between the calls:
 *   pass 0..3: spa_summary_pass (pass 0 zero-initialised hist [1][q][256],
 *              acc_mean [q], acc_in [ndelta][q], total [1]; pass p > 0 a
 *              zeroed hist [nlev][q][256]), then spa_summary_select;
 *   then spa_summary_finish -> out_mean [q], out_quant [nlev][q],
 *   out_conc [ndelta][q] (float64). */
int spa_summary_pass(const float* beta, int64_t m, int32_t ldb, int32_t q, const double* w, int32_t nlev,
                     const double* levels, int32_t ndelta, const double* deltas, int32_t pass, const uint32_t* prefix,
                     unsigned long long* hist, unsigned long long* acc_mean, unsigned long long* acc_in,
                     unsigned long long* total, void* stream);
int spa_summary_select(const unsigned long long* hist, int32_t q, int32_t nlev, const double* levels, int32_t pass,
                       const unsigned long long* total, uint32_t* prefix, unsigned long long* below, void* stream);
int spa_summary_finish(int32_t q, int32_t nlev, int32_t ndelta, const uint32_t* prefix,
                       const unsigned long long* acc_mean, const unsigned long long* acc_in,
                       const unsigned long long* total, double* out_mean, double* out_quant, double* out_conc,
                       void* stream);

/* ---- f2: run-directory writer fast path (host, smc.py:532-549) -----------
 * Rows "i,weight,p_0,...,p_{q-1}\n" for i = index0 .. index0+n-1 with every
 * value as f"{v:.17g}" (byte-identical to the reference writer), formatted
 * on `threads` host threads into buf (cap bytes; *used = bytes written, or
 * needed when the status is the workspace-too-small code).  particles is
 * float64 [n][q] row-major.  Needs no GPU. */
int spa_format_particle_rows(const double* weights, const double* particles, int64_t n, int32_t q, int64_t index0,
                             char* buf, size_t cap, size_t* used, int32_t threads);

/* ---- f3: batched EM MAP (emmap.py:117-165; summary.py:173-211) ----------
 * `problems` independent local-mode searches, problem k from seeds[k][q]
 * (float64) under GtPrior(a[k], c[k]): EM with adaptive L1 weights
 * (emmap.py:48-56) around weighted-L1 logistic solves by cyclic coordinate
 * descent with curvature curv[j] = 0.25 sum_i x_ij^2 (emmap.py:69-108), all
 * float64.  Outputs beta_out[k][q], the final log posterior, info[k] (bit 0
 * EM converged, bit 1 every inner solve converged) and the EM iteration
 * count.  Genotype-coded designs only. */
int spa_em_map(const spa_design* d, int32_t problems, const double* seeds, const double* a, const double* c,
               const double* curv, double tol, int32_t max_iter, double inner_tol, int32_t inner_max_sweeps,
               double* beta_out, double* log_post, int32_t* info, int32_t* iters, void* stream);

/* Load every kernel of the library on the current device now (instead of
 * lazily at first launch) -- run_sampler calls it during initialisation. */
int spa_prepare(void);

/* ---- test hook: the raw tcgen05 GEMM engine --------------------------
 * C[m][ldc] = sum_t A_t B^T for A = [A_0 | A_1] (terms_a bf16 blocks of kp
 * columns, K-major) and B [rows_b][kp] bf16; float32 C (ldc % 4 == 0, TMA
 * store epilogue).  Used by the GEMM
 * unit tests (tests/test_gpu_kernels.py::test_tc_gemm_*). */
int spa_tc_gemm_f32(const void* A, int64_t m, int32_t terms_a, const void* B, int32_t rows_b, int32_t kp, float* C,
                    int32_t ldc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPA_B200_H_ */
