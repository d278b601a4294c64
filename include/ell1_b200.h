/*
 * ell1_b200.h — C ABI of the B200 (sm_100a) l1-minimization solver library.
 *
 * Plain C: device pointers, sizes, an opaque cudaStream_t (void*), int status.
 * No torch / C++ types cross this boundary.  Every entry point names the
 * reference interface it replaces (paths relative to /root/reference/pkg/src/ell1).
 *
 * Memory conventions
 *   - Dictionaries live on the device COLUMN-MAJOR (element (i, j) at
 *     A[j * ld + i]), ld >= d, ld % 32 == 0, rows d..ld-1 zero.  Build one from
 *     a row-major float64 device copy with ell1_dict_build().
 *   - d-vectors are allocated with ld entries (padding zero); n-vectors with
 *     n (+ d for the [A, sI] extension) entries.  All solver vectors are float64.
 *   - The library never allocates: callers query workspace sizes and pass
 *     caller-owned device buffers.
 *
 * Status codes (return value of every call; solver state.status likewise)
 */
#ifndef ELL1_B200_H
#define ELL1_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ELL1_OK = 0,
  ELL1_ZERO_DATA = 1,          /* ||A^T b||_inf == 0: x = 0 is optimal (early exit) */
  ELL1_LAMBDA_NONPOS = 2,      /* resolved lambda <= 0 -> ValueError */
  ELL1_BREAKDOWN = 3,          /* NumericalBreakdownError (backtracking / line search) */
  ELL1_ILL_CONDITIONED = 4,    /* IllConditionedError */
  ELL1_NOT_PD = 5,             /* NotPositiveDefiniteError */
  ELL1_DEGENERATE = 6,         /* DegenerateSupportError */
  ELL1_RUNNING = 7,            /* step budget of this launch used up; resumable */
  ELL1_ERR_ARG = -1,           /* bad argument */
  ELL1_ERR_CUDA = -2,          /* CUDA launch / runtime error */
  ELL1_ERR_TIMEOUT = -3,       /* grid barrier timed out (kernel aborted cleanly) */
  ELL1_ERR_NOCOOP = -4         /* device cannot co-schedule the persistent grid */
};

enum { ELL1_F64 = 0, ELL1_F32 = 1 };

enum {                       /* user stopping rules (model.py:18-19) */
  ELL1_STOP_NONE = 0,
  ELL1_STOP_REL_OBJECTIVE = 1,
  ELL1_STOP_REL_ESTIMATE = 2,
  ELL1_STOP_GROUND_TRUTH = 3,
  ELL1_STOP_KKT = 4
};

/* Device dictionary view: D = A (d x n) or the implicit [A, s I] (d x (n+d))
 * of robust.ExtendedDictionary (robust.py:57-155) when ext != 0. */
typedef struct {
  const void* A;      /* column-major, ld-strided, dtype ELL1_F64 | ELL1_F32 */
  int32_t dtype;
  int32_t ext;        /* 1: append s*I columns */
  int64_t d, n, ld;
  double ext_scale;   /* s */
} ell1_dict_t;

/* Resumable solver state (device resident; the host reads it after a run). */
typedef struct {
  int32_t status;     /* ELL1_* */
  int32_t phase;      /* 0 fresh, 1 iterating, 2 finished */
  int32_t iterations;
  int32_t converged;
  int32_t hist;       /* stop-rule history length (0..2) */
  int32_t ntrace;     /* trace rows written */
  int32_t rot[10];    /* buffer rotation (internal) */
  double scal[24];    /* solver scalars (internal; documented per solver) */
} ell1_state_t;

/* Common solver controls (SolverConfig, model.py:75-105). */
typedef struct {
  double lam;          /* lambda; < 0 => default 1e-2 * ||D^T b||_inf (model.py:126-129) */
  double tol;
  int32_t max_iter;
  int32_t stop_kind;   /* ELL1_STOP_* */
  double stop_thr;
  const double* ground_truth;  /* device, n entries, or NULL */
  double gt_norm;      /* ||ground_truth||_2 (host-computed) */
} ell1_ctrl_t;

/* FISTA options (shrinkage.py:251-260). */
typedef struct {
  double L0, eta, beta;
  int32_t continuation;
  int32_t exact_L;     /* 1: L fixed to L_exact (host passes spectral_norm_sq * (1 + 1e-9)) */
  double L_exact;
  const double* x0;    /* probe mode only: the point y to backtrack from (device, n(+d)) */
  int32_t probe;       /* 1: shrinkage.backtrack_L (shrinkage.py:216-228): one backtracking
                          search from y = x0 at fixed lambda, no zero-data / lambda checks */
  int32_t _pad;
} ell1_fista_opts_t;

/* Output / scratch buffers of one solve (all device). */
typedef struct {
  void* workspace; size_t workspace_bytes;
  ell1_state_t* state;
  double* trace;       /* [max_iter + 2][4]: iteration, objective, residual_norm, support */
  double* x;           /* n(+d): current iterate (valid at any exit) */
  double* x_prev;      /* n(+d): previous iterate (observer payload) or NULL */
  double* y;           /* n(+d): extrapolated point (observer payload) or NULL */
  int32_t max_steps;   /* iterations this launch may take (<= 0: unlimited); resumable */
  int32_t blocks;      /* persistent grid size (0: one CTA per SM) */
  unsigned long long* phase_ns;  /* optional diagnostics: [blocks][16] per-phase ns (NULL: off) */
} ell1_io_t;

/* ---------------------------------------------------------------- setup */

/* Convert a row-major float64 d x n device matrix into the column-major
 * dictionary layout (dtype conversion included).  Replaces the host-side
 * np.ascontiguousarray(A, float64) (model.py:51) + upload. */
int ell1_dict_build(const double* A_rowmajor, int64_t d, int64_t n, int64_t ld,
                    int32_t dtype, void* A_out, void* stream);

/* max_j |(D^T b)_j| and ||b||_2 into out[0], out[1] (device).  Replaces the
 * np.max(np.abs(A.T @ b)) of model.py:128 / shrinkage.py:245. */
int ell1_correlation_max(const ell1_dict_t* D, const double* b, double* out,
                         void* workspace, size_t workspace_bytes, void* stream);
size_t ell1_correlation_workspace(const ell1_dict_t* D);

/* Largest eigenvalue of D^T D by power iteration on the smaller Gram side
 * (numerics.py:224-261); v0 = host-drawn default_rng(218751) start (length
 * min(d, n_cols)), extra redraws in v0 + k*min(d,n_cols) (nredraw of them).
 * out[0] = theta, out[1] = steps. */
int ell1_spectral_norm_sq(const ell1_dict_t* D, const double* v0, int32_t nredraw,
                          double tol, int32_t max_iter, double* out,
                          void* workspace, size_t workspace_bytes, void* stream);
size_t ell1_power_workspace(const ell1_dict_t* D);

/* ------------------------------------------------------- _accel kernels */

/* out = sgn(u) max(|u| - a, 0)  (_accel/_fastkernels.pyx:14-27). */
int ell1_soft_threshold(const double* u, double a, double* out, int64_t n, void* stream);
/* out = clamp(z, -1, 1)  (_accel/_fastkernels.pyx:30-43). */
int ell1_project_box_linf(const double* z, double* out, int64_t n, void* stream);
/* In-place LINPACK rank-1 update / downdate of an upper factor (row-major m x m),
 * consuming v (_accel/_fastkernels.pyx:46-78).  status (device int) receives 0
 * or failing pivot + 1 (downdate only). */
int ell1_chol_update(double* R, double* v, int64_t m, int32_t* status, void* stream);
int ell1_chol_downdate(double* R, double* v, int64_t m, int32_t* status, void* stream);

/* ------------------------------------------------ numerics / operator utilities
 * (csrc/linalg.cu).  Factors are row-major m x m
 * upper triangles R with R^T R = G. */
/* R = chol(G) upper; *status 0, or 1 when G is not positive definite
 * (numerics.chol_factor, numerics.py:75-87). */
int ell1_chol_factor(const double* G, double* R, int64_t m, int32_t* status, void* stream);
/* out = (R^T R)^{-1} rhs by two triangular solves (CholFactor.solve, numerics.py:62-65). */
int ell1_chol_solve(const double* R, const double* rhs, double* out, int64_t m, void* stream);
/* Rout ((m+1) x (m+1)) = factor of [[G, g], [g^T, diag]]; work: m doubles;
 * *status 1 when the extension is not PD (numerics.chol_append, numerics.py:115-137). */
int ell1_chol_append(const double* R, int64_t m, const double* g, double diag, double* Rout,
                     double* work, int32_t* status, void* stream);
/* out[j] = sum_i A_ij^2 (DenseDictionary.column_norms_sq, operators.py:44-45). */
int ell1_column_norms_sq(const ell1_dict_t* D, double* out, void* stream);
/* G (d x d) = A diag(w) A^T, w == NULL -> A A^T (operators.py:53-58; cuBLAS DGEMM). */
size_t ell1_gram_dd_workspace(const ell1_dict_t* D);
int ell1_gram_dd(const ell1_dict_t* D, const double* w, double* G, void* ws, size_t ws_bytes, void* stream);
/* out = a x + b y (y may be NULL) and *out = sum x_i^2 (fixed order) — the
 * vector steps of dual_y_solve (alm.py:172-189). */
int ell1_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, void* stream);
int ell1_sumsq(int64_t n, const double* x, double* out, void* stream);
/* Jacobi-preconditioned CG on a dense symmetric M (D with d == n; diag NULL ->
 * identity); out4 = {converged, iterations, residual / ||rhs||, status}
 * (numerics.pcg_solve, numerics.py:164-221; status ELL1_BREAKDOWN on
 * non-finite curvature / residual). */
size_t ell1_pcg_workspace(const ell1_dict_t* M);
int ell1_pcg_dense(const ell1_dict_t* M, const double* rhs, const double* diag, double tol,
                   int32_t max_iter, double* x, double* out4, void* ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- solvers */

/* Accelerated proximal gradient with backtracking and continuation —
 * replaces shrinkage.fista_solve (shrinkage.py:231-298). */
size_t ell1_fista_workspace(const ell1_dict_t* D, const ell1_ctrl_t* C, int32_t blocks);
int ell1_fista(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
               const ell1_fista_opts_t* O, const ell1_io_t* io, void* stream);

/* Dual ALM options (alm.py:206-230).  M = G^{-1} A (A columns, same layout and
 * dtype as the dictionary) and Ginv = G^{-1} (d x d, column-major, ld rows,
 * float64), G = A A^T (+ s^2 I for the [A, sI] extension): the row-Gram
 * factorisation of alm._gram_factor (alm.py:162-169) done once per dictionary
 * (see ell1_gram_prepare). */
typedef struct {
  double beta;
  double y_tol;        /* y-step residual certificate (alm.py:24: 1e-10; f32 storage: 1e-5) */
  int32_t y_cg_step;   /* 1: one warm-started CG step instead of the exact y solve */
  int32_t _pad;
  const void* M;
  const double* Ginv;
  double* y_out;       /* optional (observer): multiplier y, ld entries */
  double* z_out;       /* optional (observer): z, n(+d) entries */
  const double* G;     /* optional (batched): G itself, column-major d x ld, float64 — the y-step
                          certificate then uses G y (d^2 per instance) instead of A (A^T y) */
} ell1_dalm_opts_t;

/* Dual augmented Lagrangian — replaces alm.dalm_solve (alm.py:206-272)
 * (with dual_y_solve alm.py:172-189 / _y_cg_step alm.py:192-203 fused in). */
size_t ell1_dalm_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_dalm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
              const ell1_dalm_opts_t* O, const ell1_io_t* io, void* stream);

/* Primal ALM options (alm.py:115-122): mu0, rho and tau = 1.01 * ||D||^2
 * (numerics.spectral_norm_sq / ExtendedDictionary.norm_sq, computed with
 * ell1_spectral_norm_sq). */
typedef struct {
  double mu0, rho, tau;
  double* y_out;       /* optional (observer): multiplier y, ld entries */
} ell1_palm_opts_t;

/* Primal ALM with accelerated inner shrinkage — replaces alm.palm_solve
 * (alm.py:96-159) and alm._inner_shrinkage (alm.py:71-93).  io->max_steps
 * counts OUTER iterations (the observer granularity). */
size_t ell1_palm_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_palm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
              const ell1_palm_opts_t* O, const ell1_io_t* io, void* stream);

/* Iterative shrinkage over a continuation schedule — replaces
 * shrinkage.ist_solve (shrinkage.py:105-181).  stages: the schedule's lambda
 * values (ContinuationSchedule.stages(), shrinkage.py:43-58), device memory.
 * io->max_steps counts accepted steps (the observer granularity). */
size_t ell1_ist_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_ist(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C,
             const double* stages, int32_t nstages, const ell1_io_t* io, void* stream);

/* Projected gradient on the nonnegative split — replaces
 * gradient_projection.gpsr_solve (gradient_projection.py:114-192).  lam is the
 * resolved penalty (> 0); z_out (optional, 2 * n(+d)) receives [x+; x-].
 * state.rot[2]: 1 = "zero projected gradient before kkt tolerance",
 * 2 = "projection backtracking stalled" (the reference's notes). */
size_t ell1_gpsr_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_gpsr(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
              double* z_out, const ell1_io_t* io, void* stream);

/* Truncated-Newton log-barrier interior point with on-device diagonally
 * preconditioned CG — replaces gradient_projection.tnipm_solve
 * (gradient_projection.py:218-339) and numerics.pcg_solve (numerics.py:164-221).
 * pcg_max_iter <= 0: the system dimension.  u_out optional.  state.rot[0] =
 * number of Newton steps whose CG hit its cap (the reference's note). */
size_t ell1_tnipm_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_tnipm(const ell1_dict_t* D, const double* b, const ell1_ctrl_t* C, double lam,
               double pcg_tol, int32_t pcg_max_iter, double* u_out, const ell1_io_t* io,
               void* stream);

/* LASSO solution path — replaces homotopy.solve_path / homotopy_solve
 * (homotopy.py:128-261) with the active-set Cholesky upkeep of numerics
 * chol_append / chol_delete (numerics.py:115-158) on the device.
 * state.scal[0] = reached lambda; state.rot[0] = support size;
 * state.rot[1] = 1 when the "ridge-regularized gram" fallback was used. */
typedef struct {
  double* c;           /* required: final correlations A^T(b - A x), n(+d) */
  double* lam_path;    /* optional: lambda after each breakpoint (max_iter) */
  int32_t* support;    /* optional: support list in insertion order (capacity) */
  double* factor;      /* optional: upper factor, m x m row-major */
} ell1_homotopy_out_t;
int ell1_homotopy_capacity(const ell1_dict_t* D);
size_t ell1_homotopy_workspace(const ell1_dict_t* D, int32_t blocks);
int ell1_homotopy(const ell1_dict_t* D, const double* b, double target_lambda, int32_t max_iter,
                  const ell1_homotopy_out_t* out, const ell1_io_t* io, void* stream);

/* ------------------------------------------------ groups (one dictionary per solve)
 * Many independent solves, each with its OWN dictionary, b, controls and
 * buffers, in one persistent launch: teams of `team` consecutive CTAs run
 * the single-solve kernel bodies round-robin over the solves, the team size
 * chosen so each dictionary panel stays resident in shared memory.  Replaces
 * the reference experiment harness's per-trial process fan-out
 * (bench.py:_run_tasks :145-151 over _phase_task :127-136, _noise_task
 * :196-220, _corruption_task :256-279), one solve per trial.
 * All arrays are host arrays of length `count` holding device pointers. */
#define ELL1_GROUP_ARG_BYTES 1024
typedef struct {
  int32_t count;
  int32_t team;                   /* CTAs per solve; 0 = max over the solves of
                                     ell1_<solver>_group_team (workspaces must be
                                     sized with blocks = the team actually used) */
  const ell1_dict_t* dicts;
  const double* const* b;         /* ld entries each, zero padded */
  const ell1_ctrl_t* ctrl;
  const ell1_io_t* io;            /* state zeroed; max_steps 0 (no observers); blocks ignored */
  void* args_ws;                  /* device scratch, ell1_group_args_bytes(count) bytes */
  size_t args_ws_bytes;
} ell1_group_t;

enum {
  ELL1_SOLVER_CORR = 0, ELL1_SOLVER_FISTA = 1, ELL1_SOLVER_IST = 2, ELL1_SOLVER_PALM = 3,
  ELL1_SOLVER_DALM = 4, ELL1_SOLVER_GPSR = 5, ELL1_SOLVER_TNIPM = 6, ELL1_SOLVER_HOMOTOPY = 7,
  ELL1_SOLVER_POWER = 8
};
size_t ell1_group_args_bytes(int32_t count);
/* auto team size of one solve (CTAs whose shared memory holds its panel) */
int32_t ell1_group_team(int32_t solver, const ell1_dict_t* D);
/* workspace of one solve run by a team of `team` CTAs */
size_t ell1_group_workspace(int32_t solver, const ell1_dict_t* D, int32_t team);
/* max |D_i^T b_i| -> out[2i], ||b_i|| -> out[2i+1] (device); model.py:126-129 per trial */
int ell1_correlation_max_group(const ell1_group_t* G, double* out, void* stream);
/* spectral_norm_sq per dictionary (numerics.py:224-261): out[2i] = value,
 * out[2i+1] = iterations; v0[i] = start vector + nredraw redraws, stride min(d, n) */
int ell1_spectral_norm_sq_group(const ell1_group_t* G, const double* const* v0, int32_t nredraw,
                                double tol, int32_t max_iter, double* out, void* stream);
/* the solver bodies of ell1_fista / _ist / _palm / _dalm / _gpsr / _tnipm /
 * _homotopy; per-solve options / parameters are host arrays [count] (the
 * FISTA probe mode is not available in groups) */
int ell1_fista_group(const ell1_group_t* G, const ell1_fista_opts_t* O, void* stream);
int ell1_ist_group(const ell1_group_t* G, const double* const* stages, const int32_t* nstages,
                   void* stream);
int ell1_palm_group(const ell1_group_t* G, const ell1_palm_opts_t* O, void* stream);
int ell1_dalm_group(const ell1_group_t* G, const ell1_dalm_opts_t* O, void* stream);
int ell1_gpsr_group(const ell1_group_t* G, const double* lam, void* stream);
int ell1_tnipm_group(const ell1_group_t* G, const double* lam, double pcg_tol, int32_t pcg_max_iter,
                     void* stream);
int ell1_homotopy_group(const ell1_group_t* G, const double* target_lambda, int32_t max_iter,
                        const ell1_homotopy_out_t* out, void* stream);

/* ------------------------------------------------ batched (shared dictionary)
 * B instances with right-hand sides b_j (columns of an ld x B device matrix,
 * zero padded) share one dictionary; element j of the result equals the
 * single-instance solver on (D, b_j).  The library's host loop sequences
 * GEMMs over the active instances and per-instance epilogue kernels,
 * compacting converged instances out of the batch.  New entry points (the
 * reference has no batched API). */
typedef struct {
  double* x;            /* N x B, column j = x_star of instance j */
  int32_t* iterations;  /* B */
  int32_t* converged;   /* B */
  int32_t* status;      /* B: ELL1_OK / ZERO_DATA / LAMBDA_NONPOS / BREAKDOWN / ... */
  double* trace;        /* optional: [B][max_iter (+1 for ALM)][4] */
} ell1_batch_out_t;

size_t ell1_batch_fista_workspace(const ell1_dict_t* D, int32_t B);
int ell1_batch_fista(const ell1_dict_t* D, const double* Bmat, int32_t B, const ell1_ctrl_t* C,
                     const ell1_fista_opts_t* O, const ell1_batch_out_t* out, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Batched dual ALM (exact y-step; y_cg_step not supported in batch mode).
 * trace rows: [B][max_iter + 1][4] (row 0 = the initial entry). */
size_t ell1_batch_dalm_workspace(const ell1_dict_t* D, int32_t B);
int ell1_batch_dalm(const ell1_dict_t* D, const double* Bmat, int32_t B, const ell1_ctrl_t* C,
                    const ell1_dalm_opts_t* O, const ell1_batch_out_t* out, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Batched Homotopy (BASELINE config 5): the LASSO path to `target` for every
 * column of Bmat (ld x B, device, zero padded) against the shared plain
 * dictionary D (ext unsupported) — element j equals homotopy_solve on (A, b_j)
 * (homotopy.py:128-261).  out->trace (optional): B x max_iter x 4.  lam_out
 * (optional, B): the lambda reached; notes (optional, B): 1 when a
 * ridge-regularised Gram was used.  Support capacity per instance:
 * ell1_batch_homotopy_capacity (exceeding it -> ELL1_DEGENERATE). */
int ell1_batch_homotopy_capacity(const ell1_dict_t* D);
size_t ell1_batch_homotopy_workspace(const ell1_dict_t* D, int32_t B);
int ell1_batch_homotopy(const ell1_dict_t* D, const double* Bmat, int32_t B, double target, int32_t max_iter,
                        const ell1_batch_out_t* out, double* lam_out, int32_t* notes, void* ws,
                        size_t ws_bytes, void* stream);

/* SRC labels for a CAB batch (BASELINE config 3): label_j = argmin_c
 * ||b_j - e_j - A_c x_{j,c}||, classes = contiguous column ranges
 * [class_offsets[c], class_offsets[c+1]); W (ldw x B, ldw >= n + d) holds the
 * stacked solutions [x; e/s] of the [A, sI] solves; nclasses <= 64. */
int ell1_src_classify(const ell1_dict_t* D, const double* Bmat, int32_t B, const double* W,
                      int64_t ldw, const int32_t* class_offsets, int32_t nclasses, int32_t* labels,
                      double* class_resid, void* stream);

/* ----------------------------------------- column-sharded FISTA (config 4)
 * One huge instance, A = [A_0 | ... | A_{G-1}] by columns, one rank per GPU
 * (SURVEY §8(e)).  Replaces shrinkage.fista_solve (shrinkage.py:231-298) with
 * its backtracking (_backtrack :199-213), momentum (fista_t_next :184-196),
 * continuation, KKT (model.kkt_from_correlation, model.py:160-173) and stop
 * rules (model.check_stop, model.py:176-224), for a dictionary no single
 * process can hold.
 *
 * Control stays on the device.  A solve is a sequence of identical ROUNDS,
 * each one backtracking trial:
 *     ell1_sfista_pre   prox x_n = soft(y - g_y/L, lam/L) on the local columns
 *                       + the rank's scalar partials into its slot of xchg,
 *                       then xchg[0:d) = A_r x_n (skipped once finished)
 *     <allreduce(sum) of xchg: ld + 16*world doubles, the ONLY collective>
 *     ell1_sfista_post  r_n = xchg - b, the rank-ordered fold of every rank's
 *                       slots, the acceptance / stop / continuation decisions
 *                       in ctl, then (if accepted) g_n = A_r^T r_n, the
 *                       iterate rotation and the KKT partials of the new
 *                       iterate (they ride on the NEXT round's allreduce; the
 *                       trace row's support count and the KKT exit are
 *                       finalised one round late).
 * Every rank holds bit-identical ctl (same allreduced inputs, fixed-order
 * folds), so all ranks run the same number of rounds; the host only polls
 * ctl->state every few rounds.  Rounds after FINISHED are no-ops.
 * xchg layout: [0, ld) partial A x | slot r (16 doubles): 8 prox partials
 * {sum|xn|, g_y.dl, dl.dl, max|xn|, ||xn-x||^2, ||x||^2, ||xn-gt||^2, 0},
 * 8 KKT partials {max_on, max_off, any_on, any_off, count, 0, 0, 0}. */
enum { ELL1_SF_RUNNING = 0, ELL1_SF_FINAL = 1, ELL1_SF_FINISHED = 2 };
typedef struct {
  /* constants (set by the host before the first round) */
  double lam_bar, tol, stop_thr, gt_norm, eta, beta;
  int64_t max_iter;
  int32_t stop_kind, exact, world, rank;
  /* state (device-owned after begin) */
  double L, lam_k, lam_used, tp, tc, m, mn, f_y, F_prev, cut;
  int64_t it, passes, trials;
  int32_t hist, growths, state, converged, status, run_trial, adv, pending;
} ell1_shard_ctl_t;
size_t ell1_gemv_workspace(const ell1_dict_t* D);
/* y (ld) = D x (n), fixed-order reduction  (DenseDictionary.apply, operators.py:27-28) */
int ell1_gemv(const ell1_dict_t* D, const double* x, double* y, void* ws, size_t ws_bytes, void* stream);
/* g (n) = D^T r (ld)  (DenseDictionary.adjoint, operators.py:30-31) */
int ell1_gemv_t(const ell1_dict_t* D, const double* r, double* g, void* ws, size_t ws_bytes, void* stream);
/* KKT / support partials of a shard: out8 = {max_on, max_off, any_on, any_off, count, ...} */
int ell1_shard_kkt(int64_t n, const double* x, const double* g, double lam, double cut, double* out8,
                   void* ws, void* stream);
/* r_next = ax - b, out8 = {||r_next||^2, ||(1+mn) r_next - mn r_x||^2, ...} */
int ell1_shard_resid(int64_t d, const double* ax, const double* b, const double* rx, double mn, double* rn,
                     double* out8, void* ws, void* stream);
/* Vectors of one rank: V[0..5] = x, x_prev, x_next, g, g_prev, g_next (n_local
 * each), V[6..7] = r, r_next (ld each), gt (n_local or NULL), b (ld); trace
 * (max_iter x 4 doubles: it, F, ||r||, support). ws >= ell1_sfista_workspace(). */
typedef struct {
  double *x, *xp, *xn, *g, *gp, *gn, *r, *rn;
  const double* gt;
  const double* b;
  double* xchg;
  double* trace;
} ell1_sfista_bufs_t;
size_t ell1_sfista_workspace(const ell1_dict_t* D);
int ell1_sfista_pre(const ell1_dict_t* D, ell1_shard_ctl_t* ctl, const ell1_sfista_bufs_t* V, void* ws,
                    size_t ws_bytes, void* stream);
int ell1_sfista_post(const ell1_dict_t* D, ell1_shard_ctl_t* ctl, const ell1_sfista_bufs_t* V, void* ws,
                     size_t ws_bytes, void* stream);

/* ------------------------------ column-sharded Homotopy (shard_hom.cu)
 * Per-rank candidates of homotopy.py:78-105 / :229-233 for the sharded path
 * (paper_1007_3753_b200/sharded_homotopy.py); first index wins ties.
 * out2 = {max |c|, first argmax}; out4 = {gamma_a, i_a, gamma_b, i_b} over the
 * columns with mask == 0 (floor 1e-10 max(lam, 1e-30), INFINITY / -1 if none);
 * gamma_minus: {min -x/d (finite, > 0), its position; ties -> lowest keys[k]};
 * xstats: {sum |x|, count |x| > 1e-10 max(max|x|, 1)}. */
int ell1_hom_absmax(int64_t n, const double* c, double* out2, void* stream);
int ell1_hom_gammas(int64_t n, const double* c, const double* w, const unsigned char* mask, double lam,
                    double* out4, void* stream);
int ell1_hom_gamma_minus(int64_t m, const double* x, const double* d, const int64_t* keys, double* out2,
                         void* stream);
int ell1_hom_xstats(int64_t m, const double* x, double* out2, void* stream);

/* Dense Cholesky of PDIPA's weighted normal matrix (pdipa.py:43-52
 * _factor_with_jitter -> numerics.chol_factor; chol.cu): L (lower, ldl) of
 * M + jitter I (M column-major, ldm); *status (device int) = 0, or k + 1 when
 * the k-th pivot is not positive (LAPACK's potrf convention). */
int ell1_chol_factor_dense(int64_t d, const double* M, int64_t ldm, double jitter, double* L, int64_t ldl,
                           int* status, void* stream);
/* x = (L L^T)^-1 rhs (factor.solve, numerics.py:62-72); d <= 25600 */
int ell1_chol_solve_dense(int64_t d, const double* L, int64_t ldl, const double* rhs, double* x, void* stream);
/* the same for nrhs right-hand sides (columns of rhs / x, leading dimensions ldr / ldx),
 * one CTA each: the dual ALM's row-Gram inverse G^-1 (alm.py:162-169 _gram_factor) */
int ell1_chol_solve_dense_multi(int64_t d, const double* L, int64_t ldl, int64_t nrhs, const double* rhs,
                                int64_t ldr, double* x, int64_t ldx, void* stream);

/* ---------------------------------------------- PDIPA vector kernels (pdipa.cu)
 * Primal-dual interior point on the split LP min 1'v, [A, -A] v = b, v >= 0
 * (pdipa.py:97-185; split = 1: vectors of length 2n against n columns; split = 0:
 * an explicit A_ext with n columns, newton_kkt_step pdipa.py:65-94).  Scalar
 * outputs are fixed-order reductions; ws >= ell1_pd_workspace() bytes. */
size_t ell1_pd_workspace(void);
/* u = x[:n] - x[n:] (or x), out[0] = max|u| */
int ell1_pd_split(int64_t n, int32_t split, const double* x, double* u, double* out, void* ws, void* stream);
/* rp = b - Ax, rd = c - A_ext^T y - z (c NULL = ones); out4 = {|rp|^2, b.y, |rd|^2, c.x} */
int ell1_pd_resid(int64_t d, int64_t n, int32_t split, const double* Ax, const double* b, const double* y,
                  const double* Aty, const double* x, const double* z, const double* c, double* rp, double* rd,
                  double* out4, void* ws, void* stream);
/* rc = mu_hat - x z, w = x / z, wsum = w+ + w-, vd = (rc/z - w rd)+ - (...)- (pdipa.py:55-58, 150-153) */
int ell1_pd_prep(int64_t n, int32_t split, const double* x, const double* z, const double* rd, double mu_hat,
                 double* rc, double* w, double* wsum, double* vd, void* stream);
/* dz = rd - A_ext^T dy, dx = rc / z - w dz; out4 = {min_{dx<0} -x/dx, min_{dz<0} -z/dz,
 * any non-finite in dx, dz, dy, |z dx + x dz - rc|^2} (pdipa.py:35-40, 59-61, 86-92) */
int ell1_pd_direction(int64_t n, int32_t split, int64_t d, const double* Atdy, const double* dy,
                      const double* rd, const double* rc, const double* x, const double* z, const double* w,
                      double* dx, double* dz, double* out4, void* ws, void* stream);
/* out[0] = (x + ap dx) . (z + ad dz)   (pdipa.py:165-169) */
int ell1_pd_mu(int64_t N2, const double* x, const double* dx, double ap, const double* z, const double* dz,
               double ad, double* out, void* ws, void* stream);
/* x += ap dx, z += ad dz, y += ad dy   (pdipa.py:176-179) */
int ell1_pd_update(int64_t N2, int64_t d, double* x, const double* dx, double ap, double* z, const double* dz,
                   double ad, double* y, const double* dy, void* stream);
/* M[i][i] += alpha v[i] (v NULL: none), *trace = sum_i M[i][i]  (jitter, robust.py:148) */
int ell1_pd_diag(int64_t d, int64_t ldm, double* M, double alpha, const double* v, double* trace, void* stream);

/* Alignment solvers batched across images (robust.py:223-515).
 * Image j: B_j (d x m, row-major with row pitch ldb >= m — numpy's layout —
 * images b_stride apart), b_j (d, images ld_rhs apart); outputs w (count x m),
 * e (count x d).
 * d <= 2048, m <= 32, d > m.  status[j]: ELL1_OK or ELL1_NOT_PD (B_j lacks full
 * column rank -> IllConditionedError, robust.py:254-258). */
typedef struct {
  int32_t count, d, m, max_iter;
  const double* B;
  int64_t ldb, b_stride;
  const double* rhs;
  int64_t ld_rhs;
  double tol;
  double mu0, rho;      /* PALM (robust.py:487-490) */
  double lam;           /* IST / homotopy / gp: <= 0 -> 1e-2 * peak least-squares residual (robust.py:270-273, 391) */
  const double* v0;     /* IST: 4 normalised power-iteration start vectors (4 x m) */
  double* w;
  double* e;
  int32_t* status;
  int32_t* iterations;  /* optional */
  double* Bstage;       /* global staging of B when (d+1) m doubles exceed the SM's
                           shared memory: ell1_align_stage_bytes() bytes, else NULL */
} ell1_align_t;
/* bytes of global B staging a launch of this shape needs (0: B fits in shared memory) */
size_t ell1_align_stage_bytes(int32_t kind, int32_t count, int32_t d, int32_t m);
/* robust.ist_block_step (robust.py:433-445): one block soft-threshold sweep on one
 * image, B row-major d x m (ldb), m <= 32; w_next (m), e_next (d) device outputs */
int ell1_align_ist_step(int32_t d, int32_t m, const double* B, int64_t ldb, const double* b, const double* w,
                        const double* e, double lam, double alpha, double* w_next, double* e_next, void* stream);
/* test hook: 1 routes every alignment launch through the large-image variant
 * (d <= 8192, 32 rows per thread) — bit-identical to the default variant where
 * both apply; 0 restores the size-based choice */
void ell1_test_align_large_rows(int32_t on);
/* align_palm_solve per image (robust.py:470-515) */
int ell1_align_palm_batch(const ell1_align_t* A, void* stream);
/* align_ist_solve per image (robust.py:427-467) */
int ell1_align_ist_batch(const ell1_align_t* A, void* stream);
/* align_homotopy_solve per image (robust.py:374-424); lam = target weight (<= 0: 1e-2 peak residual) */
int ell1_align_homotopy_batch(const ell1_align_t* A, void* stream);
/* align_gp_solve per image (robust.py:276-371); status ELL1_ILL_CONDITIONED (reduced system not PD),
 * ELL1_BREAKDOWN (line search exhausted), ELL1_LAMBDA_NONPOS */
int ell1_align_gp_batch(const ell1_align_t* A, void* stream);

/* The batched solvers' fp32 dictionary product on its own (new; the
 * reference's equivalent is the numpy `A @ X` / `A.T @ R` of its solvers,
 * e.g. alm.py:179, 239, shrinkage.py:271-272, looped over instances):
 *   trans = 0: C (M x N) = A (M x K, column-major, lda >= M) * B (K x N, ldb)
 *   trans = 1: C (M x N) = A^T (A is K x M, column-major, lda >= K) * B
 * fp32-accurate (3xTF32 on tcgen05, per-k-block fp32 accumulation).  B, C
 * column-major; lda, ldb multiples of 4; workspace holds the split A. */
size_t ell1_gemm_f32_workspace(int32_t trans, int64_t M, int64_t K);
int ell1_gemm_f32(int32_t trans, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, void* ws, size_t wsb, void* stream);
/* fp64 product on the DMMA tensor path (dmma_gemm.cu): C (M x N, column-major,
 * ldc) = op(A) op(B), transA: A is K x M (else M x K), transB: B is N x K (else
 * K x N); not both transposed.  The batched solvers' float64 dictionary
 * products (the reference's A @ X / A.T @ R, shrinkage.py:271-272, alm.py:179-181,
 * 239-249, and pdipa.py:150-153's weighted Gram) all go through it. */
int ell1_gemm_f64(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);
/* the same with a fixed tile variant (0: 64x64, 4 stages of k16; 1: 64x64, 3 x k16
 * (default); 2: 128x64, 3 x k16; 3: 64x64, 3 x k32; 4: 128x64, 2 x k32) and K split
 * (1/2/4/8 CTAs of a cluster, -1 auto); tuning */
int ell1_gemm_f64_variant(int32_t variant, int32_t split, int32_t transA, int32_t transB, int64_t M, int64_t N,
                          int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                          int64_t ldc, void* stream);


/* library / device info */
int ell1_device_sms(int32_t device);
const char* ell1_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ELL1_B200_H */
