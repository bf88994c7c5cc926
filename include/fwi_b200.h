/*
 * fwi_b200.h — C ABI of the B200-native KKT/Krylov hot path of full-space
 * Gauss-Newton FWI (arXiv 2204.06489).
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes. No C++
 * or torch types cross this boundary. Every entry point below replaces one
 * reference interface (paths relative to /root/reference/proj):
 *
 *   fwi_dev_ctx_create          fwi::make_gn_state        include/fwi/reduced_space.hpp:51-54
 *                               (+ fwi::GnState           include/fwi/reduced_space.hpp:15-41)
 *   fwi_dev_vec_*               fwi::KktVector + dot/norm/axpy/scal
 *                                                         include/fwi/kkt.hpp:12-24
 *   fwi_dev_kkt_apply           fwi::kkt_apply            include/fwi/kkt.hpp:32
 *   fwi_dev_kkt_rhs             fwi::kkt_rhs              include/fwi/kkt.hpp:36
 *   fwi_dev_precond_apply       fwi::precond_apply        include/fwi/kkt.hpp:45
 *   fwi_dev_solve               LuFactors::solve / IluFactors::solve
 *                                                         include/fwi/lu.hpp:28, include/fwi/ilu.hpp:31
 *   fwi_dev_factor_ilu          IluFactors::factor        include/fwi/ilu.hpp:26
 *   fwi_dev_solve_count         LuFactors::solve_count    include/fwi/lu.hpp:37-39
 *   fwi_dev_fsgn_gmres_step     fwi::fsgn_gmres_step      include/fwi/kkt.hpp:62
 *   fwi_dev_gmres_generic       fwi::gmres<Vec,OpA,OpM>   include/fwi/krylov.hpp:128-131
 *
 * Vector layout on the host side of upload/download is the reference's
 * KktVector flattened in its own dot order (src/kkt.cpp:15-24):
 *   [ du_0 .. du_{K-1} | ds | lambda_0 .. lambda_{K-1} ]
 * where each du_k / lambda_k is n complex numbers stored (re, im) and ds is n
 * doubles: 4*K*n + n doubles in total. The device keeps exactly this layout.
 *
 * Errors: every function returns FWI_OK (0) or an FWI_ERR_* code;
 * fwi_dev_last_error() gives the message and fwi_dev_last_error_index() the
 * pivot index carried by SingularPivotError / ZeroPivotError
 * (include/fwi/lu.hpp:11-16, include/fwi/ilu.hpp:11-17). Both are thread-local.
 * Calls on one context are serialised on the context's CUDA stream.
 */
#ifndef FWI_B200_H
#define FWI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define FWI_OK 0
#define FWI_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define FWI_ERR_SINGULAR_PIVOT 2   /* fwi::SingularPivotError */
#define FWI_ERR_ZERO_PIVOT 3       /* fwi::ZeroPivotError */
#define FWI_ERR_CUDA 4             /* CUDA runtime failure (no fallback exists) */
#define FWI_ERR_NOT_SUPPORTED 5
#define FWI_ERR_OUT_OF_MEMORY 6
#define FWI_ERR_CG_BREAKDOWN 7       /* fwi::CgBreakdownError */

/* fwi::PrecondMode (include/fwi/kkt.hpp:38) */
#define FWI_PRECOND_EXACT 0
#define FWI_PRECOND_ILU 1

/* fwi::WeightMode (include/fwi/forward.hpp:11) */
#define FWI_WEIGHT_IDENTITY 0
#define FWI_WEIGHT_OFFSET 1

/* vector precision */
#define FWI_C128 0
#define FWI_C64 1

typedef struct fwi_dev_ctx fwi_dev_ctx;
typedef struct fwi_dev_vec fwi_dev_vec;

/* fwi::Grid2D + fwi::PmlProfile (include/fwi/grid.hpp:11-42). pml_sigma_max is
 * the profile amplitude, i.e. what make_pml_profile (src/grid.cpp:21-33)
 * returns, or an explicit override. */
typedef struct fwi_grid_desc {
    int nx, nz;
    double h;
    int n_pml;
    double pml_sigma_max;
    double pml_power;
} fwi_grid_desc;

/* fwi::Survey (include/fwi/forward.hpp:16-33) flattened. */
typedef struct fwi_survey_desc {
    int num_sources;
    const int* src_ix;        /* [K] */
    const int* src_iz;        /* [K] */
    const double* src_amp;    /* [K], NULL = 1.0 */
    const int* recv_offset;   /* [K+1] data offsets */
    const int* recv_ix;       /* [recv_offset[K]] */
    const int* recv_iz;       /* [recv_offset[K]] */
    int weight_mode;          /* FWI_WEIGHT_* */
} fwi_survey_desc;

/* Inputs of one Gauss-Newton linearisation point (make_gn_state,
 * src/reduced_space.cpp:40-86). */
typedef struct fwi_state_desc {
    fwi_grid_desc grid;
    fwi_survey_desc survey;
    double freq_hz;
    double epsilon;           /* > 0 */
    int drop_reg_term;
    const double* s;          /* [n] squared slowness */
    /* Background fields u_k, K*n complex (re,im), source-major. NULL: the
     * context computes them with its exact block factorisation
     * (solve_forward, src/forward.cpp:64-76). */
    const double* u;
    /* Data residual r = d_obs - d_pred, num_data complex. If NULL and d_obs is
     * given, r is formed from the context's own d_pred; if both are NULL, r = 0. */
    const double* r;
    const double* d_obs;
    int exact_factor;         /* build the exact block factorisation */
    int ilu_level;            /* < 0: no ILU factors */
    double ilu_diag_shift;
    int precision_mask;       /* bit FWI_C64: also keep a complex64 copy of u */
} fwi_state_desc;

typedef struct fwi_state_info {
    int nx, nz, n, num_sources, num_data;
    double omega, epsilon;
    int drop_reg_term;
    int has_exact, has_ilu;
    int64_t vec_doubles;      /* 4*K*n + n */
    int64_t device_bytes;     /* resident bytes held by the context */
    int64_t exact_factor_bytes; /* exact block factorisation (0: none) */
    int64_t ilu_factor_bytes;   /* ILU(p) factors incl. transposes and schedules (0: none) */
    double exact_probe_residual; /* ||b - A A^{-1} b|| / ||b|| of the post-factorisation
                                    probe (-1: not run) */
} fwi_state_info;

/* fwi::FsgnOptions (include/fwi/kkt.hpp:47-57). */
typedef struct fwi_fsgn_options {
    int mode;                 /* FWI_PRECOND_* */
    int restart;
    double tol;
    int maxit;
    int ecg_stride;           /* normal-equation metric cadence; 0 = off */
    double ecg_stop_tol;
} fwi_fsgn_options;

/* fwi::ConvergenceLog::Entry (include/fwi/krylov.hpp:17-33). */
typedef struct fwi_log_entry {
    int iteration;
    int has_precond_residual;
    int has_normal_residual;
    int pad_;
    double residual_norm;
    double precond_residual;
    double normal_residual;
    double wall_time;
} fwi_log_entry;

typedef struct fwi_convergence_log {
    fwi_log_entry* entries;   /* caller-owned, capacity entries */
    int capacity;
    int count;                /* entries written (maxit + 1 suffices) */
    int converged;
    int stagnated;
} fwi_convergence_log;

/* ---- errors ---------------------------------------------------------- */
const char* fwi_dev_last_error(void);
int fwi_dev_last_error_index(void);
const char* fwi_dev_version(void);

/* ---- context (GnState on the device) ---------------------------------- */
int fwi_dev_ctx_create(const fwi_state_desc* desc, fwi_dev_ctx** out);
int fwi_dev_ctx_destroy(fwi_dev_ctx* ctx);
int fwi_dev_ctx_info(const fwi_dev_ctx* ctx, fwi_state_info* out);
int fwi_dev_ctx_set_epsilon(fwi_dev_ctx* ctx, double epsilon);
int fwi_dev_ctx_set_drop_reg_term(fwi_dev_ctx* ctx, int drop);
int fwi_dev_ctx_synchronize(fwi_dev_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for event timing / interop. */
int fwi_dev_ctx_stream(const fwi_dev_ctx* ctx, void** stream);
/* Downloads: u (K*n complex), r and d_pred (num_data complex), and the
 * assembled operator as 5-point coefficient planes (each n complex):
 * A(i,i), A(i,i+1), A(i,i+nx). Couplings into Dirichlet columns are 0. */
int fwi_dev_ctx_get_u(const fwi_dev_ctx* ctx, double* host);
int fwi_dev_ctx_get_residual(const fwi_dev_ctx* ctx, double* host);
int fwi_dev_ctx_get_dpred(const fwi_dev_ctx* ctx, double* host);
int fwi_dev_ctx_get_stencil(const fwi_dev_ctx* ctx, double* diag, double* east, double* south);

/* ---- factorisations --------------------------------------------------- */
int fwi_dev_factor_exact(fwi_dev_ctx* ctx);
int fwi_dev_factor_ilu(fwi_dev_ctx* ctx, int level, double diag_shift);
/* Triangular-solve pairs performed per mode (one per RHS, as the reference
 * counts them), and reset. */
int64_t fwi_dev_solve_count(const fwi_dev_ctx* ctx, int mode);
void fwi_dev_reset_solve_count(fwi_dev_ctx* ctx, int mode);
/* Name of the K1 kernel the last fwi_dev_kkt_apply at this precision
 * (FWI_C128 / FWI_C64) launched ("" before the first apply): diagnostics for
 * benchmarks and profiles, no reference counterpart. */
const char* fwi_dev_kkt_kernel(const fwi_dev_ctx* ctx, int precision);
/* nrhs block solves A x = b (A^H x = b if adjoint) on host arrays of nrhs*n
 * complex, source-major. */
int fwi_dev_solve(fwi_dev_ctx* ctx, int mode, int adjoint, int nrhs, const double* b_host,
                  double* x_host);

/* ---- KKT vectors -------------------------------------------------------- */
int fwi_dev_vec_create(fwi_dev_ctx* ctx, int precision, fwi_dev_vec** out); /* zeros */
int fwi_dev_vec_destroy(fwi_dev_vec* v);
/* Precision the vector was created with (FWI_C128 / FWI_C64); -1 for NULL. */
int fwi_dev_vec_precision(const fwi_dev_vec* v);
int fwi_dev_vec_upload(fwi_dev_vec* v, const double* host_flat);   /* 4Kn+n doubles */
int fwi_dev_vec_download(const fwi_dev_vec* v, double* host_flat);
/* complex64 vectors: host side is 4Kn+n floats */
int fwi_dev_vec_upload_f32(fwi_dev_vec* v, const float* host_flat);
int fwi_dev_vec_download_f32(const fwi_dev_vec* v, float* host_flat);
int fwi_dev_vec_copy(fwi_dev_vec* dst, const fwi_dev_vec* src);
int fwi_dev_vec_zero(fwi_dev_vec* v);
int fwi_dev_vec_dot(const fwi_dev_vec* x, const fwi_dev_vec* y, double* out);
int fwi_dev_vec_norm(const fwi_dev_vec* x, double* out);
int fwi_dev_vec_axpy(double a, const fwi_dev_vec* x, fwi_dev_vec* y);
int fwi_dev_vec_scal(double a, fwi_dev_vec* x);
/* Raw device pointer of the flat buffer (for zero-copy interop). */
int fwi_dev_vec_device_ptr(const fwi_dev_vec* v, void** out);

/* ---- the hot path ------------------------------------------------------- */
int fwi_dev_kkt_apply(fwi_dev_ctx* ctx, const fwi_dev_vec* xi, fwi_dev_vec* out);
/* kkt_apply on HOST flat buffers (4Kn+n doubles each), the reference's own
 * value-in/value-out signature: source chunks stream H2D, are applied as they
 * land and stream back D2H on separate copy engines. Pinned host memory
 * (fwi_host_register) gives full PCIe rate. Bit-identical to fwi_dev_kkt_apply. */
int fwi_dev_kkt_apply_host(fwi_dev_ctx* ctx, const double* xi_host, double* out_host);
int fwi_dev_kkt_rhs(fwi_dev_ctx* ctx, fwi_dev_vec* out);
int fwi_dev_precond_apply(fwi_dev_ctx* ctx, int mode, const fwi_dev_vec* v, fwi_dev_vec* out);
/* fsgn_gmres_step: returns delta_s (n doubles) and the convergence log. */
int fwi_dev_fsgn_gmres_step(fwi_dev_ctx* ctx, const fwi_fsgn_options* opt, double* delta_s_host,
                            fwi_convergence_log* log);

/* Reduced-space gradient and Gauss-Newton Hessian action (the RSGN / E_cg
 * building blocks): g = Re(J^H W^T W r) - eps s (gradient, src/reduced_space.cpp:
 * 141-152; K adjoint exact solves) and H v = Re(J^H W^T W J v) + eps v
 * (hessian_apply, src/reduced_space.cpp:120-139; 2K exact solves). Host arrays of
 * n doubles. */
int fwi_dev_gradient(fwi_dev_ctx* ctx, double* g_host);
int fwi_dev_hessian_apply(fwi_dev_ctx* ctx, const double* v_host, double* out_host);

/* rsgn_cg_step (src/reduced_space.cpp:163-170): CG on the reduced normal
 * equations H ds = g with device Hessian actions (2K exact solves each) — the
 * RSGN comparison path of the paper's Table 1. */
int fwi_dev_rsgn_cg_step(fwi_dev_ctx* ctx, double tol, int maxit, double* delta_s_host,
                         fwi_convergence_log* log);

/* ---- Gauss-Newton step (the caller of the hot path, src/driver.cpp:65-127) --
 * Linearise at desc->s (u computed on the device, r from desc->d_obs), solve
 * the KKT system with fsgn_gmres_step, clamp s + ds to [1/v_max^2, 1/v_min^2],
 * and re-solve at the updated model for the final misfit. */
#define FWI_SOLVER_RSGN_CG 0
#define FWI_SOLVER_FSGN_EXACT 1
#define FWI_SOLVER_FSGN_ILU 2
typedef struct fwi_gn_options {
    int solver;               /* FWI_SOLVER_RSGN_CG / FWI_SOLVER_FSGN_EXACT / FWI_SOLVER_FSGN_ILU */
    int max_inner;            /* FwiConfig::max_inner */
    double inner_tol;         /* FwiConfig::inner_tol */
    int gmres_restart;
    int ilu_level;
    double ilu_diag_shift;
    double v_min, v_max;      /* clamp bounds, m/s */
    int ecg_stride;
    double ecg_stop_tol;
} fwi_gn_options;

typedef struct fwi_gn_result {
    double misfit_ini, misfit_fin, update_relnorm, wall_seconds;
    /* split of wall_seconds: linearisation (assembly, exact factorisation, forward solves,
     * ILU(p)), of which the host ILU(p) factorisation; the Krylov solve; the re-solve at the
     * updated model */
    double setup_seconds, ilu_factor_seconds, krylov_seconds, final_seconds;
} fwi_gn_result;

int fwi_dev_gn_step(const fwi_state_desc* desc, const fwi_gn_options* opt, double* s_out,
                    fwi_gn_result* result, fwi_convergence_log* log);

/* ---- generic GMRES over flat real device vectors ------------------------
 * The same restarted left-preconditioned GMRES core as fsgn_gmres_step
 * (krylov.hpp:128-269), with caller-supplied operators. Vectors are device
 * arrays of n doubles; callbacks run on the host and must leave their result
 * in `out` (device) before returning 0. */
typedef int (*fwi_op_cb)(void* user, const double* in_dev, double* out_dev);
typedef int (*fwi_observer_cb)(void* user, int iteration, const double* x_dev);
int fwi_dev_gmres_generic(int64_t n, fwi_op_cb apply, fwi_op_cb precond, fwi_observer_cb observer,
                          void* user, const double* b_dev, double* x_dev, int restart, double tol,
                          int maxit, fwi_convergence_log* log);

/* ---- raw device memory helpers (for callback-driven use from FFI hosts) -- */
int fwi_dev_malloc(void** out, int64_t bytes);
int fwi_dev_free(void* p);
int fwi_dev_memcpy_h2d(void* dst_dev, const void* src_host, int64_t bytes);
int fwi_dev_memcpy_d2h(void* dst_host, const void* src_dev, int64_t bytes);
/* Page-lock an existing host buffer (so uploads/downloads run at DMA speed). */
int fwi_host_register(void* host, int64_t bytes);
int fwi_host_unregister(void* host);
/* Allocate / free page-locked host memory (cudaHostAlloc): the fastest source and
 * destination for fwi_dev_kkt_apply_host and the vector uploads/downloads. */
int fwi_host_alloc(void** out, int64_t bytes);
int fwi_host_free(void* host);

#ifdef __cplusplus
}
#endif

#endif /* FWI_B200_H */
