/*
 * wc4dvar_gpu.h -- C-ABI of the B200 (sm_100a) randomized-LMP hot path.
 *
 * Drop-in boundary for the reference's operator / sketch / LMP / PCG API
 * (/root/reference/proj, C++20 + Eigen 3).  Every entry point names the
 * reference interface it replaces (file:line relative to /root/reference/).
 * INTEGRATION.md shows the C++ adapter a maintainer would add on the
 * reference side (a `GpuHessianOperator : wc4dvar::LinearOperator`).
 *
 * Conventions
 *  - All matrices are column-major fp64 with an explicit leading dimension,
 *    exactly Eigen's default MatrixXd layout (types.hpp:9-11).
 *  - Functions without a `_dev` suffix take HOST pointers and copy through
 *    pinned staging buffers; `_dev` variants take device pointers on the
 *    operator's device and a cudaStream_t passed as `void*` (NULL = the
 *    handle's own stream).
 *  - Every function returns a status code; on failure the thread-local
 *    message is in wc4dvar_gpu_last_error().  Codes mirror the reference's
 *    exception types (types.hpp:14-30):
 *        1 std::invalid_argument (require), 2 NumericalError,
 *        3 device failure (no reference equivalent), 4 DenseCapError.
 *  - Handles are thread-safe: calls on one handle are serialised internally
 *    (the reference's apply/apply_block are const and reentrant,
 *    operators.hpp:30 / SPEC.md:271).
 *  - Apply accounting follows LinearOperator::count (operators.hpp:32-39):
 *    +1 per vector apply, +m per block apply of m columns.
 */
#ifndef WC4DVAR_GPU_H
#define WC4DVAR_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    WC4DVAR_OK = 0,
    WC4DVAR_INVALID_ARGUMENT = 1,
    WC4DVAR_NUMERICAL = 2,
    WC4DVAR_DEVICE = 3,
    WC4DVAR_DENSE_CAP = 4
};

/* Thread-local message of the last failing call on this thread. */
const char* wc4dvar_gpu_last_error(void);
/* Library version string and the compiled device architecture ("sm_100a"). */
const char* wc4dvar_gpu_version(void);

/* Number of kernel launches this library has issued (bench.py's gpu_launches). */
int64_t wc4dvar_gpu_launch_count(void);

/* ------------------------------------------------------------------------- */
/* Operator descriptors                                                       */
/* ------------------------------------------------------------------------- */

/* LinearizedModel kinds (operators.hpp:57-111).  ADVDIFF and substeps > 1 are
 * the BASELINE.json extensions. */
enum {
    WC4DVAR_MODEL_IDENTITY = 0,  /* IdentityLinearized, operators.hpp:100-111 */
    WC4DVAR_MODEL_ADVECTION = 1, /* AdvectionLinearized, operators.cpp:31-42 */
    WC4DVAR_MODEL_ADVDIFF = 2,   /* upwind advection + centred diffusion */
    WC4DVAR_MODEL_LORENZ96 = 3   /* Lorenz96Linearized, operators.cpp:44-59 */
};

typedef struct {
    int32_t kind;        /* WC4DVAR_MODEL_* */
    int32_t N;           /* window intervals (ModelGrid::N, operators.hpp:125) */
    int64_t n;           /* grid points (ModelGrid::n) */
    int32_t substeps;    /* TL steps per interval; 1 = reference */
    int32_t reserved;
    double courant;      /* ADVECTION / ADVDIFF: c dt / dx */
    double diffusion;    /* ADVDIFF: nu dt / dx^2 */
    double dt;           /* LORENZ96 */
    /* LORENZ96: host pointer to N*substeps stage sets, each [x1|x2|x3|x4] of
     * 4n doubles (Lorenz96Stages::at, models.cpp:80-87), sub-step-major.  NULL
     * when `trajectory` is given instead. */
    const double* stages;
    /* LORENZ96 alternative (Lorenz96Linearized ctor, operators.cpp:44-51): the
     * linearisation trajectory, n x (N*substeps + 1) col-major with leading
     * dimension ld_trajectory, host memory or (trajectory_on_device = 1) device
     * memory on the operator's device; the stages are computed on the device. */
    const double* trajectory;
    int64_t ld_trajectory;
    double forcing;
    int32_t trajectory_on_device;
    int32_t reserved2;
} wc4dvar_model_desc;

/* ObservationNetwork (models.hpp:45-56): observed times ascending, observed
 * points ascending; q = n_times * n_points. */
typedef struct {
    int64_t n;
    int32_t N;
    int32_t n_times;
    const int32_t* times;
    int32_t n_points;
    int32_t reserved;
    const int32_t* points;
} wc4dvar_network_desc;

enum {
    WC4DVAR_COV_DENSE = 0,    /* CovarianceFactor{half, half_inv}, covariance.hpp:31-38 */
    WC4DVAR_COV_CIRCULANT = 1 /* EXTENSION: first columns of C^{1/2}, C^{-1/2} */
};

typedef struct {
    int32_t kind;           /* WC4DVAR_COV_* */
    int32_t reserved;
    const double* half;     /* DENSE: n x n (symmetric); CIRCULANT: n */
    const double* half_inv; /* same shape; may be NULL if D^{-1/2} is never used */
} wc4dvar_cov_desc;

typedef struct wc4dvar_op wc4dvar_op;

/* HessianOperator ctor, operators.hpp:119-123 / operators.cpp:64-77:
 * A = I + D^{1/2} L^{-T} H^T R^{-1} H L^{-1} D^{1/2}, R = sigma_obs^2 I. */
int wc4dvar_gpu_hessian_create(const wc4dvar_model_desc* model,
                               const wc4dvar_network_desc* net,
                               const wc4dvar_cov_desc* background_half,
                               const wc4dvar_cov_desc* model_error_half,
                               double sigma_obs, int device, wc4dvar_op** out);

/* DenseOperator, operators.hpp:42-53 (test/desk-scale operator). */
int wc4dvar_gpu_dense_create(int64_t n, const double* A, int64_t lda, int device,
                             wc4dvar_op** out);

int wc4dvar_gpu_op_destroy(wc4dvar_op* op);
int64_t wc4dvar_gpu_op_dim(const wc4dvar_op* op);
/* LinearOperator::apply_count / reset_apply_count, operators.hpp:32-33. */
int64_t wc4dvar_gpu_op_apply_count(const wc4dvar_op* op);
void wc4dvar_gpu_op_reset_apply_count(wc4dvar_op* op);
int wc4dvar_gpu_op_device(const wc4dvar_op* op);

/* Frees the operator's grow-only device workspaces (block-apply, sketch and PCG buffers);
 * they re-grow on the next call.  Lets a caller bound peak HBM between the sketch (two
 * n x (k+l) blocks) and the solve (SURVEY §7 hard part 7). */
int wc4dvar_gpu_op_release_workspaces(wc4dvar_op* op);

/* LinearOperator::apply (operators.hpp:23) and apply_block (operators.hpp:30,
 * operators.cpp:9-19).  Column-major V (dim x m, ldv), out (dim x m, ldo). */
int wc4dvar_gpu_op_apply(wc4dvar_op* op, const double* in, double* out);
int wc4dvar_gpu_op_apply_block(wc4dvar_op* op, const double* V, int64_t ldv, int64_t m,
                               double* out, int64_t ldo);
int wc4dvar_gpu_op_apply_block_dev(wc4dvar_op* op, const double* V, int64_t ldv, int64_t m,
                                   double* out, int64_t ldo, void* stream);

/* HessianOperator pieces (operators.hpp:127-135), block forms (m columns):
 * which = 0 apply_Linv (operators.cpp:79-89), 1 apply_LinvT (:91-101),
 *         2 apply_D_half (:103-113), 3 apply_D_half_inv (:115-125).
 * These do not count as operator applies, as in the reference. */
enum { WC4DVAR_LINV = 0, WC4DVAR_LINVT = 1, WC4DVAR_D_HALF = 2, WC4DVAR_D_HALF_INV = 3,
       /* the middle of HessianOperator::apply (operators.cpp:132-141):
        * L^{-T} H^T R^{-1} H L^{-1} v, no D^{1/2} (row-sharded apply, distributed.py) */
       WC4DVAR_SWEEPS = 4 };
int wc4dvar_gpu_hessian_piece(wc4dvar_op* op, int which, const double* V, int64_t ldv,
                              int64_t m, double* out, int64_t ldo);
int wc4dvar_gpu_hessian_piece_dev(wc4dvar_op* op, int which, const double* V, int64_t ldv,
                                  int64_t m, double* out, int64_t ldo, void* stream);

/* Stage profiling of HessianOperator block applies (CUDA events around the
 * D^{1/2} GEMM, the fused sweep and the final D^{1/2} GEMM + identity term).
 * enable != 0 resets the accumulators; read returns ms[3] summed over calls. */
/* observe (models.cpp:184-192) with the operator's network: y (q, network order) =
 * H traj for a window trajectory traj (n(N+1), i.e. n x (N+1) col-major).  Host / device. */
int wc4dvar_gpu_observe(wc4dvar_op* op, const double* traj, double* y);
int wc4dvar_gpu_observe_dev(wc4dvar_op* op, const double* traj, double* y, void* stream);

/* HessianOperator::observation_range (operators.cpp:146-154): W (dim x q, ldw) =
 * D^{1/2} L^{-T} H^T [e_1 .. e_q], computed as one block adjoint sweep of the q
 * unit observations.  Host / device (_dev, on `stream`) outputs. */
int wc4dvar_gpu_observation_range(wc4dvar_op* op, double* W, int64_t ldw);
int wc4dvar_gpu_observation_range_dev(wc4dvar_op* op, double* W, int64_t ldw, void* stream);

/* clustered_spectrum (spectrum.cpp:31-64) of the (LMP-preconditioned) Hessian:
 * the q + k eigenvalues of C^T A C on span([W | U]) in decreasing order
 * (*n_nonunit = q + k, nonunit holds them) and the multiplicity dim - (q + k) of
 * the eigenvalue 1 elsewhere.  precond NULL = no preconditioner; obs_range NULL =
 * computed (observation_range).  Counts q + k operator applies. */
int wc4dvar_gpu_clustered_spectrum(wc4dvar_op* op, const struct wc4dvar_lmp* precond,
                                   const double* obs_range, int64_t ldw, double* nonunit,
                                   int64_t* n_nonunit, int64_t* unit_multiplicity);

/* One covariance factor of the operator (which = 0: B^{1/2}, 1: Q^{1/2}; inv != 0: the
 * inverse factor; CovarianceFactor::half / half_inv, covariance.hpp:31-38) applied to c
 * n-vectors X (n x c, ldx) -> out (n x c, ldo), device pointers on `stream`: the local step
 * of the block-sharded D^{1/2} in the row-sharded Hessian apply. */
int wc4dvar_gpu_factor_apply_dev(wc4dvar_op* op, int which, int inv, const double* X, int64_t ldx,
                                 int64_t c, double* out, int64_t ldo, void* stream);

/* Fourier-space form of HessianOperator::apply (operators.cpp:127-144), an execution
 * strategy with the same result to rounding: for a periodic constant-coefficient TL model
 * (advection / advection-diffusion, models.cpp:27-45), circulant covariance factors and the
 * regular network of ObservationNetwork::build (models.cpp:159-176) every factor of A but the
 * observation mask is diagonal in the DFT basis, so the block apply runs as one forward
 * transform, the window recurrences per frequency class and one inverse transform.
 * mode = 1 / 0 switches it on / off for this operator (on is refused with status 1 when the
 * operator is not eligible), mode < 0 only queries; *active (optional) receives the state.
 * Eligible operators start with it on unless WC4DVAR_SPECTRAL=0. */
int wc4dvar_gpu_op_spectral(wc4dvar_op* op, int mode, int* active);

int wc4dvar_gpu_op_profile(wc4dvar_op* op, int enable);
int wc4dvar_gpu_op_profile_read(wc4dvar_op* op, double* ms3, int64_t* calls);

/* Diagnostics: sustained fp64 tensor-core (DMMA) throughput of this device in
 * TFLOP/s, measured with an all-SM mma.sync.f64 loop (the roofline denominator
 * for the D^{1/2} GEMM; MEASURED_PEAKS.json carries bf16 only). */
int wc4dvar_gpu_probe_dmma_peak(int device, double* tflops);

/* ------------------------------------------------------------------------- */
/* Gaussian sketch matrix (randevd.cpp:16-21; NormalStream random.hpp:14-42)  */
/* ------------------------------------------------------------------------- */
/* Bit-exact with the reference stream (mt19937_64 + Box-Muller on glibc libm),
 * column-major fill.  Host output. */
int wc4dvar_gpu_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* Device NormalStream with MT19937-64 jump-ahead (random.hpp:14-42; randevd.cpp:16-21;
 * SURVEY §7 hard part 3).  out (rows x cols, ldo; device memory on `device`) = rows
 * [row0, row0 + rows) x columns [col0, col0 + cols) of gaussian_matrix(n_total, *, seed),
 * i.e. entry (i, j) is normal number n_total j + i of NormalStream(seed): column shards
 * (multi-GPU A*Omega) and row shards (row-sharded ritzit) of the reference's single serial
 * stream.  Raw engine outputs are bit-exact with libstdc++ std::mt19937_64; the normals
 * use the device log / cos / sqrt (within a few ulp of glibc's).  Enqueued on `stream`. */
int wc4dvar_gpu_gaussian_block_dev(int64_t n_total, int64_t row0, int64_t rows, int64_t col0,
                                   int64_t cols, uint64_t seed, double* out, int64_t ldo,
                                   int device, void* stream);
/* Test hook: `count` raw std::mt19937_64(seed) outputs starting at draw `offset` (both even),
 * generated on the device from a jump-ahead state (device pointer `out`). */
int wc4dvar_gpu_mt19937_raw_dev(uint64_t seed, uint64_t offset, int64_t count, uint64_t* out,
                                int device, void* stream);
/* Host twin of the jump-ahead (same polynomial arithmetic), for the CPU test suite. */
int wc4dvar_gpu_mt19937_raw_host(uint64_t seed, uint64_t offset, int64_t count, uint64_t* out);

/* ------------------------------------------------------------------------- */
/* Lorenz-96 nonlinear model on the device                   */
/* ------------------------------------------------------------------------- */
/* lorenz96_step (models.cpp:72-78, RK4 of lorenz96_rhs models.cpp:59-70)
 * applied `spinup` times to x0 (n), then the next `steps` states: traj is
 * n x (steps + 1) col-major (ld >= n), column 0 the spun-up state.  Bitwise
 * equal to the reference's (non-FMA) arithmetic.  Host pointers. */
int wc4dvar_gpu_l96_trajectory(int64_t n, double forcing, double dt, const double* x0,
                               int64_t spinup, int64_t steps, double* traj, int64_t ldt,
                               int device);
/* Same with device pointers, enqueued on `stream`. */
int wc4dvar_gpu_l96_trajectory_dev(int64_t n, double forcing, double dt, const double* x0,
                                   int64_t spinup, int64_t steps, double* traj, int64_t ldt,
                                   int device, void* stream);
/* AssimilationSystem::integrate_p (assimilation.cpp:21-33) for Lorenz-96 with
 * `substeps` RK4 steps per window interval (1 = reference): p is the window
 * control vector n(N+1); traj n x (N substeps + 1) holds every sub-step state,
 * x_0 = p_0 and the end of interval i gets + p_i.  A non-finite interval end
 * is NumericalError "integrate_p: non-finite trajectory at step i". */
int wc4dvar_gpu_l96_integrate_p(int64_t n, int32_t N, int32_t substeps, double forcing,
                                double dt, const double* p, double* traj, int64_t ldt,
                                int device);

/* ------------------------------------------------------------------------- */
/* Randomized eigenpairs (randevd.hpp:24-41)                                  */
/* ------------------------------------------------------------------------- */
enum { WC4DVAR_SKETCH_REVD = 0, WC4DVAR_SKETCH_NYSTROM = 1, WC4DVAR_SKETCH_RITZIT = 2 };

/* SketchConfig, randevd.hpp:13-21; p_iter is the ritzit EXTENSION (1 = reference). */
typedef struct {
    int32_t target_rank; /* k */
    int32_t oversample;  /* l */
    uint64_t seed;
    int32_t method;      /* WC4DVAR_SKETCH_* */
    int32_t p_iter;
} wc4dvar_sketch_config;

/* sketch_eigenpairs (randevd.cpp:138-148).  omega: dim x (k+l) host matrix, or
 * NULL to draw gaussian_matrix(dim, k+l, seed).  Outputs U (dim x k_out, ldu)
 * and theta (k_out), decreasing; *k_out <= k (Nystrom caps at the rank). */
int wc4dvar_gpu_sketch(wc4dvar_op* op, const wc4dvar_sketch_config* cfg, const double* omega,
                       double* U, int64_t ldu, double* theta, int64_t* k_out);
int wc4dvar_gpu_sketch_dev(wc4dvar_op* op, const wc4dvar_sketch_config* cfg,
                           const double* omega_dev, double* U_dev, int64_t ldu,
                           double* theta_dev, int64_t* k_out, void* stream);

/* rayleigh_ritz (randevd.cpp:47-60): Z dim x m orthonormal -> all m pairs. */
int wc4dvar_gpu_rayleigh_ritz(wc4dvar_op* op, const double* Z, int64_t ldz, int64_t m,
                              double* U, int64_t ldu, double* theta);

/* Per-stage device timings of the last sketch on this thread (ms):
 * [0] block applies, [1] orthonormalisation, [2] small factorizations,
 * [3] tall GEMMs, [4] total.  Used by bench.py. */
int wc4dvar_gpu_last_sketch_timing(double* ms5);

/* ------------------------------------------------------------------------- */
/* Row-sharded building blocks (multi-GPU sketches)          */
/* ------------------------------------------------------------------------- */
/* The local halves of the dense steps of randevd.cpp for a ROW shard of the
 * tall matrices; the caller all-reduces each m x m result across ranks
 * (paper_2101_07249_b200/distributed.py) and runs the replicated small steps
 * on every rank.  Same kernels as wc4dvar_gpu_sketch, so world size 1
 * reproduces it.  Device pointers on `device`; stream as void* (NULL = the
 * legacy default stream).  Sizes of the small factorizations: 1 <= m <= 512. */
/* G (m1 x m2, ldg) = A^T B for A rows x m1, B rows x m2: the local Gram of
 * householder_q / ColPivHouseholderQR (randevd.cpp:27-30,67), K = Z^T A Z
 * (randevd.cpp:54) and Z^T E1 (randevd.cpp:95); fixed-order reduction. */
int wc4dvar_gpu_la_gram_dev(int device, int64_t rows, int64_t m1, int64_t m2, const double* A,
                            int64_t lda, const double* B, int64_t ldb, double* G, int64_t ldg,
                            void* stream);
/* C (rows x ncols) = A (rows x k) W (k x ncols): U = Z W (randevd.cpp:57,133),
 * Y R^{-1} and F = E1 U^{-1} (randevd.cpp:105) with R^{-1} from tri_inv_upper.
 * C must not alias A. */
int wc4dvar_gpu_la_tall_times_small_dev(int device, int64_t rows, int64_t k, int64_t ncols,
                                        const double* A, int64_t lda, const double* W,
                                        int64_t ldw, double* C, int64_t ldc, void* stream);
/* R = upper Cholesky factor of sym(G) (Eigen::LLT, randevd.cpp:96-102); status 2
 * (NumericalError) when G is not positive definite. */
int wc4dvar_gpu_la_chol_upper_dev(int device, int64_t m, const double* G, double* R, void* stream);
/* R = chol_upper(G) and Rinv = R^{-1} in one call (the CholQR step of
 * householder_q, randevd.cpp:27-30, and the LLT + triangular solve of
 * randevd.cpp:97-105); status 2 as chol_upper.  R may alias G. */
int wc4dvar_gpu_la_chol_inv_upper_dev(int device, int64_t m, const double* G, double* R,
                                      double* Rinv, void* stream);
/* Rinv = R^{-1} for upper-triangular R (triangular solve, randevd.cpp:105). */
int wc4dvar_gpu_la_tri_inv_upper_dev(int device, int64_t m, const double* R, double* Rinv,
                                     void* stream);
/* Rank probe of ColPivHouseholderQR (randevd.cpp:67-73,89-92) as a diagonally
 * pivoted Cholesky of the (all-reduced) Gram G: *rank (host) = pivots above
 * tol_rel * max diag, perm (device, m int32) = pivot order. */
int wc4dvar_gpu_la_pivoted_rank_dev(int device, int64_t m, const double* G, double tol_rel,
                                    int64_t* rank, int32_t* perm, void* stream);
/* sorted_symmetric_evd (randevd.cpp:37-43): values decreasing, W (m x m). */
int wc4dvar_gpu_la_sym_evd_dev(int device, int64_t m, const double* K, double* vals, double* W,
                               void* stream);
/* Left singular vectors and values of a square X (BDCSVD thin U, randevd.cpp:106),
 * sigma decreasing. */
int wc4dvar_gpu_la_svd_left_dev(int device, int64_t m, const double* X, double* sigma, double* U,
                                void* stream);
/* C = alpha op(A) op(B) + beta C for small matrices (R2 R1, R3 R3^T of
 * randevd.cpp:128); op = transpose when trans_* != 0. */
int wc4dvar_gpu_la_small_gemm_dev(int device, int32_t trans_a, int32_t trans_b, int64_t M,
                                  int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                                  const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                                  void* stream);
/* out[:, j] = in[:, perm[j]], j < r: the pivoted Nystrom basis (randevd.cpp:89-92). */
int wc4dvar_gpu_la_gather_cols_dev(int device, int64_t rows, int64_t r, const double* in,
                                   int64_t ldi, const int32_t* perm, double* out, int64_t ldo,
                                   void* stream);

/* ------------------------------------------------------------------------- */
/* Spectral LMP (lmp.hpp:12-28)                                               */
/* ------------------------------------------------------------------------- */
typedef struct wc4dvar_lmp wc4dvar_lmp;

/* build_spectral_lmp (lmp.cpp:35-52): rejects theta <= 0 and an
 * orthonormality defect > 1e-8.  k = 0 gives the identity factor. */
int wc4dvar_gpu_lmp_build(int64_t n, int64_t k, const double* U, int64_t ldu,
                          const double* theta, int device, wc4dvar_lmp** out);
int wc4dvar_gpu_lmp_build_dev(int64_t n, int64_t k, const double* U_dev, int64_t ldu,
                              const double* theta_dev, int device, wc4dvar_lmp** out);
int wc4dvar_gpu_lmp_destroy(wc4dvar_lmp* lmp);
/* LmpFactor::apply (C v, lmp.cpp:8-16) / apply_transpose (C^T v, lmp.cpp:18-26). */
int wc4dvar_gpu_lmp_apply(wc4dvar_lmp* lmp, int transpose, const double* v, double* out);

/* ------------------------------------------------------------------------- */
/* Quadratic cost (assimilation.cpp:130-150) and split PCG (krylov.cpp:22-99) */
/* ------------------------------------------------------------------------- */
typedef struct wc4dvar_cost wc4dvar_cost;
/* QuadraticCost(op, b, d): stores b~ = D^{-1/2} b and d (q). */
int wc4dvar_gpu_cost_create(wc4dvar_op* hessian, const double* b, const double* d,
                            wc4dvar_cost** out);
int wc4dvar_gpu_cost_destroy(wc4dvar_cost* cost);
int wc4dvar_gpu_cost_eval(wc4dvar_cost* cost, const double* x, double* value);
int wc4dvar_gpu_cost_rhs(wc4dvar_cost* cost, double* rhs);

/* PcgOptions (krylov.hpp:32-38). */
typedef struct {
    int32_t max_iter;
    int32_t reorthogonalize;
    double rel_tol;
    int32_t store_residual_vectors; /* keep f_j = r_j / ||r_j|| (CgHistory::normalized_residuals) */
    int32_t reserved;
} wc4dvar_pcg_options;

/* CgHistory (krylov.hpp:17-30): caller-provided arrays of length max_iter + 1
 * (alphas/betas use max_iter); any pointer may be NULL. */
typedef struct {
    double* alphas;
    double* betas;
    double* residual_norms;
    double* quadratic_costs; /* filled only when a cost handle is passed */
    int32_t iterations;
    int32_t converged;
    int32_t stop_reason;     /* 0 zero initial residual, 1 tolerance, 2 max iterations */
    int32_t reserved;
    /* n x (max_iter + 1) host block (ld_residuals) for the normalised residuals, filled when
     * reorthogonalize or store_residual_vectors is set; n_residuals = columns written */
    double* normalized_residuals;
    int64_t ld_residuals;
    int32_t n_residuals;
    int32_t reserved2;
} wc4dvar_pcg_history;

/* pcg_split (krylov.cpp:22-99): precond may be NULL (identity, krylov.cpp:106-108),
 * x0 may be NULL (zero guess: no initial apply), cost may be NULL. */
int wc4dvar_gpu_pcg(wc4dvar_op* op, const double* b, wc4dvar_lmp* precond, const double* x0,
                    const wc4dvar_pcg_options* opts, wc4dvar_cost* cost, double* x,
                    wc4dvar_pcg_history* hist);

/* ------------------------------------------------------------------------- */
/* Deterministic LMP eigenpairs                              */
/* ------------------------------------------------------------------------- */
/* LanczosOptions (krylov.hpp:81-85). */
typedef struct {
    int32_t max_iter; /* 0: min(dim, 8k + 120) */
    int32_t reserved;
    double tol;       /* relative residual tolerance on each pair (1e-10) */
    uint64_t seed;    /* NormalStream seed of the start vector (0x5eed0f4d) */
} wc4dvar_lanczos_options;

/* lanczos_eigenpairs (krylov.cpp:178-278): top-k eigenpairs by matrix-free Lanczos with
 * full re-orthogonalisation, on the device.  U: dim x k host (ldu), values: k host,
 * decreasing; *steps = Krylov dimension used (may be NULL).  One apply per step. */
int wc4dvar_gpu_lanczos_eigenpairs(wc4dvar_op* op, int64_t k, const wc4dvar_lanczos_options* opts,
                                   double* U, int64_t ldu, double* values, int64_t* steps);

/* ritz_from_tridiagonal (krylov.cpp:136-176): top-k Ritz pairs from the CG-Lanczos
 * tridiagonal (gammas j, taus j-1) and the stored normalised CG residuals (n x j, ldf,
 * host); ghosts collapsed, NumericalError when the basis lost orthogonality or fewer
 * than k distinct values remain.  U: n x k host (ldu), values: k host. */
int wc4dvar_gpu_ritz_from_tridiagonal(int64_t n, int64_t j, const double* gammas, const double* taus,
                                      const double* residual_basis, int64_t ldf, int64_t k, double* U,
                                      int64_t ldu, double* values, int device);

/* ------------------------------------------------------------------------- */
/* Multi-GPU plumbing for a C++ host                    */
/* ------------------------------------------------------------------------- */
/* NCCL communicator (NCCL resolved at run time: libnccl.so.2).  Rank 0 makes the
 * 128-byte id and the caller broadcasts it out of band, as with ncclGetUniqueId. */
typedef struct wc4dvar_comm wc4dvar_comm;
int wc4dvar_gpu_comm_unique_id(unsigned char* id128);
int wc4dvar_gpu_comm_create(const unsigned char* id128, int rank, int size, int device, wc4dvar_comm** out);
int wc4dvar_gpu_comm_destroy(wc4dvar_comm* comm);
/* In-place sum of the m x m Gram-type partials (Y^T Y, Z^T A Z, Z^T E1, U^T v, ...). */
int wc4dvar_gpu_comm_allreduce_sum(wc4dvar_comm* comm, double* buf, int64_t count, void* stream);
int wc4dvar_gpu_comm_allgather(wc4dvar_comm* comm, const double* send, int64_t count, double* recv,
                               void* stream);
/* The column <-> row transposes of the row-sharded sketches: an nrows x ncols block,
 * balanced partitions (part r = [total r / G, total (r+1) / G)); rank r holds columns
 * part_r(ncols) (cols: nrows x m_r, ld nrows) or rows part_r(nrows) (rows: R_r x ncols,
 * ld R_r).  Grouped NCCL send / recv on `stream`. */
int wc4dvar_gpu_comm_cols_to_rows(wc4dvar_comm* comm, const double* cols, int64_t nrows, int64_t ncols,
                                  double* rows, void* stream);
int wc4dvar_gpu_comm_rows_to_cols(wc4dvar_comm* comm, const double* rows, int64_t nrows, int64_t ncols,
                                  double* cols, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WC4DVAR_GPU_H */
