/*
 * dynscreen.h -- C ABI of the B200-native dynamic-screening solver
 * (libdynscreen.so, built for sm_100a).
 *
 * The reference (screenlab, pure Python/NumPy) has no FFI; its operator seams
 * are Python signatures.  Each entry point below names the reference interface
 * it replaces (file:line under /root/reference/pkg/src/screenlab/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller (e.g. torch
 *    tensors).  The library never allocates device memory: solver state lives
 *    in a caller-provided workspace sized by dscr_solver_workspace_size().
 *  - Every call takes a cudaStream_t (passed as void*), is asynchronous and
 *    never synchronises, except the ones documented as blocking.
 *  - Dictionaries are column-major with leading dimension `ldd` (elements),
 *    ldd >= n_rows, ldd % 16 == 0, rows n_rows..ldd-1 zero.  Vectors in
 *    observation space (y, theta) are fp64 of length ldd (zero padded).
 *  - Return codes map to the reference's exception types:
 *      DSCR_OK                0
 *      DSCR_EINVAL           -1   ValueError          (solvers.py:65-85, problems.py:33-45)
 *      DSCR_ENONFINITE       -2   FloatingPointError  (solvers.py:157-159, 186-187)
 *      DSCR_ERADIUS          -3   RuntimeError        (screening.py:199-205, 245-246)
 *      DSCR_ECUDA            -4   RuntimeError, text in dscr_last_error()
 *      DSCR_ENOCOMM          -5   RuntimeError (NCCL unavailable)
 *  - Thread safety: distinct solver handles may be driven concurrently from
 *    distinct host threads/streams (reference re-entrancy, tests/test_solvers.py:307-323).
 */
#ifndef DYNSCREEN_H
#define DYNSCREEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSCR_ABI_VERSION 1

#define DSCR_OK 0
#define DSCR_EINVAL -1
#define DSCR_ENONFINITE -2
#define DSCR_ERADIUS -3
#define DSCR_ECUDA -4
#define DSCR_ENOCOMM -5

/* element type of the dictionary */
#define DSCR_F64 0
#define DSCR_F32 1
#define DSCR_BF16 2

/* solvers.py:32-37 */
#define DSCR_ISTA 0
#define DSCR_FISTA 1
#define DSCR_TWIST 2
#define DSCR_SPARSA 3
#define DSCR_CP 4

/* instrument.py:12-15 */
#define DSCR_NONE 0
#define DSCR_STATIC 1
#define DSCR_DYNAMIC 2

/* screening.py:21-29 */
#define DSCR_TEST_OFF -1
#define DSCR_SAFE 0
#define DSCR_DST3 1
#define DSCR_DOME 2
#define DSCR_GSAFE 3
#define DSCR_GST3 4

/* stop reasons reported in dscr_scalars.stop */
#define DSCR_RUNNING 0
#define DSCR_STOP_RELTOL 1
#define DSCR_STOP_GAP 2
#define DSCR_STOP_MAXITER 3
#define DSCR_STOP_EMPTY 4
#define DSCR_STOP_TRIVIAL 5
#define DSCR_STOP_ERROR 6

/* per-iteration trace row (dscr_solver_buffers.trace, row-major [max_iters][DSCR_TRACE_FIELDS]) */
#define DSCR_TRACE_FIELDS 10
#define DSCR_TR_T 0
#define DSCR_TR_KEPT 1      /* surviving atoms after the iteration's reduction */
#define DSCR_TR_NNZ 2       /* nonzeros of the reduced iterate */
#define DSCR_TR_OBJ 3       /* F(x_t) = 1/2||D x - y||^2 + lam*penalty(x) (solvers.py:488) */
#define DSCR_TR_GAP 4       /* F(x_t) - 1/2||y||^2 + lam^2/2 r_SAFE,t^2 */
#define DSCR_TR_RADIUS 5    /* test radius (NaN unless dynamic) */
#define DSCR_TR_L 6         /* step constant used */
#define DSCR_TR_NS 7        /* device globaltimer ns since setup start */
#define DSCR_TR_UNITS 8     /* surviving units (atoms or groups) */
#define DSCR_TR_SUPPORT 9   /* columns streamed by the residual pass */

/* Problem description (problems.py:20-57 Problem, dictionary.py:37-117 Dictionary,
 * dictionary.py:175-216 GroupPartition).  Groups must be contiguous column
 * ranges [group_ptr[g], group_ptr[g+1]); the host permutes columns to get there. */
typedef struct dscr_problem_desc {
    int32_t dtype;
    int32_t n_rows;
    int32_t n_cols;          /* columns held by this rank */
    int32_t ldd;
    const void* D;
    const double* y;
    double lam;
    int32_t n_groups;        /* 0: Lasso */
    int32_t norm_aware;      /* 1: columns not unit-norm (fp32/bf16 storage): the SAFE/DST3 tests use
                                ||a_i|| and the DST3 normal is the extremal atom over its norm
                                (reduces to the reference at unit norms) */
    const int32_t* group_ptr;   /* n_groups+1 (device) */
    const double* group_w;      /* n_groups (device) */
    const double* group_snorm;  /* n_groups (device), ||D_g||_2 */
    int32_t col_offset;      /* global index of local column 0 (sharding) */
    int32_t n_cols_total;
    int32_t group_offset;
    int32_t n_groups_total;
    const double* col_norms;    /* n_cols (device), ||d_j||_2 of the stored columns for the norm-aware
                                   tests, e.g. cached per dictionary from dscr_column_norms; null: the
                                   solver's setup computes them (a full pass over D per solve) */
} dscr_problem_desc;

/* SolverConfig (solvers.py:44-63) plus the BASELINE duality-gap stop. */
typedef struct dscr_config {
    int32_t algorithm;
    int32_t strategy;
    int32_t test;
    int32_t max_iters;
    double rel_tol;
    double gap_tol;          /* <= 0: off */
    double L0;
    double backtrack_factor;
    double twist_alpha;
    double twist_beta;
    double twist_step;       /* <= 0: 1/op_norm^2 */
    double cp_gamma;
    double cp_step_safety;
    double bb_L_min;
    double bb_L_max;
    double op_norm;          /* ||D||_2, required by CP and TwIST */
} dscr_config;

/* Device-resident scalar state; mirrors SolverState (solvers.py:89-102) and the
 * run-loop bookkeeping (solvers.py:431-501). */
typedef struct dscr_scalars {
    int32_t t, run_limit, max_iters, mode;
    int32_t stop, status, parity, xi;
    int32_t moved, have_fprev, n_units, n_units_new;
    int32_t n_support, p_eff, kept_atoms, nnz;
    int32_t dropped_nz, nonfinite, trivial, lmax_index;
    int32_t lmax_unit, any_group, static_done, trips;
    double L, l_acc, l_new, beta;
    double tau, sigma, phi, sigma_new;
    double theta_sq, theta_y, yy, lmax;
    double lmax_sign, shift_sq, corr_inf, mu;
    double rsafe_sq, radius, dome_rs, dome_cut;
    double dome_slope, dome_flat, maj_cs, maj_ss;
    double pen, ss_red, f_prev, F;
    double gap, t0_ns, gst3_coef, gst3_nsq;
    double ds_sq, fc, tw_step, spare;
    double astar_nsq, gstar_w;   /* ||a_*||^2 (norm-aware DST3); weight of the extremal group (GST3) */
    double oc_empty, oc_spare;   /* one-collective sharding: every unit screened this trip (global); spare */
} dscr_scalars;

/* Device pointers into a solver's workspace (valid while the handle lives). */
typedef struct dscr_solver_buffers {
    dscr_scalars* scalars;
    double* theta[2];        /* theta[parity] = current dual candidate */
    double* resid;           /* D x - y of the current iterate */
    double* corr;            /* D_A^T theta per local column */
    double* x[3];            /* x[xi] = current iterate (local column indexing) */
    double* u[2];
    double* y_corr;          /* D^T y */
    double* star_corr;       /* D^T a_* (DST3/Dome) */
    double* cc;              /* test centre correlations per column (SAFE/DST3) */
    double* cnorm;           /* centre group norms per group (GSAFE/GST3) */
    int32_t* act[2];         /* segmented active-unit lists, slot s at [s*cap, s*cap+cnt) */
    int32_t* act_cnt[2];
    int32_t* act_off[2];     /* exclusive scan, G+1 entries */
    uint8_t* mask;           /* per old-active flat position, last iteration's test */
    double* trace;           /* [max_iters][DSCR_TRACE_FIELDS] */
    uint64_t* kts;           /* [max_kts][8] %globaltimer stamps per trip: K1 in/out, K2 in/out, K3a in, -, K3b in/out */
    int32_t max_kts;
    int32_t G;               /* CTAs of the per-unit kernels (= number of slots) */
    int32_t cap;             /* slot capacity in units */
    int32_t comm_len;        /* doubles in `comm` (incl. 64 x 8 one-collective rank slots) */
    double* comm;            /* multi-rank exchange region: [0,8) MAX, [8,16) setup, [16,32)+[32,32+2*ldd) SUM */
    double* vec;             /* ldd: extremal atom / GST3 normal (broadcast from the owner rank) */
} dscr_solver_buffers;

typedef struct dscr_solver dscr_solver;

const char* dscr_last_error(void);
int dscr_abi_version(void);

/* ---- kernel-level entry points (unit parity) -------------------------- */

/* out[j] = ||D[:,j]||_2 in fp64 for j < k (the norms the norm-aware tests use; a property of D
 * alone, so callers cache it per dictionary and pass it as dscr_problem_desc.col_norms). */
int dscr_column_norms(int dtype, const void* D, int ldd, int n, int k, double* out, void* stream);
/* out[j] = D[:,j] . v  for j < k.  Replaces Dictionary.correlate (dictionary.py:89-94).
 * v holds n values; when 8*ldd exceeds the shared-memory staging buffer (n_rows > ~27000)
 * it is read through L2 and must hold ldd values with rows n..ldd-1 zero. */
int dscr_correlate(int dtype, const void* D, int ldd, int n, int k, const double* v,
                   double* out, void* stream);
/* out = D x (out has ldd rows).  Replaces Dictionary.apply (dictionary.py:82-87).
 * Deterministic split-K: `work` holds dscr_apply_work_size() bytes of device memory. */
size_t dscr_apply_work_size(int dtype, int ldd, int k);
int dscr_apply(int dtype, const void* D, int ldd, int n, int k, const double* x,
               double* out, void* work, size_t work_bytes, void* stream);
/* out = sign(v) max(|v|-t,0).  Replaces prox_l1 (problems.py:106-111). */
int dscr_prox_l1(const double* v, int64_t n, double t, double* out, void* stream);
/* group soft threshold, threshold t*w_g over contiguous groups.
 * Replaces GroupLayout.prox (dictionary.py:290-301). */
int dscr_prox_group(const double* v, const int32_t* group_ptr, int n_groups,
                    const double* w, double t, double* out, void* stream);
/* mask[i] = (1-|cc[kept[i]]|) - radius > 1e-12.  Replaces test_sphere_lasso (screening.py:351-359). */
int dscr_test_sphere(const double* cc, const int32_t* kept, int n_kept, double radius,
                     uint8_t* mask, void* stream);
/* Replaces test_dome (screening.py:362-388). */
int dscr_test_dome(const double* star_corr, const double* y_corr, const int32_t* kept, int n_kept,
                   double lam, double lambda_star, double radius, uint8_t* mask, void* stream);
/* mask[i] = (w_g - cnorm_g)/snorm_g - radius > 1e-12 for g = kept_groups[i].
 * Replaces test_sphere_group (screening.py:391-404). */
int dscr_test_group(const double* w, const double* cnorm, const double* snorm,
                    const int32_t* kept_groups, int n_kept, double radius, uint8_t* mask,
                    void* stream);
/* ---- inner seams of the iteration (SURVEY §8(b) kernel-level entry points) ----------------
 * Values are indexed by atom (K-length arrays); `active` lists the atoms (or groups) to touch.
 * The engine fuses the same arithmetic into its per-iteration kernels (K1: corr + prox,
 * K2: test + compaction, K3: residual). */

/* One proximal gradient step over the active atoms: corr_out[j] = D[:,j] . theta,
 * x_out[j] = soft(v, thr) with v = point[j] - corr[j] / step (mult = 0: ISTA / FISTA / SpaRSA,
 * solvers.py:178, 276) or v = point[j] - step * corr[j] (mult = 1: CP / TwIST, solvers.py:302,
 * 242); u_out[j] = x_out + beta (x_out - x_prev[j]) if u_out (FISTA momentum, solvers.py:216-218).
 * red_out[3] = max |corr|, corr . (x_out - point), ||x_out - point||^2 over the active atoms
 * (dual-scaling bound screening.py:126-140; majorization terms of _backtrack solvers.py:176-183).
 * theta: ldd doubles, rows n..ldd-1 zero.  Replaces update_ista / update_fista's step. */
int dscr_corr_prox(int dtype, const void* D, int ldd, int n, const int32_t* active, int n_active,
                   const double* theta, const double* point, const double* x_prev, double step, int mult, double thr,
                   double beta, double* x_out, double* u_out, double* corr_out, double* red_out, void* stream);
/* The group-Lasso step: correlations of `active_atoms`, then per active group g (contiguous atoms
 * group_ptr[g]..group_ptr[g+1]) the block soft threshold x_g = v_g max(1 - thr w_g / ||v_g||, 0)
 * with numpy's pairwise sum for the norm (GroupLayout.prox, dictionary.py:290-301);
 * group_cnorm[i] = ||corr_g|| of active_groups[i]; red_out[0] = min w_g / ||corr_g|| over the
 * active groups with ||corr_g|| > 0 (screening.py:143-165), red_out[1..2] as dscr_corr_prox. */
int dscr_group_corr_prox(int dtype, const void* D, int ldd, int n, const int32_t* group_ptr,
                         const int32_t* active_groups, int n_active, const int32_t* active_atoms, int n_atoms,
                         const double* group_w, const double* theta, const double* point, const double* x_prev,
                         double step, int mult, double thr, double beta, double* x_out, double* u_out,
                         double* corr_out, double* group_cnorm, double* red_out, void* stream);
/* Residuals over a compact support list (idx[e], x[e], u[e]): r_x = D_S x - y, r_u = D_S u - y
 * (r_u / u optional), entries accumulated in list order per row; red_out[3] = ||r_x||^2,
 * ||r_u||^2, r_u . y.  Replaces _residual / Dictionary.apply(x) - y (solvers.py:160-165,
 * dictionary.py:82-87). */
int dscr_residual(int dtype, const void* D, int ldd, int n, const int32_t* idx, int nnz, const double* x,
                  const double* u, const double* y, double* r_x, double* r_u, double* red_out, void* stream);
/* Order-preserving compaction of a kept list by a test mask (mask[i] = 1: screened):
 * active_out = active[~mask], *n_out (device int) = its length.  Replaces screen_update's kept
 * set (screening.py:104-112) and Dictionary.reduce's column selection (dictionary.py:99-117).
 * `work`: dscr_compact_work_size(n) bytes of device memory. */
size_t dscr_compact_work_size(int n);
int dscr_compact(const int32_t* active, int n, const uint8_t* mask, int32_t* active_out, int32_t* n_out, void* work,
                 size_t work_bytes, void* stream);

/* Largest singular value of D by 2-vector block power iteration (dictionary.py:120-171);
 * blocking; `work` must hold dscr_operator_norm_work_size() bytes of device memory. */
/* DSMX ingestion (dictionary.py:304-335: row-major little-endian fp64 payload): `nr` file rows
 * starting at row0 (device, nr x ncols row-major) transposed into the column-major dictionary
 * layout dst[col * ldd + row0 + r] in the storage dtype (fp64; fp32 round-to-nearest; bf16 bit
 * patterns via fp32, round-to-nearest-even). */
int dscr_ingest_rows_f64(const double* rows, int nr, int ncols, int row0, int dtype, void* dst, int ldd,
                         void* stream);

/* Spectral norms of column groups of D (GroupPartition.build, dictionary.py:120-160 per group):
 * group g = columns group_cols[group_ptr[g] .. group_ptr[g+1]) (device arrays).  One kernel for
 * all groups: fp64 Gram per group + the 2-vector block power iteration of dscr_operator_norm on
 * it.  out[g] (device) = ||D_g||_2, or -1 for groups of more than 32 columns or more columns
 * than rows (use dscr_operator_norm on those). */
int dscr_group_spectral_norms(int dtype, const void* D, int ldd, int n_rows, int n_groups, const int32_t* group_ptr,
                              const int32_t* group_cols, double tol, int max_iters, double* out, void* stream);

size_t dscr_operator_norm_work_size(int ldd, int k);
int dscr_operator_norm(int dtype, const void* D, int ldd, int n, int k, double tol, int max_iters,
                       void* work, double* out_host, void* stream);

/* ---- solver-level entry points (replaces solvers.run, solvers.py:358-511) ---- */

size_t dscr_solver_workspace_size(const dscr_problem_desc* prob, const dscr_config* cfg);
/* Builds the solver state and its CUDA graphs (setup graph + conditional-WHILE
 * iteration graph).  `workspace` is caller-owned device memory. */
int dscr_solver_create(const dscr_problem_desc* prob, const dscr_config* cfg, void* workspace,
                       size_t workspace_bytes, void* stream, dscr_solver** out);
/* Enqueue the per-solve setup: lambda_max, screening precomputes, static screen. */
int dscr_solver_setup(dscr_solver* h, void* stream);
/* Enqueue iterations until the solver stops or `iteration_limit` accepted iterations
 * have completed (hook mode passes t+1).  Asynchronous: one graph launch. */
int dscr_solver_run(dscr_solver* h, int iteration_limit, void* stream);
/* Blocking: synchronise `stream` and copy the scalar state to *out. */
int dscr_solver_scalars(dscr_solver* h, void* stream, dscr_scalars* out);
int dscr_solver_get_buffers(dscr_solver* h, dscr_solver_buffers* out);
/* Profiling aid: run `trips` iteration trips as direct kernel launches with CUDA
 * events between K1 | K2 | K3a | K3b; ms_out[4] gets the mean per-kernel time.
 * Blocking.  Advances the solver state like real iterations. */
int dscr_solver_profile(dscr_solver* h, int trips, void* stream, float* ms_out);
int dscr_solver_destroy(dscr_solver* h);

/* ---- batched many-observation path (BASELINE config 5) ---------------- */

/* C^T[n][m] = sum_s sum_k A[m][k] * B[s*Nb + n][k]   (bf16 in, fp32 accumulate, tcgen05)
 * A = D^T (atoms x features, row stride lda), B = S stacked bf16 terms of the residuals
 * (observations x features, row stride ldb), C^T row stride ldc (fp32).
 * M % 128 == 0, Nb % 256 == 0, K % 64 == 0.  Replaces the per-observation
 * Dictionary.correlate calls of a batch (dictionary.py:89-94). */
int dscr_batched_gemm_bf16(const void* A, int M, int lda, const void* B, int Nb, int ldb, int K,
                           int splits, float* C, int ldc, void* stream);

/* Correlations D^T V of a bf16 dictionary (D^T = atoms x rows, row stride ldd) with fp64
 * vectors (V = n_obs x rows, stride ldv) to ~fp64 accuracy on the integer tensor cores:
 * int8 slices of both operands, exact int32 products, fp64 recombination (relative error
 * ~2^-30 of sum |d||v|).  out[j][i] (stride ldo).  Atoms, observations and rows multiples of
 * 128, rows <= 2048.  The fp64 setup correlations of a batch (problems.py:75-86 lambda_max,
 * screening.py:214-231 centre correlations) for many observations at once. */
size_t dscr_corr_exact_work_size(int n_atoms, int n_rows, int n_obs);
int dscr_corr_exact_bf16(const void* Dt, int n_atoms, int n_rows, int ldd, const double* V, int n_obs, int ldv,
                         double* out, int ldo, void* work, size_t work_bytes, void* stream);

/* Batched FISTA with per-observation dynamic screening: shared bf16 dictionary
 * (stored as D^T = atoms x features, i.e. column-major D), many observations.
 * Iterates are sparse per observation; c = D^T theta runs on tcgen05 tensor cores;
 * the fp64 setup computes lambda_*, a_* and the test centres. */
typedef struct dscr_batched_desc {
    int32_t n_rows;          /* N features, multiple of 64, <= 16384 (above 2048: fp64 setup correlations, chunked residual pass) */
    int32_t n_atoms;         /* K, multiple of 128 (all-zero columns are allowed as padding: never active, not counted as kept) */
    int32_t n_obs;           /* B, multiple of 256 (pad with observations whose lam exceeds lambda_*: status 1, skipped) */
    int32_t ldd;             /* row stride of D^T (elements), multiple of 8 */
    const void* Dt;          /* bf16 [K][ldd] */
    const double* Y;         /* fp64 [B][ldy], unit-norm observations */
    int32_t ldy;             /* multiple of 64 */
    int32_t splits;          /* bf16 terms of theta per GEMM: 1 or 2 */
    const double* lam;       /* fp64 [B] (device) */
    double L;                /* step constant 1/L */
    int32_t test;            /* DSCR_TEST_OFF, DSCR_SAFE or DSCR_DST3 */
    int32_t cap;             /* max nonzeros per observation */
    int32_t max_iters;
    int32_t fused;           /* 1: the tcgen05 epilogue emits only the entries whose update can be nonzero
                                (|c| > lam_j or currently nonzero); 0: dense fp32 C round trip */
    const double* beta;      /* host [max_iters]: FISTA momentum coefficients (l_t - 1)/l_{t+1} */
} dscr_batched_desc;

typedef struct dscr_batched_buffers {
    /* support lists by parity ([B][cap]): sorted atoms with x or u nonzero, their x and u
     * values, and the count per observation; after t iterations the solution is the entries of
     * parity t & 1 with x != 0 */
    int32_t* s_idx[2]; double* s_x[2]; double* s_u[2]; int32_t* s_cnt[2];
    double* F; double* gap; int32_t* nnz; int32_t* kept; int32_t* status; double* lmax; double* radius;
    double* trace;            /* [max_iters][4]: sum F, sum gap, sum nnz, sum kept */
    int32_t* iterations;      /* device counter */
    float* C;                 /* last correlations, [B][K] fp32 */
    uint32_t* mask;           /* active atoms, [B][K/32] bits */
} dscr_batched_buffers;

typedef struct dscr_batched dscr_batched;
size_t dscr_batched_workspace_size(const dscr_batched_desc* d);
int dscr_batched_create(const dscr_batched_desc* d, void* workspace, size_t bytes, void* stream,
                        dscr_batched** out);
int dscr_batched_setup(dscr_batched* h, void* stream);
int dscr_batched_run(dscr_batched* h, int iterations, void* stream);
int dscr_batched_get_buffers(dscr_batched* h, dscr_batched_buffers* out);
/* Profiling aid: iteration t as direct launches; ms_out[3] = GEMM, update, residual (blocking). */
int dscr_batched_profile(dscr_batched* h, int t, void* stream, float* ms_out);
int dscr_batched_destroy(dscr_batched* h);

/* ---- multi-GPU (column sharding, one process per GPU) ---------------- */

/* Phases of a column-sharded solve.  Each rank owns a contiguous block of columns
 * (groups kept whole; col_offset / group_offset in the problem descriptor).  The host
 * runs the phases in this order and reduces the comm region between them:
 *   SETUP_LOCAL; all-gather comm[8..10] (local lambda_*, global index, sign), pick the
 *   max (lowest index on ties) and write comm[8..14] = {lambda_*, index, sign, trivial,
 *   is_owner, w_g*, owner's local unit}; SETUP_ADOPT; owner: SETUP_VEC; broadcast the
 *   vec buffer from the owner; SETUP_FINISH; [static: STATIC_LOCAL; MAX comm[0..7];
 *   STATIC_FINISH]; then per trip: K1; MAX comm[0..7]; K1R; K2; K3A; K3S;
 *   SUM comm[16..32+2*ldd); K3B.  Every rank computes the radius, stop flags and trip
 *   modes from identical reduced values. */
#define DSCR_PH_SETUP_LOCAL 0
#define DSCR_PH_SETUP_ADOPT 1
#define DSCR_PH_SETUP_VEC 2
#define DSCR_PH_SETUP_FINISH 3
#define DSCR_PH_STATIC_LOCAL 4
#define DSCR_PH_STATIC_FINISH 5
#define DSCR_PH_K1 10
#define DSCR_PH_K1R 11
#define DSCR_PH_K2 12
#define DSCR_PH_K3A 13
#define DSCR_PH_K3S 14
#define DSCR_PH_K3B 15
#define DSCR_PH_K2S 16     /* one-collective trips: support of x_t / u_t before the test */
#define DSCR_PH_K1R1 17    /* one-collective trips: radius, dropped-nonzero and all-screened flags */
#define DSCR_PH_K2C 18     /* one-collective trips: test and compaction after the collective */
int dscr_solver_phase(dscr_solver* h, int phase, void* stream);
/* One collective per trip (SURVEY §7 hard part 2).  The residual partials are taken on the
 * unreduced iterate, and each rank's MAX quantities (max |c|, non-finite flag), the largest
 * test value over its units with a nonzero coefficient and the smallest over its active units
 * travel in rank-indexed slots of the SUM buffer (comm[32+2*ldd + 8*rank ..+8), zeros
 * elsewhere, so the SUM is a gather).  After the SUM every rank knows the radius and whether
 * any rank screens a unit carrying a nonzero coefficient; only then (rare) a FIXUP trip
 * recomputes the residuals on the reduced iterate.  Per trip: K1; K2S; K3A; K3S;
 * SUM comm[16..32+2*ldd+8*world); K1R1; K2C; K3B.  The dome test keeps two collectives.
 * world <= 64.  rank/world also select the slot; one_collective = 0 restores the
 * two-collective phase semantics. */
int dscr_solver_set_collectives(dscr_solver* h, int rank, int world, int one_collective);
/* Native exchange over peer memory (replaces the NCCL SUM of one-collective trips): each rank
 * allocates dscr_peer_buffer_bytes(world, ldd) with dscr_peer_alloc (CUDA IPC handle out),
 * the host all-gathers the handles, opens the peers' buffers with dscr_peer_open and passes
 * every rank's base (its own included) to dscr_solver_set_peers.  The trip then runs
 * K1; K2S; K3A; K3S; K3X_PUSH; K3X_REDUCE; K1R1; K2C; K3B with no host collective: PUSH stores
 * this rank's SUM section into every peer (NVLink) and signals arrival flags (release, system
 * scope), REDUCE waits for all flags (acquire) and sums the sections in rank order. */
#define DSCR_PH_K3X_PUSH 19
#define DSCR_PH_K3X_REDUCE 20
size_t dscr_peer_buffer_bytes(int world, int ldd);
int dscr_peer_alloc(size_t bytes, void** dptr, void* handle_out_64);
int dscr_peer_open(const void* handle_64, void** dptr);
int dscr_peer_close(void* dptr);
int dscr_peer_free(void* dptr);
int dscr_solver_set_peers(dscr_solver* h, int rank, int world, void* const* recv_bases, void* const* flag_bases);

#ifdef __cplusplus
}
#endif
#endif /* DYNSCREEN_H */
