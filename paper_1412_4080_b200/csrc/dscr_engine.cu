// B200-native screened first-order solver engine (sm_100a).
//
// One solve = one setup graph launch + one loop graph launch.  The loop graph
// is a conditional WHILE node whose body is the per-iteration kernel chain
//
//   K1 corr_update  : c = D_A^T theta_t over the active units, prox/momentum
//                     candidate, block max|c| (or group norms), majorization
//                     partials; the last CTA computes mu, r_SAFE^2 and the
//                     test radius (screening.py:115-307).
//   K2 screen       : per-unit sphere/dome/group test, order-preserving
//                     compaction of the active list (warp ballot + CTA scan),
//                     momentum vectors, support list of the residual pass.
//   K3a residual    : D_S [a b] over the support S, split over (row tile x
//                     support split) CTAs, fp64 partial vectors.
//   K3b finalize    : fixed-order split reduction, residual / next dual
//                     candidate, objective, duality gap, stop flag; the last
//                     CTA runs the iteration epilogue and sets the WHILE
//                     condition (cudaGraphSetConditional).
//
// Backtracking (solvers.py:168-187) and the "dropped a nonzero coefficient"
// residual recompute (solvers.py:354-355, 486-487) are extra trips of the same
// body (mode REDO / FIXUP) instead of host round trips.
//
// Reference semantics restated here: solvers.py:190-313 (updates), 434-501
// (run loop), screening.py:115-413 (dual scaling, regions, tests),
// problems.py:75-177, dictionary.py:82-117, 280-301.

#include <map>
#include <mutex>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>
#include <functional>

#include "dynscreen.h"
#include "dscr_device.cuh"

namespace dscr {

enum { MODE_NORMAL = 0, MODE_REDO = 1, MODE_FIXUP = 2, MODE_STATIC = 3 };
static_assert(sizeof(dscr_scalars) % 8 == 0, "scalar block copied as 8-byte words");
constexpr int NP1 = 6;   // K1 partials
constexpr int NP3 = 4;   // K3b partials
constexpr int MIN_COLS_PER_SPLIT = 16;
// comm region (doubles): [0,8) MAX-reduced, [8,16) setup exchange, [16,32) SUM-reduced scalars,
// [32, 32+2*ldd) SUM-reduced partial residual vectors D_S a, D_S b
constexpr int CM_MAX = 0, CM_SETUP = 8, CM_SUM = 16, CM_VEC = 32;
constexpr int OC_SLOT = 8, OC_MAX_WORLD = 64;   // one-collective rank slots after the SUM vector
constexpr int NP2X = 8;  // K2 partials incl. the one-collective test extremes
#ifndef DSCR_TRIPS_PER_BODY
#define DSCR_TRIPS_PER_BODY 4
#endif
constexpr int TRIPS_PER_BODY = DSCR_TRIPS_PER_BODY;
constexpr int PERS_MAX_G = 2048;   // persistent engine: max CTAs (support offsets kept in smem)


static int set_err(const char* what, cudaError_t e) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    err_store() = buf;
    return DSCR_ECUDA;
}
static int set_inval(const char* what) {
    err_store() = what;
    return DSCR_EINVAL;
}
#define CK(call)                                            \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return set_err(#call, e_);   \
    } while (0)

struct Params {
    const void* D;
    int ldd, n, kcols, dtype;
    const double* y;
    double lam;
    int n_groups;
    const int* gptr;
    const double* gw;
    const double* gsn;
    int n_units;
    int algo, strategy, test;
    double rel_tol, gap_tol, bt_factor, twa, twb, cp_gamma, bb_min, bb_max;
    double L0, cp_safety, op_norm, tw_step;
    dscr_scalars* sc;
    double* theta[2];
    double* resid;
    double* corr;
    double* x[3];
    double* u[2];
    double* ycorr;
    double* star;
    double* cc;
    double* cnorm;
    double* vec;       // N-vector scratch (a_* or the GST3 normal)
    double* dn;        // K-vector scratch (D^T normal)
    double* anorm;     // per-column norms (norm-aware tests), or null
    int norm_aware;
    int* act[2];
    int* act_cnt[2];
    int* act_off[2];
    uint8_t* mask;
    int* sidx;
    double* sa;
    double* sb;
    int* sup_cnt;
    int* sup_off;
    int sup_cap;
    double* p1;
    double* p2;
    double* p3v;
    double* p3s;
    unsigned* tickets;
    double* trace;
    unsigned long long* kts;   // per-trip kernel timestamps [trips][8]
    int max_kts;
    int max_gsize;
    int min_cols;      // support columns per K3a split at least (MIN_COLS_PER_SPLIT)
    int onecoll;       // one collective per trip (dscr_solver_set_collectives)
    void** peer_tab;   // peer exchange: [0, world) receive buffers, [64, 64 + world) flag arrays
    int peer_len;      // doubles exchanged per rank (the one-collective SUM section)
    int oc_rank, oc_world;
    int k2v;           // K2 variant: 0 classic, 1 support before the test (K2S), 2 test + compaction (K2C)
    int k1_ilv;        // K1 interleaved column passes over the identity list
    int k1_tile;       // K1 tiled path: row segments per column (0 = per-warp column path)
    int theta_gl;      // theta read through L2 instead of staged in shared memory (tall dictionaries)
    int f23;           // fused graph: K2 (test / compaction) and K3a-scan (residual) run concurrently
    int P23;           // K3a-scan splits
    int* p3c;          // [P23] support entries per K3a-scan split
    int max_iters;
    int G, cap, TR, R, P, G3b;
    int col_offset, group_offset;
    int in_graph;
    int writer;        // this CTA owns the trace / timestamp writes
    int persistent;    // engine mode chosen at create
    int split;         // multi-rank: phases exchange through `comm` (see dscr_solver_phase)
    double* comm;
    float l2_keep;
    cudaGraphConditionalHandle h_main;
};

// ---------------------------------------------------------------------------
// small device utilities
// ---------------------------------------------------------------------------

// device timestamps: slot 2k = kernel k entry (CTA 0), 2k+1 = kernel k exit (last CTA)
__device__ __forceinline__ void stamp(const Params& P, int slot) {
    if (!P.writer) return;
    const int trip = P.sc->trips;
    if (P.kts && trip < P.max_kts) P.kts[(size_t)trip * 8 + slot] = globaltimer();
}

// Programmatic dependent launch: the chain kernels are launched with programmatic stream
// serialization, so the next kernel's CTAs are scheduled while this one drains; every chain
// kernel waits for its predecessor's completion (and memory flush) before touching state.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int find_slot(const int* off, int G, int f) {
    int lo = 0, hi = G;   // off[lo] <= f < off[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (off[mid] <= f) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int unit_atom_lo(const Params& P, int u) { return P.n_groups ? P.gptr[u] : u; }
__device__ __forceinline__ int unit_atom_hi(const Params& P, int u) { return P.n_groups ? P.gptr[u + 1] : u + 1; }

// Flat index -> slot of a segmented list (slot s holds entries [off[s], off[s+1])).
// A CTA stages a window of K3_WIN consecutive slot offsets in shared memory, starting at
// the slot of its first entry (one warp, 32-ary search), and resolves entries inside the
// window with a shared-memory search; entries past the window fall back to find_slot.
constexpr int K3_WIN = 256;


// slot of flat entry f (last s with off[s] <= f), one warp: 32-ary search, ~log32(G) rounds
__device__ __forceinline__ int warp_find_slot(const int* off, int G, int f, int lane) {
    int lo = 0, hi = G;   // off[lo] <= f < off[hi]
    while (hi - lo > 1) {
        const int span = hi - lo;
        const int probe = lo + (int)(((long long)span * lane) / 32);
        const bool le = (lane == 0) || (probe > lo && off[probe] <= f);
        const unsigned bal = __ballot_sync(0xffffffffu, le);
        const int l = 31 - __clz(bal);                        // last lane whose probe is <= f
        const int nlo = lo + (int)(((long long)span * l) / 32);
        const int nhi = (l == 31) ? hi : lo + (int)(((long long)span * (l + 1)) / 32);
        lo = max(nlo, lo);
        hi = max(nhi, lo + 1);
    }
    return lo;
}

// all threads: stage the window starting at the slot of flat entry f0; returns the window end
__device__ __forceinline__ int stage_window(const int* off, int G, int f0, int* s_off, int* s_s0) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int s0 = warp_find_slot(off, G, f0, threadIdx.x);
        if (threadIdx.x == 0) *s_s0 = s0;
    }
    __syncthreads();
    const int s0 = *s_s0;
    for (int i = threadIdx.x; i < K3_WIN; i += NT) s_off[i] = (s0 + i <= G) ? off[s0 + i] : INT_MAX;
    __syncthreads();
    return s_off[K3_WIN - 1];
}

__device__ __forceinline__ int window_slot(const int* off, int G, const int* s_off, int s0, int wend, int f) {
    if (f >= wend) return find_slot(off, G, f);
    int a = 0, b = K3_WIN - 1;   // s_off[a] <= f < s_off[b]
    while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (s_off[m] <= f) a = m; else b = m;
    }
    return s0 + a;
}

// Copy n doubles (n even, both pointers 16-byte aligned) global -> shared with cp.async:
// every 16-byte piece is in flight at once (no register round trip per element).  The
// caller's next cp_async_wait_all() + __syncthreads() publishes the data.
__device__ __forceinline__ void stage_async(double* dst, const double* src, int n) {
    for (int i = 2 * threadIdx.x; i < n; i += 2 * NT) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src + i) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// test radius from the dual-scaling bound; whole CTA participates.
// Restates dual_scale_lasso/group + _safe_radius_sq + _shifted_radius
// (screening.py:115-205).  bound = 1/corr_inf (Lasso) or min_g w_g/||c_g||.
__device__ void radius_epilogue(const Params& P, double bound, const double* theta, double sq,
                                double ty, double* sh) {
    dscr_scalars* sc = P.sc;
    const double lam = P.lam;
    double mu = 0.0;
    if (sq != 0.0) mu = clip(ty / (lam * sq), bound);
    double acc = 0.0;
    // 4 rows per thread loaded before any is used (same accumulation order as one at a time)
    for (int i0 = threadIdx.x; i0 < P.n; i0 += 4 * NT) {
        double th4[4], y4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * NT;
            th4[q] = (i < P.n) ? theta[i] : 0.0;
            y4[q] = (i < P.n) ? P.y[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (i0 + q * NT < P.n) {
                double v = (sq != 0.0) ? mu * th4[q] : 0.0;
                double d = y4[q] / lam - v;
                acc = fma(d, d, acc);
            }
        }
    }
    double rsq = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        sc->mu = mu;
        sc->rsafe_sq = rsq;
        double r = NAN;
        const int test = P.test;
        if (test == DSCR_SAFE || test == DSCR_GSAFE) {
            r = sqrt(rsq);
        } else if (test == DSCR_DST3 || test == DSCR_DOME || test == DSCR_GST3) {
            double arg = rsq - sc->shift_sq;
            if (arg < -RADIUS_GUARD) {
                sc->status = DSCR_ERADIUS;
                sc->stop = DSCR_STOP_ERROR;
            }
            r = sqrt(fmax(arg, 0.0));
        }
        sc->radius = r;
        if (test == DSCR_DOME) {
            const double shift = sc->lmax / lam - 1.0;
            double rs = hypot(r, shift);
            sc->dome_rs = rs;
            sc->dome_cut = (rs > 0.0) ? shift / rs : 0.0;
            sc->dome_slope = sc->lmax - lam;
            sc->dome_flat = lam * (1.0 - rs);
        }
    }
}

// ---------------------------------------------------------------------------
// K1: correlation + algorithm update over the active units
// ---------------------------------------------------------------------------

// Loads in flight per lane (U) and CTAs per SM of K1.  Measured: one CTA/SM with
// U=4 for fp32 spills (255 regs) and halves the bandwidth; 2 CTAs/SM, C=4, U=1 is best.
template <typename T> struct K1Cfg { static constexpr int U = 2, MINB = 2; };
#ifndef K1_UF32
#define K1_UF32 1
#endif
#ifndef K1_COLS
#define K1_COLS 4
#endif
template <> struct K1Cfg<float> { static constexpr int U = K1_UF32, MINB = 2; };
template <> struct K1Cfg<__nv_bfloat16> { static constexpr int U = 1, MINB = 2; };

// Vectors of ldd doubles up to this size are staged in shared memory by K1 and the setup
// correlations (next to ~5 KB of static state); taller dictionaries read them through L2 (the
// vector is 8 bytes per row against s bytes of dictionary per row and column, and stays
// resident in the 126 MB L2).
constexpr size_t THETA_SMEM_MAX = 227 * 1024 - 8192;

// K1 per-CTA work: correlations, update, per-CTA partials into P.p1[b]
// TG: theta is read through L2 (global loads) instead of being staged in shared memory -- the
// path for dictionaries taller than the shared-memory staging buffer (8 bytes per row).
template <typename T, bool GROUP, bool TG = false>
__device__ __forceinline__ void k1_body(const Params& P, int b, int G, double* s_theta) {
    __shared__ double s_red[NW][NP1];
    dscr_scalars* sc = P.sc;
    const int mode = sc->mode;
    const int p = sc->parity, xi = sc->xi;
    const int nu = sc->n_units;
    const int lo = (int)(((long long)nu * b) / G), hi = (int)(((long long)nu * (b + 1)) / G);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool need_dot = (mode == MODE_NORMAL);
    if (!TG && need_dot && hi > lo) {
        const double* th = P.theta[p];
        stage_async(s_theta, th, P.ldd);
    }
    if (TG) s_theta = P.theta[p];
    cp_async_wait_all();
    __syncthreads();

    const T* D = static_cast<const T*>(P.D);
    const int* act = P.act[p];
    const int* off = P.act_off[p];
    const double* xc = P.x[xi];
    double* xn = P.x[(xi + 1) % 3];
    const double* xp = P.x[(xi + 2) % 3];
    const double* uc = P.u[p];
    const int algo = P.algo;
    const double L = sc->L, lam = P.lam;
    const double tau = sc->tau, tws = P.tw_step;
    const bool first = (sc->t == 0);
    // prox argument scale and threshold per algorithm (solvers.py:178, 276, 302, 242)
    double thr;
    if (algo == DSCR_CP) thr = lam * tau;
    else if (algo == DSCR_TWIST) thr = lam * tws;
    else thr = lam / L;

    double wmax = GROUP ? INFINITY : 0.0;   // Lasso: max|c|; group: min w/||c_g||
    double wcs = 0.0, wss = 0.0, wnf = 0.0, wany = 0.0;

    const uint64_t pol = make_policy(P.l2_keep);
    __shared__ int s_off[K3_WIN];
    __shared__ int s_s0;
    // nothing screened yet: the order-preserving list is the identity (no slot lookups)
    const bool ident = (nu == P.n_units);
    const int wend = ident ? 0 : stage_window(off, P.G, lo, s_off, &s_s0);   // slot offsets of this CTA's range
    if (!GROUP) {
        // Lasso: each warp streams C columns at once (C*U 32-byte loads in flight per lane);
        // lane c applies the update of column c.
        constexpr int C = K1_COLS;
        // interleaved passes (identity list only): pass k of CTA b covers the 32 columns of
        // chunk b + k*G, so the columns streamed at any moment are adjacent in HBM
        const bool ilv = P.k1_ilv && ident;
        const int nchunk = (nu + NW * C - 1) / (NW * C);
        const int f_beg = ilv ? b * NW * C : lo;
        const int f_end = ilv ? nchunk * NW * C : hi;
        const int f_step = ilv ? G * NW * C : NW * C;
        const int fhi = ilv ? nu : hi;
        for (int fb = f_beg; fb < f_end; fb += f_step) {
            const int f0 = fb + warp * C;
            int myj = -1;
            if (lane < C && f0 + lane < fhi) {
                if (ident) {
                    myj = f0 + lane;
                } else {
                    const int s = window_slot(off, P.G, s_off, s_s0, wend, f0 + lane);
                    DSCR_CHECK(s >= 0 && s < P.G && f0 + lane - off[s] < P.cap);
                    myj = act[s * P.cap + (f0 + lane - off[s])];
                    DSCR_CHECK(myj >= 0 && myj < P.kcols);
                }
            }
            int js[C];
#pragma unroll
            for (int c = 0; c < C; ++c) js[c] = __shfl_sync(0xffffffffu, myj, c);
            double cs[C];
            if (need_dot) {
                const T* cols[C];
#pragma unroll
                for (int c = 0; c < C; ++c) cols[c] = js[c] >= 0 ? D + (size_t)js[c] * P.ldd : nullptr;
                warp_dots<T, C, K1Cfg<T>::U>(cols, P.n, s_theta, lane, pol, cs);
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) cs[c] = js[c] >= 0 ? P.corr[js[c]] : 0.0;
            }
            if (myj >= 0) {
                double c = cs[0];
#pragma unroll
                for (int q = 1; q < C; ++q) if (lane == q) c = cs[q];
                const int j = myj;
                if (need_dot) P.corr[j] = c;
                wmax = fmax(wmax, fabs(c));
                double point, v;
                if (algo == DSCR_FISTA) { point = uc[j]; v = point - c / L; }
                else if (algo == DSCR_CP) { point = xc[j]; v = point - tau * c; }
                else if (algo == DSCR_TWIST) { point = xc[j]; v = point - tws * c; }
                else { point = xc[j]; v = point - c / L; }
                double cand = soft(v, thr);
                if (algo == DSCR_TWIST && !first) {
                    const double a = P.twa, bb = P.twb;
                    cand = ((1.0 - a) * xp[j] + (a - bb) * xc[j]) + bb * cand;
                }
                xn[j] = cand;
                if (!isfinite(cand)) wnf = 1.0;
                const double st = cand - point;
                wcs += c * st;
                wss += st * st;
            }
        }
    }
    constexpr int GMAX = 64;                 // groups up to GMAX atoms: lane-parallel, staged in smem
    __shared__ double s_gc[GROUP ? NW : 1][GROUP ? GMAX : 1], s_gv[GROUP ? NW : 1][GROUP ? GMAX : 1];
    for (int f = lo + warp; GROUP && f < hi; f += NW) {
        int unit = f;
        if (!ident) {
            const int s = window_slot(off, P.G, s_off, s_s0, wend, f);
            unit = act[s * P.cap + (f - off[s])];
        }
        const int j0 = unit_atom_lo(P, unit), j1 = unit_atom_hi(P, unit);
        const int gs = j1 - j0;
        if (gs <= GMAX) {
            // correlations (4 columns in flight) and prox arguments staged per warp, group norms in
            // numpy's reduceat order from shared memory, the block soft threshold lane-parallel
            for (int jb = j0; jb < j1; jb += 4) {
                double cs4[4] = {0.0, 0.0, 0.0, 0.0};
                if (need_dot) {
                    const T* cols[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) cols[c] = (jb + c < j1) ? D + (size_t)(jb + c) * P.ldd : nullptr;
                    warp_dots<T, 4, (sizeof(T) == 8 ? 2 : 1)>(cols, P.n, s_theta, lane, pol, cs4);
                }
                if (lane < 4 && jb + lane < j1) {
                    double cc = cs4[0];
#pragma unroll
                    for (int q = 1; q < 4; ++q) if (lane == q) cc = cs4[q];
                    s_gc[warp][jb - j0 + lane] = need_dot ? cc : P.corr[jb + lane];
                }
            }
            __syncwarp();
            for (int c0 = lane; c0 < gs; c0 += 32) {
                const int j = j0 + c0;
                const double cc = s_gc[warp][c0];
                if (need_dot) P.corr[j] = cc;
                double v;
                if (algo == DSCR_FISTA) v = uc[j] - cc / L;
                else if (algo == DSCR_CP) v = xc[j] - tau * cc;
                else if (algo == DSCR_TWIST) v = xc[j] - tws * cc;
                else v = xc[j] - cc / L;
                s_gv[warp][c0] = v;
            }
            __syncwarp();
            double fac = 0.0;
            if (lane == 0) {   // group soft threshold (dictionary.py:290-301), numpy reduceat summation order
                const double nv = sqrt(np_segment_sum([&](int i) { double t = s_gv[warp][i - j0]; return t * t; }, j0, gs));
                const double nc = sqrt(np_segment_sum([&](int i) { double t = s_gc[warp][i - j0]; return t * t; }, j0, gs));
                if (nc > 0.0) { wmax = fmin(wmax, P.gw[unit] / nc); wany = 1.0; }
                fac = (nv > 0.0) ? fmax(1.0 - thr * P.gw[unit] / nv, 0.0) : 0.0;
            }
            fac = __shfl_sync(0xffffffffu, fac, 0);
            for (int c0 = lane; c0 < gs; c0 += 32) {
                const int j = j0 + c0;
                double cand = s_gv[warp][c0] * fac;
                if (algo == DSCR_TWIST && !first) {
                    const double a = P.twa, bb = P.twb;
                    cand = ((1.0 - a) * xp[j] + (a - bb) * xc[j]) + bb * cand;
                }
                xn[j] = cand;
                if (!isfinite(cand)) wnf = 1.0;
                const double point = (algo == DSCR_FISTA) ? uc[j] : xc[j];
                const double st = cand - point;
                wcs += s_gc[warp][c0] * st;
                wss += st * st;
            }
            __syncwarp();
            continue;
        }
        // larger groups: serial per-group path through global memory
        // correlations of the group's atoms (4 columns in flight), provisional prox argument in xn
        for (int jb = j0; jb < j1; jb += 4) {
            double cs4[4];
            if (need_dot) {
                const T* cols[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) cols[c] = (jb + c < j1) ? D + (size_t)(jb + c) * P.ldd : nullptr;
                warp_dots<T, 4, (sizeof(T) == 8 ? 2 : 1)>(cols, P.n, s_theta, lane, pol, cs4);
            }
            if (lane == 0) {
                for (int c = 0; c < 4 && jb + c < j1; ++c) {
                    const int j = jb + c;
                    const double cc = need_dot ? cs4[c] : P.corr[j];
                    if (need_dot) P.corr[j] = cc;
                    double v;
                    if (algo == DSCR_FISTA) v = uc[j] - cc / L;
                    else if (algo == DSCR_CP) v = xc[j] - tau * cc;
                    else if (algo == DSCR_TWIST) v = xc[j] - tws * cc;
                    else v = xc[j] - cc / L;
                    xn[j] = v;
                }
            }
        }
        if (lane == 0) {
            // group soft threshold (dictionary.py:290-301) with numpy's reduceat summation order
            const int gs = j1 - j0;
            double nv = sqrt(np_segment_sum([&](int i) { double t = xn[i]; return t * t; }, j0, gs));
            double nc = sqrt(np_segment_sum([&](int i) { double t = P.corr[i]; return t * t; }, j0, gs));
            if (nc > 0.0) { wmax = fmin(wmax, P.gw[unit] / nc); wany = 1.0; }
            double fac = (nv > 0.0) ? fmax(1.0 - thr * P.gw[unit] / nv, 0.0) : 0.0;
            for (int j = j0; j < j1; ++j) {
                double cand = xn[j] * fac;
                if (algo == DSCR_TWIST && !first) {
                    const double a = P.twa, bb = P.twb;
                    cand = ((1.0 - a) * xp[j] + (a - bb) * xc[j]) + bb * cand;
                }
                xn[j] = cand;
                if (!isfinite(cand)) wnf = 1.0;
                const double point = (algo == DSCR_FISTA) ? uc[j] : xc[j];
                const double st = cand - point;
                wcs += P.corr[j] * st;
                wss += st * st;
            }
        }
    }
    wmax = GROUP ? warp_min(wmax) : warp_max(wmax);
    wcs = warp_sum(wcs);
    wss = warp_sum(wss);
    wnf = warp_max(wnf);
    wany = warp_max(wany);
    if (lane == 0) {
        s_red[warp][0] = wmax; s_red[warp][1] = wcs; s_red[warp][2] = wss;
        s_red[warp][3] = wnf; s_red[warp][4] = wany;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = GROUP ? INFINITY : 0.0, cs = 0.0, ss = 0.0, nf = 0.0, any = 0.0;
        for (int w = 0; w < NW; ++w) {
            m = GROUP ? fmin(m, s_red[w][0]) : fmax(m, s_red[w][0]);
            cs += s_red[w][1]; ss += s_red[w][2]; nf = fmax(nf, s_red[w][3]); any = fmax(any, s_red[w][4]);
        }
        double* o = P.p1 + (size_t)b * NP1;
        o[0] = m; o[1] = cs; o[2] = ss; o[3] = nf; o[4] = any;
    }
}

// K1 tiled path, for short columns (at most K1T_SEGS segments of 32*V*U rows; c1-c3 shapes).
// The per-warp column path gives each warp whole columns, so a CTA whose share is a few
// columns more than a multiple of 4*NW waits a second full column chain on one warp (c2:
// 34 columns per CTA = 16 round trips).  Here the CTA's atoms are resolved into shared
// memory in batches of K1T_ATOMS, the correlations are (atom quad x row segment) items dealt
// evenly over the warps -- one round trip of 4*U loads per lane per item -- and the segment
// partials are combined in fixed segment order (independent of the grid), then the update
// runs per atom (Lasso) or per group (one warp per group, correlations read from shared).
constexpr int K1T_ATOMS = 256;
constexpr int K1T_SEGS = 16;

template <typename T>
__device__ __forceinline__ void warp_dots_seg(const T* const (&col)[4], int n, const double* sv, int lane,
                                              uint64_t pol, int row0, double (&out)[4]) {
    constexpr int V = Vec<T>::V, U = K1Cfg<T>::U;
    typename Vec<T>::Raw d[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = row0 + u * 32 * V + lane * V;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (i < n && col[c]) Vec<T>::load_raw(col[c] + i, d[u][c], pol);
            else Vec<T>::zero(d[u][c]);
        }
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int i = row0 + u * 32 * V + lane * V;
        if (i < n) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const double t = sv[i + v];
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] = fma(Vec<T>::get(d[u][c], v), t, acc[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = warp_sum(acc[c]);
}

template <typename T, bool GROUP>
__device__ __forceinline__ void k1_body_tile(const Params& P, int b, int G, double* s_theta) {
    __shared__ double s_red[NW][NP1];
    __shared__ int s_atom[K1T_ATOMS];
    __shared__ int s_unit[K1T_ATOMS], s_uoff[K1T_ATOMS + 1];
    __shared__ int s_scan[2 * NW + 1];
    __shared__ int s_off[K3_WIN];
    __shared__ int s_s0;
    constexpr int GMAX = 64;
    __shared__ double s_gv[GROUP ? NW : 1][GROUP ? GMAX : 1];
    double* s_part = s_theta + P.ldd;                 // [K1T_SEGS][K1T_ATOMS] after theta
    dscr_scalars* sc = P.sc;
    const int mode = sc->mode;
    const int p = sc->parity, xi = sc->xi;
    const int nu = sc->n_units;
    const int lo = (int)(((long long)nu * b) / G), hi = (int)(((long long)nu * (b + 1)) / G);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool need_dot = (mode == MODE_NORMAL);
    if (need_dot && hi > lo) {
        const double* th = P.theta[p];
        stage_async(s_theta, th, P.ldd);
    }
    const T* D = static_cast<const T*>(P.D);
    const int* act = P.act[p];
    const int* off = P.act_off[p];
    const double* xc = P.x[xi];
    double* xn = P.x[(xi + 1) % 3];
    const double* xp = P.x[(xi + 2) % 3];
    const double* uc = P.u[p];
    const int algo = P.algo;
    const double L = sc->L, lam = P.lam;
    const double tau = sc->tau, tws = P.tw_step;
    const bool first = (sc->t == 0);
    double thr;
    if (algo == DSCR_CP) thr = lam * tau;
    else if (algo == DSCR_TWIST) thr = lam * tws;
    else thr = lam / L;
    const int nseg = P.k1_tile;
    constexpr int SEGR = 32 * Vec<T>::V * K1Cfg<T>::U;   // rows per segment

    double wmax = GROUP ? INFINITY : 0.0;
    double wcs = 0.0, wss = 0.0, wnf = 0.0, wany = 0.0;
    const uint64_t pol = make_policy(P.l2_keep);
    const bool ident = (nu == P.n_units);
    int wend = 0;
    cp_async_wait_all();          // theta staged (published by the barrier below)
    if (ident) __syncthreads();
    else wend = stage_window(off, P.G, lo, s_off, &s_s0);   // (syncs: theta staged)
    const int ub = GROUP ? max(1, K1T_ATOMS / max(1, P.max_gsize)) : K1T_ATOMS;

    for (int b0 = lo; b0 < hi; b0 += ub) {
        const int nb = min(ub, hi - b0);
        // ---- resolve the batch's units and atoms
        int unit = -1, gs = 0;
        if (threadIdx.x < nb) {
            const int f = b0 + threadIdx.x;
            if (ident) {
                unit = f;
            } else {
                const int s = window_slot(off, P.G, s_off, s_s0, wend, f);
                unit = act[s * P.cap + (f - off[s])];
            }
            gs = GROUP ? (P.gptr[unit + 1] - P.gptr[unit]) : 1;
        }
        int na;
        const int aoff = GROUP ? block_exscan(gs, s_scan, &na) : (int)threadIdx.x;   // (syncs)
        if (!GROUP) na = nb;
        if (threadIdx.x < nb) {
            s_unit[threadIdx.x] = unit;
            s_uoff[threadIdx.x] = aoff;
            if (GROUP) { const int j0 = P.gptr[unit]; for (int k = 0; k < gs; ++k) s_atom[aoff + k] = j0 + k; }
            else s_atom[threadIdx.x] = unit;
        }
        if (threadIdx.x == 0) s_uoff[nb] = na;
        __syncthreads();
        // ---- correlation items: (atom quad, row segment), dealt round-robin over the warps
        if (need_dot) {
            const int nq = (na + 3) >> 2;
            for (int it = warp; it < nq * nseg; it += NW) {
                const int q = it / nseg, sg = it - q * nseg;
                const T* cols[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int a = 4 * q + c;
                    cols[c] = (a < na) ? D + (size_t)s_atom[a] * P.ldd : nullptr;
                }
                double cs[4];
                warp_dots_seg<T>(cols, P.n, s_theta, lane, pol, sg * SEGR, cs);
                if (lane < 4 && 4 * q + lane < na) {
                    double v = cs[0];
#pragma unroll
                    for (int c = 1; c < 4; ++c) if (lane == c) v = cs[c];
                    s_part[sg * K1T_ATOMS + 4 * q + lane] = v;
                }
            }
        }
        __syncthreads();
        // ---- fixed-order segment combination
        for (int a = threadIdx.x; a < na; a += NT) {
            const int j = s_atom[a];
            double c;
            if (need_dot) {
                c = s_part[a];
                for (int sg = 1; sg < nseg; ++sg) c += s_part[sg * K1T_ATOMS + a];
                P.corr[j] = c;
            } else {
                c = P.corr[j];
            }
            if (GROUP) { s_part[a] = c; continue; }
            // Lasso update of atom j (as in k1_body)
            wmax = fmax(wmax, fabs(c));
            double point, v;
            if (algo == DSCR_FISTA) { point = uc[j]; v = point - c / L; }
            else if (algo == DSCR_CP) { point = xc[j]; v = point - tau * c; }
            else if (algo == DSCR_TWIST) { point = xc[j]; v = point - tws * c; }
            else { point = xc[j]; v = point - c / L; }
            double cand = soft(v, thr);
            if (algo == DSCR_TWIST && !first) {
                const double a2 = P.twa, bb = P.twb;
                cand = ((1.0 - a2) * xp[j] + (a2 - bb) * xc[j]) + bb * cand;
            }
            xn[j] = cand;
            if (!isfinite(cand)) wnf = 1.0;
            const double st = cand - point;
            wcs += c * st;
            wss += st * st;
        }
        if (GROUP) {
            __syncthreads();
            // ---- group update: one warp per group (sizes <= GMAX), as the k1_body group path
            for (int t = warp; t < nb; t += NW) {
                const int u = s_unit[t], a0 = s_uoff[t], g = s_uoff[t + 1] - a0;
                const int j0 = s_atom[a0];                 // first atom (already resolved)
                const double gwu = P.gw[u];                // in flight with the x / u loads
                const double* gc = s_part + a0;
                for (int c0 = lane; c0 < g; c0 += 32) {
                    const int j = j0 + c0;
                    const double cc = gc[c0];
                    double v;
                    if (algo == DSCR_FISTA) v = uc[j] - cc / L;
                    else if (algo == DSCR_CP) v = xc[j] - tau * cc;
                    else if (algo == DSCR_TWIST) v = xc[j] - tws * cc;
                    else v = xc[j] - cc / L;
                    s_gv[warp][c0] = v;
                }
                __syncwarp();
                double fac = 0.0;
                if (lane == 0) {   // group soft threshold (dictionary.py:290-301), numpy reduceat order
                    const double nv = sqrt(np_segment_sum([&](int i) { double q = s_gv[warp][i - j0]; return q * q; }, j0, g));
                    const double nc = sqrt(np_segment_sum([&](int i) { double q = gc[i - j0]; return q * q; }, j0, g));
                    if (nc > 0.0) { wmax = fmin(wmax, gwu / nc); wany = 1.0; }
                    fac = (nv > 0.0) ? fmax(1.0 - thr * gwu / nv, 0.0) : 0.0;
                }
                fac = __shfl_sync(0xffffffffu, fac, 0);
                for (int c0 = lane; c0 < g; c0 += 32) {
                    const int j = j0 + c0;
                    double cand = s_gv[warp][c0] * fac;
                    if (algo == DSCR_TWIST && !first) {
                        const double a2 = P.twa, bb = P.twb;
                        cand = ((1.0 - a2) * xp[j] + (a2 - bb) * xc[j]) + bb * cand;
                    }
                    xn[j] = cand;
                    if (!isfinite(cand)) wnf = 1.0;
                    const double point = (algo == DSCR_FISTA) ? uc[j] : xc[j];
                    const double st = cand - point;
                    wcs += gc[c0] * st;
                    wss += st * st;
                }
                __syncwarp();
            }
        }
        __syncthreads();   // s_atom / s_part reuse by the next batch
    }
    wmax = GROUP ? warp_min(wmax) : warp_max(wmax);
    wcs = warp_sum(wcs);
    wss = warp_sum(wss);
    wnf = warp_max(wnf);
    wany = warp_max(wany);
    if (lane == 0) {
        s_red[warp][0] = wmax; s_red[warp][1] = wcs; s_red[warp][2] = wss;
        s_red[warp][3] = wnf; s_red[warp][4] = wany;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = GROUP ? INFINITY : 0.0, cs = 0.0, ss = 0.0, nf = 0.0, any = 0.0;
        for (int w = 0; w < NW; ++w) {
            m = GROUP ? fmin(m, s_red[w][0]) : fmax(m, s_red[w][0]);
            cs += s_red[w][1]; ss += s_red[w][2]; nf = fmax(nf, s_red[w][3]); any = fmax(any, s_red[w][4]);
        }
        double* o = P.p1 + (size_t)b * NP1;
        o[0] = m; o[1] = cs; o[2] = ss; o[3] = nf; o[4] = any;
    }
}

// K1 tail: fixed-order reduction of the G partials, FISTA/CP scalars, radius.  Run by the
// last CTA (graph path) or redundantly by every CTA (persistent path).
template <bool GROUP>
__device__ void k1_final(const Params& P, int G) {
    __shared__ double s_sh[64];
    dscr_scalars* sc = P.sc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int p = sc->parity;
    const int algo = P.algo;

    // ---- last CTA: fixed-order reduction of the per-CTA partials
    double m = GROUP ? INFINITY : 0.0, cs = 0.0, ss = 0.0, nf = 0.0, any = 0.0;
    for (int i0 = threadIdx.x; i0 < G; i0 += 4 * NT) {   // 4 partials per thread in flight
        double o4[4][5];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * NT;
            const double* o = P.p1 + (size_t)i * NP1;
#pragma unroll
            for (int k = 0; k < 5; ++k) o4[q][k] = (i < G) ? o[k] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (i0 + q * NT < G) {
                m = GROUP ? fmin(m, o4[q][0]) : fmax(m, o4[q][0]);
                cs += o4[q][1]; ss += o4[q][2]; nf = fmax(nf, o4[q][3]); any = fmax(any, o4[q][4]);
            }
        }
    }
    // max/min via warp + smem
    {
        double wm = GROUP ? warp_min(m) : warp_max(m);
        __shared__ double s_m[NW], s_nf[NW], s_any[NW];
        double wnf2 = warp_max(nf), wany2 = warp_max(any);
        if (lane == 0) { s_m[warp] = wm; s_nf[warp] = wnf2; s_any[warp] = wany2; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double mm = s_m[0], n2 = s_nf[0], a2 = s_any[0];
            for (int w = 1; w < NW; ++w) {
                mm = GROUP ? fmin(mm, s_m[w]) : fmax(mm, s_m[w]);
                n2 = fmax(n2, s_nf[w]); a2 = fmax(a2, s_any[w]);
            }
            s_m[0] = mm; s_nf[0] = n2; s_any[0] = a2;
        }
        __syncthreads();
        m = s_m[0]; nf = s_nf[0]; any = s_any[0];
    }
    {
        double v2[2] = {cs, ss};
        block_sum_n<2>(v2, s_sh);
        cs = v2[0]; ss = v2[1];
    }
    double bound;
    if (GROUP) bound = (any > 0.0) ? m : INFINITY;
    else bound = (m == 0.0) ? INFINITY : 1.0 / m;
    if (threadIdx.x == 0) {
        sc->corr_inf = m;
        sc->maj_cs = cs;
        sc->maj_ss = ss;
        sc->nonfinite = (nf > 0.0);
        if (algo == DSCR_FISTA) {
            const double l = sc->l_acc;
            const double ln = 0.5 * (1.0 + sqrt(1.0 + 4.0 * (l * l)));
            sc->l_new = ln;
            sc->beta = (l - 1.0) / ln;
        } else if (algo == DSCR_CP) {
            const double phi = 1.0 / sqrt(1.0 + 2.0 * P.cp_gamma * sc->tau);
            sc->phi = phi;
            sc->sigma_new = sc->sigma / phi;
        }
    }
    if (P.split) {
        if (threadIdx.x == 0) {
            P.comm[CM_MAX + 0] = GROUP ? ((any > 0.0) ? -m : -INFINITY) : m;
            P.comm[CM_MAX + 1] = nf;
            P.comm[CM_MAX + 2] = any;
        }
        return;
    }
    radius_epilogue(P, bound, P.theta[p], sc->theta_sq, sc->theta_y, s_sh);
    if (threadIdx.x == 0) stamp(P, 1);
}


// TG (tall dictionaries, theta through L2) is a separate instantiation so the common kernel
// keeps its code size (one k1_body copy: a second one in the same kernel measured +6% on c1 /
// +18% on c2's K1)
template <typename T, bool GROUP, bool TG = false>
__global__ void __launch_bounds__(NT, K1Cfg<T>::MINB) k1_corr_update(Params P) {
    extern __shared__ double s_theta[];
    __shared__ int s_flag;
    pdl_wait();
    pdl_trigger();
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    const int mode = sc->mode;
    if (mode == MODE_FIXUP || mode == MODE_STATIC) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) stamp(P, 0);
    if (TG) k1_body<T, GROUP, true>(P, blockIdx.x, gridDim.x, s_theta);
    else if (P.k1_tile) k1_body_tile<T, GROUP>(P, blockIdx.x, gridDim.x, s_theta);
    else k1_body<T, GROUP>(P, blockIdx.x, gridDim.x, s_theta);
    if (!last_block(P.tickets + 0, gridDim.x, &s_flag)) return;
    k1_final<GROUP>(P, gridDim.x);
}

// split mode: radius from the MAX-reduced correlation bound (after the collective)
__global__ void __launch_bounds__(NT) k1r_radius(Params P) {
    __shared__ double s_sh[64];
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    const int mode = sc->mode;
    if (mode == MODE_FIXUP || mode == MODE_STATIC) return;
    const double m = P.comm[CM_MAX + 0];
    double bound;
    if (P.n_groups) bound = (P.comm[CM_MAX + 2] > 0.0) ? -m : INFINITY;
    else bound = (m == 0.0) ? INFINITY : 1.0 / m;
    if (threadIdx.x == 0) {
        sc->corr_inf = P.n_groups ? -m : m;
        sc->nonfinite = P.comm[CM_MAX + 1] > 0.0;
    }
    radius_epilogue(P, bound, P.theta[sc->parity], sc->theta_sq, sc->theta_y, s_sh);
}

// split mode: sum the local split partials into the comm vector, local scalars into comm
// K3S rows per CTA and split groups per row: the split sums in exactly K3b's order (group g
// sums splits g, g+8, ...; groups combined in order), so one rank reproduces the fused engine
// bit for bit; 8 loads in flight per row instead of a serial walk over the splits (c4: 25 ->
// a few us per trip)
constexpr int K3S_ROWS = 32;
constexpr int K3S_GROUPS = NT / K3S_ROWS;

__global__ void __launch_bounds__(NT) k3s_pack(Params P) {
    __shared__ double s_pa[K3S_GROUPS][K3S_ROWS], s_pb[K3S_GROUPS][K3S_ROWS];
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    if (sc->mode == MODE_STATIC) return;
    const int pe = sc->p_eff;
    {
        const int rr = threadIdx.x % K3S_ROWS, g = threadIdx.x / K3S_ROWS;
        const int r = blockIdx.x * K3S_ROWS + rr;
        double a = 0.0, b = 0.0;
        if (r < P.n)
            for (int q = g; q < pe; q += K3S_GROUPS) {
                a += P.p3v[((size_t)q * 2) * P.ldd + r];
                b += P.p3v[((size_t)q * 2 + 1) * P.ldd + r];
            }
        s_pa[g][rr] = a;
        s_pb[g][rr] = b;
    }
    __syncthreads();
    if (threadIdx.x < K3S_ROWS) {
        const int r = blockIdx.x * K3S_ROWS + threadIdx.x;
        if (r < P.ldd) {
            double Sa = 0.0, Sb = 0.0;
#pragma unroll
            for (int g = 0; g < K3S_GROUPS; ++g) { Sa += s_pa[g][threadIdx.x]; Sb += s_pb[g][threadIdx.x]; }
            P.comm[CM_VEC + r] = Sa;
            P.comm[CM_VEC + P.ldd + r] = Sb;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double* o = P.comm + CM_SUM;
        o[0] = sc->pen; o[1] = sc->nnz; o[2] = sc->kept_atoms; o[3] = sc->ss_red;
        o[4] = sc->dropped_nz; o[5] = sc->maj_cs; o[6] = sc->maj_ss; o[7] = 0.0;
    }
    if (P.onecoll && blockIdx.x == 0) {
        // rank slots: zeros except this rank's (the SUM gathers them); this rank's MAX
        // quantities from K1, its test extremes and active-unit count from K2S
        double* slots = P.comm + CM_VEC + 2 * P.ldd;
        const bool fresh = sc->mode != MODE_FIXUP;
        for (int i = threadIdx.x; i < OC_SLOT * OC_MAX_WORLD; i += NT) {
            const int r = i / OC_SLOT, k = i % OC_SLOT;
            if (r != P.oc_rank) { slots[i] = 0.0; continue; }
            if (k < 3) slots[i] = fresh ? P.comm[CM_MAX + k] : 0.0;
            else if (k >= 6 || !fresh) slots[i] = 0.0;
        }
    }
}

// ---- native exchange over peer memory (NVLink / NVSwitch), replacing the NCCL SUM ----------
// Every rank's buffer holds 64 uint64 arrival flags then two receive areas [2][world][len]
// (parity of the exchange sequence number).  K3X_PUSH stores this rank's SUM section into its
// slot of every peer's receive area (remote stores), and the last CTA publishes the sequence
// number in every peer's flag for this rank (release, system scope).  K3X_REDUCE waits for
// every rank's flag (acquire) and sums the received sections in rank order into `comm`, so all
// ranks hold bit-identical sums.  A rank can be at most one exchange ahead of a peer (its next
// REDUCE waits for the peer's next PUSH, issued after the peer's current REDUCE), so two
// receive areas suffice.  Both kernels exit on the same stop / mode state as K3S, which every
// rank computes identically.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// The exchange sequence number lives on the device (a 64-bit word after the kernel tickets),
// so a captured trip graph replays with fresh numbers: PUSH and REDUCE use counter + 1 and
// REDUCE's last CTA stores it.  It is never reset by a new solve on the same handle (the peers'
// flags keep the last number they saw), only by dscr_solver_set_peers.
__device__ __forceinline__ unsigned long long* xseq_ptr(const Params& P) {
    return reinterpret_cast<unsigned long long*>(P.tickets + 8);
}

__global__ void __launch_bounds__(NT) k3x_push(Params P) {
    __shared__ int s_flag;
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    if (sc->mode == MODE_STATIC) return;
    const unsigned long long seq = *reinterpret_cast<volatile unsigned long long*>(xseq_ptr(P)) + 1ull;
    const int W = P.oc_world, len = P.peer_len;
    const size_t off = (size_t)(seq & 1ull) * W * len + (size_t)P.oc_rank * len;
    const double* src = P.comm + CM_SUM;
    for (int i = blockIdx.x * NT + threadIdx.x; i < len; i += gridDim.x * NT) {
        const double v = src[i];
        for (int r = 0; r < W; ++r) static_cast<double*>(P.peer_tab[r])[off + i] = v;
    }
    __threadfence_system();
    if (!last_block(P.tickets + 3, gridDim.x, &s_flag)) return;
    if (threadIdx.x < W) {
        __threadfence_system();
        st_release_sys(static_cast<unsigned long long*>(P.peer_tab[64 + threadIdx.x]) + P.oc_rank, seq);
    }
}

__global__ void __launch_bounds__(NT) k3x_reduce(Params P) {
    __shared__ int s_flag;
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    if (sc->mode == MODE_STATIC) return;
    const unsigned long long seq = *reinterpret_cast<volatile unsigned long long*>(xseq_ptr(P)) + 1ull;
    const int W = P.oc_world, len = P.peer_len;
    if (threadIdx.x < W) {   // every rank's section of this exchange has arrived
        const unsigned long long* f = static_cast<const unsigned long long*>(P.peer_tab[64 + P.oc_rank]) + threadIdx.x;
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(f) < seq) {
            if (globaltimer() - t0 > 30000000000ull) {   // 30 s watchdog: a peer never arrived
                sc->status = DSCR_ENOCOMM;
                sc->stop = DSCR_STOP_ERROR;
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    const double* rb = static_cast<const double*>(P.peer_tab[P.oc_rank]) + (size_t)(seq & 1ull) * W * len;
    double* dst = P.comm + CM_SUM;
    for (int i = blockIdx.x * NT + threadIdx.x; i < len; i += gridDim.x * NT) {
        double a = 0.0;
        for (int r = 0; r < W; ++r) a += rb[(size_t)r * len + i];   // rank order: identical on every rank
        dst[i] = a;
    }
    if (!last_block(P.tickets + 6, gridDim.x, &s_flag)) return;   // every CTA has read seq
    if (threadIdx.x == 0) *xseq_ptr(P) = seq;
}

// one-collective trips: MAX quantities and test extremes from the gathered rank slots, the
// radius (as k1r_radius), then whether any rank screens a unit carrying a nonzero coefficient
// (FIXUP) and whether every active unit is screened (the all-screened stop)
__global__ void __launch_bounds__(NT) k1r_radius_oc(Params P) {
    __shared__ double s_sh[64];
    __shared__ double s_v[4];
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    const int mode = sc->mode;
    if (mode == MODE_FIXUP || mode == MODE_STATIC) return;
    if (threadIdx.x == 0) {
        const double* slots = P.comm + CM_VEC + 2 * P.ldd;
        double m = -INFINITY, nf = 0.0, any = 0.0, tmax = -INFINITY, vmin = INFINITY, units = 0.0;
        for (int r = 0; r < P.oc_world; ++r) {
            const double* q = slots + OC_SLOT * r;
            m = fmax(m, q[0]); nf = fmax(nf, q[1]); any = fmax(any, q[2]);
            tmax = fmax(tmax, q[3]); vmin = fmin(vmin, q[4]); units += q[5];
        }
        if (!P.n_groups && m < 0.0) m = 0.0;   // every rank empty
        s_v[0] = m; s_v[1] = nf; s_v[2] = any;
        sc->oc_spare = tmax;
        sc->oc_empty = (units == 0.0) ? 1.0 : 0.0;
        s_v[3] = vmin;
    }
    __syncthreads();
    const double m = s_v[0];
    double bound;
    if (P.n_groups) bound = (s_v[2] > 0.0) ? -m : INFINITY;
    else bound = (m == 0.0) ? INFINITY : 1.0 / m;
    if (threadIdx.x == 0) {
        sc->corr_inf = P.n_groups ? -m : m;
        sc->nonfinite = s_v[1] > 0.0;
    }
    radius_epilogue(P, bound, P.theta[sc->parity], sc->theta_sq, sc->theta_y, s_sh);
    __syncthreads();
    if (threadIdx.x == 0) {
        const double r = sc->radius;
        const bool dyn = P.strategy == DSCR_DYNAMIC;
        sc->dropped_nz = dyn && (sc->oc_spare - r > SCREEN_MARGIN);
        if (dyn && s_v[3] - r > SCREEN_MARGIN) sc->oc_empty = 1.0;
    }
}

// ---------------------------------------------------------------------------
// K2: screening test + order-preserving compaction + support list
// ---------------------------------------------------------------------------

// test value of a unit for the sphere tests: screened iff value - r > SCREEN_MARGIN
// (SAFE/DST3: screening.py:359; groups: screening.py:404).  Rounding of value - r is
// monotone in value, so max / min over units decide "any" / "all" screened exactly.
__device__ __forceinline__ double unit_value(const Params& P, int unit) {
    const int test = P.test;
    if (test == DSCR_SAFE || test == DSCR_DST3) {
        if (P.norm_aware)   // max over the sphere of |a.theta| = |a.c| + r ||a||  (non-unit atoms)
            return (1.0 - fabs(P.cc[unit])) / P.anorm[unit];
        return 1.0 - fabs(P.cc[unit]);
    }
    return (P.gw[unit] - P.cnorm[unit]) / P.gsn[unit];
}

__device__ __forceinline__ bool unit_test(const Params& P, const dscr_scalars* sc, int unit) {
    const int test = P.test;
    const double r = sc->radius;
    if (test == DSCR_SAFE || test == DSCR_DST3 || test == DSCR_GSAFE || test == DSCR_GST3)
        return unit_value(P, unit) - r > SCREEN_MARGIN;
    if (test == DSCR_DOME) {                                    // screening.py:374-388
        if (r >= 1.0) return false;
        const double lam = P.lam;
        const double t = P.star[unit], u = P.ycorr[unit];
        const double arc = (lam * r) * sqrt(fmax(1.0 - t * t, 0.0));
        const double slope = sc->dome_slope, flat = sc->dome_flat, cut = sc->dome_cut;
        const double lower = (t < cut) ? (slope * t - lam) + arc : -flat;
        const double upper = (t <= -cut) ? flat : (slope * t + lam) - arc;
        const double mg = lam * SCREEN_MARGIN;
        return (u - lower > mg) && (upper - u > mg);
    }
    return false;
}

// b value of an atom for the residual pass (D b - y is theta_{t+1} or, for SpaRSA, D s): FISTA
// u = c + beta (c - x) (solvers.py:216-218), CP u = c + phi (c - x) (solvers.py:305-307),
// SpaRSA s = c - x (solvers.py:272), none for ISTA / TwIST
__device__ __forceinline__ double b_value(int algo, double c, double xc, double beta, double phi) {
    if (algo == DSCR_FISTA) return c + beta * (c - xc);
    if (algo == DSCR_CP) return c + phi * (c - xc);
    if (algo == DSCR_SPARSA) return c - xc;
    return 0.0;
}

// K2 per-CTA work: test, compaction into slot b, vectors, support list, partials.
// Variants (P.k2v): 0 classic; 1 = K2S (one collective): no test, support list and vectors
// over every active unit (the reduced list in a FIXUP trip), plus the largest test value over
// units carrying a nonzero coefficient and the smallest over all units; 2 = K2C: test and
// compaction only (after the collective), kept atoms counted; 3 = K2F (single GPU, residual
// pass running concurrently over the unreduced iterate): test, compaction, vectors and sums,
// no support list; dropped = a screened unit carries a nonzero x or b (FIXUP trip).
template <bool GROUP>
__device__ __forceinline__ void k2_body(const Params& P, int b, int G) {
    __shared__ int s_scan[2 * NW + 1];
    __shared__ double s_sh[64];
    __shared__ int s_off[K3_WIN];
    __shared__ int s_s0;
    dscr_scalars* sc = P.sc;
    const int var = P.k2v;
    const bool static_mode = (sc->mode == MODE_STATIC);
    const bool fix_pre = (var == 1 && sc->mode == MODE_FIXUP);   // K2S of a FIXUP trip: reduced list
    const int p = sc->parity, xi = sc->xi;
    const int lp = fix_pre ? (p ^ 1) : p;                         // list read
    const int nu = fix_pre ? sc->n_units_new : sc->n_units;
    const int lo = (int)(((long long)nu * b) / G), hi = (int)(((long long)nu * (b + 1)) / G);
    const int* act = P.act[lp];
    const int* off = P.act_off[lp];
    int* actn = P.act[p ^ 1] + (size_t)b * P.cap;
    const bool test_on = (var == 1) ? false : (static_mode ? true : (P.strategy == DSCR_DYNAMIC));
    const bool do_list = (var != 1);                 // compaction into the next list
    const bool do_vec = !static_mode && var != 2;    // vectors, support list, sums
    const bool do_sup = do_vec && var != 3;           // support list for K3a
    const bool want_ext = (var == 1) && P.strategy == DSCR_DYNAMIC && P.test != DSCR_DOME && !fix_pre;
    const int algo = P.algo;
    const double* xc = P.x[xi];
    const double* xn = P.x[(xi + 1) % 3];
    double* un = P.u[p ^ 1];
    const double beta = sc->beta, phi = sc->phi;
    const bool keep_masked_a = (algo == DSCR_ISTA || algo == DSCR_FISTA);
    int* sidx = P.sidx + (size_t)b * P.sup_cap;
    double* sa = P.sa + (size_t)b * P.sup_cap;
    double* sb = P.sb + (size_t)b * P.sup_cap;

    int n_keep = 0, n_sup = 0;
    double pen = 0.0, nnz = 0.0, kept_atoms = 0.0, ssr = 0.0, dropped = 0.0;
    double tmax = -INFINITY, vmin = INFINITY;
    int wend = INT_MIN;
    const bool ident = (nu == P.n_units);   // nothing screened yet: identity list
    // Lasso, identity list, more units than threads (c4: ~886 per CTA): 4 consecutive units per
    // thread and round, so one round (two block scans) covers up to 4*NT units.  Lists and
    // support entries come out in unit order, exactly as in the one-unit-per-thread rounds.
    const bool wide = !GROUP && ident && !static_mode && (hi - lo) > NT;
    for (int base = lo; wide && base < hi; base += 4 * NT) {
        constexpr int Q = 4;
        const int f0 = base + Q * threadIdx.x;
        double cand[Q], xcv[Q], bvq[Q];
        bool valid[Q], keep[Q], sup[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            valid[q] = f0 + q < hi;
            cand[q] = 0.0; xcv[q] = 0.0;
            if (valid[q] && do_vec) { cand[q] = xn[f0 + q]; xcv[q] = xc[f0 + q]; }
        }
        int nk = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const bool masked = valid[q] && test_on && unit_test(P, sc, f0 + q);
            if (valid[q] && do_list) P.mask[f0 + q] = masked ? 1 : 0;
            keep[q] = valid[q] && !masked;
            nk += keep[q] ? 1 : 0;
            if (var == 2 && keep[q]) kept_atoms += 1.0;
        }
        if (do_list) {
            int tot;
            int pos = n_keep + block_exscan(nk, s_scan, &tot);
#pragma unroll
            for (int q = 0; q < Q; ++q) if (keep[q]) { DSCR_CHECK(pos < P.cap); actn[pos++] = f0 + q; }
            n_keep += tot;
        }
        if (!do_vec) continue;
        int ns = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            bvq[q] = 0.0;
            sup[q] = false;
            if (!valid[q]) continue;
            const int j = f0 + q;
            const double c = cand[q];
            if (keep[q]) {
                double bv = 0.0;
                if (algo == DSCR_FISTA) { bv = c + beta * (c - xcv[q]); un[j] = bv; }
                else if (algo == DSCR_CP) { bv = c + phi * (c - xcv[q]); un[j] = bv; }
                else if (algo == DSCR_SPARSA) { bv = c - xcv[q]; ssr += bv * bv; }
                bvq[q] = bv;
                sup[q] = (c != 0.0 || bv != 0.0);
                pen += fabs(c);
                nnz += (c != 0.0) ? 1.0 : 0.0;
                kept_atoms += 1.0;
            } else if (var == 3) {
                if (c != 0.0 || b_value(algo, c, xcv[q], beta, phi) != 0.0) dropped = 1.0;
            } else if (c != 0.0) {
                dropped = 1.0;
                sup[q] = keep_masked_a;
            }
            if (want_ext) {
                const double v = unit_value(P, j);
                vmin = fmin(vmin, v);
                if (c != 0.0 || bvq[q] != 0.0) tmax = fmax(tmax, v);
            }
            ns += sup[q] ? 1 : 0;
        }
        if (!do_sup) continue;
        int tot;
        int w = n_sup + block_exscan(ns, s_scan, &tot);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (!sup[q]) continue;
            const int j = f0 + q;
            DSCR_CHECK(w < P.sup_cap && j >= 0 && j < P.kcols);
            if (keep[q]) { sidx[w] = j; sa[w] = cand[q]; sb[w] = bvq[q]; }
            else { sidx[w] = ~j; sa[w] = cand[q]; sb[w] = 0.0; }
            ++w;
        }
        n_sup += tot;
    }
    for (int base = lo; !wide && base < hi; base += NT) {
        if (!ident && base >= wend) wend = stage_window(off, P.G, base, s_off, &s_s0);   // uniform
        const int f = base + threadIdx.x;
        const bool valid = f < hi;
        int unit = -1;
        if (valid) {
            if (ident) {
                unit = f;
            } else {
                const int s = window_slot(off, P.G, s_off, s_s0, wend, f);
                unit = act[s * P.cap + (f - off[s])];
            }
        }
        // Lasso: the unit's x values are loaded with the test inputs (one round trip)
        double cand0 = 0.0, xc0 = 0.0;
        if (!GROUP && valid && do_vec) { cand0 = xn[unit]; xc0 = xc[unit]; }
        const bool masked = valid && test_on && unit_test(P, sc, unit);
        if (valid && !static_mode && do_list) P.mask[f] = masked ? 1 : 0;
        const bool keep = valid && !masked;
        if (do_list) {
            int tot;
            const int pos = block_exscan(keep ? 1 : 0, s_scan, &tot);
            if (keep) { DSCR_CHECK(n_keep + pos < P.cap && unit >= 0 && unit < P.n_units); actn[n_keep + pos] = unit; }
            n_keep += tot;
        }
        if (var == 2 && keep) kept_atoms += (double)(unit_atom_hi(P, unit) - unit_atom_lo(P, unit));
        if (!do_vec) continue;

        // per-atom vectors and support entries of this unit
        int my_sup = 0;
        double bv0 = 0.0;   // Lasso: b value of the unit's atom, reused for the support entry
        if (valid) {
            const int j0 = unit_atom_lo(P, unit), j1 = unit_atom_hi(P, unit);
            bool carries = false;
            // groups: the atoms' x values are loaded 4 at a time (all in flight) before use
            constexpr int GB = GROUP ? 4 : 1;
            double gxn[GB], gxc[GB];
            for (int j = j0; j < j1; ++j) {
                const int jj = (j - j0) % GB;
                if (GROUP && jj == 0) {
#pragma unroll
                    for (int q = 0; q < GB; ++q) {
                        gxn[q] = (j + q < j1) ? xn[j + q] : 0.0;
                        gxc[q] = (j + q < j1) ? xc[j + q] : 0.0;
                    }
                }
                double cand = cand0, xcj = xc0;
                if (GROUP) {
#pragma unroll
                    for (int q = 0; q < GB; ++q) if (q == jj) { cand = gxn[q]; xcj = gxc[q]; }
                }
                if (keep) {
                    double bv = 0.0;
                    if (algo == DSCR_FISTA) { bv = cand + beta * (cand - xcj); un[j] = bv; }
                    else if (algo == DSCR_CP) { bv = cand + phi * (cand - xcj); un[j] = bv; }
                    else if (algo == DSCR_SPARSA) { bv = cand - xcj; ssr += bv * bv; }
                    bv0 = bv;
                    if (cand != 0.0 || bv != 0.0) { ++my_sup; carries = true; }
                    if (!GROUP) pen += fabs(cand);
                    nnz += (cand != 0.0) ? 1.0 : 0.0;
                    kept_atoms += 1.0;
                } else if (var == 3) {
                    if (cand != 0.0 || b_value(algo, cand, xcj, beta, phi) != 0.0) dropped = 1.0;
                } else {
                    if (cand != 0.0) { dropped = 1.0; if (keep_masked_a) ++my_sup; }
                }
            }
            if (GROUP && keep) {
                const double nx = sqrt(np_segment_sum([&](int i) { double t = xn[i]; return t * t; }, j0, j1 - j0));
                pen += P.gw[unit] * nx;
            }
            if (want_ext) {
                const double v = unit_value(P, unit);
                vmin = fmin(vmin, v);
                if (carries) tmax = fmax(tmax, v);
            }
        }
        if (!do_sup) continue;
        int tot;
        const int spos = block_exscan(my_sup, s_scan, &tot);
        if (my_sup && !GROUP) {   // single atom: values from registers
            const int w = n_sup + spos;
            DSCR_CHECK(w < P.sup_cap);
            if (keep) { sidx[w] = unit; sa[w] = cand0; sb[w] = bv0; }
            else { sidx[w] = ~unit; sa[w] = cand0; sb[w] = 0.0; }
        } else if (my_sup) {
            int w = n_sup + spos;
            const int j0 = unit_atom_lo(P, unit), j1 = unit_atom_hi(P, unit);
            double gxn[4], gb[4];
            for (int j = j0; j < j1; ++j) {
                const int jj = (j - j0) % 4;
                if (jj == 0) {   // 4 atoms' values in flight at once
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool in = j + q < j1;
                        gxn[q] = in ? xn[j + q] : 0.0;
                        gb[q] = 0.0;
                        if (in && (algo == DSCR_FISTA || algo == DSCR_CP)) gb[q] = un[j + q];
                        else if (in && algo == DSCR_SPARSA) gb[q] = xc[j + q];
                    }
                }
                double cand = 0.0, gq = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) if (q == jj) { cand = gxn[q]; gq = gb[q]; }
                if (keep) {
                    double bv = 0.0;
                    if (algo == DSCR_FISTA || algo == DSCR_CP) bv = gq;
                    else if (algo == DSCR_SPARSA) bv = cand - gq;
                    if (cand != 0.0 || bv != 0.0) { DSCR_CHECK(w < P.sup_cap); sidx[w] = j; sa[w] = cand; sb[w] = bv; ++w; }
                } else if (cand != 0.0) {
                    DSCR_CHECK(w < P.sup_cap);
                    sidx[w] = ~j; sa[w] = cand; sb[w] = 0.0; ++w;
                }
            }
        }
        n_sup += tot;
    }
    // per-CTA outputs
    if (threadIdx.x == 0) {
        if (do_list) P.act_cnt[p ^ 1][b] = n_keep;
        if (do_sup) P.sup_cnt[b] = n_sup;
    }
    if (!static_mode) {
        double v5[5] = {pen, nnz, kept_atoms, ssr, dropped};
        block_sum_n<5>(v5, s_sh);
        double ext[2] = {tmax, -vmin};
        if (want_ext) block_max_n<2>(ext, s_sh);
        if (threadIdx.x == 0) {
            double* o = P.p2 + (size_t)b * NP2X;
            o[0] = v5[0]; o[1] = v5[1]; o[2] = v5[2]; o[3] = v5[3]; o[4] = v5[4];
            o[5] = ext[0]; o[6] = -ext[1];
        }
    }
}

// K2 tail: slot scans (new active list offsets, support offsets), partial reduction
template <bool GROUP>
__device__ void k2_final(const Params& P, int G) {
    __shared__ int s_scan[2 * NW + 1];
    __shared__ double s_sh[64];
    dscr_scalars* sc = P.sc;
    const int var = P.k2v;
    const bool static_mode = (sc->mode == MODE_STATIC);
    const bool do_list = (var != 1);
    const bool do_vec = !static_mode && var != 2 && var != 3;   // support-list offsets (K3a)
    const int p = sc->parity;

    // ---- last CTA: scans of the slot counts, fixed-order partial reduction.  Every count and
    // partial this thread needs is loaded up front (one round trip), then scanned.
    constexpr int KPF = 5;                       // prefetched slots per thread (G <= KPF * NT)
    const bool pf = P.G <= KPF * NT;
    int cnv[KPF], scv[KPF];
    double pv[KPF][7];
    if (pf) {
#pragma unroll
        for (int k = 0; k < KPF; ++k) {
            const int i = k * NT + threadIdx.x;
            const bool in = i < P.G;
            cnv[k] = (in && do_list) ? P.act_cnt[p ^ 1][i] : 0;
            scv[k] = (in && do_vec) ? P.sup_cnt[i] : 0;
            const double* o = P.p2 + (size_t)i * NP2X;
#pragma unroll
            for (int q = 0; q < 7; ++q) pv[k][q] = (in && !static_mode) ? o[q] : ((q == 5) ? -INFINITY : (q == 6 ? INFINITY : 0.0));
        }
    }
    {
        int carry = 0, carry_s = 0;
        int* offn = P.act_off[p ^ 1];
        const int* cn = P.act_cnt[p ^ 1];
        for (int base = 0, kk = 0; base < P.G; base += NT, ++kk) {
            const int i = base + threadIdx.x;
            int tot;
            if (do_list) {
                int v = 0;
                if (pf) {
#pragma unroll
                    for (int k = 0; k < KPF; ++k) if (k == kk) v = cnv[k];
                } else {
                    v = (i < P.G) ? cn[i] : 0;
                }
                const int e = block_exscan(v, s_scan, &tot);
                if (i < P.G && P.writer) offn[i] = carry + e;
                carry += tot;
            }
            if (do_vec) {
                int vs = 0;
                if (pf) {
#pragma unroll
                    for (int k = 0; k < KPF; ++k) if (k == kk) vs = scv[k];
                } else {
                    vs = (i < P.G) ? P.sup_cnt[i] : 0;
                }
                const int es = block_exscan(vs, s_scan, &tot);
                if (i < P.G) P.sup_off[i] = carry_s + es;
                carry_s += tot;
            }
        }
        if (threadIdx.x == 0) {
            if (do_list) {
                if (P.writer) offn[P.G] = carry;
                sc->n_units_new = carry;
            }
            if (do_vec) {
                P.sup_off[P.G] = carry_s;
                sc->n_support = carry_s;
                int pe = (carry_s + P.min_cols - 1) / P.min_cols;
                sc->p_eff = max(1, min(P.P, pe));
            }
        }
    }
    if (static_mode) {
        __syncthreads();
        if (threadIdx.x == 0) {
            sc->n_units = sc->n_units_new;
            sc->parity ^= 1;
            sc->mode = MODE_NORMAL;
            sc->static_done = 1;
        }
        return;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0, tmax = -INFINITY, vmin = INFINITY;
    if (pf) {
#pragma unroll
        for (int k = 0; k < KPF; ++k) {
            a0 += pv[k][0]; a1 += pv[k][1]; a2 += pv[k][2]; a3 += pv[k][3]; a4 += pv[k][4];
            tmax = fmax(tmax, pv[k][5]); vmin = fmin(vmin, pv[k][6]);
        }
    } else {
        for (int i = threadIdx.x; i < G; i += NT) {
            const double* o = P.p2 + (size_t)i * NP2X;
            a0 += o[0]; a1 += o[1]; a2 += o[2]; a3 += o[3]; a4 += o[4];
            tmax = fmax(tmax, o[5]); vmin = fmin(vmin, o[6]);
        }
    }
    double r5[5] = {a0, a1, a2, a3, a4};
    block_sum_n<5>(r5, s_sh);
    a0 = r5[0]; a1 = r5[1]; a2 = r5[2]; a3 = r5[3]; a4 = r5[4];
    double ext[2] = {tmax, -vmin};
    if (var == 1) block_max_n<2>(ext, s_sh);
    if (threadIdx.x == 0) {
        if (var == 2) {                    // K2C: local kept atoms after the test
            sc->kept_atoms = (int)a2;
        } else {
            sc->pen = a0;
            sc->nnz = (int)a1;
            sc->kept_atoms = (int)a2;
            sc->ss_red = a3;
            sc->dropped_nz = (a4 > 0.0);
        }
        if (var == 1 && sc->mode != MODE_FIXUP) {   // this rank's slot: test extremes, active units
            double* slot = P.comm + CM_VEC + 2 * P.ldd + OC_SLOT * P.oc_rank;
            slot[3] = ext[0];
            slot[4] = -ext[1];
            slot[5] = (double)sc->n_units;
        }
        stamp(P, 3);
    }
}

template <bool GROUP>
__global__ void __launch_bounds__(NT) k2_screen(Params P) {
    __shared__ int s_flag;
    pdl_wait();
    pdl_trigger();
    dscr_scalars* sc = P.sc;
    if (sc->stop) return;
    const int mode = sc->mode;
    if (mode == MODE_FIXUP && P.k2v != 1) return;
    const bool static_mode = (mode == MODE_STATIC);
    if (!static_mode && sc->t >= sc->run_limit) return;
    if (!static_mode && blockIdx.x == 0 && threadIdx.x == 0) stamp(P, 2);
    k2_body<GROUP>(P, blockIdx.x, gridDim.x);
    if (!last_block(P.tickets + 1, gridDim.x, &s_flag)) return;
    k2_final<GROUP>(P, gridDim.x);
}

// ---------------------------------------------------------------------------
// K3a: residual partials over the support list
// ---------------------------------------------------------------------------

constexpr int K3_CHUNK = 128;
template <typename T>
__device__ __forceinline__ void k3a_acc(const typename Vec<T>::Raw (&d)[4], const double* sa, const double* sb,
                                        double* acc_a, double* acc_b) {
    constexpr int V = Vec<T>::V;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double a = sa[q], bb = sb[q];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double x = Vec<T>::get(d[q], v);
            acc_a[v] = fma(a, x, acc_a[v]);
            acc_b[v] = fma(bb, x, acc_b[v]);
        }
    }
}

// rows r0..r0+V-1 of D_S [a b] for the cn staged entries (column s_idx[i], coefficients s_a[i],
// s_b[i]), accumulated in entry order; groups of 4 columns, the next group's loads in flight
// while this group accumulates
template <typename T>
__device__ __forceinline__ void k3a_stream(const T* D, int ldd, int r0, const int* s_idx, const double* s_a,
                                           const double* s_b, int cn, uint64_t pol, double* acc_a, double* acc_b) {
    constexpr int V = Vec<T>::V;
    const int ng = cn / 4;
    typename Vec<T>::Raw d0[4], d1[4];
    if (ng > 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) Vec<T>::load_raw(D + (size_t)s_idx[q] * ldd + r0, d0[q], pol);
    }
    int g = 0;
    for (; g + 2 <= ng; g += 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) Vec<T>::load_raw(D + (size_t)s_idx[4 * g + 4 + q] * ldd + r0, d1[q], pol);
        k3a_acc<T>(d0, s_a + 4 * g, s_b + 4 * g, acc_a, acc_b);
        if (g + 2 < ng) {
#pragma unroll
            for (int q = 0; q < 4; ++q) Vec<T>::load_raw(D + (size_t)s_idx[4 * g + 8 + q] * ldd + r0, d0[q], pol);
        }
        k3a_acc<T>(d1, s_a + 4 * g + 4, s_b + 4 * g + 4, acc_a, acc_b);
    }
    if (g < ng) k3a_acc<T>(d0, s_a + 4 * g, s_b + 4 * g, acc_a, acc_b);   // odd group count
    for (int i = 4 * ng; i < cn; ++i) {
        typename Vec<T>::Raw d;
        Vec<T>::load_raw(D + (size_t)s_idx[i] * ldd + r0, d, pol);
        const double a = s_a[i], bb = s_b[i];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double x = Vec<T>::get(d, v);
            acc_a[v] = fma(a, x, acc_a[v]);
            acc_b[v] = fma(bb, x, acc_b[v]);
        }
    }
}

template <typename T>
__device__ __forceinline__ void k3a_body(const Params& P, int tile, int split) {
    __shared__ int s_idx[K3_CHUNK];
    __shared__ double s_a[K3_CHUNK], s_b[K3_CHUNK];
    __shared__ int s_off[K3_WIN];
    __shared__ int s_s0;
    dscr_scalars* sc = P.sc;
    const bool fix = (sc->mode == MODE_FIXUP) && !P.onecoll;   // one collective: K2S rebuilt the list
    const int pe = sc->p_eff;
    if (split >= pe) return;
    const int nS = sc->n_support;
    const int lo = (int)(((long long)nS * split) / pe), hi = (int)(((long long)nS * (split + 1)) / pe);
    constexpr int V = Vec<T>::V;
    const int r0 = tile * P.TR + threadIdx.x * V;
    const bool rows_ok = r0 < P.n;
    const T* D = static_cast<const T*>(P.D);
    const uint64_t pol = make_policy(P.l2_keep);
    double acc_a[V], acc_b[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { acc_a[v] = 0.0; acc_b[v] = 0.0; }
    const int* off = P.sup_off;
    for (int c0 = lo; c0 < hi; c0 += K3_CHUNK) {
        const int cn = min(K3_CHUNK, hi - c0);
        const int wend = stage_window(off, P.G, c0, s_off, &s_s0);
        for (int i = threadIdx.x; i < cn; i += NT) {
            const int f = c0 + i;
            const int s = window_slot(off, P.G, s_off, s_s0, wend, f);
            const size_t e = (size_t)s * P.sup_cap + (f - off[s]);
            DSCR_CHECK(s >= 0 && s < P.G && f - off[s] >= 0 && f - off[s] < P.sup_cap);
            int idx = P.sidx[e];
            DSCR_CHECK((idx < 0 ? ~idx : idx) < P.kcols);
            double a = P.sa[e], bb = P.sb[e];
            if (fix) {
                if (idx < 0) a = 0.0;   // masked entry: excluded from the reduced iterate
                bb = 0.0;
            }
            s_idx[i] = idx < 0 ? ~idx : idx;
            s_a[i] = a;
            s_b[i] = bb;
        }
        __syncthreads();
        if (rows_ok) k3a_stream<T>(D, P.ldd, r0, s_idx, s_a, s_b, cn, pol, acc_a, acc_b);
    }
    if (rows_ok) {
        double* pa = P.p3v + ((size_t)split * 2) * P.ldd + r0;
        double* pb = P.p3v + ((size_t)split * 2 + 1) * P.ldd + r0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (r0 + v < P.ldd) { pa[v] = acc_a[v]; pb[v] = acc_b[v]; }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(NT) k3a_residual(Params P) {
    pdl_wait();
    pdl_trigger();
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    if (sc->mode == MODE_STATIC) return;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) stamp(P, 4);
    k3a_body<T>(P, blockIdx.x, blockIdx.y);
}

// K3a-scan (single GPU, with K2 running concurrently): the residual partials over the
// *unreduced* iterate, read straight from x_{t+1} (written by K1) and the current active list
// -- no support list from K2, so K2's test / compaction and this pass overlap.  Split `split`
// of P23 scans the active units [nu*split/P23, nu*(split+1)/P23) in rounds of K3S_UNITS
// (4 consecutive units per thread on the identity list), stages the atoms with a nonzero
// a = x_{t+1} or b (b_value) in shared memory in unit order and streams their columns.  A
// FIXUP trip (K2 found a screened unit carrying a nonzero a or b) rescans the compacted list.
constexpr int K3S_UNITS = 4 * NT;

template <typename T, bool GROUP>
__device__ __forceinline__ void k3a_scan_body(const Params& P, int tile, int split) {
    __shared__ int s_idx[K3S_UNITS];
    __shared__ double s_a[K3S_UNITS], s_b[K3S_UNITS];
    __shared__ int s_scan[2 * NW + 1];
    __shared__ int s_off[K3_WIN];
    __shared__ int s_s0;
    dscr_scalars* sc = P.sc;
    const bool fixup = (sc->mode == MODE_FIXUP);
    const int p = sc->parity, xi = sc->xi;
    const int lp = fixup ? (p ^ 1) : p;
    const int nu = fixup ? sc->n_units_new : sc->n_units;
    const int* act = P.act[lp];
    const int* off = P.act_off[lp];
    const bool ident = !fixup && (nu == P.n_units);
    const int S = P.P23;
    const int lo = (int)(((long long)nu * split) / S), hi = (int)(((long long)nu * (split + 1)) / S);
    const double* xn = P.x[(xi + 1) % 3];
    const double* xc = P.x[xi];
    const int algo = P.algo;
    const double beta = sc->beta, phi = sc->phi;
    constexpr int V = Vec<T>::V;
    const int r0 = tile * P.TR + threadIdx.x * V;
    const bool rows_ok = r0 < P.n;
    const T* D = static_cast<const T*>(P.D);
    const uint64_t pol = make_policy(P.l2_keep);
    double acc_a[V], acc_b[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { acc_a[v] = 0.0; acc_b[v] = 0.0; }
    int count = 0;
    const int upr = GROUP ? max(1, min(NT, K3S_UNITS / max(1, P.max_gsize))) : K3S_UNITS;   // units per round
    int wend = INT_MIN;
    for (int u0 = lo; u0 < hi; u0 += upr) {
        const int cu = min(upr, hi - u0);
        if (!ident && u0 + cu > wend) wend = stage_window(off, P.G, u0, s_off, &s_s0);   // uniform
        // this thread's units: 4 consecutive flat positions (Lasso) or one group
        constexpr int Q = GROUP ? 1 : 4;
        int units[Q];
        int my = 0;
        double av[GROUP ? 1 : 4], bv[GROUP ? 1 : 4];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int f = u0 + Q * threadIdx.x + q;
            units[q] = -1;
            if (f < u0 + cu) {
                if (ident) units[q] = f;
                else {
                    const int sl = window_slot(off, P.G, s_off, s_s0, wend, f);
                    units[q] = act[sl * P.cap + (f - off[sl])];
                }
            }
        }
        if (!GROUP) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                av[q] = 0.0; bv[q] = 0.0;
                if (units[q] >= 0) {
                    av[q] = xn[units[q]];
                    bv[q] = b_value(algo, av[q], xc[units[q]], beta, phi);
                }
                my += (av[q] != 0.0 || bv[q] != 0.0) ? 1 : 0;
            }
        } else if (units[0] >= 0) {
            // 8 atoms' x values in flight at a time
            const int j0 = unit_atom_lo(P, units[0]), j1 = unit_atom_hi(P, units[0]);
            for (int jb = j0; jb < j1; jb += 8) {
                double xa[8], xb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    xa[q] = (jb + q < j1) ? xn[jb + q] : 0.0;
                    xb[q] = (jb + q < j1) ? xc[jb + q] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    my += (jb + q < j1 && (xa[q] != 0.0 || b_value(algo, xa[q], xb[q], beta, phi) != 0.0)) ? 1 : 0;
            }
        }
        int tot;
        int w = block_exscan(my, s_scan, &tot);
        if (!GROUP) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (av[q] != 0.0 || bv[q] != 0.0) {
                    DSCR_CHECK(w < K3S_UNITS && units[q] < P.kcols);
                    s_idx[w] = units[q]; s_a[w] = av[q]; s_b[w] = bv[q]; ++w;
                }
        } else if (my) {
            const int j0 = unit_atom_lo(P, units[0]), j1 = unit_atom_hi(P, units[0]);
            for (int jb = j0; jb < j1; jb += 8) {
                double xa[8], xb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    xa[q] = (jb + q < j1) ? xn[jb + q] : 0.0;
                    xb[q] = (jb + q < j1) ? xc[jb + q] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double b = b_value(algo, xa[q], xb[q], beta, phi);
                    if (jb + q < j1 && (xa[q] != 0.0 || b != 0.0)) {
                        DSCR_CHECK(w < K3S_UNITS && jb + q < P.kcols);
                        s_idx[w] = jb + q; s_a[w] = xa[q]; s_b[w] = b; ++w;
                    }
                }
            }
        }
        __syncthreads();
        if (rows_ok && tot) k3a_stream<T>(D, P.ldd, r0, s_idx, s_a, s_b, tot, pol, acc_a, acc_b);
        count += tot;
        __syncthreads();
    }
    if (rows_ok) {
        double* pa = P.p3v + ((size_t)split * 2) * P.ldd + r0;
        double* pb = P.p3v + ((size_t)split * 2 + 1) * P.ldd + r0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (r0 + v < P.ldd) { pa[v] = acc_a[v]; pb[v] = acc_b[v]; }
        }
    }
    if (tile == 0 && threadIdx.x == 0) P.p3c[split] = count;
}

template <typename T, bool GROUP>
__global__ void __launch_bounds__(NT) k3a_scan(Params P) {
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) return;
    if (sc->mode == MODE_STATIC) return;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) stamp(P, 4);
    k3a_scan_body<T, GROUP>(P, blockIdx.x, blockIdx.y);
}

// ---------------------------------------------------------------------------
// K3b: split reduction, finalize rows, iteration epilogue
// ---------------------------------------------------------------------------

__device__ __forceinline__ void set_cond(const Params& P, unsigned v) {
    if (P.in_graph) cudaGraphSetConditional(P.h_main, v);
}

__device__ void iteration_epilogue(const Params& P, dscr_scalars* sc, double s_qa2, double s_tn2, double s_tny,
                                   double s_ds2) {
    const int algo = P.algo;
    const int mode = sc->mode;
    if (mode != MODE_FIXUP) {
        // reference order: the backtracking loop first (a non-finite candidate fails the
        // majorization test and is retried with a larger L, solvers.py:176-187), then the
        // finiteness check of the accepted step (solvers.py:157-159, 196), then the screening
        // radius guard (screening.py:199-205)
        const bool bt = (algo == DSCR_ISTA || algo == DSCR_FISTA);
        if (bt) {
            // majorization test of the backtracking step (solvers.py:176-187)
            const double f0 = 0.5 * sc->theta_sq;
            const double fc = 0.5 * s_qa2;
            const double L = sc->L;
            const double bound = f0 + sc->maj_cs + 0.5 * L * sc->maj_ss;
            if (!(fc <= bound + MAJ_SLACK * fmax(1.0, f0))) {
                const double Ln = L * P.bt_factor;
                sc->L = Ln;
                if (Ln > L_CEILING) {
                    sc->status = DSCR_ENONFINITE;
                    sc->stop = DSCR_STOP_ERROR;
                    set_cond(P, 0);
                    return;
                }
                sc->mode = MODE_REDO;
                sc->trips += 1;
                return;
            }
        }
        if (sc->nonfinite) {
            sc->status = DSCR_ENONFINITE;
            sc->stop = DSCR_STOP_ERROR;
            set_cond(P, 0);
            return;
        }
        if (sc->status != DSCR_OK) {   // radius guard tripped in K1
            sc->stop = DSCR_STOP_ERROR;
            set_cond(P, 0);
            return;
        }
        if (bt && !P.f23) {
            if (sc->dropped_nz && !P.onecoll) {
                // resid must be recomputed on the reduced iterate (solvers.py:354-355)
                sc->spare = s_tn2;
                sc->ds_sq = s_tny;
                sc->mode = MODE_FIXUP;
                sc->trips += 1;
                return;
            }
        }
        if ((P.onecoll || P.f23) && sc->dropped_nz) {
            // one collective / concurrent K2 + K3a-scan: the residuals were taken on the unreduced
            // iterate; a screened unit carried a nonzero x or u / s, so both are recomputed on the
            // reduced iterate
            sc->mode = MODE_FIXUP;
            sc->trips += 1;
            return;
        }
    } else if (algo == DSCR_FISTA && !P.onecoll && !P.f23) {
        s_tn2 = sc->spare;   // theta_{t+1} = D u - y from the normal trip
        s_tny = sc->ds_sq;
    }
    // ---- accept the iteration
    const double lam = P.lam;
    const double F = 0.5 * s_qa2 + lam * sc->pen;
    const double gap = F - 0.5 * sc->yy + 0.5 * lam * lam * sc->rsafe_sq;
    const double L_used = sc->L;
    if (algo == DSCR_FISTA) sc->l_acc = sc->l_new;
    if (algo == DSCR_CP) { sc->tau = sc->phi * sc->tau; sc->sigma = sc->sigma_new; }
    if (algo == DSCR_SPARSA && sc->ss_red > 0.0) {
        sc->L = fmin(fmax(s_ds2 / sc->ss_red, P.bb_min), P.bb_max);   // solvers.py:275
    }
    const int t = sc->t + 1;
    sc->t = t;
    sc->trips += 1;
    sc->F = F;
    sc->gap = gap;
    sc->fc = s_qa2;
    const int nnz = sc->nnz;
    if (t <= P.max_iters && P.writer) {
        double* row = P.trace + (size_t)(t - 1) * DSCR_TRACE_FIELDS;
        row[DSCR_TR_T] = t;
        row[DSCR_TR_KEPT] = sc->kept_atoms;
        row[DSCR_TR_NNZ] = nnz;
        row[DSCR_TR_OBJ] = F;
        row[DSCR_TR_GAP] = gap;
        row[DSCR_TR_RADIUS] = (P.strategy == DSCR_DYNAMIC) ? sc->radius : NAN;
        row[DSCR_TR_L] = L_used;
        row[DSCR_TR_NS] = (double)globaltimer() - sc->t0_ns;
        row[DSCR_TR_UNITS] = sc->n_units_new;
        row[DSCR_TR_SUPPORT] = sc->n_support;
    }
    sc->moved = sc->moved || (nnz > 0);
    int stop = DSCR_RUNNING;
    if (sc->moved && sc->have_fprev && fabs(sc->f_prev - F) / fmax(F, 1e-300) < P.rel_tol)
        stop = DSCR_STOP_RELTOL;
    else if (P.gap_tol > 0.0 && gap <= P.gap_tol)
        stop = DSCR_STOP_GAP;
    else if (P.onecoll ? (sc->oc_empty > 0.0) : (sc->kept_atoms == 0))
        stop = DSCR_STOP_EMPTY;
    else if (t >= P.max_iters)
        stop = DSCR_STOP_MAXITER;
    sc->f_prev = F;
    sc->have_fprev = 1;
    sc->theta_sq = s_tn2;
    sc->theta_y = s_tny;
    sc->n_units = sc->n_units_new;
    sc->parity ^= 1;
    sc->xi = (sc->xi + 1) % 3;
    sc->mode = MODE_NORMAL;
    sc->stop = stop;
    // the WHILE condition is 1 from k_preloop until a trip ends the loop: only the stop is
    // written (a device-side cudaGraphSetConditional every trip cost ~0.4 us per iteration on c1)
    if (!(stop == DSCR_RUNNING && t < sc->run_limit)) set_cond(P, 0u);
}

constexpr int K3B_ROWS = 32;                 // rows per CTA
constexpr int K3B_GROUPS = NT / K3B_ROWS;    // split groups per row

__device__ __forceinline__ void k3b_body(const Params& P, int rb) {
    __shared__ double s_sh[64];
    __shared__ double s_pa[K3B_GROUPS][K3B_ROWS], s_pb[K3B_GROUPS][K3B_ROWS];
    dscr_scalars* sc = P.sc;
    const int mode = sc->mode;
    const bool fix = (mode == MODE_FIXUP) && !P.onecoll && !P.f23;   // FIXUP re-derives a only
    const int algo = P.algo;
    const int p = sc->parity;
    const int pe = P.f23 ? P.P23 : sc->p_eff;
    // split reduction: group g sums splits g, g+8, ... ; groups combined in order (deterministic)
    {
        const int rr = threadIdx.x % K3B_ROWS, g = threadIdx.x / K3B_ROWS;
        const int r = rb * K3B_ROWS + rr;
        double a = 0.0, b = 0.0;
        if (r < P.n) {
            if (P.split) {
                if (g == 0) { a = P.comm[CM_VEC + r]; b = P.comm[CM_VEC + P.ldd + r]; }
            } else {
                for (int s = g; s < pe; s += K3B_GROUPS) {
                    a += P.p3v[((size_t)s * 2) * P.ldd + r];
                    b += P.p3v[((size_t)s * 2 + 1) * P.ldd + r];
                }
            }
        }
        s_pa[g][rr] = a;
        s_pb[g][rr] = b;
    }
    __syncthreads();
    double qa2 = 0.0, tn2 = 0.0, tny = 0.0, ds2 = 0.0;
    if (threadIdx.x < K3B_ROWS) {
        const int r = rb * K3B_ROWS + threadIdx.x;
        if (r < P.n) {
            double Sa = 0.0, Sb = 0.0;
#pragma unroll
            for (int g = 0; g < K3B_GROUPS; ++g) { Sa += s_pa[g][threadIdx.x]; Sb += s_pb[g][threadIdx.x]; }
            const double yr = P.y[r];
            const double qa = Sa - yr;            // D x - y (solvers.py:179, 487)
            P.resid[r] = qa;
            qa2 = qa * qa;
            double* thn = P.theta[p ^ 1];
            double tn = 0.0;
            bool have_tn = true;
            if (algo == DSCR_FISTA) {
                if (!fix) tn = Sb - yr; else have_tn = false;        // D u - y (solvers.py:212)
            } else if (algo == DSCR_CP) {
                if (!fix) {
                    const double q = Sb - yr;
                    const double sg = sc->sigma_new;
                    tn = (P.theta[p][r] + sg * q) / (1.0 + sg);          // solvers.py:299
                } else have_tn = false;
            } else {
                tn = qa;                                                   // resid carried as theta
                if (algo == DSCR_SPARSA && !fix) ds2 = Sb * Sb;
            }
            if (have_tn) {
                thn[r] = tn;
                tn2 = tn * tn;
                tny = tn * yr;
            }
        }
    }
    double q4[4] = {qa2, tn2, tny, ds2};
    block_sum_n<4>(q4, s_sh);
    qa2 = q4[0]; tn2 = q4[1]; tny = q4[2]; ds2 = q4[3];
    if (threadIdx.x == 0) {
        double* o = P.p3s + (size_t)rb * NP3;
        o[0] = qa2; o[1] = tn2; o[2] = tny; o[3] = ds2;
    }
}

__device__ void k3b_final(const Params& P, int G3) {
    __shared__ double s_sh[64];
    // the iteration epilogue is one thread's chain of scalar reads and writes: run it on a
    // shared-memory copy of the scalar block (one cooperative load, one write-back) instead of
    // a global round trip per field read after a write
    __shared__ double s_scw[sizeof(dscr_scalars) / 8];
    dscr_scalars* sc = reinterpret_cast<dscr_scalars*>(s_scw);
    {
        const double* g = reinterpret_cast<const double*>(P.sc);
        for (int i = threadIdx.x; i < (int)(sizeof(dscr_scalars) / 8); i += NT) s_scw[i] = g[i];
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, ns = 0.0;
    for (int i = threadIdx.x; i < G3; i += NT) {
        const double* o = P.p3s + (size_t)i * NP3;
        a0 += o[0]; a1 += o[1]; a2 += o[2]; a3 += o[3];
    }
    if (P.f23)                  // columns streamed by K3a-scan this trip (trace)
        for (int i = threadIdx.x; i < P.P23; i += NT) ns += (double)P.p3c[i];
    double r5[5] = {a0, a1, a2, a3, ns};
    block_sum_n<5>(r5, s_sh);   // (syncs: the scalar copy is complete)
    a0 = r5[0]; a1 = r5[1]; a2 = r5[2]; a3 = r5[3];
    if (P.f23 && threadIdx.x == 0) sc->n_support = (int)r5[4];
    if (threadIdx.x == 0) {
        stamp(P, 7);
        if (P.split) {      // global sums of the per-rank K1/K2 scalars
            const double* o = P.comm + CM_SUM;
            sc->pen = o[0]; sc->nnz = (int)llround(o[1]);
            sc->ss_red = o[3]; sc->maj_cs = o[5]; sc->maj_ss = o[6];
            if (!P.onecoll) { sc->kept_atoms = (int)llround(o[2]); sc->dropped_nz = o[4] > 0.0; }
            // one collective: kept_atoms stays this rank's count (trace; summed by the host),
            // dropped_nz comes from k1r_radius_oc
        }
        iteration_epilogue(P, sc, a0, a1, a2, a3);
    }
    __syncthreads();
    {
        double* g = reinterpret_cast<double*>(P.sc);
        for (int i = threadIdx.x; i < (int)(sizeof(dscr_scalars) / 8); i += NT) g[i] = s_scw[i];
    }
}


__global__ void __launch_bounds__(NT) k3b_finalize(Params P) {
    __shared__ int s_flag;
    pdl_wait();
    pdl_trigger();
    dscr_scalars* sc = P.sc;
    if (sc->stop || sc->t >= sc->run_limit) {
        // stopped earlier in this trip (K1: radius guard, non-finite iterate) or before it: end
        // the WHILE loop here too -- the epilogue below is skipped, so nothing else would
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(P, 0u);
        return;
    }
    if (sc->mode == MODE_STATIC) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) stamp(P, 6);
    k3b_body(P, blockIdx.x);
    if (!last_block(P.tickets + 2, gridDim.x, &s_flag)) return;
    k3b_final(P, gridDim.x);
}

// ---------------------------------------------------------------------------
// persistent engine: the whole iteration loop in one cooperative launch
// ---------------------------------------------------------------------------
//
// Every CTA runs the K1/K2/K3a/K3b bodies on its share of the work, separated by
// grid barriers; the tails (partial reductions, radius, slot scans, iteration
// epilogue) run redundantly in every CTA on a shared-memory copy of the scalar
// state.  The tails are deterministic, so all copies stay identical and no CTA
// waits on another's tail.  Four grid barriers per iteration, no launches.

// Grid barrier on a monotonic arrival counter (zeroed by the host before each launch): thread 0
// arrives with a fire-and-forget red.release and polls with ld.acquire until the count reaches
// epoch * n -- one L2 round trip to detect completion, no generation word, no fences around an
// atomic with a return value (that version measured ~3 us per barrier).  The acquire by thread 0
// followed by the CTA barrier orders every thread's later loads after all arrivals' earlier
// writes (and invalidates this SM's L1).
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned* /*gen*/, unsigned n, unsigned& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        epoch += 1u;
        const unsigned target = epoch * n;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(count) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

template <typename T, bool GROUP>
__global__ void __launch_bounds__(NT, 2) k_persistent(Params P0) {
    extern __shared__ double s_theta[];
    __shared__ dscr_scalars s_sc;
    __shared__ int s_supoff[PERS_MAX_G + 1];    // this CTA's copy of the support offsets
    Params P = P0;
    P.sc = &s_sc;
    P.sup_off = s_supoff;
    P.in_graph = 0;
    P.writer = (blockIdx.x == 0);
    const int G = gridDim.x;
    unsigned* bc = P0.tickets + 4;
    unsigned* bg = P0.tickets + 5;
    unsigned epoch = 0u;
    if (threadIdx.x == 0) {
        s_sc = *P0.sc;
        if (s_sc.stop == DSCR_RUNNING && s_sc.n_units == 0) s_sc.stop = DSCR_STOP_EMPTY;   // solvers.py:435
    }
    __syncthreads();
    for (;;) {
        if (s_sc.stop != DSCR_RUNNING || s_sc.t >= s_sc.run_limit || s_sc.t >= P.max_iters) break;
        const int mode = s_sc.mode;
        if (mode == MODE_NORMAL || mode == MODE_REDO) {
            if (threadIdx.x == 0) stamp(P, 0);
            k1_body<T, GROUP>(P, blockIdx.x, G, s_theta);
            grid_sync(bc, bg, G, epoch);
            k1_final<GROUP>(P, G);
            __syncthreads();
            if (threadIdx.x == 0) stamp(P, 2);
            k2_body<GROUP>(P, blockIdx.x, G);
            grid_sync(bc, bg, G, epoch);
            k2_final<GROUP>(P, G);
            __syncthreads();
        }
        if (threadIdx.x == 0) stamp(P, 4);
        const int nv = P.R * s_sc.p_eff;
        for (int v = blockIdx.x; v < nv; v += G) {
            k3a_body<T>(P, v % P.R, v / P.R);
            __syncthreads();
        }
        grid_sync(bc, bg, G, epoch);
        if (threadIdx.x == 0) stamp(P, 6);
        for (int v = blockIdx.x; v < P.G3b; v += G) {
            k3b_body(P, v);
            __syncthreads();
        }
        grid_sync(bc, bg, G, epoch);
        k3b_final(P, P.G3b);
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *P0.sc = s_sc;
}

// ---------------------------------------------------------------------------
// loop control and setup kernels
// ---------------------------------------------------------------------------

__global__ void k_preloop(Params P) {
    dscr_scalars* sc = P.sc;
    unsigned go = (sc->stop == DSCR_RUNNING && sc->t < sc->run_limit && sc->t < P.max_iters) ? 1u : 0u;
    if (sc->stop == DSCR_RUNNING && sc->n_units == 0) {   // solvers.py:435
        sc->stop = DSCR_STOP_EMPTY;
        go = 0u;
    }
    cudaGraphSetConditional(P.h_main, go);
}

__global__ void k_set_limit(dscr_scalars* sc, int limit) { sc->run_limit = limit; }

// zero state, active list = all units, theta_1, scalars
__global__ void k_init(Params P) {
    const size_t gt = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t gs = (size_t)gridDim.x * blockDim.x;
    for (size_t i = gt; i < (size_t)P.kcols; i += gs) {
        P.x[0][i] = 0.0; P.x[1][i] = 0.0; P.x[2][i] = 0.0;
        P.u[0][i] = 0.0; P.u[1][i] = 0.0;
        P.corr[i] = 0.0;
    }
    for (size_t f = gt; f < (size_t)P.n_units; f += gs) {
        P.act[0][f] = (int)f;   // slot f / cap, position f % cap
        P.act[1][f] = (int)f;
    }
    for (size_t s = gt; s <= (size_t)P.G; s += gs) {
        long long o = min((long long)s * P.cap, (long long)P.n_units);
        P.act_off[0][s] = (int)o;
        P.act_off[1][s] = (int)o;
        if (s < (size_t)P.G) {
            long long c = min((long long)P.cap, max(0LL, (long long)P.n_units - (long long)s * P.cap));
            P.act_cnt[0][s] = (int)c;
            P.act_cnt[1][s] = (int)c;
        }
    }
    // theta_1: -y, or (0 + sigma*(0 - y)) / (1 + sigma) for CP (solvers.py:296-299)
    const double sig = (P.algo == DSCR_CP) ? P.cp_safety / P.op_norm : 0.0;
    for (size_t r = gt; r < (size_t)P.ldd; r += gs) {
        double yr = (r < (size_t)P.n) ? P.y[r] : 0.0;
        double t;
        if (P.algo == DSCR_CP) t = (0.0 + sig * (0.0 - yr)) / (1.0 + sig);
        else t = 0.0 - yr;
        if (r >= (size_t)P.n) t = 0.0;
        P.theta[0][r] = t;
        P.theta[1][r] = t;
        P.resid[r] = 0.0 - yr;
    }
    if (gt == 0) {
        dscr_scalars* sc = P.sc;
        memset(sc, 0, sizeof(dscr_scalars));
        sc->run_limit = 0x7fffffff;
        sc->max_iters = P.max_iters;
        sc->n_units = P.n_units;
        sc->L = P.L0;
        sc->l_acc = 1.0;
        if (P.algo == DSCR_CP) { sc->tau = sig; sc->sigma = sig; }
        sc->radius = NAN;
        sc->t0_ns = (double)globaltimer();
        for (int i = 0; i < 8; ++i) P.tickets[i] = 0u;
    }
}

// ||y||^2, ||theta_1||^2, theta_1.y (single CTA)
__global__ void __launch_bounds__(NT) k_init_scalars(Params P) {
    __shared__ double s_sh[64];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int r = threadIdx.x; r < P.n; r += NT) {
        const double yr = P.y[r], t = P.theta[0][r];
        a = fma(yr, yr, a);
        b = fma(t, t, b);
        c = fma(t, yr, c);
    }
    a = block_sum(a, s_sh); b = block_sum(b, s_sh); c = block_sum(c, s_sh);
    if (threadIdx.x == 0) {
        P.sc->yy = a;
        P.sc->theta_sq = b;
        P.sc->theta_y = c;
    }
}

template <typename T>
__device__ __forceinline__ void k_correlate_cols(const T* __restrict__ D, int ldd, int n, int k, const double* sv,
                                                 double* out, uint64_t pol) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * NT) >> 5;
    // 4 adjacent columns per warp (4 x U loads of 32 B in flight per lane, U as in K1)
    for (int j0 = 4 * gw; j0 < k; j0 += 4 * nwarps) {
        const T* cols[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) cols[c] = (j0 + c < k) ? D + (size_t)(j0 + c) * ldd : nullptr;
        double cs[4];
        warp_dots<T, 4, K1Cfg<T>::U>(cols, n, sv, lane, pol, cs);
        if (lane < 4 && j0 + lane < k) {
            double c = cs[0];
#pragma unroll
            for (int q = 1; q < 4; ++q) if (lane == q) c = cs[q];
            out[j0 + lane] = c;
        }
    }
}

// out[j] = D[:, j] . v for all local columns (setup correlations, dictionary.py:94)
// VG: v read through L2 (dictionaries taller than the shared-memory staging buffer)
template <typename T, bool VG = false>
__global__ void __launch_bounds__(NT, 2) k_correlate(const T* __restrict__ D, int ldd, int n, int k,
                                                  const double* __restrict__ v, double* out,
                                                  const int* skip_flag, float l2_keep) {
    extern __shared__ double s_v[];
    if (skip_flag && *skip_flag) return;
    const uint64_t pol = make_policy(l2_keep);
    if constexpr (VG) {        // tall dictionary: v read through L2 (its padding rows are zero)
        k_correlate_cols<T>(D, ldd, n, k, v, out, pol);
    } else {
        for (int i = threadIdx.x; i < ldd; i += NT) s_v[i] = (i < n) ? v[i] : 0.0;
        __syncthreads();
        k_correlate_cols<T>(D, ldd, n, k, s_v, out, pol);
    }
}

// lambda_max with lowest-index argmax (problems.py:75-86), per-CTA partials + last CTA
__global__ void __launch_bounds__(NT) k_lmax(Params P) {
    __shared__ double s_v[NT];
    __shared__ int s_i[NT];
    __shared__ int s_flag;
    const int nu = P.n_units;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int u = blockIdx.x * NT + threadIdx.x; u < nu; u += gridDim.x * NT) {
        double val;
        if (P.n_groups) {
            const int j0 = P.gptr[u], j1 = P.gptr[u + 1];
            val = sqrt(np_segment_sum([&](int i) { double t = P.ycorr[i]; return t * t; }, j0, j1 - j0)) / P.gw[u];
        } else {
            val = fabs(P.ycorr[u]);
        }
        if (val > best || (val == best && u < bi)) { best = val; bi = u; }
    }
    s_v[threadIdx.x] = best;
    s_i[threadIdx.x] = bi;
    __syncthreads();
    for (int st = NT / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) {
            double ov = s_v[threadIdx.x + st];
            int oi = s_i[threadIdx.x + st];
            if (ov > s_v[threadIdx.x] || (ov == s_v[threadIdx.x] && oi < s_i[threadIdx.x])) {
                s_v[threadIdx.x] = ov; s_i[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        P.p1[blockIdx.x * 2] = s_v[0];
        P.p1[blockIdx.x * 2 + 1] = (double)s_i[0];
    }
    if (!last_block(P.tickets + 3, gridDim.x, &s_flag)) return;
    if (threadIdx.x == 0) {
        double bv = -1.0;
        int bidx = 0x7fffffff;
        for (int i = 0; i < (int)gridDim.x; ++i) {
            double v = P.p1[i * 2];
            int ii = (int)P.p1[i * 2 + 1];
            if (v > bv || (v == bv && ii < bidx)) { bv = v; bidx = ii; }
        }
        dscr_scalars* sc = P.sc;
        sc->lmax = bv;
        sc->lmax_unit = bidx;
        sc->lmax_index = bidx + (P.n_groups ? P.group_offset : P.col_offset);
        if (!P.n_groups) sc->lmax_sign = (P.ycorr[bidx] >= 0.0) ? 1.0 : -1.0;
        if (P.n_groups) sc->gstar_w = P.gw[bidx];
        if (P.split) {          // candidate for the cross-rank argmax (value, global index, sign)
            P.comm[CM_SETUP + 0] = bv;
            P.comm[CM_SETUP + 1] = (double)sc->lmax_index;
            P.comm[CM_SETUP + 2] = sc->lmax_sign;
        } else if (P.lam > bv) {                // solvers.py:384-397
            sc->trivial = 1;
            sc->stop = DSCR_STOP_TRIVIAL;
        }
    }
}

// a_* = sign * d_{i*} (Lasso) or the GST3 normal n = D_g* (D_g*^T y) / lambda_* (screening.py:238-243)
template <typename T>
__global__ void k_setup_vec(Params P) {
    const dscr_scalars* sc = P.sc;
    if (sc->stop) return;
    const T* D = static_cast<const T*>(P.D);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P.ldd; r += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (r < P.n) {
            if (P.n_groups == 0) {
                v = sc->lmax_sign * elem<T>(D + (size_t)sc->lmax_unit * P.ldd + r);
            } else {
                const int j0 = P.gptr[sc->lmax_unit], j1 = P.gptr[sc->lmax_unit + 1];
                double acc = 0.0;
                for (int j = j0; j < j1; ++j) acc = fma(elem<T>(D + (size_t)j * P.ldd + r), P.ycorr[j], acc);
                v = acc / sc->lmax;
            }
        }
        P.vec[r] = v;
    }
}

// GST3 scalars: ||n||^2, coef = n.y/lam - w_g*^2, shift^2 = coef^2/||n||^2 (screening.py:244-250)
__global__ void __launch_bounds__(NT) k_gst3_scalars(Params P) {
    __shared__ double s_sh[64];
    dscr_scalars* sc = P.sc;
    if (sc->stop) return;
    double a = 0.0, b = 0.0;
    for (int r = threadIdx.x; r < P.n; r += NT) {
        const double v = P.vec[r];
        a = fma(v, v, a);
        b = fma(v, P.y[r], b);
    }
    a = block_sum(a, s_sh);
    b = block_sum(b, s_sh);
    if (threadIdx.x == 0) {
        if (a == 0.0) {
            sc->status = DSCR_ERADIUS;
            sc->stop = DSCR_STOP_ERROR;
            return;
        }
        const double w = sc->gstar_w;
        const double coef = b / P.lam - w * w;
        sc->gst3_coef = coef;
        sc->gst3_nsq = a;
        sc->shift_sq = coef * coef / a;
    }
}

// ||d_j||_2 in fp64 for the norm-aware tests (reduced-precision dictionaries)
template <typename T>
__device__ __forceinline__ void colnorms_body(const T* D, int ldd, int n, int k, double* out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5, nw = (gridDim.x * NT) >> 5;
    for (int j = gw; j < k; j += nw) {
        double acc = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double d = elem<T>(D + (size_t)j * ldd + i);
            acc = fma(d, d, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) out[j] = sqrt(acc);
    }
}

template <typename T>
__global__ void __launch_bounds__(NT) k_colnorms(Params P) {
    if (P.sc->stop) return;
    colnorms_body<T>(static_cast<const T*>(P.D), P.ldd, P.n, P.kcols, P.anorm);
}

template <typename T>
__global__ void __launch_bounds__(NT) k_colnorms_op(const T* D, int ldd, int n, int k, double* out) {
    colnorms_body<T>(D, ldd, n, k, out);
}

// ||vec||^2 of the broadcast extremal atom (norm-aware DST3)
__global__ void __launch_bounds__(NT) k_vec_nsq(Params P) {
    __shared__ double s_sh[64];
    if (P.sc->stop) return;
    double a = 0.0;
    for (int r = threadIdx.x; r < P.n; r += NT) a = fma(P.vec[r], P.vec[r], a);
    a = block_sum(a, s_sh);
    if (threadIdx.x == 0) P.sc->astar_nsq = a;
}

// split mode: adopt the cross-rank lambda_* decision written by the host into comm
__global__ void k_setup_adopt(Params P) {
    dscr_scalars* sc = P.sc;
    const double* c = P.comm + CM_SETUP;
    sc->lmax = c[0];
    sc->lmax_index = (int)c[1];
    sc->lmax_sign = c[2];
    sc->gstar_w = c[5];
    sc->lmax_unit = (c[4] > 0.0) ? (int)c[6] : -1;     // owner keeps its local unit
    if (c[3] > 0.0) { sc->trivial = 1; sc->stop = DSCR_STOP_TRIVIAL; }
}

// test centre correlations (screening.py:213-255)
__global__ void k_centers(Params P) {
    dscr_scalars* sc = P.sc;
    if (sc->stop) return;
    const int test = P.test;
    const double lam = P.lam;
    const double shift = sc->lmax / lam - 1.0;
    // non-unit atoms: the DST3 half-space normal is a_*/||a_*||, at distance shift/||a_*|| from y/lam
    const double an2 = P.norm_aware ? sc->astar_nsq : 1.0;
    const double coef = P.norm_aware ? shift / an2 : shift;
    if (blockIdx.x == 0 && threadIdx.x == 0 && (test == DSCR_DST3 || test == DSCR_DOME))
        sc->shift_sq = P.norm_aware ? shift * shift / an2 : shift * shift;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.kcols; j += gridDim.x * blockDim.x) {
        const double safe = P.ycorr[j] / lam;
        double c = safe;
        if (test == DSCR_DST3) c = safe - coef * P.star[j];
        else if (test == DSCR_GST3) c = safe - (sc->gst3_coef / sc->gst3_nsq) * P.dn[j];
        P.cc[j] = c;
    }
}

__global__ void k_center_group_norms(Params P) {
    if (P.sc->stop) return;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < P.n_groups; g += gridDim.x * blockDim.x) {
        const int j0 = P.gptr[g], j1 = P.gptr[g + 1];
        P.cnorm[g] = sqrt(np_segment_sum([&](int i) { double t = P.cc[i]; return t * t; }, j0, j1 - j0));
    }
}

// static screen-once region at theta = y (screening.py:309-315)
__global__ void __launch_bounds__(NT) k_static_radius(Params P, int from_comm) {
    __shared__ double s_sh[64];
    __shared__ double s_m[NW];
    __shared__ int s_any[NW];
    dscr_scalars* sc = P.sc;
    if (sc->stop) return;
    double m = P.n_groups ? INFINITY : 0.0;
    int any = 0;
    for (int u = threadIdx.x; u < P.n_units; u += NT) {
        if (P.n_groups) {
            const int j0 = P.gptr[u], j1 = P.gptr[u + 1];
            double nc = sqrt(np_segment_sum([&](int i) { double t = P.ycorr[i]; return t * t; }, j0, j1 - j0));
            if (nc > 0.0) { m = fmin(m, P.gw[u] / nc); any = 1; }
        } else {
            m = fmax(m, fabs(P.ycorr[u]));
        }
    }
    m = P.n_groups ? warp_min(m) : warp_max(m);
    any = warp_isum(any);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { s_m[w] = m; s_any[w] = any; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = s_m[0]; int aa = s_any[0];
        for (int i = 1; i < NW; ++i) { mm = P.n_groups ? fmin(mm, s_m[i]) : fmax(mm, s_m[i]); aa += s_any[i]; }
        s_m[0] = mm; s_any[0] = aa;
    }
    __syncthreads();
    m = s_m[0];
    if (P.split && !from_comm) {      // publish the local bound, finish after the MAX collective
        if (threadIdx.x == 0) {
            P.comm[CM_MAX + 0] = P.n_groups ? (s_any[0] ? -m : -INFINITY) : m;
            P.comm[CM_MAX + 1] = 0.0;
            P.comm[CM_MAX + 2] = s_any[0] ? 1.0 : 0.0;
        }
        return;
    }
    bool any_g = s_any[0] != 0;
    if (from_comm) {
        m = P.n_groups ? -P.comm[CM_MAX + 0] : P.comm[CM_MAX + 0];
        any_g = P.comm[CM_MAX + 2] > 0.0;
    }
    double bound = P.n_groups ? (any_g ? m : INFINITY) : (m == 0.0 ? INFINITY : 1.0 / m);
    // theta = y: ||theta||^2 and theta.y are the same dot product
    radius_epilogue(P, bound, P.y, sc->yy, sc->yy, s_sh);
    if (threadIdx.x == 0) sc->mode = MODE_STATIC;
}

__global__ void k_static_done(Params P) {
    dscr_scalars* sc = P.sc;
    if (sc->mode == MODE_STATIC) sc->mode = MODE_NORMAL;   // trivial / error path
    sc->radius = NAN;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
    size_t total = 0;
    size_t add(size_t bytes) {
        size_t o = align_up(total, 256);
        total = o + bytes;
        return o;
    }
};

struct Geometry {
    int G, cap, sup_cap, TR, R, P, G3b, max_gsize, smem1, tile, theta_gl, P23;
};

static int dtype_size(int dt) { return dt == DSCR_F64 ? 8 : (dt == DSCR_F32 ? 4 : 2); }

// Fraction of the dictionary to keep L2-resident across iterations: all of it
// when it fits in ~3/4 of L2, a slice of that size when it is up to 3x L2,
// none (evict-first streaming) beyond.
static float l2_keep_fraction(size_t dict_bytes) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const double budget = 0.75 * (double)l2;
    if ((double)dict_bytes <= budget) return 1.0f;
    if ((double)dict_bytes <= 3.0 * l2) return (float)(budget / (double)dict_bytes);
    return 0.0f;
}

// Max dynamic shared memory attribute of a kernel.  The attribute is global per function and
// graphs created earlier keep launching with their own sizes, so it only ever grows (a later,
// smaller problem must not invalidate an earlier engine's launches).
static cudaError_t raise_smem(const void* fn, int smem) {
    static std::mutex mu;
    static std::map<const void*, int> cur;
    std::lock_guard<std::mutex> lk(mu);
    int& c = cur[fn];
    if (smem <= c) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) c = smem;
    return e;
}

template <typename T>
static int k1_occ_t(bool group, int smem) {
    int n = 0;
    if (group) {
        raise_smem((const void*)k1_corr_update<T, true>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_corr_update<T, true>, NT, smem);
    } else {
        raise_smem((const void*)k1_corr_update<T, false>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_corr_update<T, false>, NT, smem);
    }
    return std::max(1, n);
}

template <typename T>
static int pers_occ_t(bool group, int smem) {
    int n = 0;
    if (group) {
        raise_smem((const void*)k_persistent<T, true>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_persistent<T, true>, NT, smem);
    } else {
        raise_smem((const void*)k_persistent<T, false>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_persistent<T, false>, NT, smem);
    }
    return n;
}

static int pers_occupancy(int dtype, bool group, int smem) {
    if (dtype == DSCR_F64) return pers_occ_t<double>(group, smem);
    if (dtype == DSCR_F32) return pers_occ_t<float>(group, smem);
    return pers_occ_t<__nv_bfloat16>(group, smem);
}

template <typename T>
static int k3a_occ_t() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k3a_residual<T>, NT, 0);
    return std::max(1, n);
}

static int k3a_occupancy(int dtype) {
    if (dtype == DSCR_F64) return k3a_occ_t<double>();
    if (dtype == DSCR_F32) return k3a_occ_t<float>();
    return k3a_occ_t<__nv_bfloat16>();
}

static int k1_occupancy(int dtype, bool group, int smem) {
    if (dtype == DSCR_F64) return k1_occ_t<double>(group, smem);
    if (dtype == DSCR_F32) return k1_occ_t<float>(group, smem);
    return k1_occ_t<__nv_bfloat16>(group, smem);
}

static Geometry make_geometry(const dscr_problem_desc* pr, int n_units, int max_gsize) {
    Geometry g{};
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g.theta_gl = (size_t)pr->ldd * sizeof(double) > THETA_SMEM_MAX;   // tall: theta through L2
    g.smem1 = g.theta_gl ? 16 : pr->ldd * (int)sizeof(double);
    {   // K1 tiled path for short columns (DSCR_K1_TILE=0 forces the per-warp column path)
        const int segr = 32 * (32 / dtype_size(pr->dtype)) * (pr->dtype == DSCR_F64 ? K1Cfg<double>::U : 1);
        const int nseg = (pr->n_rows + segr - 1) / segr;
        const char* et = getenv("DSCR_K1_TILE");
        const char* em = getenv("DSCR_K1_TILE_MIN");   // experiment knob: smallest tiled segment count
        const int tmin = em ? atoi(em) : 5;
        g.tile = (nseg >= tmin && nseg <= K1T_SEGS && max_gsize <= 64 && !(et && !strcmp(et, "0"))) ? nseg : 0;
        if (g.tile) g.smem1 += K1T_ATOMS * g.tile * (int)sizeof(double);
    }
    // resident K1 CTAs per SM (registers + theta staging buffer): one full wave
    // one full wave; also co-resident for the persistent kernel (grid barriers)
    const int per_sm = std::max(1, std::min(k1_occupancy(pr->dtype, pr->n_groups > 0, g.smem1),
                                            std::max(1, pers_occupancy(pr->dtype, pr->n_groups > 0, g.smem1))));
    // >= 16 atoms per CTA (group problems: count atoms, not groups), at most one CTA per unit
    g.G = std::max(1, std::min(std::min((pr->n_cols + 15) / 16, n_units), sms * per_sm));
    if (const char* e = getenv("DSCR_MAX_CTAS")) g.G = std::max(1, std::min(g.G, atoi(e)));
    g.cap = (n_units + g.G - 1) / g.G;
    g.max_gsize = max_gsize;
    g.sup_cap = g.cap * max_gsize;
    const int V = 32 / dtype_size(pr->dtype);   // Vec<T>::V (32-byte loads)
    g.TR = NT * V;
    g.R = (pr->n_rows + g.TR - 1) / g.TR;
    g.P = std::max(1, (sms * k3a_occupancy(pr->dtype)) / g.R);   // (row tile x split) CTAs: one wave
    g.G3b = (pr->n_rows + K3B_ROWS - 1) / K3B_ROWS;
    // K3a-scan splits (fused graph): ~512 atoms scanned per split (measured on c1-c3: more splits
    // cost more in K3b's reduction and in slots taken from K2 than they save), one wave at most
    g.P23 = std::max(1, std::min(g.P, pr->n_cols / 512));
    if (const char* e = getenv("DSCR_P23")) g.P23 = std::max(1, std::min(g.P, atoi(e)));
    return g;
}

static int kts_slots(const dscr_config* cfg) { return std::min(std::max(cfg->max_iters, 1) + 64, 20000); }

struct Offsets {
    size_t sc, theta0, theta1, resid, corr, x0, x1, x2, u0, u1, ycorr, star, cc, cnorm, vec, dn;
    size_t act0, act1, cnt0, cnt1, off0, off1, mask, sidx, sa, sb, supcnt, supoff;
    size_t p1, p2, p3v, p3s, p3c, tickets, trace, kts, anorm, comm;
};

static Offsets make_offsets(const dscr_problem_desc* pr, const dscr_config* cfg, const Geometry& g,
                            int n_units, size_t* total) {
    Layout L;
    Offsets o{};
    const size_t K = (size_t)pr->n_cols, ldd = (size_t)pr->ldd, G = (size_t)g.G;
    const size_t ng = (size_t)std::max(pr->n_groups, 1);
    o.sc = L.add(sizeof(dscr_scalars));
    o.theta0 = L.add(ldd * 8); o.theta1 = L.add(ldd * 8); o.resid = L.add(ldd * 8);
    o.corr = L.add(K * 8);
    o.x0 = L.add(K * 8); o.x1 = L.add(K * 8); o.x2 = L.add(K * 8);
    o.u0 = L.add(K * 8); o.u1 = L.add(K * 8);
    o.ycorr = L.add(K * 8); o.star = L.add(K * 8); o.cc = L.add(K * 8); o.cnorm = L.add(ng * 8);
    o.vec = L.add(ldd * 8); o.dn = L.add(K * 8);
    const size_t slots = G * (size_t)g.cap;
    o.act0 = L.add(slots * 4); o.act1 = L.add(slots * 4);
    o.cnt0 = L.add(G * 4); o.cnt1 = L.add(G * 4);
    o.off0 = L.add((G + 1) * 4); o.off1 = L.add((G + 1) * 4);
    o.mask = L.add((size_t)n_units);
    const size_t ss = G * (size_t)g.sup_cap;
    o.sidx = L.add(ss * 4); o.sa = L.add(ss * 8); o.sb = L.add(ss * 8);
    o.supcnt = L.add(G * 4); o.supoff = L.add((G + 1) * 4);
    o.p1 = L.add(std::max<size_t>(G * NP1, 2 * (size_t)4096) * 8);
    o.p2 = L.add(G * NP2X * 8);
    o.p3v = L.add((size_t)g.P * 2 * ldd * 8);
    o.p3s = L.add((size_t)g.G3b * NP3 * 8);
    o.p3c = L.add((size_t)g.P * 4);
    o.tickets = L.add(64);
    o.trace = L.add((size_t)std::max(cfg->max_iters, 1) * DSCR_TRACE_FIELDS * 8);
    o.kts = L.add((size_t)kts_slots(cfg) * 8 * 8);
    o.anorm = L.add(K * 8);
    o.comm = L.add((CM_VEC + 2 * ldd + OC_SLOT * OC_MAX_WORLD) * 8);
    *total = L.total + 256;
    return o;
}

}  // namespace dscr

using namespace dscr;

struct dscr_solver {
    Params P;
    Geometry geo;
    dscr_problem_desc prob;
    dscr_config cfg;
    void* ws;
    cudaStream_t cap_stream = nullptr;
    cudaGraph_t g_setup = nullptr, g_loop = nullptr;
    cudaGraphExec_t e_setup = nullptr, e_loop = nullptr;
    int world = 1, rank = 0;
    void* comm = nullptr;
    bool pdl = false;   // chain kernels launched with programmatic dependent launch
    void** peer_tab_dev = nullptr;   // device copy of the peer pointer table
    cudaStream_t fork_stream = nullptr;          // K3a-scan branch of the captured trip (f23)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

extern "C" const char* dscr_last_error(void) { return err_store().c_str(); }
extern "C" int dscr_abi_version(void) { return DSCR_ABI_VERSION; }

// largest group size (1 for the Lasso); reads the device group pointer
static int group_max_size(const dscr_problem_desc* pr, int* out) {
    *out = 1;
    if (pr->n_groups <= 0) return DSCR_OK;
    if (!pr->group_ptr) return set_inval("group problems need group_ptr");
    std::vector<int> ptr(pr->n_groups + 1);
    CK(cudaMemcpy(ptr.data(), pr->group_ptr, ptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int g = 0; g < pr->n_groups; ++g) *out = std::max(*out, ptr[g + 1] - ptr[g]);
    return DSCR_OK;
}

// atoms any `cap` active units can hold: sum of the `cap` largest group sizes
static int max_atoms_per_slot(const dscr_problem_desc* pr, int cap, int* out) {
    if (pr->n_groups <= 0) { *out = cap; return DSCR_OK; }
    std::vector<int> ptr(pr->n_groups + 1);
    CK(cudaMemcpy(ptr.data(), pr->group_ptr, ptr.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<int> sz(pr->n_groups);
    for (int g = 0; g < pr->n_groups; ++g) {
        sz[g] = ptr[g + 1] - ptr[g];
        if (sz[g] < 1) return set_inval("groups must be nonempty");
    }
    if (ptr[0] != 0 || ptr[pr->n_groups] != pr->n_cols) return set_inval("groups must cover every column");
    std::sort(sz.begin(), sz.end(), std::greater<int>());
    long long acc = 0;
    for (int i = 0; i < std::min(cap, pr->n_groups); ++i) acc += sz[i];
    *out = (int)std::min<long long>(acc, pr->n_cols);
    return DSCR_OK;
}

static int validate(const dscr_problem_desc* pr, const dscr_config* cfg, int* n_units, int* max_gsize) {
    if (!pr || !cfg) return set_inval("null argument");
    if (pr->dtype < DSCR_F64 || pr->dtype > DSCR_BF16) return set_inval("unknown dtype");
    if (pr->n_rows < 1 || pr->n_cols < 1) return set_inval("dictionary must have at least one row and one column");
    if (pr->ldd < pr->n_rows || pr->ldd % 16) return set_inval("ldd must be >= n_rows and a multiple of 16");
    if (pr->ldd > (1 << 28)) return set_inval("n_rows too large");
    if (!(pr->lam > 0)) return set_inval("lam must be strictly positive");
    if (!pr->D || !pr->y) return set_inval("null device pointer");
    if (cfg->algorithm < DSCR_ISTA || cfg->algorithm > DSCR_CP) return set_inval("unknown algorithm");
    if (cfg->strategy < DSCR_NONE || cfg->strategy > DSCR_DYNAMIC) return set_inval("unknown strategy");
    if (cfg->max_iters < 1) return set_inval("max_iters must be at least 1");
    if (!(cfg->rel_tol > 0)) return set_inval("rel_tol must be positive");
    if (!(cfg->backtrack_factor > 1)) return set_inval("backtrack_factor must exceed 1");
    if (!(cfg->L0 > 0)) return set_inval("L0 must be positive");
    if (!(cfg->cp_step_safety > 0 && cfg->cp_step_safety < 1)) return set_inval("cp_step_safety must lie in (0, 1)");
    const bool group = pr->n_groups > 0;
    if (pr->norm_aware && cfg->strategy != DSCR_NONE && cfg->test == DSCR_DOME)
        return set_inval("the dome test requires unit-norm columns (norm_aware dictionaries: use safe or dst3)");
    if (cfg->strategy != DSCR_NONE) {
        if (cfg->test < 0) return set_inval("screening strategies require a test kind");
        bool lasso_test = cfg->test <= DSCR_DOME;
        if (group == lasso_test) return set_inval("test does not apply to this problem kind");
    }
    if ((cfg->algorithm == DSCR_CP || (cfg->algorithm == DSCR_TWIST && !(cfg->twist_step > 0))) && !(cfg->op_norm > 0))
        return set_inval("op_norm (||D||_2 > 0) is required for this algorithm");
    *n_units = group ? pr->n_groups : pr->n_cols;
    *max_gsize = 1;
    return DSCR_OK;
}

extern "C" size_t dscr_solver_workspace_size(const dscr_problem_desc* pr, const dscr_config* cfg) {
    int nu, mg;
    if (validate(pr, cfg, &nu, &mg) != DSCR_OK) return 0;
    if (group_max_size(pr, &mg) != DSCR_OK) return 0;
    Geometry g = make_geometry(pr, nu, mg);
    if (pr->n_groups > 0 && (!pr->group_ptr || max_atoms_per_slot(pr, g.cap, &g.sup_cap) != DSCR_OK)) return 0;
    size_t total;
    make_offsets(pr, cfg, g, nu, &total);
    return total;
}

// K1 kernel of a problem: dtype x (Lasso | groups) x (theta in shared memory | through L2)
static void (*k1_kernel(int dtype, bool group, bool tall))(Params) {
#define DSCR_K1_SEL(T) (group ? (tall ? k1_corr_update<T, true, true> : k1_corr_update<T, true>) \
                              : (tall ? k1_corr_update<T, false, true> : k1_corr_update<T, false>))
    switch (dtype) {
        case DSCR_F64: return DSCR_K1_SEL(double);
        case DSCR_F32: return DSCR_K1_SEL(float);
        default: return DSCR_K1_SEL(__nv_bfloat16);
    }
#undef DSCR_K1_SEL
}

// Kernel launch with optional programmatic stream serialization (PDL edges when captured).
template <typename... KArgs>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, size_t smem, cudaStream_t s, bool pdl,
                              const Params& P, int priority = INT_MIN) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (priority != INT_MIN) {   // graph node priority (the loop graph is instantiated with node priorities)
        at[na].id = cudaLaunchAttributePriority;
        at[na].val.priority = priority;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, P);
}

// greatest / least stream priority of the device (numerically lowest = greatest)
static void priority_range(int* greatest, int* least) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);   // (least, greatest)
    *least = lo;
    *greatest = hi;
}

// Off by default: measured on B200 (c1, in-graph stamps) the chain is latency-bound inside
// the kernels, and PDL edges left the loop time unchanged (39.1 vs 38.5 us/iteration).
static bool pdl_enabled() {
    const char* e = getenv("DSCR_PDL");
    return e && !strcmp(e, "1");
}

static int launch_iteration(dscr_solver* h, const Params& P, cudaStream_t s, cudaEvent_t* ev = nullptr) {
    const Geometry& g = h->geo;
    const bool group = P.n_groups > 0;
    const size_t smem1 = (size_t)g.smem1;
    const bool pdl = h->pdl && !ev;   // timed per-kernel runs keep plain launches
    void (*k1)(Params);
    void (*k3a)(Params);
    k1 = k1_kernel(P.dtype, group, P.theta_gl != 0);
    switch (P.dtype) {
        case DSCR_F64: k3a = k3a_residual<double>; break;
        case DSCR_F32: k3a = k3a_residual<float>; break;
        default: k3a = k3a_residual<__nv_bfloat16>;
    }
    cudaError_t le = launch_pdl(k1, dim3(g.G), smem1, s, pdl, P);
    if (le != cudaSuccess) return set_err("K1 launch", le);
    if (ev) CK(cudaEventRecord(ev[1], s));
    if (P.f23) {
        // K2 (test, compaction, vectors) and K3a-scan (residual partials of the unreduced
        // iterate) have no dependency on each other: two branches of the trip graph, joined
        // before K3b (timed runs launch them one after the other)
        void (*k3s)(Params);
        switch (P.dtype) {
            case DSCR_F64: k3s = group ? k3a_scan<double, true> : k3a_scan<double, false>; break;
            case DSCR_F32: k3s = group ? k3a_scan<float, true> : k3a_scan<float, false>; break;
            default: k3s = group ? k3a_scan<__nv_bfloat16, true> : k3a_scan<__nv_bfloat16, false>;
        }
        Params P2 = P;
        P2.k2v = 3;
        if (ev) {      // timed: K2, then K3a-scan, each between events
            le = launch_pdl(group ? k2_screen<true> : k2_screen<false>, dim3(g.G), 0, s, false, P2);
            if (le != cudaSuccess) return set_err("K2 launch", le);
            CK(cudaEventRecord(ev[2], s));
            k3s<<<dim3(g.R, g.P23), NT, 0, s>>>(P);
            CK(cudaGetLastError());
            CK(cudaEventRecord(ev[3], s));
        } else {
            // K2 at the greatest priority, so its CTAs are dispatched first and K3a-scan fills the
            // slots they free (a K3a-scan CTA holding a slot first delayed K2 by 2-6 us)
            int hi_pr = 0, lo_pr = 0;
            priority_range(&hi_pr, &lo_pr);
            CK(cudaEventRecord(h->ev_fork, s));
            CK(cudaStreamWaitEvent(h->fork_stream, h->ev_fork, 0));
            le = launch_pdl(k3s, dim3(g.R, g.P23), 0, h->fork_stream, false, P, lo_pr);
            if (le != cudaSuccess) return set_err("K3a-scan launch", le);
            le = launch_pdl(group ? k2_screen<true> : k2_screen<false>, dim3(g.G), 0, s, false, P2, hi_pr);
            if (le != cudaSuccess) return set_err("K2 launch", le);
            CK(cudaEventRecord(h->ev_join, h->fork_stream));
            CK(cudaStreamWaitEvent(s, h->ev_join, 0));
        }
        le = launch_pdl(k3b_finalize, dim3(g.G3b), 0, s, false, P);
        if (le != cudaSuccess) return set_err("K3b launch", le);
        return DSCR_OK;
    }
    le = launch_pdl(group ? k2_screen<true> : k2_screen<false>, dim3(g.G), 0, s, pdl, P);
    if (le != cudaSuccess) return set_err("K2 launch", le);
    if (ev) CK(cudaEventRecord(ev[2], s));
    le = launch_pdl(k3a, dim3(g.R, g.P), 0, s, pdl, P);
    if (le != cudaSuccess) return set_err("K3a launch", le);
    if (ev) CK(cudaEventRecord(ev[3], s));
    le = launch_pdl(k3b_finalize, dim3(g.G3b), 0, s, pdl, P);
    if (le != cudaSuccess) return set_err("K3b launch", le);
    return DSCR_OK;
}

template <typename T>
static int set_smem_attrs(size_t smem, bool k1 = true) {
    if (k1) {
        CK(raise_smem((const void*)k1_corr_update<T, false>, (int)smem));
        CK(raise_smem((const void*)k1_corr_update<T, true>, (int)smem));
    }
    CK(raise_smem((const void*)k_correlate<T>, (int)smem));
    return DSCR_OK;
}

template <typename T>
static int launch_correlate_t(const T* D, int ldd, int n, int k, const double* v, double* out, const int* skip,
                              float keep, cudaStream_t s, int grid) {
    const size_t smem = (size_t)ldd * 8;
    if (smem > THETA_SMEM_MAX) {
        k_correlate<T, true><<<grid, NT, 0, s>>>(D, ldd, n, k, v, out, skip, keep);
    } else {
        int rc;
        if ((rc = set_smem_attrs<T>(smem, false))) return rc;
        k_correlate<T><<<grid, NT, smem, s>>>(D, ldd, n, k, v, out, skip, keep);
    }
    return DSCR_OK;
}

// v: ldd doubles (rows n..ldd-1 zero)
static int launch_correlate(int dtype, const void* D, int ldd, int n, int k, const double* v, double* out,
                            const int* skip, float keep, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min((k + 4 * NW - 1) / (4 * NW), sms * 2));
    int rc;
    switch (dtype) {
        case DSCR_F64: rc = launch_correlate_t((const double*)D, ldd, n, k, v, out, skip, keep, s, grid); break;
        case DSCR_F32: rc = launch_correlate_t((const float*)D, ldd, n, k, v, out, skip, keep, s, grid); break;
        default: rc = launch_correlate_t((const __nv_bfloat16*)D, ldd, n, k, v, out, skip, keep, s, grid);
    }
    if (rc) return rc;
    CK(cudaGetLastError());
    return DSCR_OK;
}

static int enqueue_setup(dscr_solver* h, cudaStream_t s) {
    Params& P = h->P;
    const Geometry& g = h->geo;
    const int test = P.test;
    const bool group = P.n_groups > 0;
    int rc;
    k_init<<<256, NT, 0, s>>>(P);
    CK(cudaGetLastError());
    k_init_scalars<<<1, NT, 0, s>>>(P);
    CK(cudaGetLastError());
    if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.y, P.ycorr, nullptr, P.l2_keep, s))) return rc;
    int lgrid = std::max(1, std::min((P.n_units + NT - 1) / NT, 2048));
    k_lmax<<<lgrid, NT, 0, s>>>(P);
    CK(cudaGetLastError());
    const int* stop_flag = &P.sc->stop;
    if (P.strategy != DSCR_NONE) {
        if (test == DSCR_DST3 || test == DSCR_DOME) {
            switch (P.dtype) {
                case DSCR_F64: k_setup_vec<double><<<32, NT, 0, s>>>(P); break;
                case DSCR_F32: k_setup_vec<float><<<32, NT, 0, s>>>(P); break;
                default: k_setup_vec<__nv_bfloat16><<<32, NT, 0, s>>>(P);
            }
            CK(cudaGetLastError());
            k_vec_nsq<<<1, NT, 0, s>>>(P);
            if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.vec, P.star, stop_flag, P.l2_keep, s))) return rc;
        } else if (test == DSCR_GST3) {
            switch (P.dtype) {
                case DSCR_F64: k_setup_vec<double><<<32, NT, 0, s>>>(P); break;
                case DSCR_F32: k_setup_vec<float><<<32, NT, 0, s>>>(P); break;
                default: k_setup_vec<__nv_bfloat16><<<32, NT, 0, s>>>(P);
            }
            CK(cudaGetLastError());
            k_gst3_scalars<<<1, NT, 0, s>>>(P);
            CK(cudaGetLastError());
            if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.vec, P.dn, stop_flag, P.l2_keep, s))) return rc;
        }
        if (P.norm_aware && !h->prob.col_norms) {   // not cached by the caller: one pass over D
            const int cg = std::max(1, std::min((P.kcols + NW - 1) / NW, 2048));
            switch (P.dtype) {
                case DSCR_F64: k_colnorms<double><<<cg, NT, 0, s>>>(P); break;
                case DSCR_F32: k_colnorms<float><<<cg, NT, 0, s>>>(P); break;
                default: k_colnorms<__nv_bfloat16><<<cg, NT, 0, s>>>(P);
            }
            CK(cudaGetLastError());
        }
        k_centers<<<std::max(1, std::min((P.kcols + NT - 1) / NT, 1024)), NT, 0, s>>>(P);
        CK(cudaGetLastError());
        if (group) {
            k_center_group_norms<<<std::max(1, std::min((P.n_groups + NT - 1) / NT, 1024)), NT, 0, s>>>(P);
            CK(cudaGetLastError());
        }
        if (P.strategy == DSCR_STATIC) {
            k_static_radius<<<1, NT, 0, s>>>(P, 0);
            CK(cudaGetLastError());
            if (group) k2_screen<true><<<g.G, NT, 0, s>>>(P);
            else k2_screen<false><<<g.G, NT, 0, s>>>(P);
            CK(cudaGetLastError());
            k_static_done<<<1, 1, 0, s>>>(P);
            CK(cudaGetLastError());
        }
    }
    return DSCR_OK;
}

template <typename T>
static int launch_colnorms(const void* D, int ldd, int n, int k, double* out, cudaStream_t s) {
    const int cg = std::max(1, std::min((k + NW - 1) / NW, 2048));
    k_colnorms_op<T><<<cg, NT, 0, s>>>(static_cast<const T*>(D), ldd, n, k, out);
    CK(cudaGetLastError());
    return DSCR_OK;
}

extern "C" int dscr_column_norms(int dtype, const void* D, int ldd, int n, int k, double* out, void* stream) {
    if (!D || !out || n < 1 || k < 1 || ldd < n) return set_inval("bad column-norm arguments");
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
        case DSCR_F64: return launch_colnorms<double>(D, ldd, n, k, out, s);
        case DSCR_F32: return launch_colnorms<float>(D, ldd, n, k, out, s);
        case DSCR_BF16: return launch_colnorms<__nv_bfloat16>(D, ldd, n, k, out, s);
        default: return set_inval("unknown dtype");
    }
}

extern "C" {
int dscr_solver_create(const dscr_problem_desc* pr, const dscr_config* cfg, void* workspace,
                       size_t workspace_bytes, void* stream, dscr_solver** out) {
    int nu, mg;
    int rc = validate(pr, cfg, &nu, &mg);
    if (rc) return rc;
    if (!out || !workspace) return set_inval("null output or workspace");
    if (pr->n_groups > 0 && !(pr->group_ptr && pr->group_w && pr->group_snorm))
        return set_inval("group problems need group_ptr, group_w and group_snorm");
    if ((rc = group_max_size(pr, &mg))) return rc;
    Geometry g = make_geometry(pr, nu, mg);
    if ((rc = max_atoms_per_slot(pr, g.cap, &g.sup_cap))) return rc;
    size_t total;
    Offsets o = make_offsets(pr, cfg, g, nu, &total);
    if (workspace_bytes < total) return set_inval("workspace too small");
    dscr_solver* h = new dscr_solver();
    h->pdl = pdl_enabled();
    h->prob = *pr;
    h->cfg = *cfg;
    h->geo = g;
    h->ws = workspace;
    char* base = (char*)align_up((size_t)workspace, 256);
    Params& P = h->P;
    memset(&P, 0, sizeof P);
    P.D = pr->D; P.ldd = pr->ldd; P.n = pr->n_rows; P.kcols = pr->n_cols; P.dtype = pr->dtype;
    P.y = pr->y; P.lam = pr->lam;
    P.n_groups = pr->n_groups; P.gptr = pr->group_ptr; P.gw = pr->group_w; P.gsn = pr->group_snorm;
    P.n_units = nu;
    P.algo = cfg->algorithm; P.strategy = cfg->strategy;
    P.test = (cfg->strategy == DSCR_NONE) ? DSCR_TEST_OFF : cfg->test;
    P.rel_tol = cfg->rel_tol; P.gap_tol = cfg->gap_tol; P.bt_factor = cfg->backtrack_factor;
    P.twa = cfg->twist_alpha; P.twb = cfg->twist_beta; P.cp_gamma = cfg->cp_gamma;
    P.bb_min = cfg->bb_L_min; P.bb_max = cfg->bb_L_max;
    P.L0 = cfg->L0; P.cp_safety = cfg->cp_step_safety; P.op_norm = cfg->op_norm;
    P.tw_step = (cfg->twist_step > 0) ? cfg->twist_step : (cfg->op_norm > 0 ? 1.0 / (cfg->op_norm * cfg->op_norm) : 0.0);
    P.sc = (dscr_scalars*)(base + o.sc);
    P.theta[0] = (double*)(base + o.theta0); P.theta[1] = (double*)(base + o.theta1);
    P.resid = (double*)(base + o.resid); P.corr = (double*)(base + o.corr);
    P.x[0] = (double*)(base + o.x0); P.x[1] = (double*)(base + o.x1); P.x[2] = (double*)(base + o.x2);
    P.u[0] = (double*)(base + o.u0); P.u[1] = (double*)(base + o.u1);
    P.ycorr = (double*)(base + o.ycorr); P.star = (double*)(base + o.star); P.cc = (double*)(base + o.cc);
    P.cnorm = (double*)(base + o.cnorm); P.vec = (double*)(base + o.vec); P.dn = (double*)(base + o.dn);
    P.act[0] = (int*)(base + o.act0); P.act[1] = (int*)(base + o.act1);
    P.act_cnt[0] = (int*)(base + o.cnt0); P.act_cnt[1] = (int*)(base + o.cnt1);
    P.act_off[0] = (int*)(base + o.off0); P.act_off[1] = (int*)(base + o.off1);
    P.mask = (uint8_t*)(base + o.mask);
    P.sidx = (int*)(base + o.sidx); P.sa = (double*)(base + o.sa); P.sb = (double*)(base + o.sb);
    P.sup_cnt = (int*)(base + o.supcnt); P.sup_off = (int*)(base + o.supoff); P.sup_cap = g.sup_cap;
    P.p1 = (double*)(base + o.p1); P.p2 = (double*)(base + o.p2); P.p3v = (double*)(base + o.p3v);
    P.p3s = (double*)(base + o.p3s); P.tickets = (unsigned*)(base + o.tickets);
    P.p3c = (int*)(base + o.p3c);
    P.trace = (double*)(base + o.trace);
    P.kts = (unsigned long long*)(base + o.kts);
    P.anorm = pr->col_norms ? const_cast<double*>(pr->col_norms) : (double*)(base + o.anorm);
    P.comm = (double*)(base + o.comm);
    P.norm_aware = pr->norm_aware;
    P.max_kts = kts_slots(cfg);
    P.max_iters = cfg->max_iters;
    P.G = g.G; P.cap = g.cap; P.TR = g.TR; P.R = g.R; P.P = g.P; P.G3b = g.G3b;
    P.k1_tile = g.tile; P.max_gsize = g.max_gsize;
    P.theta_gl = g.theta_gl;
    P.min_cols = MIN_COLS_PER_SPLIT;
    P.k1_ilv = 1;   // measured on c4: K1 1241 -> 1222 us (DSCR_K1_INTERLEAVE=0 restores contiguous passes)
    if (const char* ei = getenv("DSCR_K1_INTERLEAVE")) P.k1_ilv = atoi(ei);
    if (const char* em = getenv("DSCR_K3A_MIN_COLS")) P.min_cols = std::max(1, atoi(em));   // experiment knob
    P.col_offset = pr->col_offset;
    P.group_offset = pr->group_offset;
    P.in_graph = 1;
    P.writer = 1;
    {
        // engine mode: the conditional-graph chain (default) or, with DSCR_ENGINE=persistent, one
        // cooperative launch with grid barriers (measured slower on B200 -- c1 70 vs 32 us per
        // iteration even with the ~1 us arrival-counter barrier: K1 inside the all-in-one kernel runs
        // at half speed and the redundant tails exceed the launch gaps it removes; an alternative)
        const char* env = getenv("DSCR_ENGINE");
        int dev = 0, coop = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int occ = pers_occupancy(pr->dtype, pr->n_groups > 0, g.smem1);
        P.persistent = coop && occ * sms >= g.G && g.G <= PERS_MAX_G && !g.theta_gl && env &&
                       strcmp(env, "persistent") == 0;
    }
    P.P23 = g.P23;
    // K2 concurrent with the K3a-scan residual: measured c1 37.0 -> 32.2, c2 58.0 -> 52.4,
    // c3 67.8 -> 64.8, c4 proxy (128 MB) 61.4 -> 57.7 us per iteration; neutral on c4 (8.6 GB,
    // K3a streams ~160 MB per trip and waits for K2's slots anyway), so the bandwidth-bound
    // sizes keep the support-list K3a.  DSCR_F23=0/1 overrides.
    const size_t dict_bytes = (size_t)pr->ldd * pr->n_cols * dtype_size(pr->dtype);
    P.f23 = (!P.persistent && dict_bytes <= ((size_t)1 << 30)) ? 1 : 0;
    if (const char* ef = getenv("DSCR_F23")) P.f23 = P.persistent ? 0 : atoi(ef);
    P.l2_keep = l2_keep_fraction((size_t)pr->ldd * pr->n_cols * dtype_size(pr->dtype));
    if (const char* ek = getenv("DSCR_L2_KEEP")) P.l2_keep = (float)atof(ek);   // experiment knob

    cudaStream_t us = (cudaStream_t)stream;
    // smem attributes for the K1 instantiations
    switch (P.dtype) {
        case DSCR_F64: rc = set_smem_attrs<double>(g.smem1); break;
        case DSCR_F32: rc = set_smem_attrs<float>(g.smem1); break;
        default: rc = set_smem_attrs<__nv_bfloat16>(g.smem1);
    }
    if (rc) { delete h; return rc; }
    cudaError_t e = cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete h; return set_err("cudaStreamCreate", e); }
    if (P.f23) {
        e = cudaStreamCreateWithFlags(&h->fork_stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
        if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("fork stream / events", e); }
    }
    // tickets must start at zero before any kernel runs
    e = cudaMemsetAsync(P.tickets, 0, 64, us);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("cudaMemsetAsync", e); }

    // ---- setup graph (plain capture)
    cudaStream_t cs = h->cap_stream;
    e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("capture setup", e); }
    rc = enqueue_setup(h, cs);
    cudaGraph_t gs = nullptr;
    e = cudaStreamEndCapture(cs, &gs);
    if (rc || e != cudaSuccess) { if (gs) cudaGraphDestroy(gs); dscr_solver_destroy(h); return rc ? rc : set_err("end capture setup", e); }
    h->g_setup = gs;
    e = cudaGraphInstantiate(&h->e_setup, gs, 0);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("instantiate setup", e); }

    // ---- loop graph: k_preloop -> WHILE(h_main) { K1; K2; K3a; K3b }
    cudaGraph_t gl;
    e = cudaGraphCreate(&gl, 0);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("graph create", e); }
    h->g_loop = gl;
    e = cudaGraphConditionalHandleCreate(&P.h_main, gl, 0, 0);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("conditional handle", e); }
    e = cudaStreamBeginCaptureToGraph(cs, gl, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("capture preloop", e); }
    k_preloop<<<1, 1, 0, cs>>>(P);
    e = cudaGetLastError();
    cudaGraph_t tmp = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cs, &tmp);
    if (e != cudaSuccess || e2 != cudaSuccess) { dscr_solver_destroy(h); return set_err("capture preloop", e != cudaSuccess ? e : e2); }
    size_t nn = 0;
    cudaGraphGetNodes(gl, nullptr, &nn);
    cudaGraphNode_t pre = nullptr;
    if (nn != 1 || cudaGraphGetNodes(gl, &pre, &nn) != cudaSuccess) { dscr_solver_destroy(h); return set_inval("unexpected preloop graph"); }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = P.h_main;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    e = cudaGraphAddNode(&cnode, gl, &pre, 1, &cp);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("add WHILE node", e); }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("capture body", e); }
    // TRIPS_PER_BODY trips per body launch amortise the conditional-node relaunch;
    // trips after a stop or pause return at entry.
    for (int r = 0; r < TRIPS_PER_BODY && rc == DSCR_OK; ++r) rc = launch_iteration(h, h->P, cs);
    e = cudaStreamEndCapture(cs, &tmp);
    if (rc || e != cudaSuccess) {
        // an invalidated capture leaves the conditional body unusable and cudaGraphDestroy on its
        // parent crashes in the driver: leak the loop graph on this error path
        h->g_loop = nullptr;
        dscr_solver_destroy(h);
        return rc ? rc : set_err("end capture body", e);
    }
    e = cudaGraphInstantiate(&h->e_loop, gl, cudaGraphInstantiateFlagUseNodePriority);
    if (e != cudaSuccess) { dscr_solver_destroy(h); return set_err("instantiate loop", e); }
    *out = h;
    return DSCR_OK;
}

int dscr_solver_setup(dscr_solver* h, void* stream) {
    if (!h) return set_inval("null handle");
    CK(cudaGraphLaunch(h->e_setup, (cudaStream_t)stream));
    return DSCR_OK;
}

static int launch_persistent(dscr_solver* h, cudaStream_t s) {
    Params P = h->P;
    P.persistent = 1;
    void* args[] = {&P};
    const bool group = P.n_groups > 0;
    const void* fn;
    switch (P.dtype) {
        case DSCR_F64: fn = group ? (const void*)k_persistent<double, true> : (const void*)k_persistent<double, false>; break;
        case DSCR_F32: fn = group ? (const void*)k_persistent<float, true> : (const void*)k_persistent<float, false>; break;
        default: fn = group ? (const void*)k_persistent<__nv_bfloat16, true> : (const void*)k_persistent<__nv_bfloat16, false>;
    }
    CK(cudaMemsetAsync(P.tickets + 4, 0, 8, s));     // grid-barrier arrival counter
    CK(cudaLaunchCooperativeKernel(fn, dim3(h->geo.G), dim3(NT), args, (size_t)h->geo.smem1, s));
    return DSCR_OK;
}

int dscr_solver_run(dscr_solver* h, int iteration_limit, void* stream) {
    if (!h) return set_inval("null handle");
    cudaStream_t s = (cudaStream_t)stream;
    k_set_limit<<<1, 1, 0, s>>>(h->P.sc, iteration_limit > 0 ? iteration_limit : 0x7fffffff);
    CK(cudaGetLastError());
    if (h->P.persistent) return launch_persistent(h, s);
    CK(cudaGraphLaunch(h->e_loop, s));
    return DSCR_OK;
}

// Direct (non-graph) launches of `trips` iteration trips with CUDA events
// between the four kernels; ms_out[0..3] receive the mean duration of K1, K2,
// K3a and K3b.  Used by bench.py for the live roofline measurement.
int dscr_solver_profile(dscr_solver* h, int trips, void* stream, float* ms_out) {
    if (!h || !ms_out || trips < 1) return set_inval("bad profile arguments");
    cudaStream_t s = (cudaStream_t)stream;
    Params P = h->P;
    P.in_graph = 0;
    cudaEvent_t ev[5];
    for (int i = 0; i < 5; ++i) CK(cudaEventCreate(&ev[i]));
    double acc[4] = {0, 0, 0, 0};
    int rc = DSCR_OK;
    for (int t = 0; t < trips && rc == DSCR_OK; ++t) {
        CK(cudaEventRecord(ev[0], s));
        rc = launch_iteration(h, P, s, ev);
        CK(cudaEventRecord(ev[4], s));
        CK(cudaEventSynchronize(ev[4]));
        for (int k = 0; k < 4; ++k) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
            acc[k] += ms;
        }
    }
    for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
    for (int k = 0; k < 4; ++k) ms_out[k] = (float)(acc[k] / trips);
    return rc;
}

// Multi-rank (column-sharded) execution: the host runs these phases in order and
// performs the collectives on the comm region between them (Multi-GPU).
int dscr_solver_phase(dscr_solver* h, int phase, void* stream) {
    if (!h) return set_inval("null handle");
    cudaStream_t s = (cudaStream_t)stream;
    Params P = h->P;
    P.in_graph = 0;
    P.split = 1;
    P.f23 = 0;   // split mode: K2S / K2 build the support list, K3A reads it
    const Geometry& g = h->geo;
    const bool group = P.n_groups > 0;
    const int test = P.test;
    int rc = DSCR_OK;
    switch (phase) {
        case DSCR_PH_SETUP_LOCAL: {
            k_init<<<256, NT, 0, s>>>(P);
            k_init_scalars<<<1, NT, 0, s>>>(P);
            if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.y, P.ycorr, nullptr, P.l2_keep, s))) return rc;
            k_lmax<<<std::max(1, std::min((P.n_units + NT - 1) / NT, 2048)), NT, 0, s>>>(P);
            break;
        }
        case DSCR_PH_SETUP_ADOPT:
            k_setup_adopt<<<1, 1, 0, s>>>(P);
            break;
        case DSCR_PH_SETUP_VEC:     // owner rank only: extremal atom or GST3 normal into vec
            switch (P.dtype) {
                case DSCR_F64: k_setup_vec<double><<<32, NT, 0, s>>>(P); break;
                case DSCR_F32: k_setup_vec<float><<<32, NT, 0, s>>>(P); break;
                default: k_setup_vec<__nv_bfloat16><<<32, NT, 0, s>>>(P);
            }
            break;
        case DSCR_PH_SETUP_FINISH: {
            if (P.strategy == DSCR_NONE) break;
            const int* stop_flag = &P.sc->stop;
            if (test == DSCR_DST3 || test == DSCR_DOME) {
                k_vec_nsq<<<1, NT, 0, s>>>(P);
                if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.vec, P.star, stop_flag, P.l2_keep, s))) return rc;
            } else if (test == DSCR_GST3) {
                k_gst3_scalars<<<1, NT, 0, s>>>(P);
                if ((rc = launch_correlate(P.dtype, P.D, P.ldd, P.n, P.kcols, P.vec, P.dn, stop_flag, P.l2_keep, s))) return rc;
            }
            if (P.norm_aware && !h->prob.col_norms) {
                const int cg = std::max(1, std::min((P.kcols + NW - 1) / NW, 2048));
                switch (P.dtype) {
                    case DSCR_F64: k_colnorms<double><<<cg, NT, 0, s>>>(P); break;
                    case DSCR_F32: k_colnorms<float><<<cg, NT, 0, s>>>(P); break;
                    default: k_colnorms<__nv_bfloat16><<<cg, NT, 0, s>>>(P);
                }
            }
            k_centers<<<std::max(1, std::min((P.kcols + NT - 1) / NT, 1024)), NT, 0, s>>>(P);
            if (group) k_center_group_norms<<<std::max(1, std::min((P.n_groups + NT - 1) / NT, 1024)), NT, 0, s>>>(P);
            break;
        }
        case DSCR_PH_STATIC_LOCAL:
            k_static_radius<<<1, NT, 0, s>>>(P, 0);
            break;
        case DSCR_PH_STATIC_FINISH:
            k_static_radius<<<1, NT, 0, s>>>(P, 1);
            if (group) k2_screen<true><<<g.G, NT, 0, s>>>(P);
            else k2_screen<false><<<g.G, NT, 0, s>>>(P);
            k_static_done<<<1, 1, 0, s>>>(P);
            break;
        case DSCR_PH_K1: {
            const size_t smem1 = (size_t)g.smem1;
            k1_kernel(P.dtype, group, P.theta_gl != 0)<<<g.G, NT, smem1, s>>>(P);
            break;
        }
        case DSCR_PH_K1R:
            k1r_radius<<<1, NT, 0, s>>>(P);
            break;
        case DSCR_PH_K2:
        case DSCR_PH_K2S:
        case DSCR_PH_K2C:
            if (phase != DSCR_PH_K2 && !P.onecoll) return set_inval("K2S/K2C need one-collective mode");
            P.k2v = (phase == DSCR_PH_K2S) ? 1 : (phase == DSCR_PH_K2C ? 2 : 0);
            if (group) k2_screen<true><<<g.G, NT, 0, s>>>(P);
            else k2_screen<false><<<g.G, NT, 0, s>>>(P);
            break;
        case DSCR_PH_K1R1:
            if (!P.onecoll) return set_inval("K1R1 needs one-collective mode");
            k1r_radius_oc<<<1, NT, 0, s>>>(P);
            break;
        case DSCR_PH_K3A: {
            dim3 g3(g.R, g.P);
            switch (P.dtype) {
                case DSCR_F64: k3a_residual<double><<<g3, NT, 0, s>>>(P); break;
                case DSCR_F32: k3a_residual<float><<<g3, NT, 0, s>>>(P); break;
                default: k3a_residual<__nv_bfloat16><<<g3, NT, 0, s>>>(P);
            }
            break;
        }
        case DSCR_PH_K3S:
            k3s_pack<<<(P.ldd + K3S_ROWS - 1) / K3S_ROWS, NT, 0, s>>>(P);
            break;
        case DSCR_PH_K3X_PUSH:
        case DSCR_PH_K3X_REDUCE: {
            if (!P.peer_tab || !P.onecoll) return set_inval("peer exchange needs dscr_solver_set_peers and one-collective mode");
            const int grid = std::max(1, std::min((P.peer_len + NT - 1) / NT, 148));
            if (phase == DSCR_PH_K3X_PUSH) k3x_push<<<grid, NT, 0, s>>>(P);
            else k3x_reduce<<<grid, NT, 0, s>>>(P);
            break;
        }
        case DSCR_PH_K3B:
            k3b_finalize<<<g.G3b, NT, 0, s>>>(P);
            break;
        default:
            return set_inval("unknown phase");
    }
    CK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_solver_set_collectives(dscr_solver* h, int rank, int world, int one_collective) {
    if (!h) return set_inval("null handle");
    if (world < 1 || world > OC_MAX_WORLD || rank < 0 || rank >= world) return set_inval("rank / world out of range");
    if (one_collective && h->P.test == DSCR_DOME && h->P.strategy == DSCR_DYNAMIC)
        return set_inval("the dome test needs the two-collective trips");
    h->P.onecoll = one_collective ? 1 : 0;
    h->P.oc_rank = rank;
    h->P.oc_world = world;
    return DSCR_OK;
}

int dscr_solver_set_peers(dscr_solver* h, int rank, int world, void* const* recv_bases, void* const* flag_bases) {
    if (!h || !recv_bases || !flag_bases) return set_inval("null argument");
    if (world < 1 || world > OC_MAX_WORLD || rank < 0 || rank >= world) return set_inval("rank / world out of range");
    void* tab[128] = {};
    for (int r = 0; r < world; ++r) { tab[r] = recv_bases[r]; tab[64 + r] = flag_bases[r]; }
    if (!h->peer_tab_dev) CK(cudaMalloc(&h->peer_tab_dev, sizeof tab));
    CK(cudaMemcpy(h->peer_tab_dev, tab, sizeof tab, cudaMemcpyHostToDevice));
    h->P.peer_tab = h->peer_tab_dev;
    h->P.peer_len = (CM_VEC - CM_SUM) + 2 * h->P.ldd + OC_SLOT * world;
    h->P.onecoll = 1;
    h->P.oc_rank = rank;
    h->P.oc_world = world;
    CK(cudaMemset(h->P.tickets + 8, 0, sizeof(unsigned long long)));   // exchange sequence number
    return DSCR_OK;
}

size_t dscr_peer_buffer_bytes(int world, int ldd) {
    if (world < 1 || world > OC_MAX_WORLD || ldd < 1) return 0;
    const size_t len = (size_t)(CM_VEC - CM_SUM) + 2 * (size_t)ldd + (size_t)OC_SLOT * world;
    return 64 * 8 + 2 * (size_t)world * len * 8;
}

int dscr_solver_scalars(dscr_solver* h, void* stream, dscr_scalars* out) {
    if (!h || !out) return set_inval("null argument");
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    CK(cudaMemcpy(out, h->P.sc, sizeof(dscr_scalars), cudaMemcpyDeviceToHost));
    return DSCR_OK;
}

int dscr_solver_get_buffers(dscr_solver* h, dscr_solver_buffers* b) {
    if (!h || !b) return set_inval("null argument");
    const Params& P = h->P;
    b->scalars = P.sc;
    b->theta[0] = P.theta[0]; b->theta[1] = P.theta[1];
    b->resid = P.resid; b->corr = P.corr;
    b->x[0] = P.x[0]; b->x[1] = P.x[1]; b->x[2] = P.x[2];
    b->u[0] = P.u[0]; b->u[1] = P.u[1];
    b->y_corr = P.ycorr; b->star_corr = P.star; b->cc = P.cc; b->cnorm = P.cnorm;
    b->act[0] = P.act[0]; b->act[1] = P.act[1];
    b->act_cnt[0] = P.act_cnt[0]; b->act_cnt[1] = P.act_cnt[1];
    b->act_off[0] = P.act_off[0]; b->act_off[1] = P.act_off[1];
    b->mask = P.mask; b->trace = P.trace;
    b->kts = (uint64_t*)P.kts; b->max_kts = P.max_kts;
    b->comm = P.comm; b->comm_len = CM_VEC + 2 * P.ldd + OC_SLOT * OC_MAX_WORLD;
    b->vec = P.vec;
    b->G = P.G; b->cap = P.cap;
    return DSCR_OK;
}

int dscr_solver_destroy(dscr_solver* h) {
    if (!h) return DSCR_OK;
    if (h->e_loop) cudaGraphExecDestroy(h->e_loop);
    if (h->e_setup) cudaGraphExecDestroy(h->e_setup);
    if (h->g_loop) cudaGraphDestroy(h->g_loop);
    if (h->g_setup) cudaGraphDestroy(h->g_setup);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->fork_stream) cudaStreamDestroy(h->fork_stream);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->peer_tab_dev) cudaFree(h->peer_tab_dev);
    delete h;
    return DSCR_OK;
}

}  // extern "C"
