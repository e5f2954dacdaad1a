// Kernel-level entry points for the reference's inner seams: the fused
// correlation + prox step of update_ista / update_fista (solvers.py:168-225) and its
// group-Lasso form (dictionary.py:290-301), the sparse residual (solvers.py:160-165 /
// dictionary.py:82-87) and the order-preserving compaction of the kept set after a test
// (screening.py:104-112, dictionary.py:99-117).  The solver engine runs the same arithmetic
// inside its per-iteration kernels; these standalone versions serve unit parity and callers
// that drive the iteration themselves.  All reductions are fixed-order (deterministic).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include <algorithm>
#include <cmath>

#include "dynscreen.h"
#include "dscr_device.cuh"

namespace dscr {
namespace seams {

static int inval(const char* what) {
    err_store() = what;
    return DSCR_EINVAL;
}
static int cuda_check(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return DSCR_OK;
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    err_store() = buf;
    return DSCR_ECUDA;
}

constexpr size_t VEC_SMEM_MAX = 200 * 1024;   // theta staged in shared memory up to this size

template <typename T> struct SeamU { static constexpr int U = 2; };
template <> struct SeamU<__nv_bfloat16> { static constexpr int U = 1; };

// c_j = D[:, j] . theta for the atoms listed in `atoms` (4 per warp); theta staged in shared
// memory unless too tall (VG: read through L2, rows n..ldd-1 must be zero)
template <typename T, bool VG>
__global__ void __launch_bounds__(NT) k_seam_corr(const T* __restrict__ D, int ldd, int n, const int* atoms,
                                                 int na, const double* __restrict__ theta, double* corr) {
    extern __shared__ double s_t[];
    const double* tv = theta;
    if (!VG) {
        for (int i = threadIdx.x; i < ldd; i += NT) s_t[i] = (i < n) ? theta[i] : 0.0;
        __syncthreads();
        tv = s_t;
    }
    const uint64_t pol = make_policy(0.5f);
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5, nw = (gridDim.x * NT) >> 5;
    for (int i0 = 4 * gw; i0 < na; i0 += 4 * nw) {
        const T* cols[4];
        int js[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            js[c] = (i0 + c < na) ? atoms[i0 + c] : -1;
            cols[c] = js[c] >= 0 ? D + (size_t)js[c] * ldd : nullptr;
        }
        double cs[4];
        warp_dots<T, 4, SeamU<T>::U>(cols, n, tv, lane, pol, cs);
        if (lane < 4 && js[lane] >= 0) {
            double v = cs[0];
#pragma unroll
            for (int c = 1; c < 4; ++c) if (lane == c) v = cs[c];
            corr[js[lane]] = v;
        }
    }
}

template <typename T>
static int launch_seam_corr(const void* D, int ldd, int n, const int* atoms, int na, const double* theta,
                            double* corr, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min((na + 4 * NW - 1) / (4 * NW), sms * 2));
    const size_t smem = (size_t)ldd * 8;
    if (smem > VEC_SMEM_MAX) {
        k_seam_corr<T, true><<<grid, NT, 0, s>>>(static_cast<const T*>(D), ldd, n, atoms, na, theta, corr);
    } else {
        cudaFuncSetAttribute(k_seam_corr<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_seam_corr<T, false><<<grid, NT, smem, s>>>(static_cast<const T*>(D), ldd, n, atoms, na, theta, corr);
    }
    return cuda_check("seam correlations");
}

static int seam_corr(int dtype, const void* D, int ldd, int n, const int* atoms, int na, const double* theta,
                     double* corr, cudaStream_t s) {
    switch (dtype) {
        case DSCR_F64: return launch_seam_corr<double>(D, ldd, n, atoms, na, theta, corr, s);
        case DSCR_F32: return launch_seam_corr<float>(D, ldd, n, atoms, na, theta, corr, s);
        case DSCR_BF16: return launch_seam_corr<__nv_bfloat16>(D, ldd, n, atoms, na, theta, corr, s);
        default: return inval("unknown dtype");
    }
}

// gradient step of the prox argument with the reference's own operation: point - c / L
// (ISTA/FISTA/SpaRSA, solvers.py:178, 276) or point - tau * c (CP / TwIST, solvers.py:302, 242)
__device__ __forceinline__ double grad_step(double point, double c, double s, int mult) {
    return mult ? point - s * c : point - c / s;
}

// Lasso prox step per active atom: x = soft(grad_step, thr), u = x + beta (x - x_prev)
__global__ void k_seam_prox(const int* active, int na, const double* corr, const double* point,
                            const double* x_prev, double step, int mult, double thr, double beta, double* x_out,
                            double* u_out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
        const int j = active[i];
        const double xo = soft(grad_step(point[j], corr[j], step, mult), thr);   // prox_l1 of the step
        x_out[j] = xo;
        if (u_out) u_out[j] = xo + beta * (xo - x_prev[j]);       // solvers.py:216-218
    }
}

// Group prox per active group g (contiguous atoms group_ptr[g]..group_ptr[g+1]): v_g = point_g -
// step*c_g, x_g = v_g max(1 - thr w_g / ||v_g||, 0) with numpy's pairwise sum for the norm
// (dictionary.py:290-301); also ||c_g|| for the dual-scaling bound
__global__ void k_seam_group_prox(const int* gptr, const int* groups, int ng, const double* w, const double* corr,
                                  const double* point, const double* x_prev, double step, int mult, double thr,
                                  double beta, double* x_out, double* u_out, double* cnorm) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x) {
        const int g = groups[i];
        const int j0 = gptr[g], n = gptr[g + 1] - j0;
        const double nv = sqrt(np_segment_sum([&](int j) {
            double t = grad_step(point[j], corr[j], step, mult); return t * t; }, j0, n));
        const double nc = sqrt(np_segment_sum([&](int j) { double t = corr[j]; return t * t; }, j0, n));
        const double fac = (nv > 0.0) ? fmax(1.0 - thr * w[g] / nv, 0.0) : 0.0;
        for (int j = j0; j < j0 + n; ++j) {
            const double xo = grad_step(point[j], corr[j], step, mult) * fac;
            x_out[j] = xo;
            if (u_out) u_out[j] = xo + beta * (xo - x_prev[j]);
        }
        cnorm[i] = nc;
    }
}

// Fixed-order reduction (one CTA) of the step's scalars over the active atoms:
// red[0] = max|c_j| (Lasso) or min_g w_g / ||c_g|| over groups with ||c_g|| > 0 (inf if none;
// screening.py:126-165), red[1] = c . (x - point), red[2] = ||x - point||^2 (the majorization
// terms of _backtrack, solvers.py:176-183)
__global__ void __launch_bounds__(NT) k_seam_step_red(const int* atoms, int na, const double* corr, const double* point,
                                                      const double* x_out, const int* groups, int ng, const double* w,
                                                      const double* cnorm, double* red) {
    __shared__ double s_sh[64];
    double m = groups ? INFINITY : 0.0, cs = 0.0, ss = 0.0;
    for (int i = threadIdx.x; i < na; i += NT) {
        const int j = atoms[i];
        const double c = corr[j], d = x_out[j] - point[j];
        if (!groups) m = fmax(m, fabs(c));
        cs = fma(c, d, cs);
        ss = fma(d, d, ss);
    }
    for (int i = threadIdx.x; groups && i < ng; i += NT)
        if (cnorm[i] > 0.0) m = fmin(m, w[groups[i]] / cnorm[i]);
    double v2[2] = {cs, ss};
    block_sum_n<2>(v2, s_sh);
    double mm[1] = {groups ? -m : m};
    block_max_n<1>(mm, s_sh);
    if (threadIdx.x == 0) {
        red[0] = groups ? -mm[0] : mm[0];
        red[1] = v2[0];
        red[2] = v2[1];
    }
}

// r_x = D_S x - y, r_u = D_S u - y over a compact support list (idx[e], x[e], u[e]): one thread
// per row, entries accumulated in list order
template <typename T>
__global__ void __launch_bounds__(NT) k_seam_residual(const T* __restrict__ D, int ldd, int n, const int* idx, int nnz,
                                                      const double* x, const double* u, const double* y,
                                                      double* r_x, double* r_u) {
    __shared__ int s_i[NT];
    __shared__ double s_x[NT], s_u[NT];
    const int r = blockIdx.x * NT + threadIdx.x;
    double ax = 0.0, au = 0.0;
    for (int e0 = 0; e0 < nnz; e0 += NT) {
        __syncthreads();
        if (e0 + threadIdx.x < nnz) {
            s_i[threadIdx.x] = idx[e0 + threadIdx.x];
            s_x[threadIdx.x] = x[e0 + threadIdx.x];
            s_u[threadIdx.x] = u ? u[e0 + threadIdx.x] : 0.0;
        }
        __syncthreads();
        const int m = min(NT, nnz - e0);
        if (r < n) {
            for (int e = 0; e < m; ++e) {
                const double d = elem<T>(D + (size_t)s_i[e] * ldd + r);
                ax = fma(s_x[e], d, ax);
                au = fma(s_u[e], d, au);
            }
        }
    }
    if (r < n) {
        r_x[r] = ax - y[r];
        if (r_u) r_u[r] = au - y[r];
    }
}

__global__ void __launch_bounds__(NT) k_seam_residual_red(int n, const double* r_x, const double* r_u, const double* y,
                                                          double* red) {
    __shared__ double s_sh[64];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
        a = fma(r_x[i], r_x[i], a);
        if (r_u) { b = fma(r_u[i], r_u[i], b); c = fma(r_u[i], y[i], c); }
    }
    double v3[3] = {a, b, c};
    block_sum_n<3>(v3, s_sh);
    if (threadIdx.x == 0) { red[0] = v3[0]; red[1] = v3[1]; red[2] = v3[2]; }
}

// order-preserving compaction: pass 1 per-CTA kept counts, pass 2 (one CTA) exclusive scan,
// pass 3 scatter in order
constexpr int CMP_CHUNK = 4 * NT;

__global__ void __launch_bounds__(NT) k_cmp_count(const uint8_t* mask, int n, int* cnt) {
    __shared__ double s_sh[64];
    const int base = blockIdx.x * CMP_CHUNK;
    int c = 0;
    for (int i = base + threadIdx.x; i < min(n, base + CMP_CHUNK); i += NT) c += mask[i] ? 0 : 1;
    const double t = block_sum((double)c, s_sh);
    if (threadIdx.x == 0) cnt[blockIdx.x] = (int)t;
}

__global__ void __launch_bounds__(NT) k_cmp_scan(int* cnt, int nb, int* n_out) {
    __shared__ int s_scan[2 * NW + 1];
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += NT) {
        const int v = (b0 + (int)threadIdx.x < nb) ? cnt[b0 + threadIdx.x] : 0;
        int tot;
        const int e = block_exscan(v, s_scan, &tot);
        if (b0 + (int)threadIdx.x < nb) cnt[b0 + threadIdx.x] = carry + e;
        carry += tot;
    }
    if (threadIdx.x == 0) *n_out = carry;
}

__global__ void __launch_bounds__(NT) k_cmp_scatter(const int* active, const uint8_t* mask, int n, const int* off,
                                                    int* out) {
    __shared__ int s_scan[2 * NW + 1];
    const int base = blockIdx.x * CMP_CHUNK;
    int pos = off[blockIdx.x];
    for (int i0 = base; i0 < min(n, base + CMP_CHUNK); i0 += NT) {
        const int i = i0 + threadIdx.x;
        const bool keep = i < n && !mask[i];
        int tot;
        const int e = block_exscan(keep ? 1 : 0, s_scan, &tot);
        if (keep) out[pos + e] = active[i];
        pos += tot;
    }
}

}  // namespace seams
}  // namespace dscr

using namespace dscr;
using namespace dscr::seams;

extern "C" {

int dscr_corr_prox(int dtype, const void* D, int ldd, int n, const int32_t* active, int n_active,
                   const double* theta, const double* point, const double* x_prev, double step, int mult, double thr,
                   double beta, double* x_out, double* u_out, double* corr_out, double* red_out, void* stream) {
    if (!D || (n_active > 0 && !active) || !theta || !point || !x_out || !corr_out || !red_out || n < 1 || ldd < n ||
        n_active < 0)
        return inval("bad corr_prox arguments");
    if (u_out && !x_prev) return inval("u_out needs x_prev");
    if (!(step > 0.0) || !(thr >= 0.0)) return inval("step must be positive and the threshold nonnegative");
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    if (n_active > 0) {
        if ((rc = seam_corr(dtype, D, ldd, n, active, n_active, theta, corr_out, s))) return rc;
        const int grid = std::max(1, std::min((n_active + NT - 1) / NT, 1024));
        k_seam_prox<<<grid, NT, 0, s>>>(active, n_active, corr_out, point, x_prev, step, mult, thr, beta, x_out,
                                        u_out);
    }
    k_seam_step_red<<<1, NT, 0, s>>>(active, n_active, corr_out, point, x_out, nullptr, 0, nullptr, nullptr, red_out);
    return cuda_check("corr_prox");
}

int dscr_group_corr_prox(int dtype, const void* D, int ldd, int n, const int32_t* group_ptr,
                         const int32_t* active_groups, int n_active, const int32_t* active_atoms, int n_atoms,
                         const double* group_w, const double* theta, const double* point, const double* x_prev,
                         double step, int mult, double thr, double beta, double* x_out, double* u_out,
                         double* corr_out, double* group_cnorm, double* red_out, void* stream) {
    if (!D || !group_ptr || (n_active > 0 && !active_groups) || (n_atoms > 0 && !active_atoms) || !group_w ||
        !theta || !point || !x_out || !corr_out || !group_cnorm || !red_out || n < 1 || ldd < n || n_active < 0 ||
        n_atoms < 0)
        return inval("bad group_corr_prox arguments");
    if (u_out && !x_prev) return inval("u_out needs x_prev");
    if (!(step > 0.0) || !(thr >= 0.0)) return inval("step must be positive and the threshold nonnegative");
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    if (n_atoms > 0 && (rc = seam_corr(dtype, D, ldd, n, active_atoms, n_atoms, theta, corr_out, s))) return rc;
    if (n_active > 0) {
        const int grid = std::max(1, std::min((n_active + NT - 1) / NT, 1024));
        k_seam_group_prox<<<grid, NT, 0, s>>>(group_ptr, active_groups, n_active, group_w, corr_out, point, x_prev,
                                              step, mult, thr, beta, x_out, u_out, group_cnorm);
    }
    k_seam_step_red<<<1, NT, 0, s>>>(active_atoms, n_atoms, corr_out, point, x_out, active_groups, n_active, group_w,
                                     group_cnorm, red_out);
    return cuda_check("group_corr_prox");
}

int dscr_residual(int dtype, const void* D, int ldd, int n, const int32_t* idx, int nnz, const double* x,
                  const double* u, const double* y, double* r_x, double* r_u, double* red_out, void* stream) {
    if (!D || (nnz > 0 && (!idx || !x)) || !y || !r_x || !red_out || n < 1 || ldd < n || nnz < 0)
        return inval("bad residual arguments");
    if (r_u && !u) return inval("r_u needs u");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (n + NT - 1) / NT;
    switch (dtype) {
        case DSCR_F64: k_seam_residual<double><<<grid, NT, 0, s>>>((const double*)D, ldd, n, idx, nnz, x, u, y, r_x, r_u); break;
        case DSCR_F32: k_seam_residual<float><<<grid, NT, 0, s>>>((const float*)D, ldd, n, idx, nnz, x, u, y, r_x, r_u); break;
        case DSCR_BF16:
            k_seam_residual<__nv_bfloat16><<<grid, NT, 0, s>>>((const __nv_bfloat16*)D, ldd, n, idx, nnz, x, u, y, r_x, r_u);
            break;
        default: return inval("unknown dtype");
    }
    k_seam_residual_red<<<1, NT, 0, s>>>(n, r_x, r_u, y, red_out);
    return cuda_check("residual");
}

size_t dscr_compact_work_size(int n) {
    return (size_t)std::max(1, (n + CMP_CHUNK - 1) / CMP_CHUNK) * sizeof(int);
}

int dscr_compact(const int32_t* active, int n, const uint8_t* mask, int32_t* active_out, int32_t* n_out, void* work,
                 size_t work_bytes, void* stream) {
    if ((n > 0 && (!active || !mask || !active_out)) || !n_out || !work || n < 0) return inval("bad compact arguments");
    if (work_bytes < dscr_compact_work_size(n)) return inval("compact workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = std::max(1, (n + CMP_CHUNK - 1) / CMP_CHUNK);
    int* cnt = static_cast<int*>(work);
    k_cmp_count<<<nb, NT, 0, s>>>(mask, n, cnt);
    k_cmp_scan<<<1, NT, 0, s>>>(cnt, nb, n_out);
    k_cmp_scatter<<<nb, NT, 0, s>>>(active, mask, n, cnt, active_out);
    return cuda_check("compact");
}

}  // extern "C"
