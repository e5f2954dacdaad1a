// Kernel-level C-ABI entry points of libdynscreen.so.  Each one replaces a
// reference per-op function (cited at the entry point) and uses the same
// device building blocks as the solver engine, so unit parity here covers the
// engine's arithmetic.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "dynscreen.h"
#include "dscr_device.cuh"

namespace dscr {
namespace ops {


static int cuda_err(const char* what, cudaError_t e) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    err_store() = buf;
    return DSCR_ECUDA;
}
static int inval(const char* what) {
    err_store() = what;
    return DSCR_EINVAL;
}
#define OCK(call)                                            \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_err(#call, e_);   \
    } while (0)

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// VG: the vectors are read through L2 (too tall for shared memory); they then need zero rows
// n..roundup(n, 16)-1, as every ldd-padded vector of the library has.
template <typename T, bool VG = false>
__global__ void __launch_bounds__(NT) k_corr(const T* __restrict__ D, int ldd, int n, int k,
                                             const double* __restrict__ v, double* out, int nvec,
                                             int ldv, int ldo) {
    extern __shared__ double s_v[];
    const uint64_t pol = make_policy(0.5f);
    if (!VG) {
        for (int q = 0; q < nvec; ++q)
            for (int i = threadIdx.x; i < ldd; i += NT) s_v[q * ldd + i] = (i < n) ? v[(size_t)q * ldv + i] : 0.0;
        __syncthreads();
    }
    const double* vb = VG ? v : s_v;
    const size_t vs = VG ? (size_t)ldv : (size_t)ldd;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * NT) >> 5;
    for (int j = gw; j < k; j += nwarps) {
        for (int q = 0; q < nvec; ++q) {
            double c = warp_dot<T, 2>(D + (size_t)j * ldd, n, vb + q * vs, lane, pol);
            if (lane == 0) out[(size_t)q * ldo + j] = c;
        }
    }
}

constexpr size_t CORR_SMEM_MAX = 227 * 1024 - 1024;   // larger vector sets are read through L2

// Split-K GEMV: CTA (tile, split) accumulates rows [tile*TR, +TR) of
// D[:, cols of split] x[cols of split, q] in fp64 and writes a partial vector;
// k_apply_reduce sums the splits in index order (deterministic).
constexpr int APPLY_CHUNK = NT;

template <typename T>
__global__ void __launch_bounds__(NT) k_apply_part(const T* __restrict__ D, int ldd, int n, int k,
                                                   const double* __restrict__ x, int nvec, int ldx,
                                                   double* part, int nsplit) {
    constexpr int V = Vec<T>::V;
    __shared__ double s_x[2][APPLY_CHUNK];
    __shared__ int s_j[APPLY_CHUNK];
    __shared__ int s_scan[2 * NW + 1];
    const int split = blockIdx.y;
    const int c0 = (int)(((long long)k * split) / nsplit), c1 = (int)(((long long)k * (split + 1)) / nsplit);
    const int r0 = (blockIdx.x * NT + threadIdx.x) * V;
    const uint64_t pol = make_policy(0.5f);
    double acc[2][V];
#pragma unroll
    for (int v = 0; v < V; ++v) { acc[0][v] = 0.0; acc[1][v] = 0.0; }
    for (int base = c0; base < c1; base += APPLY_CHUNK) {
        const int cn = min(APPLY_CHUNK, c1 - base);
        __syncthreads();
        // compact the chunk's nonzero columns (order preserved)
        const int i0 = threadIdx.x;
        double a = 0.0, b = 0.0;
        bool nz = false;
        if (i0 < cn) {
            a = x[base + i0];
            b = nvec > 1 ? x[(size_t)ldx + base + i0] : 0.0;
            nz = (a != 0.0 || b != 0.0);
        }
        int m;
        const int pos = block_exscan(nz ? 1 : 0, s_scan, &m);
        if (nz) { s_j[pos] = base + i0; s_x[0][pos] = a; s_x[1][pos] = b; }
        __syncthreads();
        if (r0 < n) {
            int i = 0;
            for (; i + 4 <= m; i += 4) {
                double d[4][V];
#pragma unroll
                for (int q = 0; q < 4; ++q) Vec<T>::load(D + (size_t)s_j[i + q] * ldd + r0, d[q], pol);
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        acc[0][v] = fma(s_x[0][i + q], d[q][v], acc[0][v]);
                        acc[1][v] = fma(s_x[1][i + q], d[q][v], acc[1][v]);
                    }
            }
            for (; i < m; ++i) {
                double d[V];
                Vec<T>::load(D + (size_t)s_j[i] * ldd + r0, d, pol);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    acc[0][v] = fma(s_x[0][i], d[v], acc[0][v]);
                    acc[1][v] = fma(s_x[1][i], d[v], acc[1][v]);
                }
            }
        }
    }
    if (r0 < ldd) {
        for (int q = 0; q < nvec; ++q)
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (r0 + v < ldd) part[((size_t)split * 2 + q) * ldd + r0 + v] = (r0 + v < n) ? acc[q][v] : 0.0;
    }
}

__global__ void k_apply_reduce(const double* part, int nsplit, int ldd, int nvec, double* out, int ldo) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ldd * nvec; i += gridDim.x * blockDim.x) {
        const int q = i / ldd, r = i % ldd;
        double s = 0.0;
        for (int p = 0; p < nsplit; ++p) s += part[((size_t)p * 2 + q) * ldd + r];
        out[(size_t)q * ldo + r] = s;
    }
}

static int apply_splits(int k, int ldd, int V) {
    const int R = (ldd + NT * V - 1) / (NT * V);
    return std::max(1, std::min((k + 63) / 64, std::max(1, (sm_count() * 4) / R)));
}

__global__ void k_soft(const double* v, int64_t n, double t, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = soft(v[i], t);
}

__global__ void k_group_shrink(const double* v, const int* gptr, int ng, const double* w, double t,
                               double* out) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        const int j0 = gptr[g], j1 = gptr[g + 1];
        const double nv = sqrt(np_segment_sum([&](int i) { double a = v[i]; return a * a; }, j0, j1 - j0));
        const double fac = (nv > 0.0) ? fmax(1.0 - t * w[g] / nv, 0.0) : 0.0;   // dictionary.py:297-300
        for (int j = j0; j < j1; ++j) out[j] = v[j] * fac;
    }
}

__global__ void k_test_sphere(const double* cc, const int* kept, int nk, double r, uint8_t* m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += gridDim.x * blockDim.x)
        m[i] = ((1.0 - fabs(cc[kept[i]])) - r > SCREEN_MARGIN) ? 1 : 0;
}

__global__ void k_test_dome(const double* tcorr, const double* ucorr, const int* kept, int nk,
                            double lam, double lstar, double radius, uint8_t* m) {
    const double shift = lstar / lam - 1.0;
    const double rs = hypot(radius, shift);
    const double cut = (rs > 0.0) ? shift / rs : 0.0;
    const double slope = lstar - lam, flat = lam * (1.0 - rs), mg = lam * SCREEN_MARGIN;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += gridDim.x * blockDim.x) {
        if (radius >= 1.0) { m[i] = 0; continue; }
        const double t = tcorr[kept[i]], u = ucorr[kept[i]];
        const double arc = (lam * radius) * sqrt(fmax(1.0 - t * t, 0.0));
        const double lower = (t < cut) ? (slope * t - lam) + arc : -flat;
        const double upper = (t <= -cut) ? flat : (slope * t + lam) - arc;
        m[i] = ((u - lower > mg) && (upper - u > mg)) ? 1 : 0;
    }
}

__global__ void k_test_group(const double* w, const double* cn, const double* sn, const int* kg, int nk,
                             double r, uint8_t* m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += gridDim.x * blockDim.x) {
        const int g = kg[i];
        m[i] = ((w[g] - cn[g]) / sn[g] - r > SCREEN_MARGIN) ? 1 : 0;
    }
}

// sums[0..4] = q1.z1, q1.z2, q2.z1, q2.z2 (h), and z1.z1, z1.z2, z2.z2 (for QR)
__global__ void __launch_bounds__(NT) k_pw_dots(const double* q, const double* z, int dim, int ld,
                                                int nvec, double* sums) {
    __shared__ double s_sh[64];
    double a[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < dim; i += NT) {
        const double q1 = q[i], z1 = z[i];
        const double q2 = nvec > 1 ? q[ld + i] : 0.0, z2 = nvec > 1 ? z[ld + i] : 0.0;
        a[0] = fma(q1, z1, a[0]); a[1] = fma(q1, z2, a[1]); a[2] = fma(q2, z1, a[2]); a[3] = fma(q2, z2, a[3]);
        a[4] = fma(z1, z1, a[4]); a[5] = fma(z1, z2, a[5]); a[6] = fma(z2, z2, a[6]);
    }
    for (int k = 0; k < 7; ++k) {
        double r = block_sum(a[k], s_sh);
        if (threadIdx.x == 0) sums[k] = r;
    }
}

// q1 = z1 / r11 ; q2 = (z2 - r12 q1) / r22  (Gram-Schmidt of the 2-column block)
__global__ void k_pw_qr(double* q, const double* z, int dim, int ld, int nvec, double r11, double r12,
                        double r22) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += gridDim.x * blockDim.x) {
        const double q1 = z[i] / r11;
        q[i] = q1;
        if (nvec > 1) q[ld + i] = (z[ld + i] - r12 * q1) / r22;
    }
}

// ---- operator norm, device-resident loop --------------------------------------
// State of the block power iteration (dictionary.py:120-160) kept on the device.
struct PwState {
    double val;        // previous top Rayleigh value
    double result;     // ||D||_2 when done
    int have;          // val valid
    int it;            // iterations done
    int done;
    int pad;
};

// Gram of the smaller side, fp64, upper-triangle tiles mirrored:
//   ROWS = true : H[a][b] = sum_k D[a][k] D[b][k]   (dim = n; rows of Dt are atoms)
//   ROWS = false: H[i][j] = sum_n D[n][i] D[n][j]   (dim = k; contraction along Dt rows)
// 128 x 128 tile per CTA, 8 x 8 outputs per thread strided by 16, 16-deep slices in smem.
constexpr int GR_T = 128, GR_K = 16;
template <typename T, bool ROWS>
__global__ void __launch_bounds__(256) k_gram(const T* D, int ldd, int n, int k, int dim, double* H) {
    __shared__ double sA[GR_K][GR_T], sB[GR_K][GR_T];
    const int bx = blockIdx.x, by = blockIdx.y;
    if (bx > by) return;                       // upper triangle of tiles
    const int i0 = bx * GR_T, j0 = by * GR_T;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[8][8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int p = 0; p < 8; ++p) acc[q][p] = 0.0;
    const int klen = ROWS ? k : n;             // contraction length
    for (int c0 = 0; c0 < klen; c0 += GR_K) {
        if (ROWS) {   // slice = rows c0..c0+15 of Dt, columns i0.. / j0.. (contiguous along n)
            const int kk = threadIdx.x / 16, cc = (threadIdx.x % 16) * 8;
            const int row = c0 + kk;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int a = i0 + cc + q, b = j0 + cc + q;
                sA[kk][cc + q] = (row < k && a < dim) ? elem(D + (size_t)row * ldd + a) : 0.0;
                sB[kk][cc + q] = (row < k && b < dim) ? elem(D + (size_t)row * ldd + b) : 0.0;
            }
        } else {      // slice = entries c0..c0+15 of Dt rows i0.. / j0..
            const int la = threadIdx.x >> 1, lk = (threadIdx.x & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int nn = c0 + lk + q;
                const int a = i0 + la, b = j0 + la;
                sA[lk + q][la] = (nn < n && a < dim) ? elem(D + (size_t)a * ldd + nn) : 0.0;
                sB[lk + q][la] = (nn < n && b < dim) ? elem(D + (size_t)b * ldd + nn) : 0.0;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GR_K; ++kk) {
            double a8[8], b8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) { a8[q] = sA[kk][tx + 16 * q]; b8[q] = sB[kk][ty + 16 * q]; }
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[q][p] = fma(a8[p], b8[q], acc[q][p]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int j = j0 + ty + 16 * q;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const int i = i0 + tx + 16 * p;
            if (i < dim && j < dim) {
                H[(size_t)j * dim + i] = acc[q][p];
                H[(size_t)i * dim + j] = acc[q][p];
            }
        }
    }
}

// z_v = H q_v for the two block vectors (H symmetric dim x dim, one warp per row)
__global__ void __launch_bounds__(NT) k_gram_mv(const double* H, int dim, const double* q, double* z, int ld,
                                                 int nvec, const PwState* st) {
    if (st->done) return;
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * NT + threadIdx.x) >> 5;
    if (r >= dim) return;
    const double* row = H + (size_t)r * dim;
    double a1 = 0.0, a2 = 0.0;
    for (int c = lane; c < dim; c += 32) {
        const double h = row[c];
        a1 = fma(h, q[c], a1);
        if (nvec > 1) a2 = fma(h, q[ld + c], a2);
    }
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) { z[r] = a1; if (nvec > 1) z[ld + r] = a2; }
}

__global__ void __launch_bounds__(NT) k_pw_init(double* q, int dim, int ld, int nvec, PwState* st) {
    __shared__ double s_sh[64];
    // start block [ones, (+1, -1, +1, ...)], orthonormalised (same span as np.linalg.qr)
    const double n1 = sqrt((double)dim);
    double dot = 0.0;
    for (int i = threadIdx.x; i < dim; i += NT) dot += ((i & 1) ? -1.0 : 1.0) / n1;
    dot = block_sum(dot, s_sh);
    double n2 = 0.0;
    for (int i = threadIdx.x; i < dim; i += NT) {
        const double v = ((i & 1) ? -1.0 : 1.0) - dot * (1.0 / n1);
        n2 = fma(v, v, n2);
    }
    n2 = sqrt(block_sum(n2, s_sh));
    for (int i = threadIdx.x; i < dim; i += NT) {
        q[i] = 1.0 / n1;
        if (nvec > 1) q[ld + i] = n2 > 0.0 ? (((i & 1) ? -1.0 : 1.0) - dot * (1.0 / n1)) / n2 : 0.0;
    }
    if (threadIdx.x == 0) { st->val = NAN; st->result = NAN; st->have = 0; st->it = 0; st->done = 0; }
}

// one step after z = op(q): Rayleigh 2 x 2 top value, stop test, restart, q <- QR(z); single CTA
__global__ void __launch_bounds__(NT) k_pw_step(double* q, const double* z, int dim, int ld, int nvec, double tol,
                                                 int max_iters, PwState* st, cudaGraphConditionalHandle h) {
    __shared__ double s_sh[64];
    if (st->done) return;
    double a[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < dim; i += NT) {
        const double q1 = q[i], z1 = z[i];
        const double q2 = nvec > 1 ? q[ld + i] : 0.0, z2 = nvec > 1 ? z[ld + i] : 0.0;
        a[0] = fma(q1, z1, a[0]); a[1] = fma(q1, z2, a[1]); a[2] = fma(q2, z1, a[2]); a[3] = fma(q2, z2, a[3]);
        a[4] = fma(z1, z1, a[4]); a[5] = fma(z1, z2, a[5]); a[6] = fma(z2, z2, a[6]);
    }
    block_sum_n<7>(a, s_sh);
    double top;
    if (nvec > 1) {
        const double b = 0.5 * (a[1] + a[2]);
        top = 0.5 * (a[0] + a[3]) + sqrt(0.25 * (a[0] - a[3]) * (a[0] - a[3]) + b * b);
    } else {
        top = a[0];
    }
    const int it = st->it;
    const bool conv = st->have && fabs(top - st->val) <= tol * fmax(1.0, fabs(top));
    const double r11 = sqrt(a[4]);
    const bool restart = !conv && !(r11 > 0.0);
    __syncthreads();
    if (conv) {
        if (threadIdx.x == 0) { st->result = sqrt(fmax(top, 0.0)); st->done = 1; cudaGraphSetConditional(h, 0); }
        return;
    }
    if (restart) {   // block fell into the null space: restart on basis axes
        for (int i = threadIdx.x; i < dim; i += NT) {
            q[i] = (i == it % dim) ? 1.0 : 0.0;
            if (nvec > 1) q[ld + i] = (i == (it + 1) % dim) ? 1.0 : 0.0;
        }
    } else {
        const double r12 = a[5] / r11;
        const double r22 = sqrt(fmax(a[6] - r12 * r12, 0.0));
        const double d22 = r22 > 0.0 ? r22 : 1.0;
        for (int i = threadIdx.x; i < dim; i += NT) {
            const double q1 = z[i] / r11;
            q[i] = q1;
            if (nvec > 1) q[ld + i] = (z[ld + i] - r12 * q1) / d22;
        }
    }
    if (threadIdx.x == 0) {
        st->val = top;
        st->have = restart ? 0 : 1;
        st->it = it + 1;
        if (it + 1 >= max_iters) {
            st->result = sqrt(fmax(restart ? NAN : top, 0.0));
            st->done = 1;
            cudaGraphSetConditional(h, 0);
        }
    }
}

template <typename T>
static int corr_launch(const void* D, int ldd, int n, int k, const double* v, double* out, int nvec,
                       int ldv, int ldo, cudaStream_t s) {
    const size_t smem = (size_t)ldd * 8 * nvec;
    const int grid = std::max(1, std::min((k + NW - 1) / NW, sm_count() * 4));
    if (smem > CORR_SMEM_MAX) {
        k_corr<T, true><<<grid, NT, 0, s>>>((const T*)D, ldd, n, k, v, out, nvec, ldv, ldo);
    } else {
        OCK(cudaFuncSetAttribute(k_corr<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_corr<T><<<grid, NT, smem, s>>>((const T*)D, ldd, n, k, v, out, nvec, ldv, ldo);
    }
    OCK(cudaGetLastError());
    return DSCR_OK;
}

template <typename T>
static int apply_launch(const void* D, int ldd, int n, int k, const double* x, double* out, int nvec,
                        int ldx, int ldo, double* part, cudaStream_t s) {
    constexpr int V = Vec<T>::V;
    const int R = (ldd + NT * V - 1) / (NT * V);
    const int P = apply_splits(k, ldd, V);
    k_apply_part<T><<<dim3(R, P), NT, 0, s>>>((const T*)D, ldd, n, k, x, nvec, ldx, part, P);
    OCK(cudaGetLastError());
    k_apply_reduce<<<std::max(1, std::min((ldd * nvec + 255) / 256, 2048)), 256, 0, s>>>(part, P, ldd, nvec, out, ldo);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

static int corr_any(int dt, const void* D, int ldd, int n, int k, const double* v, double* out, int nvec,
                    int ldv, int ldo, cudaStream_t s) {
    if (dt == DSCR_F64) return corr_launch<double>(D, ldd, n, k, v, out, nvec, ldv, ldo, s);
    if (dt == DSCR_F32) return corr_launch<float>(D, ldd, n, k, v, out, nvec, ldv, ldo, s);
    return corr_launch<__nv_bfloat16>(D, ldd, n, k, v, out, nvec, ldv, ldo, s);
}
static int apply_any(int dt, const void* D, int ldd, int n, int k, const double* x, double* out, int nvec,
                     int ldx, int ldo, double* part, cudaStream_t s) {
    if (dt == DSCR_F64) return apply_launch<double>(D, ldd, n, k, x, out, nvec, ldx, ldo, part, s);
    if (dt == DSCR_F32) return apply_launch<float>(D, ldd, n, k, x, out, nvec, ldx, ldo, part, s);
    return apply_launch<__nv_bfloat16>(D, ldd, n, k, x, out, nvec, ldx, ldo, part, s);
}

static size_t apply_part_bytes(int dt, int ldd, int k) {
    const int V = 32 / (dt == DSCR_F64 ? 8 : (dt == DSCR_F32 ? 4 : 2));   // Vec<T>::V (32-byte loads)
    return (size_t)apply_splits(k, ldd, V) * 2 * ldd * sizeof(double);
}

// Spectral norms of many small column groups at once (GroupPartition.build,
// dictionary.py:120-160 _power_top_eig per group): one CTA per group forms the m x m
// Gram D_g^T D_g in fp64 (columns staged through shared memory, fixed-order sums), then
// one warp runs the reference's 2-vector block power iteration on it (start block
// [ones, alternating] orthonormalised, Rayleigh 2 x 2 top eigenvalue, stop when stable to
// tol * max(1, value), basis-axis restart if the block falls into the null space).
// Groups with m > GN_MAXM or m > n get -1 (the host runs the general path for them).
constexpr int GN_MAXM = 32, GN_ROWS = 64, GN_PAIRS = 3;   // 3 x 256 >= 32 * 33 / 2

template <typename T>
__global__ void __launch_bounds__(NT) k_group_norms(const T* D, int ldd, int n, int ng, const int* gptr,
                                                     const int* gcols, double tol, int max_iters, double* out) {
    __shared__ double sX[GN_ROWS][GN_MAXM + 1];
    __shared__ double sG[GN_MAXM][GN_MAXM + 1];
    __shared__ int scol[GN_MAXM];
    const int g = blockIdx.x;
    if (g >= ng) return;
    const int c0 = gptr[g], m = gptr[g + 1] - c0;
    if (m < 1 || m > GN_MAXM || m > n) {
        if (threadIdx.x == 0) out[g] = -1.0;
        return;
    }
    if (threadIdx.x < m) scol[threadIdx.x] = gcols[c0 + threadIdx.x];
    const int npairs = m * (m + 1) / 2;
    int pk[GN_PAIRS], pl[GN_PAIRS];
    double acc[GN_PAIRS];
#pragma unroll
    for (int q = 0; q < GN_PAIRS; ++q) {
        int e = threadIdx.x + q * NT, k = 0;
        pk[q] = -1; pl[q] = -1; acc[q] = 0.0;
        if (e < npairs) {           // row-major upper triangle: (k, l), k <= l
            while (e >= m - k) { e -= m - k; ++k; }
            pk[q] = k; pl[q] = k + e;
        }
    }
    for (int r0 = 0; r0 < n; r0 += GN_ROWS) {
        __syncthreads();
        for (int e = threadIdx.x; e < GN_ROWS * m; e += NT) {
            const int rr = e % GN_ROWS, kk = e / GN_ROWS, row = r0 + rr;
            sX[rr][kk] = row < n ? elem(D + (size_t)scol[kk] * ldd + row) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < GN_PAIRS; ++q) {
            if (pk[q] < 0) continue;
            double a = acc[q];
            for (int rr = 0; rr < GN_ROWS; ++rr) a = fma(sX[rr][pk[q]], sX[rr][pl[q]], a);
            acc[q] = a;
        }
    }
#pragma unroll
    for (int q = 0; q < GN_PAIRS; ++q)
        if (pk[q] >= 0) { sG[pk[q]][pl[q]] = acc[q]; sG[pl[q]][pk[q]] = acc[q]; }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const bool in = lane < m;
    const int nvec = m > 1 ? 2 : 1;
    // start block: ones and (+1, -1, +1, ...), Gram-Schmidt
    const double n1 = sqrt((double)m);
    double q1 = in ? 1.0 / n1 : 0.0;
    double alt = in ? ((lane & 1) ? -1.0 : 1.0) : 0.0;
    const double dot0 = warp_sum(alt * q1);
    double q2 = alt - dot0 * q1;
    const double n2 = sqrt(warp_sum(q2 * q2));
    q2 = (nvec > 1 && n2 > 0.0) ? q2 / n2 : 0.0;
    double val = NAN;
    bool have = false;
    for (int it = 0; it < max_iters; ++it) {
        double z1 = 0.0, z2 = 0.0;
        for (int j = 0; j < m; ++j) {
            const double a = in ? sG[lane][j] : 0.0;
            z1 = fma(a, __shfl_sync(0xffffffffu, q1, j), z1);
            z2 = fma(a, __shfl_sync(0xffffffffu, q2, j), z2);
        }
        const double h11 = warp_sum(q1 * z1), h12 = warp_sum(q1 * z2), h21 = warp_sum(q2 * z1),
                     h22 = warp_sum(q2 * z2);
        double top;
        if (nvec > 1) {
            const double b = 0.5 * (h12 + h21);
            top = 0.5 * (h11 + h22) + sqrt(0.25 * (h11 - h22) * (h11 - h22) + b * b);
        } else {
            top = h11;
        }
        if (have && fabs(top - val) <= tol * fmax(1.0, fabs(top))) {
            if (lane == 0) out[g] = sqrt(fmax(top, 0.0));
            return;
        }
        val = top;
        have = true;
        const double z11 = warp_sum(z1 * z1), z12 = warp_sum(z1 * z2), z22 = warp_sum(z2 * z2);
        const double r11 = sqrt(z11);
        if (!(r11 > 0.0)) {   // block fell into the null space: restart on basis axes
            q1 = (lane == it % m) ? 1.0 : 0.0;
            q2 = (nvec > 1 && lane == (it + 1) % m) ? 1.0 : 0.0;
            have = false;
            continue;
        }
        const double r12 = z12 / r11;
        const double r22 = sqrt(fmax(z22 - r12 * r12, 0.0));
        q1 = z1 / r11;
        q2 = (nvec > 1) ? (z2 - r12 * q1) / (r22 > 0.0 ? r22 : 1.0) : 0.0;
    }
    if (lane == 0) out[g] = sqrt(fmax(val, 0.0));
}

// DSMX ingestion (dictionary.py:304-335 layout: row-major fp64): a block of `nr` file rows
// (nr x ncols, row-major, on the device) transposed into the column-major dictionary layout
// dst[col][row0 + r] (row stride ldd) with the storage conversion: fp64 as is, fp32 round to
// nearest, bf16 = fp64 -> fp32 -> bf16 round-to-nearest-even (workloads.bf16_round).
// 32 x 32 tiles through shared memory so both sides are coalesced.
template <typename T>
__device__ __forceinline__ T ingest_cvt(double v);
template <>
__device__ __forceinline__ double ingest_cvt<double>(double v) { return v; }
template <>
__device__ __forceinline__ float ingest_cvt<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ uint16_t ingest_cvt<uint16_t>(double v) {
    const uint32_t b = __float_as_uint(__double2float_rn(v));
    return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

template <typename T>
__global__ void __launch_bounds__(256) k_ingest_rows(const double* __restrict__ src, int nr, int ncols, int row0,
                                                     T* __restrict__ dst, int ldd) {
    __shared__ double tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8
    for (int j = ty; j < 32; j += 8) {
        const int r = r0 + j, c = c0 + tx;
        tile[j][tx] = (r < nr && c < ncols) ? src[(size_t)r * ncols + c] : 0.0;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int c = c0 + j, r = r0 + tx;
        if (c < ncols && r < nr) dst[(size_t)c * ldd + row0 + r] = ingest_cvt<T>(tile[tx][j]);
    }
}

static int check_dict(int dt, const void* D, int ldd, int n, int k) {
    if (dt < DSCR_F64 || dt > DSCR_BF16) return inval("unknown dtype");
    if (!D || n < 1 || k < 1 || ldd < n || ldd % 16) return inval("bad dictionary shape or ldd");
    return DSCR_OK;
}

// Gram path when one side is small and the other much longer: iterate on the dim x dim
// Gram (L2 / HBM resident) instead of two passes over D per iteration.
static bool pw_use_gram(int n, int k) {
    const long long dim = std::min(n, k), other = std::max(n, k);
    return dim <= 16384 && other >= 4 * dim;
}

static size_t pw_layout(int ldd, int n, int k, size_t* off_q, size_t* off_z, size_t* off_w, size_t* off_st,
                        size_t* off_part, size_t* off_h, int dt) {
    const size_t M = (size_t)std::max(ldd, k);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) / 256 * 256; return r; };
    *off_q = take(2 * M * 8);
    *off_z = take(2 * M * 8);
    *off_w = take(2 * M * 8);
    *off_st = take(sizeof(PwState));
    if (pw_use_gram(n, k)) {
        const size_t dim = (size_t)std::min(n, k);
        *off_part = 0;
        *off_h = take(dim * dim * 8);
    } else {
        *off_h = 0;
        *off_part = take(apply_part_bytes(dt, ldd, k) * 2);
    }
    return o;
}

template <typename T>
static void gram_launch(const void* D, int ldd, int n, int k, int dim, double* H, cudaStream_t s) {
    const int tiles = (dim + GR_T - 1) / GR_T;
    if (k >= n) k_gram<T, true><<<dim3(tiles, tiles), 256, 0, s>>>((const T*)D, ldd, n, k, dim, H);
    else k_gram<T, false><<<dim3(tiles, tiles), 256, 0, s>>>((const T*)D, ldd, n, k, dim, H);
}

}  // namespace ops
}  // namespace dscr

using namespace dscr;
using namespace dscr::ops;

extern "C" {


int dscr_correlate(int dtype, const void* D, int ldd, int n, int k, const double* v, double* out,
                   void* stream) {
    int rc = check_dict(dtype, D, ldd, n, k);
    if (rc) return rc;
    return corr_any(dtype, D, ldd, n, k, v, out, 1, ldd, k, (cudaStream_t)stream);
}

size_t dscr_apply_work_size(int dtype, int ldd, int k) { return apply_part_bytes(dtype, ldd, k) + 256; }

int dscr_apply(int dtype, const void* D, int ldd, int n, int k, const double* x, double* out, void* work,
               size_t work_bytes, void* stream) {
    int rc = check_dict(dtype, D, ldd, n, k);
    if (rc) return rc;
    if (!work || work_bytes < apply_part_bytes(dtype, ldd, k)) return inval("apply workspace too small");
    return apply_any(dtype, D, ldd, n, k, x, out, 1, k, ldd, (double*)work, (cudaStream_t)stream);
}

int dscr_prox_l1(const double* v, int64_t n, double t, double* out, void* stream) {
    if (t < 0) return inval("threshold must be nonnegative");
    if (n <= 0) return DSCR_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
    k_soft<<<grid, 256, 0, (cudaStream_t)stream>>>(v, n, t, out);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_prox_group(const double* v, const int32_t* gptr, int ng, const double* w, double t, double* out,
                    void* stream) {
    if (t < 0) return inval("threshold must be nonnegative");
    if (ng <= 0) return DSCR_OK;
    k_group_shrink<<<std::max(1, std::min((ng + 255) / 256, 4096)), 256, 0, (cudaStream_t)stream>>>(v, gptr, ng, w, t, out);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_test_sphere(const double* cc, const int32_t* kept, int nk, double r, uint8_t* m, void* stream) {
    if (nk <= 0) return DSCR_OK;
    k_test_sphere<<<std::max(1, std::min((nk + 255) / 256, 4096)), 256, 0, (cudaStream_t)stream>>>(cc, kept, nk, r, m);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_test_dome(const double* tc, const double* uc, const int32_t* kept, int nk, double lam, double lstar,
                   double radius, uint8_t* m, void* stream) {
    if (nk <= 0) return DSCR_OK;
    k_test_dome<<<std::max(1, std::min((nk + 255) / 256, 4096)), 256, 0, (cudaStream_t)stream>>>(tc, uc, kept, nk, lam, lstar, radius, m);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_test_group(const double* w, const double* cn, const double* sn, const int32_t* kg, int nk, double r,
                    uint8_t* m, void* stream) {
    if (nk <= 0) return DSCR_OK;
    k_test_group<<<std::max(1, std::min((nk + 255) / 256, 4096)), 256, 0, (cudaStream_t)stream>>>(w, cn, sn, kg, nk, r, m);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_ingest_rows_f64(const double* rows, int nr, int ncols, int row0, int dtype, void* dst, int ldd,
                         void* stream) {
    if (!rows || !dst || nr < 0 || ncols < 1 || row0 < 0 || row0 + nr > ldd) return inval("bad ingestion block");
    if (nr == 0) return DSCR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const dim3 grid((ncols + 31) / 32, (nr + 31) / 32);
    if (dtype == DSCR_F64) k_ingest_rows<double><<<grid, 256, 0, s>>>(rows, nr, ncols, row0, (double*)dst, ldd);
    else if (dtype == DSCR_F32) k_ingest_rows<float><<<grid, 256, 0, s>>>(rows, nr, ncols, row0, (float*)dst, ldd);
    else if (dtype == DSCR_BF16) k_ingest_rows<uint16_t><<<grid, 256, 0, s>>>(rows, nr, ncols, row0, (uint16_t*)dst, ldd);
    else return inval("unknown dtype");
    OCK(cudaGetLastError());
    return DSCR_OK;
}

int dscr_group_spectral_norms(int dtype, const void* D, int ldd, int n, int n_groups, const int32_t* group_ptr,
                              const int32_t* group_cols, double tol, int max_iters, double* out, void* stream) {
    if (dtype < DSCR_F64 || dtype > DSCR_BF16) return inval("unknown dtype");
    if (!D || n < 1 || ldd < n || ldd % 16) return inval("bad dictionary shape or ldd");
    if (n_groups <= 0) return DSCR_OK;
    if (!group_ptr || !group_cols || !out || max_iters < 1 || !(tol >= 0)) return inval("bad group arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == DSCR_F64)
        k_group_norms<double><<<n_groups, NT, 0, s>>>((const double*)D, ldd, n, n_groups, group_ptr, group_cols, tol, max_iters, out);
    else if (dtype == DSCR_F32)
        k_group_norms<float><<<n_groups, NT, 0, s>>>((const float*)D, ldd, n, n_groups, group_ptr, group_cols, tol, max_iters, out);
    else
        k_group_norms<__nv_bfloat16><<<n_groups, NT, 0, s>>>((const __nv_bfloat16*)D, ldd, n, n_groups, group_ptr, group_cols, tol, max_iters, out);
    OCK(cudaGetLastError());
    return DSCR_OK;
}

size_t dscr_operator_norm_work_size(int ldd, int k) {
    // n <= ldd < n + 16: size for n = ldd (largest Gram) and the apply partials of the widest dtype
    size_t q, z, w, st, part, h;
    const size_t a = pw_layout(ldd, ldd, k, &q, &z, &w, &st, &part, &h, DSCR_BF16);
    const size_t b = pw_layout(ldd, std::max(1, ldd - 15), k, &q, &z, &w, &st, &part, &h, DSCR_BF16);
    const size_t c = pw_layout(ldd, ldd, k, &q, &z, &w, &st, &part, &h, DSCR_F64);
    return std::max(a, std::max(b, c)) + 256;
}

// 2-vector block power iteration for the top eigenvalue of D^T D (dictionary.py:120-160):
// start block [ones, alternating], orthonormalised; stop when the top Rayleigh value is
// stable to tol * max(1, value); basis-axis restart when the block falls into the null space.
// The loop runs on the device inside a CUDA graph (conditional WHILE node, 4 steps per body):
// one host synchronisation per call.
int dscr_operator_norm(int dtype, const void* D, int ldd, int n, int k, double tol, int max_iters, void* work,
                       double* out_host, void* stream) {
    int rc = check_dict(dtype, D, ldd, n, k);
    if (rc) return rc;
    if (!work || !out_host) return inval("null work or output");
    if (max_iters < 1 || !(tol >= 0)) return inval("bad tolerance or iteration cap");
    cudaStream_t s = (cudaStream_t)stream;
    const bool small_cols = k <= n;           // operate on the smaller side of the Gram operator
    const int dim = small_cols ? k : n;
    const int ldq = small_cols ? k : ldd;     // leading dim of q and z (length-dim vectors)
    const int ldw = small_cols ? ldd : k;     // leading dim of the intermediate
    const int nvec = dim > 1 ? 2 : 1;
    const bool gram = pw_use_gram(n, k);
    size_t oq, oz, ow, ost, opart, oh;
    pw_layout(ldd, n, k, &oq, &oz, &ow, &ost, &opart, &oh, dtype);
    char* base = (char*)work;
    double* q = (double*)(base + oq);
    double* z = (double*)(base + oz);
    double* w = (double*)(base + ow);
    PwState* st = (PwState*)(base + ost);
    double* part = (double*)(base + opart);
    double* H = (double*)(base + oh);
    // function attributes before capture
    if (!gram && (size_t)ldd * 8 * nvec <= CORR_SMEM_MAX) {
        const size_t smem = (size_t)ldd * 8 * nvec;
        if (dtype == DSCR_F64) OCK(cudaFuncSetAttribute(k_corr<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else if (dtype == DSCR_F32) OCK(cudaFuncSetAttribute(k_corr<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else OCK(cudaFuncSetAttribute(k_corr<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStream_t cs = nullptr;
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    auto fail = [&](const char* what, cudaError_t err) {
        if (ge) cudaGraphExecDestroy(ge);
        if (g) cudaGraphDestroy(g);
        if (cs) cudaStreamDestroy(cs);
        return cuda_err(what, err);
    };
    if (e != cudaSuccess) return fail("stream create", e);
    if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) return fail("graph create", e);
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess)
        return fail("conditional handle", e);
    // prologue: Gram (if used) and the start block
    if ((e = cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return fail("capture", e);
    if (gram) {
        if (dtype == DSCR_F64) gram_launch<double>(D, ldd, n, k, dim, H, cs);
        else if (dtype == DSCR_F32) gram_launch<float>(D, ldd, n, k, dim, H, cs);
        else gram_launch<__nv_bfloat16>(D, ldd, n, k, dim, H, cs);
    }
    k_pw_init<<<1, NT, 0, cs>>>(q, dim, ldq, nvec, st);
    cudaGraph_t tmp = nullptr;
    e = cudaStreamEndCapture(cs, &tmp);
    if (e != cudaSuccess) return fail("end capture", e);
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    cudaGraphNode_t last = nodes.back();
    // WHILE node: body = 4 x (op; step)
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    if ((e = cudaGraphAddNode(&cnode, g, &last, 1, &cp)) != cudaSuccess) return fail("add WHILE node", e);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return fail("capture body", e);
    for (int r = 0; r < 4 && rc == DSCR_OK; ++r) {
        if (gram) {
            k_gram_mv<<<(dim + NW - 1) / NW, NT, 0, cs>>>(H, dim, q, z, ldq, nvec, st);
        } else if (small_cols) {
            if ((rc = apply_any(dtype, D, ldd, n, k, q, w, nvec, ldq, ldw, part, cs)) == DSCR_OK)
                rc = corr_any(dtype, D, ldd, n, k, w, z, nvec, ldw, ldq, cs);
        } else {
            if ((rc = corr_any(dtype, D, ldd, n, k, q, w, nvec, ldq, ldw, cs)) == DSCR_OK)
                rc = apply_any(dtype, D, ldd, n, k, w, z, nvec, ldw, ldq, part, cs);
        }
        k_pw_step<<<1, NT, 0, cs>>>(q, z, dim, ldq, nvec, tol, max_iters, st, h);
    }
    e = cudaStreamEndCapture(cs, &tmp);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cs);
        return rc;
    }
    if (e != cudaSuccess) return fail("end capture body", e);
    if ((e = cudaGraphInstantiate(&ge, g, 0)) != cudaSuccess) return fail("instantiate", e);
    if ((e = cudaGraphLaunch(ge, s)) != cudaSuccess) return fail("launch", e);
    PwState hs;
    if ((e = cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail("read result", e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail("sync", e);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    *out_host = hs.result;
    return DSCR_OK;
}
}
