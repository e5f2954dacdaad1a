// Device helpers shared by the engine and the kernel-level entry points.
// Compiled with -fmad=false: every multiply-add that should fuse says fma()
// explicitly, so elementwise formulas round exactly like the reference's numpy
// expressions (one rounding per operation, same evaluation order).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#ifdef DSCR_CHECKS
#include <assert.h>
// bounds checks of the checked build (libdynscreen_checked.so, DSCR_LIB=checked): a failed check
// traps the kernel (cudaErrorAssert) with the file and line; compiled out of the default build
#define DSCR_CHECK(cond) assert(cond)
#else
#define DSCR_CHECK(cond) ((void)0)
#endif

namespace dscr {

// error text shared by every translation unit of the library (thread local)
inline std::string& err_store() {
    static thread_local std::string s;
    return s;
}

constexpr int NT = 256;          // threads per CTA of the per-unit kernels
constexpr int NW = NT / 32;
constexpr double SCREEN_MARGIN = 1e-12;     // screening.py:40
constexpr double RADIUS_GUARD = 1e-8;       // screening.py:33
constexpr double MAJ_SLACK = 1e-12;         // solvers.py:39
constexpr double L_CEILING = 1e300;         // solvers.py:40

// ---- 32-byte vector loads of dictionary elements, widened to fp64 ---------
// LDG.E.NA.256 with an L2 cache-policy descriptor: the dictionary is streamed
// once per iteration, so it bypasses L1; the L2 policy (see make_policy) keeps
// a resident fraction when the dictionary is near L2 size and evicts first
// when it is far larger.
__device__ __forceinline__ uint64_t make_policy(float keep_frac) {
    uint64_t pol;
    if (keep_frac >= 1.0f) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    } else if (keep_frac <= 0.0f) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    } else {
        asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(pol) : "f"(keep_frac));
    }
    return pol;
}

// Vec<T>: Raw = 32 bytes as loaded; get(raw, i) widens element i to fp64.
template <typename T> struct Vec;
template <> struct Vec<double> {
    static constexpr int V = 4;
    struct Raw { double w[4]; };
    __device__ __forceinline__ static void load_raw(const double* p, Raw& r, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(r.w[0]), "=d"(r.w[1]), "=d"(r.w[2]), "=d"(r.w[3]) : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double get(const Raw& r, int i) { return r.w[i]; }
    __device__ __forceinline__ static void zero(Raw& r) { for (int i = 0; i < 4; ++i) r.w[i] = 0.0; }
    __device__ __forceinline__ static void load(const double* p, double (&o)[4], uint64_t pol) {
        Raw r; load_raw(p, r, pol);
        for (int i = 0; i < 4; ++i) o[i] = r.w[i];
    }
};
template <> struct Vec<float> {
    static constexpr int V = 8;
    struct Raw { float w[8]; };
    __device__ __forceinline__ static void load_raw(const float* p, Raw& r, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=f"(r.w[0]), "=f"(r.w[1]), "=f"(r.w[2]), "=f"(r.w[3]), "=f"(r.w[4]), "=f"(r.w[5]),
                       "=f"(r.w[6]), "=f"(r.w[7])
                     : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double get(const Raw& r, int i) { return (double)r.w[i]; }
    __device__ __forceinline__ static void zero(Raw& r) { for (int i = 0; i < 8; ++i) r.w[i] = 0.f; }
    __device__ __forceinline__ static void load(const float* p, double (&o)[8], uint64_t pol) {
        Raw r; load_raw(p, r, pol);
        for (int i = 0; i < 8; ++i) o[i] = (double)r.w[i];
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int V = 16;
    struct Raw { uint32_t w[8]; };
    __device__ __forceinline__ static void load_raw(const __nv_bfloat16* p, Raw& r, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                       "=r"(r.w[6]), "=r"(r.w[7])
                     : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double get(const Raw& r, int i) {
        const uint32_t x = r.w[i >> 1];
        return (double)__uint_as_float((i & 1) ? (x & 0xffff0000u) : (x << 16));
    }
    __device__ __forceinline__ static void zero(Raw& r) { for (int i = 0; i < 8; ++i) r.w[i] = 0u; }
    __device__ __forceinline__ static void load(const __nv_bfloat16* p, double (&o)[16], uint64_t pol) {
        Raw r; load_raw(p, r, pol);
        for (int i = 0; i < 16; ++i) o[i] = get(r, i);
    }
};

template <typename T>
__device__ __forceinline__ double elem(const T* p) { return (double)p[0]; }
template <>
__device__ __forceinline__ double elem<__nv_bfloat16>(const __nv_bfloat16* p) {
    return (double)__bfloat162float(p[0]);
}

// ---- warp / block reductions (fixed order => bitwise reproducible) -------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum over the CTA (NT threads); result valid in every thread.
template <int NTH = NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = (l < NTH / 32) ? sh[l] : 0.0;
        r = warp_sum(r);
        if (l == 0) sh[0] = r;
    }
    __syncthreads();
    r = sh[0];
    __syncthreads();
    return r;
}

// Sum of M values over the CTA in one smem exchange; results valid in every thread.
// sh must hold NW*M doubles.  Fixed order => bitwise reproducible.
template <int M>
__device__ __forceinline__ void block_sum_n(double (&v)[M], double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = warp_sum(v[m]);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) sh[m * NW + w] = v[m];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) r += sh[m * NW + q];
        v[m] = r;
    }
    __syncthreads();
}

// Max of M values over the CTA (every thread gets the results).
template <int M>
__device__ __forceinline__ void block_max_n(double (&v)[M], double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = warp_max(v[m]);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) sh[m * NW + w] = v[m];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double r = -INFINITY;
#pragma unroll
        for (int q = 0; q < NW; ++q) r = fmax(r, sh[m * NW + q]);
        v[m] = r;
    }
    __syncthreads();
}

// block_sum_n for a CTA of TPB threads (TPB a multiple of 32); sh holds (TPB/32)*M doubles
template <int M, int TPB>
__device__ __forceinline__ void block_sum_nt(double (&v)[M], double* sh) {
    constexpr int W = TPB / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = warp_sum(v[m]);
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) sh[m * W + w] = v[m];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < W; ++q) r += sh[m * W + q];
        v[m] = r;
    }
    __syncthreads();
}

// Exclusive scan of an int over the CTA; returns prefix, *total gets the sum.
__device__ __forceinline__ int block_exscan(int v, int* sh, int* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (l >= o) inc += t;
    }
    __syncthreads();
    if (l == 31) sh[w] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        int s = (l < NW) ? sh[l] : 0;
        int si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, si, o);
            if (l >= o) si += t;
        }
        if (l < NW) sh[NW + l] = si - s;   // exclusive warp offsets
        if (l == NW - 1) sh[2 * NW] = si;
    }
    __syncthreads();
    int res = sh[NW + w] + inc - v;
    *total = sh[2 * NW];
    __syncthreads();
    return res;
}

// "Last CTA done" ticket.  Returns true in every thread of the last CTA.
__device__ __forceinline__ bool last_block(unsigned* ticket, unsigned nblocks, int* flag_sh) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = atomicAdd(ticket, 1u);
        *flag_sh = (t == nblocks - 1);
    }
    __syncthreads();
    bool last = *flag_sh != 0;
    if (last) {
        __threadfence();
        if (threadIdx.x == 0) *ticket = 0u;   // re-arm for the next launch
    }
    return last;
}

// ---- reference elementwise maps, one rounding per numpy operation ---------

// np.sign(v) * np.maximum(np.abs(v) - t, 0.0)   (problems.py:106-111)
__device__ __forceinline__ double soft(double v, double t) {
    double a = fabs(v) - t;
    double m = (a > 0.0 || a != a) ? a : 0.0;           // np.maximum propagates NaN
    if (v > 0.0) return m;
    if (v < 0.0) return -m;
    return (v == 0.0) ? 0.0 * m : v;                     // sign(0)=0, sign(nan)=nan
}

// np.clip(r, -b, b)
__device__ __forceinline__ double clip(double r, double b) {
    return fmin(fmax(r, -b), b);
}

// numpy pairwise summation of n contiguous doubles starting at index 1 of a
// reduceat segment: the segment value is a[0] + pairwise(a[1..n)).  Only used
// for group norms (dictionary.py:280-284), where n is the group size.
template <typename F>
__device__ __forceinline__ double np_pairwise_leaf(F get, int lo, int n) {   // n <= 128
    if (n < 8) {
        double r = -0.0;
        for (int i = 0; i < n; ++i) r += get(lo + i);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] += get(lo + i + j);
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += get(lo + i);
    return res;
}

// numpy's pairwise_sum: blocks of <= 128 summed 8-way, larger n split at n/2 (rounded down to a
// multiple of 8) and the halves added.  The recursion runs on an explicit stack so the whole
// function inlines: a recursive device function taking the accessor lambda forces the kernel
// parameters it captures into local memory (a ~700-byte Params copy per thread per launch).
template <typename F>
__device__ __forceinline__ double np_pairwise(F get, int lo, int n) {
    if (n <= 128) return np_pairwise_leaf(get, lo, n);
    int slo[32], sn[32], sst[32];
    double sleft[32];
    int sp = 0;
    slo[0] = lo; sn[0] = n; sst[0] = 0; sp = 1;
    double ret = 0.0;
    bool have = false;   // ret holds the value of the frame just popped
    while (sp > 0) {
        const int k = sp - 1;
        const int fl = slo[k], fn = sn[k];
        int n2 = fn / 2;
        n2 -= n2 % 8;
        if (!have) {
            if (fn <= 128) { ret = np_pairwise_leaf(get, fl, fn); have = true; --sp; continue; }
            sst[k] = 1;                                   // descend left
            slo[sp] = fl; sn[sp] = n2; sst[sp] = 0; ++sp;
        } else if (sst[k] == 1) {                         // left done: descend right
            sleft[k] = ret; sst[k] = 2; have = false;
            slo[sp] = fl + n2; sn[sp] = fn - n2; sst[sp] = 0; ++sp;
        } else {                                          // both done
            ret = sleft[k] + ret;
            --sp;
        }
    }
    return ret;
}

template <typename F>
__device__ __forceinline__ double np_segment_sum(F get, int lo, int n) {
    if (n <= 0) return 0.0;
    if (n == 1) return get(lo);
    return get(lo) + np_pairwise(get, lo + 1, n - 1);
}

// ---- warp dot products of dictionary columns with an smem vector ---------
// Columns are contiguous (column-major, leading dimension ldd).  Each lane
// streams 32-byte vectors; all C*U loads of a step are issued before any is
// consumed, and the smem vector is read once per step for all C columns.
template <typename T, int C, int U>
__device__ __forceinline__ void warp_dots(const T* const (&col)[C], int n, const double* sv, int lane,
                                          uint64_t pol, double (&out)[C]) {
    constexpr int V = Vec<T>::V;
    double acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    for (int base = lane * V; base < n; base += 32 * V * U) {
        typename Vec<T>::Raw d[U][C];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + u * 32 * V;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (i < n && col[c]) Vec<T>::load_raw(col[c] + i, d[u][c], pol);
                else Vec<T>::zero(d[u][c]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + u * 32 * V;
            if (i < n) {
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double t = sv[i + v];
#pragma unroll
                    for (int c = 0; c < C; ++c) acc[c] = fma(Vec<T>::get(d[u][c], v), t, acc[c]);
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) out[c] = warp_sum(acc[c]);
}

template <typename T, int U>
__device__ __forceinline__ double warp_dot(const T* __restrict__ col, int n, const double* sv, int lane,
                                           uint64_t pol) {
    const T* cols[1] = {col};
    double out[1];
    warp_dots<T, 1, U>(cols, n, sv, lane, pol, out);
    return out[0];
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace dscr
