// Batched many-observation path (BASELINE config 5): the correlation of every
// atom with every observation's residual, C = D^T Theta, is a dense
// contraction done on the 5th-generation tensor cores:
//
//   TMA (128B-swizzled tiles of D^T and Theta) -> 4-stage smem ring (mbarriers)
//   -> one elected thread issues tcgen05.mma (bf16 x bf16 -> fp32 in TMEM,
//      M=128 atoms x N=256 observations x K=16 per instruction)
//   -> double-buffered TMEM accumulators (2 x 256 columns)
//   -> 4 epilogue warps: tcgen05.ld -> fp32 C^T[obs][atom] (coalesced).
//
// Persistent: one CTA per SM walks the (atom-block, obs-block) tiles.
// Theta may be split into S bf16 terms (hi/lo) accumulated into the same TMEM
// tile, trading tensor-core time for accuracy of the fp64 residual.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include <algorithm>

#include "dynscreen.h"
#include "dscr_device.cuh"
#include "dscr_umma.cuh"

namespace dscr {
namespace batched {

using namespace umma;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 2 * BN;
constexpr int GEMM_THREADS = 192;   // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr size_t GEMM_SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;

struct GemmArgs {
    int Nb;          // observations per split (rows of one Theta block)
    int KB;          // 64-wide k-blocks per split
    int S;           // number of Theta splits accumulated
    int num_m, num_n, num_tiles;
    float* C;        // C^T [obs][atom]
    int ldc;
};

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_dt(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = base;
    uint8_t* sB = base + STAGES * A_BYTES;
    uint64_t* full = (uint64_t*)(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tslot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int kbs = g.KB * g.S;

    if (warp == 0) {
        if (lane == 0) {   // ---- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x) {
                const int mb = tile % g.num_m, nb = tile / g.num_m;
                for (int kb = 0; kb < kbs; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
                    const int s = kb / g.KB, k = (kb % g.KB) * BK;
                    tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], k, mb * BM);
                    tma_load_2d(sB + stage * B_BYTES, &tmB, &full[stage], k, s * g.Nb + nb * BN);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---- MMA issuer (single thread)
            const uint32_t idesc = idesc_bf16_f32(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int lt = 0;
            for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++lt) {
                const int ab = lt & 1;
                const uint32_t aphase = (lt >> 1) & 1;
                mbar_wait(&tempty[ab], aphase ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + ab * BN;
                for (int kb = 0; kb < kbs; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t da = desc_kmajor_sw128(smem_u32(sA + stage * A_BYTES));
                    const uint64_t db = desc_kmajor_sw128(smem_u32(sB + stage * B_BYTES));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)   // +32 B along K inside the swizzle atom
                        mma_bf16(dcol, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[ab]);
            }
        }
    } else {   // ---- epilogue: TMEM -> registers -> C^T[obs][atom]
        const int q = warp & 3;   // TMEM lane quarter this warp may access
        int lt = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++lt) {
            const int mb = tile % g.num_m, nb = tile / g.num_m;
            const int ab = lt & 1;
            const uint32_t aphase = (lt >> 1) & 1;
            mbar_wait(&tfull[ab], aphase);
            tc_fence_after();
            const int m = mb * BM + q * 32 + lane;
            float* crow = g.C + (size_t)(nb * BN) * g.ldc + m;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + ab * BN + c0, r);
#pragma unroll
                for (int i = 0; i < 32; ++i) crow[(size_t)(c0 + i) * g.ldc] = __uint_as_float(r[i]);
            }
            tc_fence_before();
            mbar_arrive(&tempty[ab]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 2-D bf16 tensor [rows][ld] (inner dimension `inner` elements), box = box_inner x box_rows, 128B swizzle
static int make_map(CUtensorMap* map, const void* ptr, int inner, int rows, int ld, int box_inner, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) { err_store() = "cuTensorMapEncodeTiled unavailable"; return DSCR_ECUDA; }
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[128];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        err_store() = buf;
        return DSCR_ECUDA;
    }
    return DSCR_OK;
}

int gemm_dt(const void* A, int M, int lda, const void* B, int Nb, int ldb, int K, int S, float* C, int ldc,
            cudaStream_t s) {
    if (M % BM || Nb % BN || K % BK || S < 1 || lda < K || ldb < K || lda % 8 || ldb % 8 || ldc < M) {
        err_store() = "batched gemm: need M%128==0, N%256==0, K%64==0, 16-byte aligned rows";
        return DSCR_EINVAL;
    }
    CUtensorMap ma, mb;
    int rc = make_map(&ma, A, K, M, lda, BK, BM);
    if (rc) return rc;
    rc = make_map(&mb, B, K, Nb * S, ldb, BK, BN);
    if (rc) return rc;
    GemmArgs g;
    g.Nb = Nb;
    g.KB = K / BK;
    g.S = S;
    g.num_m = M / BM;
    g.num_n = Nb / BN;
    g.num_tiles = g.num_m * g.num_n;
    g.C = C;
    g.ldc = ldc;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(k_gemm_dt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    if (e != cudaSuccess) { err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    k_gemm_dt<<<std::min(g.num_tiles, sms), GEMM_THREADS, GEMM_SMEM, s>>>(ma, mb, g);
    e = cudaGetLastError();
    if (e != cudaSuccess) { err_store() = cudaGetErrorString(e); return DSCR_ECUDA; }
    return DSCR_OK;
}

}  // namespace batched
}  // namespace dscr

extern "C" int dscr_batched_gemm_bf16(const void* A, int M, int lda, const void* B, int Nb, int ldb, int K,
                                      int splits, float* C, int ldc, void* stream) {
    return dscr::batched::gemm_dt(A, M, lda, B, Nb, ldb, K, splits, C, ldc, (cudaStream_t)stream);
}
