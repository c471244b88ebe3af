// glx_tc.cu -- tcgen05 (5th-gen tensor core) GEMM for the wide configuration
// (1024 -> 1024 -> 16 on 16M rows), BF16 operands, FP32
// accumulation in TMEM.
//
//   D[M x N] = A[M x K] . B[N x K]^T      (A, B row-major = K-major, bf16)
//
// One CTA per 128 x BN output tile. Warp 0 (one lane) drives TMA: 2-D tiles
// of 64 K-elements (128 B rows, 128-byte swizzle) into a 4-stage shared ring
// with mbarrier complete_tx. Warp 1 allocates TMEM and one lane issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16 per instruction),
// releasing each ring slot with tcgen05.commit. Warps 2-5 are the epilogue:
// tcgen05.ld 32x32b.x32 TMEM -> registers (each warp owns its 32-lane TMEM
// quadrant), then the fused epilogue (plain f32 store, or bias + sigmoid ->
// bf16 for the forward hidden layer).
#include <cuda.h>
#include <cuda_bf16.h>

#include "glx_common.cuh"
#include "glx_kernels.h"

#include <cstdio>

namespace glx {

constexpr int kTcBM = 128;
constexpr int kTcBK = 64;  // bf16 elements per 128-byte swizzled row
constexpr int kTcStages = 4;
constexpr int kTcThreads = 192;

// ------------------------------------------------------------- descriptors
// UMMA shared-memory descriptor, K-major, 128-byte swizzle (canonical layout:
// 8-row x 128-byte atoms, atoms 1024 B apart): start>>4 | LBO=1 | SBO=1024>>4 |
// version 1 (sm100) | layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor: BF16 x BF16 -> F32, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

struct TcEpilogue {
    int kind;            // 0: D f32 store; 1: bias + sigmoid -> bf16 store
    float* d_f32;        // kind 0
    __nv_bfloat16* d_bf16;  // kind 1
    const float* bias;   // kind 1: per column (length N)
    int ldd;             // leading dimension of D (elements)
};

template <int BN>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                                                  const __grid_constant__ CUtensorMap map_b, int M,
                                                                  int N, int K, TcEpilogue ep) {
    constexpr uint32_t kABytes = kTcBM * kTcBK * 2;
    constexpr uint32_t kBBytes = BN * kTcBK * 2;
    constexpr uint32_t kStage = kABytes + kBBytes;
    constexpr uint32_t kCols = BN < 32 ? 32 : BN;  // TMEM allocation: power of two >= 32
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128-byte swizzle atoms
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTcStages * kStage);
    uint64_t* empty = full + kTcStages;
    uint64_t* done = empty + kTcStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * kTcBM, n0 = blockIdx.x * BN;
    const int nk = K / kTcBK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kTcStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (int kb = 0; kb < nk; kb++) {
                const int s = kb % kTcStages;
                if (kb >= kTcStages) mbar_wait(&empty[s], ((kb / kTcStages) - 1) & 1);
                unsigned char* st = sm + s * kStage;
                mbar_arrive_expect_tx(&full[s], kStage);
                tma_load_2d(st, &map_a, kb * kTcBK, m0, &full[s]);
                tma_load_2d(st + kABytes, &map_b, kb * kTcBK, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(kTcBM, BN);
            for (int kb = 0; kb < nk; kb++) {
                const int s = kb % kTcStages;
                mbar_wait(&full[s], (kb / kTcStages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a_addr = smem_u32(sm + s * kStage);
                const uint32_t b_addr = a_addr + kABytes;
#pragma unroll
                for (int kk = 0; kk < kTcBK / 16; kk++) {  // 32-byte K steps inside the 128-byte row
                    umma_bf16(tmem, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                              (kb | kk) != 0);
                }
                umma_commit(&empty[s]);  // slot free once these MMAs have read it
            }
            umma_commit(done);  // accumulator complete
        }
    } else {
        // epilogue: warp w owns TMEM lanes [32*(w%4), 32*(w%4)+32)
        const int quad = warp & 3;
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int row = m0 + quad * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + c, v);
            if (row < M) {
                if (ep.kind == 0) {
                    float4* dst = reinterpret_cast<float4*>(ep.d_f32 + (int64_t)row * ep.ldd + n0 + c);
#pragma unroll
                    for (int q = 0; q < 8; q++) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                } else {
                    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(ep.d_bf16 + (int64_t)row * ep.ldd + n0 + c);
#pragma unroll
                    for (int q = 0; q < 16; q++) {
                        const float z0 = v[2 * q] + ep.bias[n0 + c + 2 * q];
                        const float z1 = v[2 * q + 1] + ep.bias[n0 + c + 2 * q + 1];
                        dst[q] = __floats2bfloat162_rn(1.0f / (1.0f + __expf(-z0)), 1.0f / (1.0f + __expf(-z1)));
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
    }
}

// -------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// row-major [rows x cols] bf16 matrix, box [box_rows x 64 cols], 128-byte swizzle
static bool make_map_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static cudaError_t tc_launch(const void* A, const void* B, int M, int N, int K, const TcEpilogue& ep,
                             cudaStream_t st) {
    CUtensorMap ma, mb;
    if (!make_map_bf16(&ma, A, M, K, kTcBM) || !make_map_bf16(&mb, B, N, K, BN)) return cudaErrorInvalidValue;
    const size_t smem = 1024 + (size_t)kTcStages * (kTcBM + BN) * kTcBK * 2 + 256;
    auto k = tc_gemm_kernel<BN>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(N / BN, (M + kTcBM - 1) / kTcBM);
    k<<<grid, kTcThreads, smem, st>>>(ma, mb, M, N, K, ep);
    return cudaGetLastError();
}

cudaError_t launch_tc_gemm(const void* A, const void* B, int M, int N, int K, int epi, float* d_f32,
                           void* d_bf16, const float* bias, int ldd, cudaStream_t st) {
    if (K % kTcBK != 0) return cudaErrorInvalidValue;
    TcEpilogue ep{epi, d_f32, reinterpret_cast<__nv_bfloat16*>(d_bf16), bias, ldd};
    if (N % 256 == 0) return tc_launch<256>(A, B, M, N, K, ep, st);
    if (N % 128 == 0) return tc_launch<128>(A, B, M, N, K, ep, st);
    if (N % 64 == 0) return tc_launch<64>(A, B, M, N, K, ep, st);
    if (N % 32 == 0) return tc_launch<32>(A, B, M, N, K, ep, st);
    return cudaErrorInvalidValue;
}

}  // namespace glx
