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

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>

namespace glx {

constexpr int kTcBM = 128;
constexpr int kTcBK = 64;  // bf16 elements per 128-byte swizzled row
#ifndef GLX_TC_MAXBN
#define GLX_TC_MAXBN 256  // widest N tile (TMEM columns) per CTA
#endif
#ifndef GLX_TC_STAGES
#define GLX_TC_STAGES 4  // persistent kernel, 1 CTA per SM: the TMEM double buffer overlaps epilogue and MMA
#endif
// ring depth per tile width: 4 x 48 KB stages at BN = 256, up to 8 for narrow tiles
__host__ __device__ constexpr int tc_stages(int BN) {
    return (GLX_TC_STAGES * (kTcBM + 256) * kTcBK * 2) / ((kTcBM + BN) * kTcBK * 2) > 8
               ? 8
               : (GLX_TC_STAGES * (kTcBM + 256) * kTcBK * 2) / ((kTcBM + BN) * kTcBK * 2);
}
// per-epilogue-warp staging for TMA stores of bf16 results: two 32 x 32 bf16
// blocks (2 KB each) per warp, used alternately
#ifndef GLX_TC_STG_SETS
#define GLX_TC_STG_SETS 1  // staging sets of 2 blocks per epilogue warp
#endif
constexpr int kTcStgSets = GLX_TC_STG_SETS;
constexpr int kTcStgBlk = 32 * 32;  // bf16 elements per staged block
constexpr int kTcStgBytes = 8 * 2 * kTcStgSets * kTcStgBlk * 2;
constexpr int kTcThreads = 320;  // TMA warp + MMA warp + 8 epilogue warps

// ------------------------------------------------------------- descriptors
// UMMA shared-memory descriptor, K-major, 128-byte swizzle (canonical layout:
// 8-row x 128-byte atoms, atoms 1024 B apart): start>>4 | LBO=1 | SBO=1024>>4 |
// version 1 (sm100) | layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// MN-major operand (M contiguous): 128-byte swizzled rows of 64 M-elements, one
// row per K index; LBO = byte stride between 64-element M atoms, SBO = 1024
// (8 K rows) -- the A operand of dW2 read straight from row-major H
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor: BF16 x BF16 -> F32, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// instruction descriptor: TF32 x TF32 -> F32, both K-major, M x N (tf32 MMAs take no
// MN-major operands: every operand of the tf32 path is stored K-major)
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// K-blocked operand ([K/64][rows][64]): box {64, rows, 1} is one contiguous span
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
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

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
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

// tcgen05.ld without the wait: the 32 registers are valid only after tmem_wait()
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct TcEpilogue {
    int kind;               // 0: f32 store; 1: bias+sigmoid -> bf16; 2: output layer; 3: delta_h; 4: f32 accumulate
    float* d_f32;           // 0, 4 (4: + blockIdx.z * zstride)
    __nv_bfloat16* d_bf16;  // 1
    __nv_bfloat16* d_t;     // 1 (optional): transposed copy of the bf16 result, row stride ldt
    const float* bias;      // 1, 2
    int ldd;
    int64_t zstride;
    // 2: output neuron per row (wide config): K sigmoid outputs, one-hot targets from labels
    const uint8_t* labels;
    int K;
    __nv_bfloat16* do_b;  // [M][64] bf16, columns >= K stay zero
    __nv_bfloat16* do_t;  // delta_o transposed, K-blocked [M/64][32][64] bf16 (the dW2 GEMM operand)
    double* stats;        // [loss, correct, wrong]
    // 3: delta_h = v * h (1 - h), row-major into d_bf16 (or transposed into dht)
    const __nv_bfloat16* h;
    int ldh;
    __nv_bfloat16* dht;
    int64_t ldt;  // row stride of the transposed outputs (d_t, dht) when t_blk == 0
    int t_blk;    // R > 0: transposed outputs K-blocked [M/64][R][64]
    // tf32 path (f32 storage; transposed outputs K-blocked [M/32][t_blk][32], written
    // with plain coalesced stores: a warp's 32 lanes are the 32 rows of one K block)
    float* h32;         // 1: sigmoid(v + bias) row-major, row stride ldd (may be null)
    float* t32;         // 1: the same transposed; 3: delta_h transposed
    const float* hin32; // 3: h row-major, row stride ldh
    float* do32;        // 2: delta_o row-major [M][32] (columns >= K zero)
    float* doT32;       // 2: delta_o transposed [M/32][32][32]
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Per-warp TMA store staging: two 2 KB blocks used alternately; a block is
// rewritten only after the bulk store issued from it two stores ago has read it.
struct EpiStage {
    uint16_t* buf;  // this warp's 2 x kTcStgBlk bf16
    int next;
    const CUtensorMap* map_d;  // row-major bf16 result (kind 1), box 32 x 32
    const CUtensorMap* map_t;  // transposed bf16 result (kinds 1, 3), box 32 x 32 (x 1 when K-blocked)
    bool t_blocked;
    __device__ __forceinline__ uint16_t* acquire(int lane) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(2 * kTcStgSets - 1) : "memory");
        __syncwarp();
        uint16_t* b = buf + next * kTcStgBlk;
        next = next + 1 == 2 * kTcStgSets ? 0 : next + 1;
        return b;
    }
    // make the generic-proxy writes of this warp visible to the bulk copy, then issue it
    __device__ __forceinline__ void release(const CUtensorMap* map, const uint16_t* b, int c0, int c1, int lane,
                                            bool blocked = false) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            if (blocked) tma_store_3d(map, b, c0 & 63, c1, c0 >> 6);
            else tma_store_2d(map, b, c0, c1);
        }
    }
    __device__ __forceinline__ void drain(int lane) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
};

// kind 1: the row-major block and (optionally) its transpose from one staging
// pass with a single proxy fence; both staging blocks are reused only after
// the previous chunk's bulk stores have read them
__device__ __forceinline__ void store_rows_cols_bf16(EpiStage& sg, const uint32_t (&pk)[16], int row0, int col0,
                                                     int lane, bool with_t) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(2 * (kTcStgSets - 1)) : "memory");
    __syncwarp();
    uint16_t* br = sg.buf + sg.next * kTcStgBlk;
    uint16_t* bt = br + kTcStgBlk;
    sg.next = sg.next + 2 == 2 * kTcStgSets ? 0 : sg.next + 2;
    uint4* d = reinterpret_cast<uint4*>(br + lane * 32);
#pragma unroll
    for (int q = 0; q < 4; q++) d[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    if (with_t) {
#pragma unroll
        for (int e = 0; e < 16; e++) {
            bt[(2 * e) * 32 + lane] = (uint16_t)(pk[e] & 0xFFFFu);
            bt[(2 * e + 1) * 32 + lane] = (uint16_t)(pk[e] >> 16);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(sg.map_d, br, col0, row0);
        if (with_t) {
            if (sg.t_blocked) tma_store_3d(sg.map_t, bt, row0 & 63, col0, row0 >> 6);
            else tma_store_2d(sg.map_t, bt, row0, col0);
        }
    }
}

struct TcGemm {
    const void* A;  // [M x K] bf16, row stride lda
    const void* B;  // [N x K] bf16, row stride ldb
    int M, N, K;
    int64_t lda, ldb;
    int splits;         // split-K: blockIdx.z takes K / splits
    int a_blk, b_blk;   // 0: row-major; R > 0: K-blocked [K/64][R][64] (lda/ldb unused)
    int a_mn = 0;       // 1: A stored [K][M] (M contiguous, row stride lda): MN-major operand
    int b_mn = 0;       // 1: B stored [K][N] (N contiguous, row stride ldb): MN-major operand
};

// lane = row, pk[e] = columns 2e, 2e+1 of that row; stored transposed
__device__ __forceinline__ void store_cols_bf16(EpiStage& sg, const uint32_t (&pk)[16], int row0, int col0, int lane) {
    uint16_t* b = sg.acquire(lane);
#pragma unroll
    for (int e = 0; e < 16; e++) {
        b[(2 * e) * 32 + lane] = (uint16_t)(pk[e] & 0xFFFFu);
        b[(2 * e + 1) * 32 + lane] = (uint16_t)(pk[e] >> 16);
    }
    sg.release(sg.map_t, b, row0, col0, lane, sg.t_blocked);
}

// f32 accumulate into global memory without the load round trip: one writer per element
// per launch (split-K slab), so the sum is the same a + b as a read-modify-write
__device__ __forceinline__ void red_add_v4(float* dst, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
#ifndef GLX_TC_F32_TMA_H
#define GLX_TC_F32_TMA_H 1  // tf32 hidden layer: H rows leave through staged TMA stores (0: per-lane float4 stores)
#endif
#ifndef GLX_TC_RED
#define GLX_TC_RED 1  // kind 4 (split-K accumulate) with vector reductions (0: load + add + store)
#endif

// tf32 path epilogues (f32 results): lane = row, v = 32 consecutive columns n0 + c ..
__device__ __forceinline__ void tc_epilogue_chunk_f32(const TcEpilogue& ep, const float (&v)[32], int M, int row,
                                                      int n0, int c, int lane, EpiStage& sg) {
    const bool rv = row < M;
    const int64_t kb = (int64_t)(row >> 5) * ep.t_blk;  // K block of this row (transposed outputs)
    if (GLX_TC_RED && ep.kind == 4) {
        if (rv) {
            float* dst = ep.d_f32 + (int64_t)row * ep.ldd + n0 + c;
#pragma unroll
            for (int q = 0; q < 8; q++) red_add_v4(dst + 4 * q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
    } else if (ep.kind == 0 || ep.kind == 4) {
        if (rv) {
            float4* dst = reinterpret_cast<float4*>(ep.d_f32 + (int64_t)row * ep.ldd + n0 + c);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                if (ep.kind == 4) {
                    const float4 p = dst[q];
                    o.x += p.x;
                    o.y += p.y;
                    o.z += p.z;
                    o.w += p.w;
                }
                dst[q] = o;
            }
        }
    } else if (ep.kind == 1) {
        float h[32];
        const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n0 + c);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const float4 b = __ldg(b4 + q);
            const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int e = 0; e < 4; e++) h[4 * q + e] = 1.0f / (1.0f + __expf(-(v[4 * q + e] + bv[e])));
        }
        if (ep.h32) {
#if GLX_TC_F32_TMA_H
            // the warp's 32 rows x 32 columns through a 128-byte-swizzled staging block and one
            // TMA store (per-lane row stores were 32 half-sector writes per instruction);
            // the block is reused once the previous chunk's store has read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            const uint32_t b = smem_u32(sg.buf) + lane * 128;
#pragma unroll
            for (int q = 0; q < 8; q++)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(b + ((q ^ (lane & 7)) << 4)),
                             "f"(h[4 * q]), "f"(h[4 * q + 1]), "f"(h[4 * q + 2]), "f"(h[4 * q + 3])
                             : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tma_store_2d(sg.map_d, sg.buf, n0 + c, row - lane);  // clips rows >= M
#else
            if (rv) {
                float4* dst = reinterpret_cast<float4*>(ep.h32 + (int64_t)row * ep.ldd + n0 + c);
#pragma unroll
                for (int q = 0; q < 8; q++) dst[q] = make_float4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
            }
#endif
        }
        if (rv && ep.t32) {
#pragma unroll
            for (int j = 0; j < 32; j++) ep.t32[(kb + n0 + c + j) * 32 + (row & 31)] = h[j];
        }
    } else if (ep.kind == 2) {
        // output neuron (kernels.py:352-375 generalised to K outputs)
        float loss = 0.f, correct = 0.f, wrong = 0.f;
        if (rv) {
            const int lab = ep.labels[row];
            float best = -1.f;
            int arg = 0;
#pragma unroll
            for (int k = 0; k < 32; k++) {
                if (k >= ep.K) break;
                const float o = 1.0f / (1.0f + __expf(-(v[k] + ep.bias[k])));
                const float t = (k == lab) ? 1.f : 0.f;
                const float d = (o - t) * o * (1.0f - o);
                loss = fmaf(0.5f * (t - o), t - o, loss);
                if (o > best) {
                    best = o;
                    arg = k;
                }
                ep.do32[(int64_t)row * 32 + k] = d;
                ep.doT32[((int64_t)(row >> 5) * 32 + k) * 32 + (row & 31)] = d;
            }
            correct = arg == lab ? 1.f : 0.f;
            wrong = 1.f - correct;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            loss += __shfl_xor_sync(0xffffffffu, loss, o);
            correct += __shfl_xor_sync(0xffffffffu, correct, o);
            wrong += __shfl_xor_sync(0xffffffffu, wrong, o);
        }
        if (lane == 0 && ep.stats) {
            atomicAdd(ep.stats + 0, (double)loss);
            atomicAdd(ep.stats + 1, (double)correct);
            atomicAdd(ep.stats + 2, (double)wrong);
        }
    } else if (rv) {
        // delta_h = (delta_o W2)_j * h (1 - h), transposed (the dW1 GEMM's K-major B operand)
        const float4* hp = reinterpret_cast<const float4*>(ep.hin32 + (int64_t)row * ep.ldh + n0 + c);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const float4 h4 = hp[q];
            const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
            for (int e = 0; e < 4; e++)
                ep.t32[(kb + n0 + c + 4 * q + e) * 32 + (row & 31)] = v[4 * q + e] * hv[e] * (1.f - hv[e]);
        }
    }
}

template <int BN>
__device__ __forceinline__ void tc_epilogue_chunk(const TcEpilogue& ep, const float (&v)[32], int M, int row, int n0,
                                                  int c, int lane, EpiStage& sg) {
    const bool rv = row < M;
    if (GLX_TC_RED && ep.kind == 4) {
        if (rv) {
            float* dst = ep.d_f32 + (int64_t)row * ep.ldd + n0 + c;
#pragma unroll
            for (int q = 0; q < 8; q++) red_add_v4(dst + 4 * q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
    } else if (ep.kind == 0 || ep.kind == 4) {
        if (rv) {
            float4* dst = reinterpret_cast<float4*>(ep.d_f32 + (int64_t)row * ep.ldd +
                                                    n0 + c);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                if (ep.kind == 4) {
                    const float4 p = dst[q];
                    o.x += p.x;
                    o.y += p.y;
                    o.z += p.z;
                    o.w += p.w;
                }
                dst[q] = o;
            }
        }
    } else if (ep.kind == 1) {
        // 16-byte stores: 8 bf16 per store, 4 per 32-column chunk
        uint32_t pall[16];
        {
            const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n0 + c);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float4 ba = __ldg(b4 + 2 * q), bb = __ldg(b4 + 2 * q + 1);
                const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
                uint32_t* pk = pall + 4 * q;
                // sigmoid(z) = 1 / (1 + 2^(-log2e z)): MUFU ex2 + rcp, ample for a bf16 result
                const float2 nl2e = bcast2(-1.4426950408889634f);
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const float2 zs = __fmul2_rn(__fadd2_rn(make_float2(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]),
                                                            make_float2(bv[2 * e], bv[2 * e + 1])),
                                                 nl2e);
                    const __nv_bfloat162 h2 = __floats2bfloat162_rn(sigmoid_scaled(zs.x), sigmoid_scaled(zs.y));
                    pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
                }
            }
        }
        // TMA stores clip rows >= M of a tail tile
        store_rows_cols_bf16(sg, pall, row - lane, n0 + c, lane, ep.d_t != nullptr);
    } else if (ep.kind == 2) {
        // output neuron (kernels.py:352-375 generalised to K outputs)
        float loss = 0.f, correct = 0.f, wrong = 0.f;
        if (rv) {
            const int lab = ep.labels[row];
            float best = -1.f;
            int arg = 0;
#pragma unroll
            for (int k = 0; k < 32; k++) {
                if (k >= ep.K) break;
                const float o = 1.0f / (1.0f + __expf(-(v[k] + ep.bias[k])));
                const float t = (k == lab) ? 1.f : 0.f;
                const float d = (o - t) * o * (1.0f - o);
                loss = fmaf(0.5f * (t - o), t - o, loss);
                if (o > best) {
                    best = o;
                    arg = k;
                }
                const __nv_bfloat16 db = __float2bfloat16_rn(d);
                ep.do_b[(int64_t)row * 64 + k] = db;
                ep.do_t[((int64_t)(row >> 6) * 32 + k) * 64 + (row & 63)] = db;
            }
            correct = arg == lab ? 1.f : 0.f;
            wrong = 1.f - correct;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            loss += __shfl_xor_sync(0xffffffffu, loss, o);
            correct += __shfl_xor_sync(0xffffffffu, correct, o);
            wrong += __shfl_xor_sync(0xffffffffu, wrong, o);
        }
        if (lane == 0 && ep.stats) {
            atomicAdd(ep.stats + 0, (double)loss);
            atomicAdd(ep.stats + 1, (double)correct);
            atomicAdd(ep.stats + 2, (double)wrong);
        }
    } else {
        // delta_h = (delta_o W2)_j * h (1 - h): row-major (the dW1 GEMM reads it MN-major)
        uint32_t pall[16];
        uint4 hv[4] = {};
        if (rv) {
            const uint4* hp = reinterpret_cast<const uint4*>(ep.h + (int64_t)row * ep.ldh + n0 + c);
#pragma unroll
            for (int q4 = 0; q4 < 4; q4++) hv[q4] = hp[q4];
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; q4++) {
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hv[q4]);
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const float2 hf = __bfloat1622float2(h2[e]);
                const __nv_bfloat162 d2 = __floats2bfloat162_rn(v[q4 * 8 + 2 * e] * hf.x * (1.f - hf.x),
                                                                v[q4 * 8 + 2 * e + 1] * hf.y * (1.f - hf.y));
                pall[q4 * 4 + e] = *reinterpret_cast<const uint32_t*>(&d2);
            }
        }
        if (ep.d_bf16) store_rows_cols_bf16(sg, pall, row - lane, n0 + c, lane, false);  // row-major dH
        else store_cols_bf16(sg, pall, row - lane, n0 + c, lane);                         // transposed dH^T
    }
}

// Persistent tcgen05 GEMM: warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer, warps 2..9 = epilogue. The accumulator is double-buffered in TMEM
// (2 x BN columns), so the epilogue of tile i overlaps the MMAs of tile i+1.
// Tiles are walked (split z, M, N) with N fastest, so concurrently running
// CTAs share their A tile through L2.
// TF: the tf32 variant (f32 operands, kind::tf32, 32 K-elements per 128-byte row, f32
// epilogues); same stage bytes, same 4 MMAs (32 bytes of K each) per k-block.
template <int BN, bool TF>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                                                                  const __grid_constant__ CUtensorMap map_b,
                                                                  const __grid_constant__ CUtensorMap map_d,
                                                                  const __grid_constant__ CUtensorMap map_t, int flags,
                                                                  int M,
                                                                  int N, int K, int kb_per_split, int n_mt, int n_nt,
                                                                  int n_zt, TcEpilogue ep) {
    constexpr int kBKe = TF ? 32 : kTcBK;  // K elements per 128-byte row
    constexpr uint32_t kABytes = kTcBM * 128;
    constexpr uint32_t kBBytes = BN * 128;
    constexpr uint32_t kStage = kABytes + kBBytes;
    constexpr int kTcStages = tc_stages(BN);
    constexpr uint32_t kCols = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulators
    constexpr int kEpiCols = BN >= 64 ? BN / 2 : BN;        // columns per epilogue warp
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTcStages * kStage);
    uint64_t* empty = full + kTcStages;
    uint64_t* tfull = empty + kTcStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // staging blocks start 1024-aligned (the tf32 path's 128-byte-swizzled TMA stores)
    uint16_t* stg_all = reinterpret_cast<uint16_t*>(sm + kTcStages * kStage + 1024);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkt = K / kBKe;
    const int tiles = n_mt * n_nt * n_zt;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kTcStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);  // one arrival per epilogue warp
        }
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

    auto decode = [&](int t, int& z, int& m0, int& n0, int& kb0, int& nk) {
        z = t / (n_mt * n_nt);
        const int rem = t - z * (n_mt * n_nt);
        m0 = (rem / n_nt) * kTcBM;
        n0 = (rem % n_nt) * BN;
        kb0 = z * kb_per_split;
        nk = min(nkt - kb0, kb_per_split);
    };

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int z, m0, n0, kb0, nk;
                decode(t, z, m0, n0, kb0, nk);
                for (int kb = 0; kb < nk; kb++, it++) {
                    const int s = it % kTcStages;
                    if (it >= kTcStages) mbar_wait(&empty[s], ((it / kTcStages) - 1) & 1);
                    unsigned char* st = sm + s * kStage;
                    mbar_arrive_expect_tx(&full[s], kStage);
                    if (!TF && (flags & 8)) {  // MN-major A: two 64 (M) x 64 (K) swizzled atoms
                        tma_load_2d(st, &map_a, m0, (kb0 + kb) * kBKe, &full[s]);
                        tma_load_2d(st + kABytes / 2, &map_a, m0 + 64, (kb0 + kb) * kBKe, &full[s]);
                    } else if (flags & 1) tma_load_3d(st, &map_a, 0, m0, kb0 + kb, &full[s]);
                    else tma_load_2d(st, &map_a, (kb0 + kb) * kBKe, m0, &full[s]);
                    if (!TF && (flags & 16)) {  // MN-major B: BN / 64 atoms of 64 (N) x 64 (K)
#pragma unroll
                        for (int i = 0; i < BN / 64; i++)
                            tma_load_2d(st + kABytes + i * 8192, &map_b, n0 + 64 * i, (kb0 + kb) * kBKe, &full[s]);
                    } else if (flags & 2) tma_load_3d(st + kABytes, &map_b, 0, n0, kb0 + kb, &full[s]);
                    else tma_load_2d(st + kABytes, &map_b, (kb0 + kb) * kBKe, n0, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            const bool a_mn = !TF && (flags & 8) != 0, b_mn = !TF && (flags & 16) != 0;
            const uint32_t idesc = TF ? umma_idesc_tf32(kTcBM, BN)
                                      : umma_idesc_bf16(kTcBM, BN) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, lt++) {
                int z, m0, n0, kb0, nk;
                decode(t, z, m0, n0, kb0, nk);
                const int acc = lt & 1;
                if (lt >= 2) mbar_wait(&tempty[acc], ((lt / 2) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dcol = tmem + acc * BN;
                for (int kb = 0; kb < nk; kb++, it++) {
                    const int s = it % kTcStages;
                    mbar_wait(&full[s], (it / kTcStages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a_addr = smem_u32(sm + s * kStage);
                    const uint32_t b_addr = a_addr + kABytes;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) {  // 32 bytes of K per MMA
                        if constexpr (TF)
                            umma_tf32(dcol, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                                      idesc, (kb | kk) != 0);
                        else
                            umma_bf16(dcol,
                                      a_mn ? umma_desc_sw128_mn(a_addr + kk * 16 * 128, kABytes / 2)
                                           : umma_desc_sw128(a_addr + kk * 32),
                                      b_mn ? umma_desc_sw128_mn(b_addr + kk * 16 * 128, 8192)
                                           : umma_desc_sw128(b_addr + kk * 32),
                                      idesc, (kb | kk) != 0);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        // epilogue warps 2..9: TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4
        const int ew = warp - 2;
        const int quad = warp & 3;
        const int c0 = (BN >= 64) ? (ew >> 2) * kEpiCols : 0;
        const bool work = (BN >= 64) || ew < 4;
        EpiStage sg{stg_all + ew * 2 * kTcStgSets * kTcStgBlk, 0, &map_d, &map_t, (flags & 4) != 0};
        int lt = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, lt++) {
            int z, m0, n0, kb0, nk;
            decode(t, z, m0, n0, kb0, nk);
            const int acc = lt & 1;
            mbar_wait(&tfull[acc], (lt / 2) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (work) {
                TcEpilogue e2 = ep;
                if (ep.kind == 4) e2.d_f32 = ep.d_f32 + z * ep.zstride;
                const int row = m0 + quad * 32 + lane;
                // software pipeline: the TMEM load of chunk c + 32 is in flight
                // while chunk c goes through the epilogue math and stores
                const uint32_t tbase = tmem + acc * BN + ((uint32_t)(quad * 32) << 16);
                uint32_t ra[32], rb[32];
                tmem_ld32_async(tbase + c0, ra);
                tmem_wait();
#pragma unroll 1
                for (int c = c0; c < c0 + kEpiCols; c += 64) {
                    const bool more = c + 32 < c0 + kEpiCols;
                    if (more) tmem_ld32_async(tbase + c + 32, rb);
                    {
                        float v[32];
#pragma unroll
                        for (int i = 0; i < 32; i++) v[i] = __uint_as_float(ra[i]);
                        if constexpr (TF) tc_epilogue_chunk_f32(e2, v, M, row, n0, c, lane, sg);
                        else tc_epilogue_chunk<BN>(e2, v, M, row, n0, c, lane, sg);
                    }
                    if (!more) break;
                    tmem_wait();
                    if (c + 64 < c0 + kEpiCols) tmem_ld32_async(tbase + c + 64, ra);
                    {
                        float v[32];
#pragma unroll
                        for (int i = 0; i < 32; i++) v[i] = __uint_as_float(rb[i]);
                        if constexpr (TF) tc_epilogue_chunk_f32(e2, v, M, row, n0, c + 32, lane, sg);
                        else tc_epilogue_chunk<BN>(e2, v, M, row, n0, c + 32, lane, sg);
                    }
                    tmem_wait();
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        sg.drain(lane);
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

// row-major [rows x cols] bf16 matrix with row stride ld (elements), box
// [box_rows x box_cols]; loads: 64 cols, 128-byte swizzle, rows beyond `rows`
// read as zero; stores: 32 x 32, no swizzle, out-of-range elements skipped
static bool make_map_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                          int box_cols = kTcBK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K-blocked [nkb][R][64] bf16 operand: box {64 | box_k, box_rows, 1}
static bool make_map_blk(CUtensorMap* map, const void* base, int64_t R, int64_t nkb, int box_rows, int box_k,
                         CUtensorMapSwizzle swz) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)R, (cuuint64_t)nkb};
    cuuint64_t strides[2] = {64 * 2, (cuuint64_t)R * 64 * 2};
    cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// f32 (tf32 operand) maps: row-major [rows x cols] with 32-column 128-byte-swizzled
// boxes, and the K-blocked [nkb][R][32] layout
static bool make_map_f32(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool make_map_blk32(CUtensorMap* map, const void* base, int64_t R, int64_t nkb, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {32, (cuuint64_t)R, (cuuint64_t)nkb};
    cuuint64_t strides[2] = {32 * 4, (cuuint64_t)R * 32 * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static cudaError_t tc_launch_tf32(const TcGemm& g, const TcEpilogue& ep, cudaStream_t st) {
    CUtensorMap ma, mb, md, mt;
    memset(&md, 0, sizeof(md));
    memset(&mt, 0, sizeof(mt));
    const int64_t nkb = g.K / 32;
    const bool oka = g.a_blk ? make_map_blk32(&ma, g.A, g.a_blk, nkb, kTcBM) : make_map_f32(&ma, g.A, g.M, g.K, g.lda, kTcBM);
    const bool okb = g.b_blk ? make_map_blk32(&mb, g.B, g.b_blk, nkb, BN) : make_map_f32(&mb, g.B, g.N, g.K, g.ldb, BN);
    if (!oka || !okb || g.a_mn || g.b_mn) return cudaErrorInvalidValue;
    if (GLX_TC_F32_TMA_H && ep.kind == 1 && ep.h32) {  // H (f32, row-major) stores: 32 x 32 boxes, 128-byte swizzle
        EncodeTiledFn fn = encode_fn();
        cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)g.M};
        cuuint64_t strides[1] = {(cuuint64_t)ep.ldd * 4};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t estr[2] = {1, 1};
        if (!fn || fn(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ep.h32, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const int flags = (g.a_blk ? 1 : 0) | (g.b_blk ? 2 : 0);
    const size_t smem = 1024 + (size_t)tc_stages(BN) * (kTcBM + BN) * 128 + 1024 + kTcStgBytes;
    auto k = tc_gemm_kernel<BN, true>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nk = g.K / 32;
    const int splits = g.splits < 1 ? 1 : g.splits;
    const int kps = (nk + splits - 1) / splits;
    const int n_nt = g.N / BN, n_mt = (g.M + kTcBM - 1) / kTcBM, n_zt = (nk + kps - 1) / kps;
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = n_nt * n_mt * n_zt;
    const int grid = tiles < sms ? tiles : sms;
    k<<<grid, kTcThreads, smem, st>>>(ma, mb, md, mt, flags, g.M, g.N, g.K, kps, n_mt, n_nt, n_zt, ep);
    return cudaGetLastError();
}

// the tf32 GEMM: D = A . B^T with f32 operands rounded to tf32 by the tensor core
cudaError_t launch_tc_tf32(const TcGemm& g, const TcEpilogue& ep, cudaStream_t st) {
    if (g.K % 32 != 0) return cudaErrorInvalidValue;
    if (GLX_TC_MAXBN >= 256 && g.N % 256 == 0 && ep.kind != 2) return tc_launch_tf32<256>(g, ep, st);
    if (GLX_TC_MAXBN >= 128 && g.N % 128 == 0 && ep.kind != 2) return tc_launch_tf32<128>(g, ep, st);
    if (g.N % 64 == 0 && ep.kind != 2) return tc_launch_tf32<64>(g, ep, st);
    if (g.N % 32 == 0) return tc_launch_tf32<32>(g, ep, st);
    return cudaErrorInvalidValue;
}

template <int BN>
static cudaError_t tc_launch(const TcGemm& g, const TcEpilogue& ep, cudaStream_t st) {
    CUtensorMap ma, mb, md, mt;
    memset(&md, 0, sizeof(md));
    memset(&mt, 0, sizeof(mt));
    const int64_t nkb = g.K / kTcBK;
    const bool oka = g.a_mn    ? make_map_bf16(&ma, g.A, g.K, g.lda, g.lda, kTcBK, 64, CU_TENSOR_MAP_SWIZZLE_128B)
                     : g.a_blk ? make_map_blk(&ma, g.A, g.a_blk, nkb, kTcBM, kTcBK, CU_TENSOR_MAP_SWIZZLE_128B)
                               : make_map_bf16(&ma, g.A, g.M, g.K, g.lda, kTcBM);
    const bool okb = g.b_mn    ? (BN % 64 == 0 && make_map_bf16(&mb, g.B, g.K, g.ldb, g.ldb, kTcBK, 64,
                                                               CU_TENSOR_MAP_SWIZZLE_128B))
                     : g.b_blk ? make_map_blk(&mb, g.B, g.b_blk, nkb, BN, kTcBK, CU_TENSOR_MAP_SWIZZLE_128B)
                               : make_map_bf16(&mb, g.B, g.N, g.K, g.ldb, BN);
    if (!oka || !okb) return cudaErrorInvalidValue;
    if ((ep.kind == 1 || (ep.kind == 3 && ep.d_bf16)) &&
        !make_map_bf16(&md, ep.d_bf16, g.M, g.N, ep.ldd, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return cudaErrorInvalidValue;
    __nv_bfloat16* tdst = ep.kind == 1 ? ep.d_t : ep.kind == 3 ? ep.dht : nullptr;
    if (tdst) {
        const bool ok = ep.t_blk ? (g.M % 64 == 0 &&
                                    make_map_blk(&mt, tdst, ep.t_blk, g.M / 64, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE))
                                 : make_map_bf16(&mt, tdst, g.N, g.M, ep.ldt, 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (!ok) return cudaErrorInvalidValue;
    }
    const int flags = (g.a_blk ? 1 : 0) | (g.b_blk ? 2 : 0) | (ep.t_blk ? 4 : 0) | (g.a_mn ? 8 : 0) | (g.b_mn ? 16 : 0);
    const size_t smem = 1024 + (size_t)tc_stages(BN) * (kTcBM + BN) * kTcBK * 2 + 1024 + kTcStgBytes;
    auto k = tc_gemm_kernel<BN, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nk = g.K / kTcBK;
    const int splits = g.splits < 1 ? 1 : g.splits;
    const int kps = (nk + splits - 1) / splits;
    const int n_nt = g.N / BN, n_mt = (g.M + kTcBM - 1) / kTcBM, n_zt = (nk + kps - 1) / kps;
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = n_nt * n_mt * n_zt;
    const int grid = tiles < sms ? tiles : sms;
    k<<<grid, kTcThreads, smem, st>>>(ma, mb, md, mt, flags, g.M, g.N, g.K, kps, n_mt, n_nt, n_zt, ep);
    return cudaGetLastError();
}

cudaError_t launch_tc(const TcGemm& g, const TcEpilogue& ep, cudaStream_t st) {
    if (g.K % kTcBK != 0) return cudaErrorInvalidValue;
    if (GLX_TC_MAXBN >= 256 && g.N % 256 == 0 && ep.kind != 2) return tc_launch<256>(g, ep, st);
    if (GLX_TC_MAXBN >= 128 && g.N % 128 == 0 && ep.kind != 2) return tc_launch<128>(g, ep, st);
    if (g.N % 64 == 0 && ep.kind != 2) return tc_launch<64>(g, ep, st);
    if (g.N % 32 == 0) return tc_launch<32>(g, ep, st);
    return cudaErrorInvalidValue;
}


// =========================================================== wide config
// D = 1024 inputs, H = 1024 hidden, K = 16 sigmoid outputs,
// full-batch GD. Per epoch, in row chunks of C rows:
//   1. H     = sigmoid(X W1^T + b1)                 tcgen05, epilogue 1 -> bf16
//   2. delta_o per row (one-hot targets, K outputs)  tcgen05 (N=32 padded), epilogue 2
//   3. dH    = (delta_o W2) * h(1-h), row-major        tcgen05 (K=64 padded), epilogue 3
//   4. dW1^T += [X,1]^T dH                            tcgen05 split-K, epilogue 4 (dH read MN-major)
//   5. dW2^T += [H,1]^T delta_o                       tcgen05 split-K, epilogue 4 (H read MN-major)
// then W <- f32(W - lr/N grad) on the f32 master weights (reference layout).
constexpr int kWD = 1024, kWH = 1024, kWK = 16;
constexpr int kWMi = 1152;
constexpr int kWP = kWH * (kWD + 1) + kWK * (kWH + 1);  // 1,066,000 weights  // [X,1]^T rows padded to a multiple of 128 (rows > 1024 read as zero)

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return (uint32_t)x;
}
__device__ __forceinline__ float unit_u01(uint64_t seed, uint64_t idx) {
    return (mix32(seed * 0x9E3779B97F4A7C15ULL + idx) >> 8) * (1.0f / 16777216.0f);
}

// X[r][i] ~ U[0,1) (counter-based hash), bf16; labels = argmax_k of 16 planted
// linear scores over 32 fixed columns (a K-class analogue of synthetic_matrix's
// planted-linear labels)
template <typename T>
__global__ void wide_gen_kernel(T* __restrict__ X, uint8_t* __restrict__ labels, int64_t N,
                                uint64_t seed, int64_t row0) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
    if (r >= N) return;
    const int64_t rg = row0 + r;  // global row index: a shard is a slice of the full data set
    float score[kWK];
#pragma unroll
    for (int k = 0; k < kWK; k++) score[k] = 0.f;
    for (int i = threadIdx.x; i < kWD; i += 32) {
        const float v = unit_u01(seed, (uint64_t)rg * kWD + i);
        float xv;  // the stored value (bf16 path: rounded to bf16; tf32 path: the f32 U[0,1) draw)
        if constexpr (sizeof(T) == 2) {
            const __nv_bfloat16 b = __float2bfloat16_rn(v);
            X[r * kWD + i] = b;
            xv = __bfloat162float(b);
        } else {
            X[r * kWD + i] = v;
            xv = v;
        }
        if ((i & 31) == 7) {  // 32 planted columns
            const float vb = xv - 0.5f;  // centred: classes come out balanced
#pragma unroll
            for (int k = 0; k < kWK; k++) score[k] += (unit_u01(seed ^ 0xABCDEFULL, (uint64_t)k * kWD + i) - 0.5f) * vb;
        }
    }
#pragma unroll
    for (int k = 0; k < kWK; k++)
        for (int o = 16; o > 0; o >>= 1) score[k] += __shfl_xor_sync(0xffffffffu, score[k], o);
    if (threadIdx.x == 0) {
        int best = 0;
        for (int k = 1; k < kWK; k++)
            if (score[k] > score[best]) best = k;
        labels[r] = (uint8_t)best;
    }
}

// [X,1]^T in the K-blocked layout of the split-K operands: element (i, r) at
// ((r / 64) * 1025 + i) * 64 + r % 64; row i = 1024 is the bias input (1)
__device__ __forceinline__ int64_t kblk_index(int64_t r, int i, int R) { return ((r >> 6) * R + i) * 64 + (r & 63); }

__global__ void wide_transpose_kernel(const __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ XT, int64_t N) {
    __shared__ __nv_bfloat16 tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t r = r0 + dy;
        tile[dy][threadIdx.x] = r < N ? X[r * kWD + i0 + threadIdx.x] : __float2bfloat16_rn(0.f);
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t r = r0 + threadIdx.x;
        if (r < N) XT[kblk_index(r, i0 + dy, kWD + 1)] = tile[threadIdx.x][dy];
    }
    if (blockIdx.y == 0 && threadIdx.y == 0) {
        const int64_t r = r0 + threadIdx.x;
        if (r < N) XT[kblk_index(r, kWD, kWD + 1)] = __float2bfloat16_rn(1.f);
    }
}

// bf16 operand copies of the f32 master weights for this epoch
__global__ void wide_derive_kernel(const float* __restrict__ W1, const float* __restrict__ W2,
                                   __nv_bfloat16* __restrict__ W1b, float* __restrict__ b1,
                                   __nv_bfloat16* __restrict__ W2b, float* __restrict__ b2,
                                   __nv_bfloat16* __restrict__ W2T) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kWH * kWD) {
        const int j = e / kWD, i = e % kWD;
        W1b[e] = __float2bfloat16_rn(W1[(int64_t)j * (kWD + 1) + i]);
    }
    if (e < kWH) b1[e] = W1[(int64_t)e * (kWD + 1) + kWD];
    if (e < 32 * kWH) {
        const int k = e / kWH, j = e % kWH;
        W2b[e] = __float2bfloat16_rn(k < kWK ? W2[k * (kWH + 1) + j] : 0.f);
    }
    if (e < kWH * 64) {
        const int j = e / 64, k = e % 64;
        W2T[e] = __float2bfloat16_rn(k < kWK ? W2[k * (kWH + 1) + j] : 0.f);
    }
    if (e < kWK) b2[e] = W2[e * (kWH + 1) + kWH];
}

// grad (f64, reference layout: dW1 [1024][1025] then dW2 [16][1025]) = the
// split-K partial sums reduced in fixed slab order (dW1^T: [split][1152][1024],
// dW2^T: [split][1152][32], row 1024 = bias)
__global__ void wide_reduce_kernel(const float* __restrict__ dW1T, int splits, int64_t zstride,
                                   const float* __restrict__ dW2T, int splits2, int64_t zstride2,
                                   double* __restrict__ grad) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kWH * (kWD + 1)) {
        const int j = e / (kWD + 1), i = e % (kWD + 1);
        double g = 0.0;
        for (int z = 0; z < splits; z++) g += (double)dW1T[z * zstride + (int64_t)i * kWH + j];
        grad[e] = g;
    } else if (e < kWP) {
        const int e2 = e - kWH * (kWD + 1);
        const int k = e2 / (kWH + 1), j = e2 % (kWH + 1);
        double g = 0.0;
        for (int z = 0; z < splits2; z++) g += (double)dW2T[z * zstride2 + (int64_t)j * 32 + k];
        grad[e] = g;
    }
}

// W <- f32(f64(W) - lr/N * grad) over both layers (the reference's unfused op order)
__global__ void wide_apply_kernel(float* __restrict__ W1, float* __restrict__ W2, const double* __restrict__ grad,
                                  double lr_over_n, int* __restrict__ nonfinite) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= kWP) return;
    float* w = e < kWH * (kWD + 1) ? W1 + e : W2 + (e - kWH * (kWD + 1));
    const float v = __double2float_rn((double)*w - lr_over_n * grad[e]);
    *w = v;
    if (!isfinite(v) && nonfinite) atomicOr(nonfinite, 1);
}

cudaError_t launch_wide_gen(void* Xb, void* XT, uint8_t* labels, int64_t N, uint64_t seed, int64_t row0,
                            cudaStream_t st) {
    dim3 blk(32, 8);
    wide_gen_kernel<__nv_bfloat16><<<(unsigned)((N + 7) / 8), blk, 0, st>>>(reinterpret_cast<__nv_bfloat16*>(Xb),
                                                                           labels, N, seed, row0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((N + 31) / 32), kWD / 32);
    wide_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(Xb),
                                                       reinterpret_cast<__nv_bfloat16*>(XT), N);
    return cudaGetLastError();
}

constexpr int kWSplits2 = 16;  // split-K of the dW2 GEMM (9 M tiles x 16 = 144 CTAs)
constexpr int kWHL = 1088;     // row stride of H: 1024 units, the bias column, zero padding to 64

// H columns 1024.. of every row: 1 (the bias input of dW2), then zeros
__global__ void h_bias_cols_kernel(__nv_bfloat16* __restrict__ H, int64_t C) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= C * (kWHL - kWH)) return;
    const int64_t r = i / (kWHL - kWH);
    const int c = (int)(i - r * (kWHL - kWH));
    H[r * kWHL + kWH + c] = __float2bfloat16_rn(c == 0 ? 1.f : 0.f);
}

// ------------------------------------------------ wide tail: GEMMs 2, 3, 5 fused
// One persistent kernel per row chunk takes the chain that follows the hidden
// layer, so H is read from HBM once (GEMMs 2, 3 and 5 read it three times) and
// delta_o never leaves the SM. Per 128-row tile:
//   A  D_o[128 rows][16]  = H . W2^T              (SS, M=128 N=16, K = 1024: 16 H k-blocks)
//   B  epilogue: o = sigmoid(D_o + b2), delta_o, loss, argmax, sum delta_o (the
//      dW2 bias row); delta_o -> shared memory as the A operand of C and the B
//      operand of E (bf16, no-swizzle core-matrix layouts)
//   C  D_h[128 rows][64 units] = delta_o . W2      (SS, M=128 N=64 K=16, W2 read MN-major), per 64-unit chunk
//   E  dW2^T[128 units][16] += H^T . delta_o       (SS, A = the H k-block pair read MN-major,
//      M=128 units N=16 K=128 rows), accumulated in TMEM over the CTA's tiles
//   D  epilogue: dH = D_h * h (1 - h) with h from the k-block still in shared memory,
//      written over h in place (same 128-byte swizzle) and TMA-stored row-major
// The H k-blocks of a tile are streamed twice: pass 1 (from HBM) through ring 1
// for A, pass 2 (L2-hot: the tile was just read) through ring 2 for C/D/E, so a
// tile's 256 KB of H never has to stay resident. Each ring has its own producer
// thread and A and C/E their own MMA-issuing threads (tcgen05 operations of
// different threads touch disjoint TMEM columns and shared memory here), so the
// next tile's output layer streams in from HBM while this tile's deltas are
// written. TMEM: D_o [0,16), dW2^T [32,160) (8 unit blocks x 16 outputs), D_h
// 4 x 64 columns at 256.
#ifndef GLX_TL_S1
#define GLX_TL_S1 3
#endif
#ifndef GLX_TL_S2
#define GLX_TL_S2 8
#endif
#ifndef GLX_TL_GATE
#define GLX_TL_GATE 1  // pass 2 of a tile waits for its pass 1 (L2 reuse)
#endif
constexpr int kTlS1 = GLX_TL_S1;        // ring 1 stages (one H k-block of 128 rows x 64 units each)
constexpr int kTlS2 = GLX_TL_S2;        // ring 2 stages (even: E reads contiguous stage pairs)
static_assert(kTlS2 % 2 == 0, "ring 2 holds stage pairs");
constexpr int kTlKB = kWH / 64;         // 16 k-blocks per pass
constexpr int kTlSlabs = 160;           // per-CTA dW2 partial slabs (>= the SM count)
constexpr int kTlThreads = 384;         // P1 producer, A issuer, 8 epilogue warps, P2 producer, C/E issuer
constexpr uint32_t kTlStage = 128 * 128;
constexpr uint32_t kTlW2b = kTlKB * 16 * 128;  // W2 rows 0..15 as 16 k-blocks of 2 KB (128-byte swizzle)
constexpr uint32_t kTlDo = 128 * 16 * 2;       // delta_o tile, one layout
constexpr size_t kTlSmem = 1024 + (kTlS1 + kTlS2) * kTlStage + kTlW2b + 2 * kTlDo + 512;
static_assert(kTlSmem <= 232448, "wide tail shared memory");

// UMMA descriptor, no swizzle: core matrices of 8 rows x 16 B; LBO = K-direction
// stride, SBO = M/N-direction stride
__device__ __forceinline__ uint64_t umma_desc_ns(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}

// TMA with an L2 cache policy (createpolicy): pass 1 keeps its lines for pass 2
// (evict_last), pass 2 and the dH stores let theirs go first
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                 uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                     map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

#ifndef GLX_TL_HINTS
#define GLX_TL_HINTS 1
#endif

__global__ void __launch_bounds__(kTlThreads, 1) wide_tail_kernel(const __grid_constant__ CUtensorMap map_h,
                                                                    const __grid_constant__ CUtensorMap map_w2,
                                                                    const __grid_constant__ CUtensorMap map_dh,
                                                                    const float* __restrict__ b2,
                                                                    const uint8_t* __restrict__ labels, int M,
                                                                    float* __restrict__ slabs,
                                                                    double* __restrict__ stats) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned base, kept as an offset into the shared array (shared-space accesses)
    unsigned char* sm = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
    unsigned char* ring1 = sm;
    unsigned char* ring2 = ring1 + kTlS1 * kTlStage;
    unsigned char* w2b = ring2 + kTlS2 * kTlStage;
    unsigned char* doa = w2b + kTlW2b;  // delta_o [128 rows][K = 16]: (k/8) 2048 + (r/8) 128 + (r%8) 16 + (k%8) 2
    unsigned char* dot = doa + kTlDo;   // delta_o^T [16][K = 128 rows]: (r/8) 256 + (k/8) 128 + (k%8) 16 + (r%8) 2
    uint64_t* full1 = reinterpret_cast<uint64_t*>(dot + kTlDo);
    uint64_t* empty1 = full1 + kTlS1;   // A's MMAs read the stage
    uint64_t* full2 = empty1 + kTlS1;
    uint64_t* empty2 = full2 + kTlS2;   // one arrival per row quadrant (its dH store read the stage)
    uint64_t* ofull = empty2 + kTlS2;   // D_o written
    uint64_t* ofree = ofull + 1;        // D_o read (4 warps)
    uint64_t* doready = ofree + 1;      // delta_o in shared memory (4 warps)
    uint64_t* dhfull = doready + 1;     // [4] D_h buffer written (and every earlier C/E MMA done)
    uint64_t* dhfree = dhfull + 4;      // [4] D_h buffer read (8 warps)
    uint64_t* wbar = dhfree + 4;        // W2 loaded
    // pass 2 of a tile is issued only after its pass 1 landed (p1land), so it hits L2;
    // p2got (the pass-2 producer saw p1land) keeps A at most one tile ahead of it
    uint64_t* p1land = wbar + 1;
    uint64_t* p2got = p1land + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p2got + 1);
    float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [4 quadrants][16] bias-row partials

    constexpr uint32_t kColO = 0, kColW2 = 32, kColDH = 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (M + 127) / 128;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTlS1; s++) {
            mbar_init(&full1[s], 1);
            mbar_init(&empty1[s], 1);
        }
        for (int s = 0; s < kTlS2; s++) {
            mbar_init(&full2[s], 1);
            mbar_init(&empty2[s], 4);
        }
        mbar_init(ofull, 1);
        mbar_init(ofree, 4);
        mbar_init(doready, 4);
        for (int b = 0; b < 4; b++) {
            mbar_init(&dhfull[b], 1);
            mbar_init(&dhfree[b], 8);
        }
        mbar_init(wbar, 1);
        mbar_init(p1land, 1);
        mbar_init(p2got, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_h) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_dh) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t w2b_a = smem_u32(w2b), doa_a = smem_u32(doa), dot_a = smem_u32(dot);

    if (warp == 0) {
        if (lane == 0) {  // pass-1 producer (HBM): W2, then the tiles' k-blocks
            const uint64_t pol = l2_policy_evict_last();
            mbar_arrive_expect_tx(wbar, kTlW2b);
            for (int kb = 0; kb < kTlKB; kb++) tma_load_2d(w2b + kb * 2048, &map_w2, kb * 64, 0, wbar);
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
                for (int kb = 0; kb < kTlKB; kb++, it++) {
                    const int s = it % kTlS1;
                    if (it >= kTlS1) mbar_wait(&empty1[s], ((it / kTlS1) - 1) & 1);
                    mbar_arrive_expect_tx(&full1[s], kTlStage);
                    if (GLX_TL_HINTS) tma_load_2d_hint(ring1 + s * kTlStage, &map_h, kb * 64, t * 128, &full1[s], pol);
                    else tma_load_2d(ring1 + s * kTlStage, &map_h, kb * 64, t * 128, &full1[s]);
                }
        }
    } else if (warp == 10) {
        if (lane == 0) {  // pass-2 producer (L2)
            const uint64_t pol = l2_policy_evict_first();
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                if (GLX_TL_GATE) {
                    mbar_wait(p1land, lt & 1);
                    mbar_arrive(p2got);
                }
                for (int kb = 0; kb < kTlKB; kb++, it++) {
                    const int s = it % kTlS2;
                    if (it >= kTlS2) mbar_wait(&empty2[s], ((it / kTlS2) - 1) & 1);
                    mbar_arrive_expect_tx(&full2[s], kTlStage);
                    if (GLX_TL_HINTS) tma_load_2d_hint(ring2 + s * kTlStage, &map_h, kb * 64, t * 128, &full2[s], pol);
                    else tma_load_2d(ring2 + s * kTlStage, &map_h, kb * 64, t * 128, &full2[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // A issuer: the output layer of each tile
            mbar_wait(wbar, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t idO = umma_idesc_bf16(128, 16);
            const uint32_t r1 = smem_u32(ring1);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                if (lt > 0) {
                    mbar_wait(ofree, (lt - 1) & 1);
                    if (GLX_TL_GATE) mbar_wait(p2got, (lt - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                for (int kb = 0; kb < kTlKB; kb++, it++) {
                    const int s = it % kTlS1;
                    mbar_wait(&full1[s], (it / kTlS1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        umma_bf16(tmem + kColO, umma_desc_sw128(r1 + s * kTlStage + kk * 32),
                                  umma_desc_sw128(w2b_a + kb * 2048 + kk * 32), idO, (kb | kk) != 0);
                    umma_commit(&empty1[s]);
                }
                mbar_arrive(p1land);  // every pass-1 k-block of this tile has landed
                umma_commit(ofull);
            }
        }
    } else if (warp == 11) {
        if (lane == 0) {  // C/E issuer: hidden-delta pre-activations and dW2 of each tile
            mbar_wait(wbar, 0);
            const uint32_t idC = umma_idesc_bf16(128, 64) | (1u << 16);  // B (W2, [k][units]) MN-major
            const uint32_t idE = umma_idesc_bf16(128, 16) | (1u << 15);  // A (H^T) MN-major
            const uint32_t r2 = smem_u32(ring2);
            int it = 0, ct = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                mbar_wait(doready, lt & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int p = 0; p < kTlKB / 2; p++, it += 2) {
                    const int s0 = it % kTlS2;  // even: the pair (s0, s0 + 1) is contiguous
                    mbar_wait(&full2[s0], (it / kTlS2) & 1);
                    mbar_wait(&full2[s0 + 1], ((it + 1) / kTlS2) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int kk = 0; kk < 8; kk++)  // E: dW2^T for units 128p .. 128p + 127
                        umma_bf16(tmem + kColW2 + 16 * p, umma_desc_sw128_mn(r2 + s0 * kTlStage + kk * 2048, kTlStage),
                                  umma_desc_ns(dot_a + kk * 512, 256, 128), idE, (lt > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
                    for (int c2 = 0; c2 < 2; c2++, ct++) {  // C: units 64c .. 64c + 63
                        const int c = 2 * p + c2, b = ct & 3;
                        if (ct >= 4) {
                            mbar_wait(&dhfree[b], ((ct >> 2) - 1) & 1);
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        }
                        umma_bf16(tmem + kColDH + 64 * b, umma_desc_ns(doa_a, 2048, 128),
                                  umma_desc_sw128_mn(w2b_a + c * 2048, 2048), idC, 0u);
                        umma_commit(&dhfull[b]);
                    }
                }
            }
        }
    } else {
        // epilogue warps 2..9: TMEM lane quadrant = warp % 4 (rows 32 quad ..), column half hlf
        const int ew = warp - 2, quad = warp & 3, hlf = ew >> 2;
        const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
        const int r = quad * 32 + lane;  // row within the tile
        const uint32_t r2 = smem_u32(ring2);
        float bk[kWK];
#pragma unroll
        for (int k = 0; k < kWK; k++) bk[k] = b2[k];
        float dbias[kWK];
#pragma unroll
        for (int k = 0; k < kWK; k++) dbias[k] = 0.f;
        float loss = 0.f, correct = 0.f, valid = 0.f;
        int ct = 0, lt = 0, pend = -1;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
            const int row = t * 128 + r;
            if (hlf == 0) {  // B: output neuron per row (kernels.py:352-375 generalised to K outputs)
                const int lab = row < M ? labels[row] : 0;
                mbar_wait(ofull, lt & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t ro[16];
                tmem_ld16_async(tmem + lanebase + kColO, ro);
                tmem_wait();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(ofree);
                uint32_t pk[8];
                if (row < M) {
                    float best = -1.f;
                    int arg = 0;
                    float d[kWK];
#pragma unroll
                    for (int k = 0; k < kWK; k++) {
                        const float o = 1.0f / (1.0f + __expf(-(__uint_as_float(ro[k]) + bk[k])));
                        const float tk = (k == lab) ? 1.f : 0.f;
                        d[k] = (o - tk) * o * (1.0f - o);
                        loss = fmaf(0.5f * (tk - o), tk - o, loss);
                        if (o > best) {
                            best = o;
                            arg = k;
                        }
                    }
                    correct += arg == lab ? 1.f : 0.f;
                    valid += 1.f;
#pragma unroll
                    for (int e = 0; e < 8; e++) pk[e] = pack_bf16x2(d[2 * e], d[2 * e + 1]);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; e++) pk[e] = 0u;
                }
#pragma unroll
                for (int e = 0; e < 8; e++) {  // the dW2 bias row sums the bf16 delta_o the MMAs use
                    dbias[2 * e] += __uint_as_float(pk[e] << 16);
                    dbias[2 * e + 1] += __uint_as_float(pk[e] & 0xFFFF0000u);
                }
                sts128(doa_a + (r >> 3) * 128 + (r & 7) * 16, make_uint4(pk[0], pk[1], pk[2], pk[3]));
                sts128(doa_a + 2048 + (r >> 3) * 128 + (r & 7) * 16, make_uint4(pk[4], pk[5], pk[6], pk[7]));
                const uint32_t dt = dot_a + (r >> 3) * 256 + (r & 7) * 2;
#pragma unroll
                for (int k = 0; k < kWK; k++)
                    sts16(dt + (k >> 3) * 128 + (k & 7) * 16,
                          (uint16_t)((k & 1) ? (pk[k >> 1] >> 16) : (pk[k >> 1] & 0xFFFFu)));
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(doready);
            }
            // D: dH = D_h * h (1 - h), 16 chunks of 64 units; this warp takes 32 of them
            for (int c = 0; c < kTlKB; c++, ct++) {
                const int b = ct & 3;
                mbar_wait(&dhfull[b], (ct >> 2) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t v[32];
                tmem_ld32_async(tmem + lanebase + kColDH + 64 * b + 32 * hlf, v);
                const int it = lt * kTlKB + c, s = it % kTlS2;
                mbar_wait(&full2[s], (it / kTlS2) & 1);  // complete already (the MMAs read it)
                const uint32_t rowa = r2 + s * kTlStage + r * 128;
                uint4 hv[4];
#pragma unroll
                for (int q = 0; q < 4; q++) hv[q] = lds128(rowa + (((4 * hlf + q) ^ (r & 7)) << 4));
                tmem_wait();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&dhfree[b]);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    uint32_t* hw = reinterpret_cast<uint32_t*>(&hv[q]);
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[e]));
                        hw[e] = pack_bf16x2(__uint_as_float(v[8 * q + 2 * e]) * hf.x * (1.f - hf.x),
                                            __uint_as_float(v[8 * q + 2 * e + 1]) * hf.y * (1.f - hf.y));
                    }
                    sts128(rowa + (((4 * hlf + q) ^ (r & 7)) << 4), hv[q]);
                }
                fence_proxy_async();
                bar_sync(1 + quad, 64);  // both column halves of these 32 rows are written
                if (hlf == 0 && lane == 0) {
                    if (GLX_TL_HINTS)
                        tma_store_2d_hint(&map_dh, ring2 + s * kTlStage + quad * 32 * 128, c * 64, t * 128 + quad * 32,
                                          l2_policy_evict_first());
                    else
                        tma_store_2d(&map_dh, ring2 + s * kTlStage + quad * 32 * 128, c * 64, t * 128 + quad * 32);
                    // a stage is released once its store has read it, one chunk late; the
                    // tile's last stage at once (keeps the release independent of the next tile)
                    if (c + 1 < kTlKB) {
                        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        if (pend >= 0) mbar_arrive(&empty2[pend]);
                        pend = s;
                    } else {
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        if (pend >= 0) mbar_arrive(&empty2[pend]);
                        mbar_arrive(&empty2[s]);
                        pend = -1;
                    }
                }
            }
        }
        if (hlf == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        // dW2^T partials (TMEM lanes = units) into this CTA's slab: units 128p + 32 quad + lane
        float* slab = slabs + (int64_t)blockIdx.x * kWMi * 32;
        for (int p = 4 * hlf; p < 4 * hlf + 4; p++) {
            uint32_t w[16];
            tmem_ld16_async(tmem + lanebase + kColW2 + 16 * p, w);
            tmem_wait();
            float4* dst = reinterpret_cast<float4*>(slab + (int64_t)(128 * p + r) * 32);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                float4 a = dst[q];
                a.x += __uint_as_float(w[4 * q]);
                a.y += __uint_as_float(w[4 * q + 1]);
                a.z += __uint_as_float(w[4 * q + 2]);
                a.w += __uint_as_float(w[4 * q + 3]);
                dst[q] = a;
            }
        }
        if (hlf == 0) {  // bias row (unit 1024) and the statistics
#pragma unroll
            for (int k = 0; k < kWK; k++)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dbias[k] += __shfl_xor_sync(0xffffffffu, dbias[k], o);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                loss += __shfl_xor_sync(0xffffffffu, loss, o);
                correct += __shfl_xor_sync(0xffffffffu, correct, o);
                valid += __shfl_xor_sync(0xffffffffu, valid, o);
            }
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < kWK; k++) red[quad * kWK + k] = dbias[k];
                if (stats) {
                    atomicAdd(stats + 0, (double)loss);
                    atomicAdd(stats + 1, (double)correct);
                    atomicAdd(stats + 2, (double)(valid - correct));
                }
            }
            bar_sync(5, 128);
            if (quad == 0 && lane < kWK)
                slab[kWH * 32 + lane] += red[lane] + red[kWK + lane] + red[2 * kWK + lane] + red[3 * kWK + lane];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

struct WideWork {
    void* W1b;
    float* b1;
    void* W2b;
    float* b2;
    void* W2T;
    void* Hb;   // [C][kWHL] bf16: h in columns 0..1023, column 1024 = 1 (bias input of dW2), 1025.. = 0
    void* dob;  // [C][64] bf16
    void* doT;  // delta_o^T, K-blocked [C/64][32][64] bf16, rows >= 16 zero
    void* dht;  // dH, row-major [C][1024] bf16 (read MN-major by the dW1 GEMM)
    float* dW1T;
    float* dW2T;
    double* grad;  // [kWP + 3]: gradient sums, then loss, correct, wrong
    int64_t C;
    int splits;
};

static size_t carve(WideWork* w, unsigned char* base, int64_t C, int splits) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
        void* p = base ? base + o : nullptr;
        o += (bytes + 255) / 256 * 256;
        return p;
    };
    WideWork t;
    t.W1b = take((size_t)kWH * kWD * 2);
    t.b1 = (float*)take(kWH * 4);
    t.W2b = take(32 * kWH * 2);
    t.b2 = (float*)take(64);
    t.W2T = take((size_t)kWH * 64 * 2);
    t.Hb = take((size_t)C * kWHL * 2);
    t.dob = take((size_t)C * 64 * 2);
    t.doT = take((size_t)32 * C * 2);
    t.dht = take((size_t)kWH * C * 2);
    t.dW1T = (float*)take((size_t)splits * kWMi * kWH * 4);
    t.dW2T = (float*)take((size_t)std::max(kWSplits2, kTlSlabs) * kWMi * 32 * 4);
    t.grad = (double*)take((size_t)(kWP + 3) * 8);
    t.C = C;
    t.splits = splits;
    if (w) *w = t;
    return o;
}

size_t wide_work_bytes(int64_t C, int splits) { return carve(nullptr, nullptr, C, splits); }

// GLX_WIDE_TAIL=0 selects the unfused GEMMs 2, 3, 5 (A/B measurements)
bool wide_tail_enabled() {
    const char* v = getenv("GLX_WIDE_TAIL");
    return !(v && v[0] == '0');
}

static int sm_count() {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// the fused tail over the Cc rows of a chunk: dH -> dht, dW2^T partials -> slabs[blockIdx],
// stats += loss, correct, wrong
static cudaError_t launch_wide_tail(const WideWork& w, int Cc, const uint8_t* labels, double* stats, cudaStream_t st) {
    CUtensorMap mh, mw, md;
    if (!make_map_bf16(&mh, w.Hb, Cc, kWH, kWHL, 128) || !make_map_bf16(&mw, w.W2b, 32, kWH, kWH, 16) ||
        !make_map_bf16(&md, w.dht, Cc, kWH, kWH, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(wide_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTlSmem);
    if (e != cudaSuccess) return e;
    const int ntiles = (Cc + 127) / 128;
    const int grid = std::min(std::min(sm_count(), kTlSlabs), ntiles);
    wide_tail_kernel<<<grid, kTlThreads, kTlSmem, st>>>(mh, mw, md, w.b2, labels, Cc, w.dW2T, stats);
    return cudaGetLastError();
}

int wide_launches_per_chunk() { return wide_tail_enabled() ? 3 : 5; }
int wide32_launches_per_chunk() { return wide_tail_enabled() ? 4 : 5; }

// one epoch; stats (device, may be null): [loss, correct, wrong] accumulated
// gradient SUM over the N rows at the current weights -> grad[0, kWP) (f64),
// grad[kWP .. kWP+3) = loss, correct, wrong (grad may be the workspace's own)
cudaError_t wide_grad(const float* W1, const float* W2, const void* Xb, const void* XT, const uint8_t* labels,
                      int64_t N, unsigned char* work, int64_t C, int splits, double* grad, cudaStream_t st,
                      const std::function<void(bool)>& prof) {
    WideWork w;
    carve(&w, work, C, splits);
    cudaError_t e;
    if (!grad) grad = w.grad;
    double* stats = grad + kWP;
    if ((e = cudaMemsetAsync(stats, 0, 3 * sizeof(double), st)) != cudaSuccess) return e;
    const int n_derive = kWH * kWD;
    wide_derive_kernel<<<(n_derive + 255) / 256, 256, 0, st>>>(W1, W2, (__nv_bfloat16*)w.W1b, w.b1,
                                                               (__nv_bfloat16*)w.W2b, w.b2, (__nv_bfloat16*)w.W2T);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int64_t zstride = (int64_t)kWMi * kWH;
    if ((e = cudaMemsetAsync(w.dW1T, 0, (size_t)splits * zstride * 4, st)) != cudaSuccess) return e;
    const int64_t zstride2 = (int64_t)kWMi * 32;
    const bool tail = wide_tail_enabled();
    const int slabs2 = tail ? kTlSlabs : kWSplits2;
    if ((e = cudaMemsetAsync(w.dW2T, 0, (size_t)slabs2 * zstride2 * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.dob, 0, (size_t)C * 64 * 2, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.doT, 0, (size_t)32 * C * 2, st)) != cudaSuccess) return e;
    if (!tail) {  // the bias input column of H (only GEMM 5 reads it)
        h_bias_cols_kernel<<<(unsigned)((C * (kWHL - kWH) + 255) / 256), 256, 0, st>>>((__nv_bfloat16*)w.Hb, C);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    for (int64_t r0 = 0; r0 < N; r0 += C) {
        const int Cc = (int)std::min<int64_t>(C, N - r0);
        const __nv_bfloat16* Xc = reinterpret_cast<const __nv_bfloat16*>(Xb) + r0 * kWD;
        prof(true);
        {  // 1. hidden layer
            TcGemm g{Xc, w.W1b, Cc, kWH, kWD, kWD, kWD, 1};
            TcEpilogue ep{};
            ep.kind = 1;
            ep.d_bf16 = (__nv_bfloat16*)w.Hb;
            ep.bias = w.b1;
            ep.ldd = kWHL;
            if ((e = launch_tc(g, ep, st)) != cudaSuccess) return e;
        }
        if (tail) {  // 2, 3, 5 fused: delta_o, loss, accuracy, dH, dW2 partials
            if ((e = launch_wide_tail(w, Cc, labels + r0, stats, st)) != cudaSuccess) return e;
        }
        if (!tail) {  // 2. output layer -> delta_o, loss, accuracy
            TcGemm g{w.Hb, w.W2b, Cc, 32, kWH, kWHL, kWH, 1};
            TcEpilogue ep{};
            ep.kind = 2;
            ep.bias = w.b2;
            ep.labels = labels + r0;
            ep.K = kWK;
            ep.do_b = (__nv_bfloat16*)w.dob;
            ep.do_t = (__nv_bfloat16*)w.doT;
            ep.stats = stats;
            if ((e = launch_tc(g, ep, st)) != cudaSuccess) return e;
        }
        if (!tail) {  // 3. hidden deltas, row-major
            TcGemm g{w.dob, w.W2T, Cc, kWH, 64, 64, 64, 1};
            TcEpilogue ep{};
            ep.kind = 3;
            ep.h = (const __nv_bfloat16*)w.Hb;
            ep.ldh = kWHL;
            ep.d_bf16 = (__nv_bfloat16*)w.dht;  // dH row-major [C][1024]
            ep.ldd = kWH;
            if ((e = launch_tc(g, ep, st)) != cudaSuccess) return e;
        }
        {  // 4. dW1^T += [X,1]^T dH (split-K over the chunk's rows)
            const __nv_bfloat16* XTc = reinterpret_cast<const __nv_bfloat16*>(XT) + r0 * (kWD + 1);
            TcGemm g{XTc, w.dht, kWD + 1, kWH, Cc, 0, kWH, splits, kWD + 1, 0, 0, 1};  // B = dH read MN-major
            TcEpilogue ep{};
            ep.kind = 4;
            ep.d_f32 = w.dW1T;
            ep.ldd = kWH;
            ep.zstride = zstride;
            if ((e = launch_tc(g, ep, st)) != cudaSuccess) return e;
        }
        if (!tail) {  // 5. dW2^T += [H,1]^T delta_o (split-K; N = 32 with delta_o^T rows >= 16 zero); A = H read
           //    MN-major (rows = K), the bias column supplies the "1" input
            TcGemm g{w.Hb, w.doT, kWH + 1, 32, Cc, kWHL, 0, kWSplits2, 0, 32, 1};
            TcEpilogue ep{};
            ep.kind = 4;
            ep.d_f32 = w.dW2T;
            ep.ldd = 32;
            ep.zstride = zstride2;
            if ((e = launch_tc(g, ep, st)) != cudaSuccess) return e;
        }
        prof(false);
    }
    wide_reduce_kernel<<<(kWP + 255) / 256, 256, 0, st>>>(w.dW1T, splits, zstride, w.dW2T, slabs2, zstride2, grad);
    return cudaGetLastError();
}

cudaError_t wide_apply(float* W1, float* W2, const double* grad, double lr_over_n, int* nonfinite, cudaStream_t st) {
    wide_apply_kernel<<<(kWP + 255) / 256, 256, 0, st>>>(W1, W2, grad, lr_over_n, nonfinite);
    return cudaGetLastError();
}

// one fused epoch (single device): gradient into the workspace, then the update;
// stats (device, may be null) receives [loss, correct, wrong]
cudaError_t wide_epoch(float* W1, float* W2, const void* Xb, const void* XT, const uint8_t* labels, int64_t N,
                       double lr, unsigned char* work, int64_t C, int splits, double* stats, int* nonfinite,
                       cudaStream_t st, const std::function<void(bool)>& prof) {
    WideWork w;
    carve(&w, work, C, splits);
    cudaError_t e = wide_grad(W1, W2, Xb, XT, labels, N, work, C, splits, w.grad, st, prof);
    if (e != cudaSuccess) return e;
    if (stats && (e = cudaMemcpyAsync(stats, w.grad + kWP, 3 * sizeof(double), cudaMemcpyDeviceToDevice, st)) !=
                     cudaSuccess)
        return e;
    return wide_apply(W1, W2, w.grad, lr / (double)N, nonfinite, st);
}

// =============================================== wide config, tf32 path
// The same five GEMMs on tcgen05 kind::tf32 with f32 storage, for f32 U[0,1) rows
// (SURVEY.md C5 "evaluated against the FP32 tolerance"): every operand K-major
// (tf32 MMAs take no MN-major operands), so the epilogues write the transposed,
// K-blocked ([rows/32][R][32]) copies the split-K GEMMs read:
//   1. H = sigmoid(X W1^T + b1)   -> H (f32 row-major) and [H,1]^T (K-blocked, R = 1025)
//   2. output layer (N = 32)      -> delta_o row-major [C][32] and K-blocked [C/32][32][32]
//   3. dH = (delta_o W2) h(1-h)   -> dH^T K-blocked [C/32][1024][32]
//   4. dW1^T += [X,1]^T dH        (A = [X,1]^T K-blocked, stored with the data)
//   5. dW2^T += [H,1]^T delta_o
// Rows >= 1025 of a 128-row M tile of the [.,1]^T operands read as zero (TMA OOB).
constexpr int kWR = kWD + 1;  // rows of the [X,1]^T and [H,1]^T operands

// [X,1]^T, K-blocked by 32 rows: element (i, r) at ((r / 32) * 1025 + i) * 32 + r % 32
__global__ void wide_transpose32_kernel(const float* __restrict__ X, float* __restrict__ XT, int64_t N) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t r = r0 + dy;
        tile[dy][threadIdx.x] = r < N ? X[r * kWD + i0 + threadIdx.x] : 0.f;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t r = r0 + threadIdx.x;
        if (r < N) XT[((r >> 5) * kWR + i0 + dy) * 32 + (r & 31)] = tile[threadIdx.x][dy];
    }
    if (blockIdx.y == 0 && threadIdx.y == 0) {
        const int64_t r = r0 + threadIdx.x;
        if (r < N) XT[((r >> 5) * kWR + kWD) * 32 + (r & 31)] = 1.f;
    }
}

cudaError_t launch_wide_gen_tf32(float* X, float* XT, uint8_t* labels, int64_t N, uint64_t seed, int64_t row0,
                                 cudaStream_t st) {
    wide_gen_kernel<float><<<(unsigned)((N + 7) / 8), dim3(32, 8), 0, st>>>(X, labels, N, seed, row0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((N + 31) / 32), kWD / 32);
    wide_transpose32_kernel<<<grid, dim3(32, 8), 0, st>>>(X, XT, N);
    return cudaGetLastError();
}

// f32 operand copies of the master weights for this epoch: W1 without its bias
// column (16-byte rows for TMA), W2 padded to 32 outputs, W2^T [1024][32]
__global__ void wide_derive32_kernel(const float* __restrict__ W1, const float* __restrict__ W2,
                                     float* __restrict__ W1p, float* __restrict__ b1, float* __restrict__ W2p,
                                     float* __restrict__ b2, float* __restrict__ W2T) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kWH * kWD) {
        const int j = e / kWD, i = e % kWD;
        W1p[e] = W1[(int64_t)j * kWR + i];
    }
    if (e < kWH) b1[e] = W1[(int64_t)e * kWR + kWD];
    if (e < 32 * kWH) {
        const int k = e / kWH, j = e % kWH;
        W2p[e] = k < kWK ? W2[k * (kWH + 1) + j] : 0.f;
        const int j2 = e / 32, k2 = e % 32;
        W2T[e] = k2 < kWK ? W2[k2 * (kWH + 1) + j2] : 0.f;
    }
    if (e < kWK) b2[e] = W2[e * (kWH + 1) + kWH];
}

// row 1024 of the K-blocked [H,1]^T chunk buffer: the bias input 1
__global__ void ht_bias_row_kernel(float* __restrict__ HT, int64_t C) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < C) HT[((r >> 5) * kWR + kWD) * 32 + (r & 31)] = 1.f;
}

struct WideWork32 {
    float *W1p, *b1, *W2p, *b2, *W2T;
    float* H;    // [C][1024]
    float* HT;   // [C/32][1025][32]
    float* dob;  // [C][32]
    float* doT;  // [C/32][32][32]
    float* dhT;  // [C/32][1024][32]
    float* dW1T;
    float* dW2T;
    double* grad;
};

// ------------------------------------------- wide tail, tf32 path (CUDA cores)
// GEMMs 2 and 3 of the tf32 epoch fused into one streaming pass per 128-row tile. Both
// contractions are 16 wide (the K = 16 outputs), and tf32 MMAs take no MN-major
// operands (a second, transposed W2 copy would be needed), so this runs on the FP32
// pipe: 32 FMA per H element against 8 bytes of HBM traffic (H in, dH^T out).
//   pass 1 (H from HBM): o_pre[r][k] = sum_j H[r][j] W2[k][j] (fp32, more exact than the
//          tf32 GEMM it replaces); o = sigmoid(o_pre + b2), delta_o, loss, argmax;
//          delta_o -> the K-blocked delta_o^T operand of the dW2 GEMM
//   pass 2 (H again, L2-hot): dH[r][j] = (sum_k delta_o[r][k] W2[k][j]) h (1 - h) ->
//          dH^T K-blocked [rows/32][1024][32] (the dW1 GEMM's operand; a warp's lanes are
//          32 consecutive rows: one 128-byte store per unit)
// Thread (row r, half) takes 16 of each k-block's 32 units; W2^T sits in shared memory
// ([1024][16], read as broadcasts).
#ifndef GLX_T3_TPR
#define GLX_T3_TPR 4  // threads per row (2: 8 compute warps, 4: 16)
#endif
constexpr int kT3S = 8;                     // H k-block stages (128 rows x 32 f32 each)
constexpr int kT3KB = kWH / 32;             // 32 k-blocks per pass
constexpr int kT3P = GLX_T3_TPR;            // threads per row
constexpr int kT3U = 32 / kT3P;             // units per thread per k-block
constexpr uint32_t kT3Stage = 128 * 128;
constexpr int kT3Threads = 32 + 128 * kT3P;  // producer warp + compute warps
constexpr size_t kT3Smem = 1024 + kT3S * kT3Stage + kWH * 16 * 4 + kT3P * 128 * 16 * 4 + 64 + 256;
static_assert(kT3Smem <= 232448, "tf32 tail shared memory");

__global__ void __launch_bounds__(kT3Threads, 1) wide_tail32_kernel(const __grid_constant__ CUtensorMap map_h,
                                                                     const float* __restrict__ W2T,
                                                                     const float* __restrict__ b2,
                                                                     const uint8_t* __restrict__ labels, int M,
                                                                     float* __restrict__ doT, float* __restrict__ dhT,
                                                                     double* __restrict__ stats) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
    unsigned char* ring = sm;
    float* w2t = reinterpret_cast<float*>(ring + kT3S * kT3Stage);  // [1024 units][16]
    float* xo = w2t + kWH * 16;                                      // [kT3P - 1][128][16] pass-1 partials
    float* dob = xo + (kT3P - 1) * 128 * 16;                         // [128][16] delta_o
    float* b2s = dob + 128 * 16;                                     // [16]
    uint64_t* full = reinterpret_cast<uint64_t*>(b2s + 16);
    uint64_t* empty = full + kT3S;
    constexpr int kCW = 4 * kT3P;  // compute warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (M + 127) / 128;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kT3S; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kCW);
        }
        fence_mbar_init();
    }
    for (int e = threadIdx.x; e < kWH * 16; e += blockDim.x) w2t[e] = W2T[(e >> 4) * 32 + (e & 15)];
    if (threadIdx.x < 16) b2s[threadIdx.x] = b2[threadIdx.x];
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {  // producer: pass 1 then pass 2 of each tile through one ring
            const uint64_t keep = l2_policy_evict_last(), drop = l2_policy_evict_first();
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
                for (int j = 0; j < 2 * kT3KB; j++, it++) {
                    const int s = it % kT3S;
                    if (it >= kT3S) mbar_wait(&empty[s], ((it / kT3S) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], kT3Stage);
                    tma_load_2d_hint(ring + s * kT3Stage, &map_h, (j % kT3KB) * 32, t * 128, &full[s],
                                     j < kT3KB ? keep : drop);
                }
        }
        return;
    }
    // thread (row r, part): units kT3U part .. of every 32-unit k-block
    const int c = threadIdx.x - 32, r = c & 127, part = c >> 7;
    const uint32_t ring_a = smem_u32(ring);
    float loss = 0.f, correct = 0.f, valid = 0.f;
    int it = 0;
    auto load_h = [&](int s, float (&hv)[kT3U]) {
        const uint32_t rowa = ring_a + s * kT3Stage + r * 128;
#pragma unroll
        for (int q = 0; q < kT3U / 4; q++) {
            const uint4 v = lds128(rowa + ((((kT3U / 4) * part + q) ^ (r & 7)) << 4));
            hv[4 * q] = __uint_as_float(v.x);
            hv[4 * q + 1] = __uint_as_float(v.y);
            hv[4 * q + 2] = __uint_as_float(v.z);
            hv[4 * q + 3] = __uint_as_float(v.w);
        }
    };
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int row = t * 128 + r;
        const int lab = (part == 0 && row < M) ? labels[row] : 0;
        // pass 1: output-layer pre-activations over this thread's units
        float2 acc[8];
#pragma unroll
        for (int k = 0; k < 8; k++) acc[k] = make_float2(0.f, 0.f);
        for (int kb = 0; kb < kT3KB; kb++, it++) {
            const int s = it % kT3S;
            mbar_wait(&full[s], (it / kT3S) & 1);
            float hv[kT3U];
            load_h(s, hv);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            const float4* wj = reinterpret_cast<const float4*>(w2t + (kb * 32 + kT3U * part) * 16);
#pragma unroll
            for (int u = 0; u < kT3U; u++) {
                const float2 h2 = bcast2(hv[u]);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const float4 w = wj[u * 4 + q];
                    acc[2 * q] = ffma2(h2, make_float2(w.x, w.y), acc[2 * q]);
                    acc[2 * q + 1] = ffma2(h2, make_float2(w.z, w.w), acc[2 * q + 1]);
                }
            }
        }
        // the parts of each row meet; part 0 owns the output neuron of its row
        if (part > 0) {
#pragma unroll
            for (int k = 0; k < 8; k++) *reinterpret_cast<float2*>(xo + ((part - 1) * 128 + r) * 16 + 2 * k) = acc[k];
        }
        bar_sync(1, kCW * 32);
        if (part == 0) {
#pragma unroll
            for (int p = 1; p < kT3P; p++)
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const float2 o2 = *reinterpret_cast<const float2*>(xo + ((p - 1) * 128 + r) * 16 + 2 * k);
                    acc[k].x += o2.x;
                    acc[k].y += o2.y;
                }
            float d[kWK];
            if (row < M) {
                float best = -1.f;
                int arg = 0;
#pragma unroll
                for (int k = 0; k < kWK; k++) {
                    const float pre = k & 1 ? acc[k >> 1].y : acc[k >> 1].x;
                    const float o = 1.0f / (1.0f + __expf(-(pre + b2s[k])));
                    const float tk = (k == lab) ? 1.f : 0.f;
                    d[k] = (o - tk) * o * (1.0f - o);
                    loss = fmaf(0.5f * (tk - o), tk - o, loss);
                    if (o > best) {
                        best = o;
                        arg = k;
                    }
                }
                correct += arg == lab ? 1.f : 0.f;
                valid += 1.f;
#pragma unroll
                for (int k = 0; k < kWK; k++) doT[((int64_t)(row >> 5) * 32 + k) * 32 + (row & 31)] = d[k];
            } else {
#pragma unroll
                for (int k = 0; k < kWK; k++) d[k] = 0.f;
            }
#pragma unroll
            for (int k = 0; k < kWK; k += 4)
                *reinterpret_cast<float4*>(dob + r * 16 + k) = make_float4(d[k], d[k + 1], d[k + 2], d[k + 3]);
        }
        bar_sync(1, kCW * 32);
        float2 dd[8];
#pragma unroll
        for (int k = 0; k < 8; k++) dd[k] = *reinterpret_cast<const float2*>(dob + r * 16 + 2 * k);
        // pass 2: dH = (delta_o W2) h (1 - h) -> dH^T
        float* dst = dhT + (int64_t)(row >> 5) * kWH * 32 + (row & 31);
        for (int kb = 0; kb < kT3KB; kb++, it++) {
            const int s = it % kT3S;
            mbar_wait(&full[s], (it / kT3S) & 1);
            float hv[kT3U];
            load_h(s, hv);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            const int j0 = kb * 32 + kT3U * part;
            const float4* wj = reinterpret_cast<const float4*>(w2t + j0 * 16);
#pragma unroll
            for (int u = 0; u < kT3U; u++) {
                float2 p = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const float4 w = wj[u * 4 + q];
                    p = ffma2(dd[2 * q], make_float2(w.x, w.y), p);
                    p = ffma2(dd[2 * q + 1], make_float2(w.z, w.w), p);
                }
                const float h = hv[u];
                if (row < M) dst[(int64_t)(j0 + u) * 32] = (p.x + p.y) * h * (1.f - h);
            }
        }
    }
    if (part == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            loss += __shfl_xor_sync(0xffffffffu, loss, o);
            correct += __shfl_xor_sync(0xffffffffu, correct, o);
            valid += __shfl_xor_sync(0xffffffffu, valid, o);
        }
        if (lane == 0 && stats) {
            atomicAdd(stats + 0, (double)loss);
            atomicAdd(stats + 1, (double)correct);
            atomicAdd(stats + 2, (double)(valid - correct));
        }
    }
}

// tf32 tail with the output layer on the tensor cores: pass 1 is an SS kind::tf32 MMA
// chain (D_o[128 rows][16] = H . W2^T over 32 k-blocks, as in the bf16 tail's phase A),
// so the CUDA cores only run pass 2. Pass 1 streams H from HBM through ring 1 (its own
// producer, MMA-issuing thread and TMEM accumulator); pass 2 re-reads the tile from L2
// through ring 2 once pass 1 landed (p1land / p2got as in wide_tail_kernel).
#ifndef GLX_T4_P1HINT
#define GLX_T4_P1HINT 1  // pass-1 loads evict_last (0: default policy)
#endif
#ifndef GLX_T4_DHCS
#define GLX_T4_DHCS 0    // 1: dH^T / delta_o^T stores with the streaming (evict-first) cache operator
#endif
#ifndef GLX_T4_LAG
#define GLX_T4_LAG 0     // > 0: pass 1 of tile t + 1 starts once pass 2 of tile t issued this many k-blocks
#endif
constexpr int kT4S1 = 3, kT4S2 = 2;
constexpr int kT4CW = 16;                        // compute warps (4 per row, 8 units each per k-block)
constexpr int kT4Threads = 32 * (3 + kT4CW);     // P1 producer, MMA, compute warps, P2 producer
constexpr size_t kT4Smem = 1024 + (kT4S1 + kT4S2) * kT3Stage + kT3KB * 2048 + kWH * 16 * 4 + 128 * 16 * 4 + 64 + 512;
static_assert(kT4Smem <= 232448, "tf32 tc tail shared memory");

__global__ void __launch_bounds__(kT4Threads, 1) wide_tail32tc_kernel(const __grid_constant__ CUtensorMap map_h,
                                                                       const __grid_constant__ CUtensorMap map_w2,
                                                                       const float* __restrict__ W2T,
                                                                       const float* __restrict__ b2,
                                                                       const uint8_t* __restrict__ labels, int M,
                                                                       float* __restrict__ doT, float* __restrict__ dhT,
                                                                       double* __restrict__ stats) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
    unsigned char* ring1 = sm;
    unsigned char* ring2 = ring1 + kT4S1 * kT3Stage;
    unsigned char* w2m = ring2 + kT4S2 * kT3Stage;                  // W2 [16][1024] as 32 sw128 k-blocks of 2 KB
    float* w2t = reinterpret_cast<float*>(w2m + kT3KB * 2048);      // [1024 units][16]
    float* dob = w2t + kWH * 16;                                     // [128][16] delta_o
    float* b2s = dob + 128 * 16;                                     // [16]
    uint64_t* full1 = reinterpret_cast<uint64_t*>(b2s + 16);
    uint64_t* empty1 = full1 + kT4S1;
    uint64_t* full2 = empty1 + kT4S1;
    uint64_t* empty2 = full2 + kT4S2;
    uint64_t* wbar = empty2 + kT4S2;
    uint64_t* ofull = wbar + 1;
    uint64_t* ofree = ofull + 1;
    uint64_t* p1land = ofree + 1;
    uint64_t* p2got = p1land + 1;
    uint64_t* p2lag = p2got + 1;  // GLX_T4_LAG: pass 2 of a tile issued its first GLX_T4_LAG k-blocks
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p2lag + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (M + 127) / 128;
    if (threadIdx.x == 0) {
        mbar_init(p2lag, 1);
        for (int i = 0; i < kT4S1; i++) {
            mbar_init(&full1[i], 1);
            mbar_init(&empty1[i], 1);
        }
        for (int i = 0; i < kT4S2; i++) {
            mbar_init(&full2[i], 1);
            mbar_init(&empty2[i], kT4CW);
        }
        mbar_init(wbar, 1);
        mbar_init(ofull, 1);
        mbar_init(ofree, 4);
        mbar_init(p1land, 1);
        mbar_init(p2got, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(32)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int e = threadIdx.x; e < kWH * 16; e += blockDim.x) w2t[e] = W2T[(e >> 4) * 32 + (e & 15)];
    if (threadIdx.x < 16) b2s[threadIdx.x] = b2[threadIdx.x];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // pass-1 producer (HBM): W2, then the tiles' k-blocks
            const uint64_t keep = l2_policy_evict_last();
            mbar_arrive_expect_tx(wbar, kT3KB * 2048);
            for (int kb = 0; kb < kT3KB; kb++) tma_load_2d(w2m + kb * 2048, &map_w2, kb * 32, 0, wbar);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                if (GLX_T4_LAG > 0 && lt > 0) mbar_wait(p2lag, (lt - 1) & 1);
                for (int kb = 0; kb < kT3KB; kb++, it++) {
                    const int s = it % kT4S1;
                    if (it >= kT4S1) mbar_wait(&empty1[s], ((it / kT4S1) - 1) & 1);
                    mbar_arrive_expect_tx(&full1[s], kT3Stage);
                    if (GLX_T4_P1HINT) tma_load_2d_hint(ring1 + s * kT3Stage, &map_h, kb * 32, t * 128, &full1[s], keep);
                    else tma_load_2d(ring1 + s * kT3Stage, &map_h, kb * 32, t * 128, &full1[s]);
                }
            }
        }
    } else if (warp == 2 + kT4CW) {
        if (lane == 0) {  // pass-2 producer (L2)
            const uint64_t drop = l2_policy_evict_first();
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                mbar_wait(p1land, lt & 1);
                mbar_arrive(p2got);
                for (int kb = 0; kb < kT3KB; kb++, it++) {
                    const int s = it % kT4S2;
                    if (it >= kT4S2) mbar_wait(&empty2[s], ((it / kT4S2) - 1) & 1);
                    mbar_arrive_expect_tx(&full2[s], kT3Stage);
                    tma_load_2d_hint(ring2 + s * kT3Stage, &map_h, kb * 32, t * 128, &full2[s], drop);
                    if (GLX_T4_LAG > 0 && kb + 1 == GLX_T4_LAG) mbar_arrive(p2lag);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // output-layer MMAs
            mbar_wait(wbar, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t idO = umma_idesc_tf32(128, 16);
            const uint32_t r1 = smem_u32(ring1), wa = smem_u32(w2m);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                if (lt > 0) {
                    mbar_wait(ofree, (lt - 1) & 1);
                    mbar_wait(p2got, (lt - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                for (int kb = 0; kb < kT3KB; kb++, it++) {
                    const int s = it % kT4S1;
                    mbar_wait(&full1[s], (it / kT4S1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                        umma_tf32(tmem, umma_desc_sw128(r1 + s * kT3Stage + kk * 32), umma_desc_sw128(wa + kb * 2048 + kk * 32),
                                  idO, (kb | kk) != 0);
                    umma_commit(&empty1[s]);
                }
                mbar_arrive(p1land);
                umma_commit(ofull);
            }
        }
    } else {
        // compute warps 2 .. 17: TMEM lane quadrant = warp % 4 -> rows 32 quad ..; part = (warp - 2) / 4
        const int quad = warp & 3, part = (warp - 2) >> 2;
        const int r = quad * 32 + lane;
        const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
        const uint32_t r2 = smem_u32(ring2);
        constexpr int kU = 8;  // units per thread per k-block
        float loss = 0.f, correct = 0.f, valid = 0.f;
        int it = 0, lt = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
            const int row = t * 128 + r;
            if (part == 0) {
                const int lab = row < M ? labels[row] : 0;
                mbar_wait(ofull, lt & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t ro[16];
                tmem_ld16_async(tmem + lanebase, ro);
                tmem_wait();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(ofree);
                float d[kWK];
                if (row < M) {
                    float best = -1.f;
                    int arg = 0;
#pragma unroll
                    for (int k = 0; k < kWK; k++) {
                        const float o = 1.0f / (1.0f + __expf(-(__uint_as_float(ro[k]) + b2s[k])));
                        const float tk = (k == lab) ? 1.f : 0.f;
                        d[k] = (o - tk) * o * (1.0f - o);
                        loss = fmaf(0.5f * (tk - o), tk - o, loss);
                        if (o > best) {
                            best = o;
                            arg = k;
                        }
                    }
                    correct += arg == lab ? 1.f : 0.f;
                    valid += 1.f;
#pragma unroll
                    for (int k = 0; k < kWK; k++) {
                        float* q = doT + ((int64_t)(row >> 5) * 32 + k) * 32 + (row & 31);
                        if (GLX_T4_DHCS) __stcs(q, d[k]);
                        else *q = d[k];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < kWK; k++) d[k] = 0.f;
                }
#pragma unroll
                for (int k = 0; k < kWK; k += 4)
                    *reinterpret_cast<float4*>(dob + r * 16 + k) = make_float4(d[k], d[k + 1], d[k + 2], d[k + 3]);
            }
            bar_sync(1, kT4CW * 32);
            float2 dd[8];
#pragma unroll
            for (int k = 0; k < 8; k++) dd[k] = *reinterpret_cast<const float2*>(dob + r * 16 + 2 * k);
            // pass 2: dH = (delta_o W2) h (1 - h) -> dH^T
            float* dst = dhT + (int64_t)(row >> 5) * kWH * 32 + (row & 31);
            for (int kb = 0; kb < kT3KB; kb++, it++) {
                const int s = it % kT4S2;
                mbar_wait(&full2[s], (it / kT4S2) & 1);
                const uint32_t rowa = r2 + s * kT3Stage + r * 128;
                float hv[kU];
#pragma unroll
                for (int q = 0; q < kU / 4; q++) {
                    const uint4 v = lds128(rowa + ((((kU / 4) * part + q) ^ (r & 7)) << 4));
                    hv[4 * q] = __uint_as_float(v.x);
                    hv[4 * q + 1] = __uint_as_float(v.y);
                    hv[4 * q + 2] = __uint_as_float(v.z);
                    hv[4 * q + 3] = __uint_as_float(v.w);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty2[s]);
                const int j0 = kb * 32 + kU * part;
                const float4* wj = reinterpret_cast<const float4*>(w2t + j0 * 16);
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    float2 p = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const float4 w = wj[u * 4 + q];
                        p = ffma2(dd[2 * q], make_float2(w.x, w.y), p);
                        p = ffma2(dd[2 * q + 1], make_float2(w.z, w.w), p);
                    }
                    const float h = hv[u];
                    if (row < M) {
                        if (GLX_T4_DHCS) __stcs(dst + (int64_t)(j0 + u) * 32, (p.x + p.y) * h * (1.f - h));
                        else dst[(int64_t)(j0 + u) * 32] = (p.x + p.y) * h * (1.f - h);
                    }
                }
            }
        }
        if (part == 0) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                loss += __shfl_xor_sync(0xffffffffu, loss, o);
                correct += __shfl_xor_sync(0xffffffffu, correct, o);
                valid += __shfl_xor_sync(0xffffffffu, valid, o);
            }
            if (lane == 0 && stats) {
                atomicAdd(stats + 0, (double)loss);
                atomicAdd(stats + 1, (double)correct);
                atomicAdd(stats + 2, (double)(valid - correct));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32) : "memory");
    }
}

// GLX_WIDE_TAIL32=cuda selects the CUDA-core tf32 tail (output layer on the FP32 pipe too)
static bool wide_tail32_tc() {
    const char* v = getenv("GLX_WIDE_TAIL32");
    return !(v && v[0] == 'c');
}

static size_t carve32(WideWork32* w, unsigned char* base, int64_t C, int splits) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
        void* p = base ? base + o : nullptr;
        o += (bytes + 255) / 256 * 256;
        return (float*)p;
    };
    WideWork32 t;
    t.W1p = take((size_t)kWH * kWD * 4);
    t.b1 = take(kWH * 4);
    t.W2p = take(32 * kWH * 4);
    t.b2 = take(64 * 4);
    t.W2T = take((size_t)kWH * 32 * 4);
    t.H = take((size_t)C * kWH * 4);
    t.HT = take((size_t)C * kWR * 4);
    t.dob = take((size_t)C * 32 * 4);
    t.doT = take((size_t)C * 32 * 4);
    t.dhT = take((size_t)C * kWH * 4);
    t.dW1T = take((size_t)splits * kWMi * kWH * 4);
    t.dW2T = take((size_t)kWSplits2 * kWMi * 32 * 4);
    t.grad = (double*)take((size_t)(kWP + 3) * 8);
    if (w) *w = t;
    return o;
}

size_t wide32_work_bytes(int64_t C, int splits) { return carve32(nullptr, nullptr, C, splits); }

cudaError_t wide_grad_tf32(const float* W1, const float* W2, const float* X, const float* XT, const uint8_t* labels,
                           int64_t N, unsigned char* work, int64_t C, int splits, double* grad, cudaStream_t st,
                           const std::function<void(bool)>& prof) {
    WideWork32 w;
    carve32(&w, work, C, splits);
    cudaError_t e;
    if (!grad) grad = w.grad;
    double* stats = grad + kWP;
    if ((e = cudaMemsetAsync(stats, 0, 3 * sizeof(double), st)) != cudaSuccess) return e;
    const bool tail = wide_tail_enabled();
    wide_derive32_kernel<<<(kWH * kWD + 255) / 256, 256, 0, st>>>(W1, W2, w.W1p, w.b1, w.W2p, w.b2, w.W2T);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int64_t zstride = (int64_t)kWMi * kWH, zstride2 = (int64_t)kWMi * 32;
    if ((e = cudaMemsetAsync(w.dW1T, 0, (size_t)splits * zstride * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.dW2T, 0, (size_t)kWSplits2 * zstride2 * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.dob, 0, (size_t)C * 32 * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.doT, 0, (size_t)C * 32 * 4, st)) != cudaSuccess) return e;
    ht_bias_row_kernel<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(w.HT, C);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    for (int64_t r0 = 0; r0 < N; r0 += C) {
        const int Cc = (int)std::min<int64_t>(C, N - r0);
        prof(true);
        {  // 1. hidden layer -> H, [H,1]^T
            TcGemm g{X + r0 * kWD, w.W1p, Cc, kWH, kWD, kWD, kWD, 1};
            TcEpilogue ep{};
            ep.kind = 1;
            ep.bias = w.b1;
            ep.h32 = w.H;
            ep.ldd = kWH;
            ep.t32 = w.HT;
            ep.t_blk = kWR;
            if ((e = launch_tc_tf32(g, ep, st)) != cudaSuccess) return e;
        }
        if (tail && wide_tail32_tc()) {  // 2 + 3 fused, output layer on tcgen05: delta_o, loss, accuracy, dH^T
            CUtensorMap mh, mw;
            if (!make_map_f32(&mh, w.H, Cc, kWH, kWH, 128) || !make_map_f32(&mw, w.W2p, 32, kWH, kWH, 16))
                return cudaErrorInvalidValue;
            if ((e = cudaFuncSetAttribute(wide_tail32tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kT4Smem)) != cudaSuccess)
                return e;
            const int grid = std::min(sm_count(), (Cc + 127) / 128);
            wide_tail32tc_kernel<<<grid, kT4Threads, kT4Smem, st>>>(mh, mw, w.W2T, w.b2, labels + r0, Cc, w.doT,
                                                                    w.dhT, stats);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        } else if (tail) {  // 2 + 3 fused (CUDA cores): delta_o, loss, accuracy, dH^T
            CUtensorMap mh;
            if (!make_map_f32(&mh, w.H, Cc, kWH, kWH, 128)) return cudaErrorInvalidValue;
            if ((e = cudaFuncSetAttribute(wide_tail32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kT3Smem)) != cudaSuccess)
                return e;
            const int grid = std::min(sm_count(), (Cc + 127) / 128);
            wide_tail32_kernel<<<grid, kT3Threads, kT3Smem, st>>>(mh, w.W2T, w.b2, labels + r0, Cc, w.doT, w.dhT,
                                                                  stats);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        if (!tail) {  // 2. output layer -> delta_o, loss, accuracy
            TcGemm g{w.H, w.W2p, Cc, 32, kWH, kWH, kWH, 1};
            TcEpilogue ep{};
            ep.kind = 2;
            ep.bias = w.b2;
            ep.labels = labels + r0;
            ep.K = kWK;
            ep.do32 = w.dob;
            ep.doT32 = w.doT;
            ep.stats = stats;
            if ((e = launch_tc_tf32(g, ep, st)) != cudaSuccess) return e;
        }
        if (!tail) {  // 3. hidden deltas -> dH^T (K-blocked)
            TcGemm g{w.dob, w.W2T, Cc, kWH, 32, 32, 32, 1};
            TcEpilogue ep{};
            ep.kind = 3;
            ep.hin32 = w.H;
            ep.ldh = kWH;
            ep.t32 = w.dhT;
            ep.t_blk = kWH;
            if ((e = launch_tc_tf32(g, ep, st)) != cudaSuccess) return e;
        }
        {  // 4. dW1^T += [X,1]^T dH (split-K over the chunk's rows)
            TcGemm g{XT + r0 * kWR, w.dhT, kWR, kWH, Cc, 0, 0, splits, kWR, kWH};
            TcEpilogue ep{};
            ep.kind = 4;
            ep.d_f32 = w.dW1T;
            ep.ldd = kWH;
            ep.zstride = zstride;
            if ((e = launch_tc_tf32(g, ep, st)) != cudaSuccess) return e;
        }
        {  // 5. dW2^T += [H,1]^T delta_o (split-K; N = 32, delta_o columns >= 16 zero)
            TcGemm g{w.HT, w.doT, kWR, 32, Cc, 0, 0, kWSplits2, kWR, 32};
            TcEpilogue ep{};
            ep.kind = 4;
            ep.d_f32 = w.dW2T;
            ep.ldd = 32;
            ep.zstride = zstride2;
            if ((e = launch_tc_tf32(g, ep, st)) != cudaSuccess) return e;
        }
        prof(false);
    }
    wide_reduce_kernel<<<(kWP + 255) / 256, 256, 0, st>>>(w.dW1T, splits, zstride, w.dW2T, kWSplits2, zstride2,
                                                         grad);
    return cudaGetLastError();
}

cudaError_t wide_epoch_tf32(float* W1, float* W2, const float* X, const float* XT, const uint8_t* labels, int64_t N,
                            double lr, unsigned char* work, int64_t C, int splits, double* stats, int* nonfinite,
                            cudaStream_t st, const std::function<void(bool)>& prof) {
    WideWork32 w;
    carve32(&w, work, C, splits);
    cudaError_t e = wide_grad_tf32(W1, W2, X, XT, labels, N, work, C, splits, w.grad, st, prof);
    if (e != cudaSuccess) return e;
    if (stats && (e = cudaMemcpyAsync(stats, w.grad + kWP, 3 * sizeof(double), cudaMemcpyDeviceToDevice, st)) !=
                     cudaSuccess)
        return e;
    return wide_apply(W1, W2, w.grad, lr / (double)N, nonfinite, st);
}

cudaError_t launch_tc_gemm(const void* A, const void* B, int M, int N, int K, int epi, float* d_f32,
                           void* d_bf16, const float* bias, int ldd, cudaStream_t st) {
    TcGemm g{A, B, M, N, K, K, K, 1};
    TcEpilogue ep{};
    ep.kind = epi;
    ep.d_f32 = d_f32;
    ep.d_bf16 = reinterpret_cast<__nv_bfloat16*>(d_bf16);
    ep.bias = bias;
    ep.ldd = ldd;
    return launch_tc(g, ep, st);
}

}  // namespace glx
