// glx_batchtc.cu -- full-batch gradient-descent epoch (configs 2 and 4:
// D <= 33 inputs -> H = 128 or 256 sigmoid units -> 1 output) on the
// 5th-generation tensor cores, fp32-accurate through 3xTF32.
//
// Same contract as batch3_kernel (glx_batch3.cu): one persistent CTA per SM
// walks row tiles and writes one per-CTA partial record
//   [dW1acc (H*(D+1)) | dW2acc (H) | dsum | loss | c0 c1 c2 c3]
// that batch_update_kernel reduces in f64 and applies (kernels.py:264-295
// batch semantics).
//
// Both GEMMs of the epoch run on tcgen05 with the hidden units on the TMEM
// lanes (M = 128 units per half):
//   forward   Z^T[j][r]  = W1s[j][:] . x_r            (SS: A = W1s, B = x tile, K-major)
//   backward  dW1[j][k] += sum_r dh[j][r] x_r[k]       (TS: A = dh^T from TMEM, B = x tile, MN-major)
// so the delta of every hidden unit stays in TMEM between the two MMAs. Both
// shared-memory operands are K-major no-swizzle core matrices (8 rows x 16 B):
// the forward reads the x tile as [rows x features], the backward a transposed
// copy [features x rows] written by the converter warps (tf32 MMAs with an
// MN-major B operand return zeros on sm_100a, tools/umma_probe.cu).
// Each operand is split hi = tf32(v) (bit truncation), lo = v - hi and the
// products are accumulated as lo.hi + hi.lo + hi.hi in the fp32 TMEM
// accumulator: the dropped lo.lo term is 2^-22 relative, so results track the
// fp32 CUDA-core kernel (tests/test_gpu_batch.py, 1e-5 against the f64 oracle).
//
// Per 64-row tile, 16 epilogue warps (4 TMEM lane quadrants x 2 unit halves x
// 2 row blocks; thread = hidden unit, 32 rows) read Z^T from TMEM, apply the
// sigmoid (MUFU, with 3 of 8 exponential pairs on the FMA pipe), reduce the
// output partials w2s_j h_j with a warp reduce-scatter plus one shared-memory
// pass per row block, compute delta_o for their own rows, and write
// dh = delta_o h (1 - h) back to TMEM as tf32 hi/lo for the backward MMA. Z^T is
// double-buffered so the forward MMA of tile t+1 overlaps the epilogue of tile
// t, and the backward of tile t overlaps the epilogue of tile t+1. Warp 0 bulk-
// copies the packed rows, warps 2-3 convert them into the two operand layouts,
// warp 1 issues the MMAs (converged, one elect.sync lane). DESIGN.md §4 has the
// measured path and the per-phase timeline.
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

namespace glx {

namespace {

constexpr int kR = 64;                      // rows per tile (forward MMA N)
constexpr int kFC = 10;                     // 4-feature chunks of the forward operands (K = 40)
constexpr int kNB = 48;                     // features in the backward (MMA N, multiple of 16)
constexpr int kXF = kR / 8 * kFC * 128;     // bytes per forward x tile (tf32): [r/8][k/4][r%8][k%4]
constexpr int kXT = kNB / 8 * kR / 4 * 128; // bytes per transposed tile (tf32): [k/8][r/4][k%8][r%4]
constexpr int kWT = 16 * kFC * 128;         // bytes per 128-unit weight copy (hi or lo)
// Two precisions (template FULL): FAST (large N) uses tf32(x) only, forward
// hi(W) tf32(x) + lo(W) tf32(x), backward tf32(dh) tf32(x); FULL (small N, where
// too few rows average the operand rounding out) is 3xTF32 on both GEMMs (x and dh
// split into hi + lo as well), which needs the lo copies of x and a dh lo TMEM
// buffer. Stage counts per precision (shared memory, TMEM):
template <bool FULL>
struct Pipe {
    static constexpr int XFS = FULL ? 2 : 4;  // forward x stages (free once the forward MMA completes)
    static constexpr int XS = FULL ? 3 : 4;   // transposed x stages (free once the backward MMA completes)
    static constexpr int XR = FULL ? 3 : 4;   // raw x stages (TMA bulk targets)
    static constexpr int ZB = FULL ? 2 : 3;   // Z^T buffers (FAST: the forward runs two tiles ahead)
    static constexpr int NX = FULL ? 2 : 1;   // x operand copies: hi (+ lo)
};
constexpr int kMaxLD = 36;
constexpr int kRawBytes = kR * kMaxLD * 4;
constexpr uint32_t kTf32Mask = 0xFFFFE000u;
constexpr int kColZ = 0;     // Z^T, then dh (tf32 hi) in place: buffer b at 128 b, half hf at + 64 hf
constexpr int kColLo = 256;  // FULL: dh lo, half hf at + 64 hf (Z uses buffers 0, 1)
constexpr int kColW = 384;   // dW1 accumulators: half hf at + 48 hf
constexpr uint32_t kTmemCols = 512;
constexpr int kEpiBar = 1;
// the dW1 TMEM accumulator restarts every kDrain tiles after being added (round
// to nearest) into per-thread fp32 registers: tensor-core fp32 accumulation over
// ~10^5 rows per CTA drifted by ~1e-3 relative at 64Mi rows; short partials keep
// the sum at the fp32 CUDA-core kernel's accuracy (tests/test_gpu_fullsize.py)
#ifndef GLX_BTC_DRAIN
#define GLX_BTC_DRAIN 8
#endif
constexpr int kDrain = GLX_BTC_DRAIN;
constexpr int kD1 = 34;  // dW1 columns kept per unit (D + 1 <= 34)
#ifndef GLX_BTC_OFFSET
#define GLX_BTC_OFFSET 1  // 0: the two row blocks start together
#endif
#ifndef GLX_BTC_EXP
#define GLX_BTC_EXP 0  // diagnostic builds only: 1 no MUFU sigmoid, 2 no backward MMAs, 3 no forward MMAs
#endif

#ifdef GLX_BTC_TIMING
__device__ unsigned long long g_btc_dbg[4096];
#define BTT(slot)                                                                                      \
    do {                                                                                               \
        if (blockIdx.x == 0 && lane == 0 && lt >= 8 && lt < 24) g_btc_dbg[((lt - 8) * 16 + (slot)) * 2 + (warp == 4 ? 0 : 1)] = clock64(); \
    } while (0)
#else
#define BTT(slot) \
    do {          \
    } while (0)
#endif

struct BtcArgs {
    const float* Xp;
    const float* Wk;
    float* part;
    int64_t N, ntiles;
    int D, DP, LD, H, P1, PS;
};

struct BtcSmem {  // byte offsets
    int w, xf, xc, raw, tgt, opart, dob, stat, bars;
    int total;
};

__host__ __device__ constexpr int btc_threads(int NH) { return (4 + 8 * NH) * 32; }

template <bool FULL>
__host__ __device__ constexpr BtcSmem btc_smem(int NH) {
    using P = Pipe<FULL>;
    BtcSmem s{};
    s.w = 0;
    s.xf = s.w + 2 * NH * kWT;
    s.xc = s.xf + P::XFS * P::NX * kXF;
    s.raw = s.xc + P::XS * P::NX * kXT;
    s.tgt = s.raw + P::XR * kRawBytes;
    s.opart = s.tgt + P::XS * kR * 4;
    s.dob = s.opart + 2 * 8 * NH * 32 * 4;  // output partials, double-buffered by tile parity
    s.stat = s.dob + 8 * NH * 32 * 4;  // dob: one 32-row slot per epilogue warp
    s.bars = s.stat;                   // (the row statistics reuse the partials buffer at the end)
    s.total = s.bars + 256;
    return s;
}

// UMMA shared-memory descriptor, no swizzle (canonical core matrices of
// 8 rows x 16 B): start | LBO (K-direction stride) | SBO (M/N-direction
// stride) | version 1 (sm100) | layout type 0
__device__ __forceinline__ uint64_t desc_ns(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// instruction descriptor: TF32 x TF32 -> F32, M = 128
__host__ __device__ constexpr uint32_t idesc_tf32(int N, bool b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}

// The MMA warp runs its loop converged (warp-uniform operands stay in uniform
// registers); `e` is the elect.sync flag: one lane issues each instruction.
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(e));
    return e;
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t e) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(e)
        : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc,
                                       uint32_t e) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(e)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar, uint32_t e) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %1, 0;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)),
        "r"(e)
        : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
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

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void ld1(uint32_t taddr, uint32_t& r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void ld2(uint32_t taddr, uint32_t (&r)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// round-to-nearest (ties away from zero) tf32, as cvt.rna.tf32.f32: unbiased operand
// rounding is what lets single-product terms meet the 1e-5 parity bar
// (tools/tf32_split_error.py); the MMA ignores the 13 low bits of any operand
__device__ __forceinline__ uint32_t tf32_rn(float v) { return (__float_as_uint(v) + 0x1000u) & kTf32Mask; }

// 2^x for a pair on the FMA/ALU pipes (pass 1 is MUFU-bound): round-to-nearest by
// the 1.5 * 2^23 magic add, degree-5 polynomial on [-1/2, 1/2] (max rel. error 2.3e-7
// in fp32 Horner, on par with ex2.approx), exponent inserted with an integer add;
// |x| clamped to 125 (1 + 2^-125 == 1 and 1 / (1 + 2^125) ~ 0 in fp32 either way)
#ifndef GLX_BTC_POLY
#define GLX_BTC_POLY 3  // element pairs per GLX_BTC_POLY_DEN that take the polynomial (0: all MUFU)
#endif
#ifndef GLX_BTC_POLY_DEN
#define GLX_BTC_POLY_DEN 8
#endif
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    x.x = fminf(fmaxf(x.x, -125.f), 125.f);
    x.y = fminf(fmaxf(x.y, -125.f), 125.f);
    const float2 t = __fadd2_rn(x, bcast2(12582912.0f));
    const float2 fi = __fadd2_rn(t, bcast2(-12582912.0f));
    const float2 f = __fadd2_rn(x, make_float2(-fi.x, -fi.y));
    float2 p = ffma2(bcast2(0.001327646430581808f), f, bcast2(0.009675540961325169f));
    p = ffma2(p, f, bcast2(0.05550713464617729f));
    p = ffma2(p, f, bcast2(0.24022120237350464f));
    p = ffma2(p, f, bcast2(0.6931469440460205f));
    p = ffma2(p, f, bcast2(1.0000001192092896f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

template <int NH, bool FULL>
__global__ void __launch_bounds__(btc_threads(NH), 1) batchtc_kernel(const BtcArgs a) {
    constexpr int NEW = 8 * NH;  // epilogue warps: 4 lane quadrants x NH unit halves x 2 row blocks
    constexpr BtcSmem L = btc_smem<FULL>(NH);
    constexpr int kXFS = Pipe<FULL>::XFS, kXS = Pipe<FULL>::XS, kXR = Pipe<FULL>::XR, kZB = Pipe<FULL>::ZB;
    constexpr int kNX = Pipe<FULL>::NX;
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = raw_full + kXR;
    uint64_t* xf_full = raw_empty + kXR;
    uint64_t* xf_empty = xf_full + kXFS;
    uint64_t* xc_full = xf_empty + kXFS;
    uint64_t* xc_empty = xc_full + kXS;
    uint64_t* z_full = xc_empty + kXS;
    uint64_t* dh_ready = z_full + kZB;
    uint64_t* drain_bar = dh_ready + 1;  // the backward of the last tile before a dW1 drain completed
    uint64_t* fin_bar = drain_bar + 1;   // the last backward completed
    uint64_t* bwd_done = fin_bar + 1;    // FULL: every backward completed (the single dh lo buffer is free)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bwd_done + 1);
    float* tgt = reinterpret_cast<float*>(sm + L.tgt);
    float* opart = reinterpret_cast<float*>(sm + L.opart);
    float* dob = reinterpret_cast<float*>(sm + L.dob);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nt = (a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA (>= 1)
    const int D = a.D, LD = a.LD, DP = a.DP;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kXR; s++) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], 2);
        }
        for (int s = 0; s < kXFS; s++) {
            mbar_init(&xf_full[s], 2);
            mbar_init(&xf_empty[s], 1);
        }
        for (int s = 0; s < kXS; s++) {
            mbar_init(&xc_full[s], 2);
            mbar_init(&xc_empty[s], 1);
        }
        for (int b = 0; b < kZB; b++) mbar_init(&z_full[b], 1);
        mbar_init(dh_ready, NEW);
        mbar_init(drain_bar, 1);
        mbar_init(fin_bar, 1);
        mbar_init(bwd_done, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // weights -> hi/lo core-matrix copies (K-major A operand of the forward MMA)
    for (int e = threadIdx.x; e < NH * 128 * kFC; e += blockDim.x) {
        const int j = e / kFC, q = e - (e / kFC) * kFC;  // unit, 4-feature chunk
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int k = 4 * q + i;
            v[i] = (k <= D) ? a.Wk[(int64_t)j * DP + k] : 0.f;
        }
        const int hf = j >> 7, jj = j & 127;
        const int off = hf * kWT + (jj >> 3) * (kFC * 128) + q * 128 + (jj & 7) * 16;
        uint4 hi, lo;
        hi.x = tf32_rn(v[0]);
        hi.y = tf32_rn(v[1]);
        hi.z = tf32_rn(v[2]);
        hi.w = tf32_rn(v[3]);
        lo.x = __float_as_uint(v[0] - __uint_as_float(hi.x));
        lo.y = __float_as_uint(v[1] - __uint_as_float(hi.y));
        lo.z = __float_as_uint(v[2] - __uint_as_float(hi.z));
        lo.w = __float_as_uint(v[3] - __uint_as_float(hi.w));
        *reinterpret_cast<uint4*>(sm + L.w + off) = hi;
        *reinterpret_cast<uint4*>(sm + L.w + NH * kWT + off) = lo;
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            for (int64_t lt = 0; lt < nt; lt++) {
                const int rs = (int)(lt % kXR);
                if (lt >= kXR) mbar_wait(&raw_empty[rs], (uint32_t)((lt / kXR) - 1) & 1);
                const int64_t row0 = (blockIdx.x + lt * gridDim.x) * kR;
                const int64_t rem = a.N - row0;
                const int nr = rem < kR ? (int)rem : kR;
                const uint32_t bytes = (uint32_t)(nr * LD * 4);
                mbar_arrive_expect_tx(&raw_full[rs], bytes);
                bulk_g2s(sm + L.raw + rs * kRawBytes, a.Xp + row0 * LD, bytes, &raw_full[rs]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        {
            const uint32_t el = elect_one();
            constexpr uint32_t idf = idesc_tf32(kR, false);
            constexpr uint32_t idb = idesc_tf32(kNB, false);
            // descriptors are built once and advanced by (byte offset >> 4) in the start
            // field (shared addresses < 256 KB: no carry out of the 14-bit field)
            const uint64_t dwh = desc_ns(smem_u32(sm + L.w), 128, kFC * 128);
            const uint64_t dwl = desc_ns(smem_u32(sm + L.w + NH * kWT), 128, kFC * 128);
            // backward of tile lt: dW1[j][k] += sum_r dh[j][r] x_r[k] (one tf32 product: the
            // rounding errors of dh and x average out over the rows, tools/tf32_split_error.py)
            auto backward = [&](int64_t lt) {
                const int cs = (int)(lt % kXS), zb = (int)(lt % kZB);
                BTT(8);
                mbar_wait(dh_ready, (uint32_t)lt & 1);
                mbar_wait(&xc_full[cs], (uint32_t)(lt / kXS) & 1);
                tc_fence_after();
                BTT(9);
                const uint64_t dth = desc_ns(smem_u32(sm + L.xc + cs * kNX * kXT), 128, kR / 4 * 128);
                const uint64_t dtl = dth + (kXT >> 4);  // FULL: the lo copy follows the hi copy
#pragma unroll
                for (int hf = 0; hf < NH; hf++) {
                    const uint32_t d = tmem + kColW + 48 * hf;
                    const uint32_t ahi = tmem + kColZ + 128 * zb + 64 * hf, alo = tmem + kColLo + 64 * hf;
#pragma unroll
                    for (int s = 0; s < kR / 8; s++) {
                        const uint32_t acc = (lt % kDrain) != 0 || s != 0;
#if GLX_BTC_EXP == 2
                        if (s == 0) mma_ts(d, ahi, dth, idb, 0, el);
#else
                        if constexpr (FULL) {
                            mma_ts(d, alo + 8 * s, dth + (s * 256 >> 4), idb, acc, el);
                            mma_ts(d, ahi + 8 * s, dtl + (s * 256 >> 4), idb, 1, el);
                            mma_ts(d, ahi + 8 * s, dth + (s * 256 >> 4), idb, 1, el);
                        } else {
                            mma_ts(d, ahi + 8 * s, dth + (s * 256 >> 4), idb, acc, el);
                        }
#endif
                    }
                }
                commit(&xc_empty[cs], el);
                if constexpr (FULL) commit(bwd_done, el);
                if ((lt + 1) % kDrain == 0) commit(drain_bar, el);
                if (lt == nt - 1) commit(fin_bar, el);
                BTT(10);
            };
            // forward of tile lt: Z^T = W1s . x as tf32 hi(W) hi(x) + lo(W) hi(x) (the small
            // term first); x is rounded once (the dropped hi(W) lo(x) term is unbiased)
            auto forward = [&](int64_t lt) {
                const int fs = (int)(lt % kXFS), zb = (int)(lt % kZB);
                BTT(11);
                mbar_wait(&xf_full[fs], (uint32_t)(lt / kXFS) & 1);
                tc_fence_after();
                BTT(12);
                const uint64_t dx = desc_ns(smem_u32(sm + L.xf + fs * kNX * kXF), 128, kFC * 128);
                const uint64_t dxl = dx + (kXF >> 4);  // FULL: lo copy
#pragma unroll
                for (int hf = 0; hf < NH; hf++) {
                    const uint32_t d = tmem + kColZ + 128 * zb + 64 * hf;
                    const uint64_t wh = dwh + (hf * kWT >> 4), wl = dwl + (hf * kWT >> 4);
#if GLX_BTC_EXP == 3
                    mma_ss(d, wh, dx, idf, 0, el);
                    if (false)
#endif
                    {
#pragma unroll
                        for (int s = 0; s < kFC / 2; s++) {
                            mma_ss(d, wl + (s * 256 >> 4), dx + (s * 256 >> 4), idf, s != 0, el);
                            if constexpr (FULL) mma_ss(d, wh + (s * 256 >> 4), dxl + (s * 256 >> 4), idf, 1, el);
                        }
#pragma unroll
                        for (int s = 0; s < kFC / 2; s++) mma_ss(d, wh + (s * 256 >> 4), dx + (s * 256 >> 4), idf, 1, el);
                    }
                }
                commit(&xf_empty[fs], el);
                commit(&z_full[zb], el);
                BTT(13);
            };
            // Z^T is triple-buffered: forward(lt + 2) reuses the buffer of tile lt - 1, whose
            // backward was issued (tensor-pipe order) in the previous iteration
            forward(0);
            if (nt > 1) forward(1);
            for (int64_t lt = 0; lt < nt; lt++) {
                backward(lt);
                if (lt + 2 < nt) forward(lt + 2);
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------------------ converters
        const int r = threadIdx.x - 64;  // row within the tile (forward copy); item base (transposed copy)
        for (int64_t lt = 0; lt < nt; lt++) {
            const int rs = (int)(lt % kXR), cs = (int)(lt % kXS), fs = (int)(lt % kXFS);
            mbar_wait(&raw_full[rs], (uint32_t)(lt / kXR) & 1);
            const int64_t row0 = (blockIdx.x + lt * gridDim.x) * kR;
            const int64_t rem = a.N - row0;
            const int nr = rem < kR ? (int)rem : kR;
            const float* rawt = reinterpret_cast<const float*>(sm + L.raw + rs * kRawBytes);
            // forward copy [r/8][k/4][r%8][k%4], tf32 (round to nearest)
            if (lt >= kXFS) mbar_wait(&xf_empty[fs], (uint32_t)((lt / kXFS) - 1) & 1);
            {
                const float* raw = rawt + r * LD;
                unsigned char* xh = sm + L.xf + fs * kNX * kXF + (r >> 3) * (kFC * 128) + (r & 7) * 16;
#pragma unroll
                for (int q = 0; q < kFC; q++) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (r < nr && 4 * q < LD) v = *reinterpret_cast<const float4*>(raw + 4 * q);
                    uint4 hi;
                    hi.x = tf32_rn(v.x);
                    hi.y = tf32_rn(v.y);
                    hi.z = tf32_rn(v.z);
                    hi.w = tf32_rn(v.w);
                    *reinterpret_cast<uint4*>(xh + q * 128) = hi;
                    if constexpr (FULL) {
                        uint4 lo;
                        lo.x = __float_as_uint(v.x - __uint_as_float(hi.x));
                        lo.y = __float_as_uint(v.y - __uint_as_float(hi.y));
                        lo.z = __float_as_uint(v.z - __uint_as_float(hi.z));
                        lo.w = __float_as_uint(v.w - __uint_as_float(hi.w));
                        *reinterpret_cast<uint4*>(xh + kXF + q * 128) = lo;
                    }
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&xf_full[fs]);
            // transposed copy [k/8][r/4][k%8][r%4]: one 16-byte core-matrix row (4 rows of
            // feature k) per item; 8 consecutive items fill one 128-byte core matrix
            if (lt >= kXS) mbar_wait(&xc_empty[cs], (uint32_t)((lt / kXS) - 1) & 1);
            unsigned char* xt = sm + L.xc + cs * kNX * kXT;
#pragma unroll 4
            for (int it = r; it < kNB * kR / 4; it += 64) {
                const int k = ((it >> 3) % (kNB / 8)) * 8 + (it & 7);
                const int rq = (it >> 3) / (kNB / 8);
                float v[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int rr = 4 * rq + i;
                    v[i] = (rr < nr && k < LD) ? rawt[rr * LD + k] : 0.f;
                }
                uint4 hi;
                hi.x = tf32_rn(v[0]);
                hi.y = tf32_rn(v[1]);
                hi.z = tf32_rn(v[2]);
                hi.w = tf32_rn(v[3]);
                const int off = (k >> 3) * (kR / 4 * 128) + rq * 128 + (k & 7) * 16;
                *reinterpret_cast<uint4*>(xt + off) = hi;
                if constexpr (FULL) {
                    uint4 lo;
                    lo.x = __float_as_uint(v[0] - __uint_as_float(hi.x));
                    lo.y = __float_as_uint(v[1] - __uint_as_float(hi.y));
                    lo.z = __float_as_uint(v[2] - __uint_as_float(hi.z));
                    lo.w = __float_as_uint(v[3] - __uint_as_float(hi.w));
                    *reinterpret_cast<uint4*>(xt + kXT + off) = lo;
                }
            }
            tgt[cs * kR + r] = (r < nr) ? rawt[r * LD + D + 1] : 0.f;
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&xc_full[cs]);
                mbar_arrive(&raw_empty[rs]);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // warp ew: TMEM lane quadrant quad = warp % 4 -> units 32 quad .. + 31 of half hf;
        // row block rb -> rows 32 rb .. 32 rb + 31 of the tile
        const int ew = warp - 4, quad = warp & 3, hf = (ew >> 2) % NH, rb = ew / (4 * NH);
        const int j = hf * 128 + quad * 32 + lane;  // this thread's hidden unit
        const int et = ew * 32 + lane;              // epilogue thread index; < kR: also owns row et
        const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
        const float w2s = a.Wk[a.H * DP + j];
        const float b2s = a.Wk[a.H * DP + a.H];
        float2 acc2 = make_float2(0.f, 0.f);
        float* out = a.part + (int64_t)blockIdx.x * a.PS;
        const uint32_t wcol = tmem + lanebase + kColW + 48 * hf;
        constexpr int kDH = kD1 / 2;  // dW1 columns drained by each row block (0..16 | 17..33)
        float acc1[kDH];
#pragma unroll
        for (int k = 0; k < kDH; k++) acc1[k] = 0.f;
        auto drain = [&]() {  // dW1 TMEM partial (this thread's unit) -> registers
            if (rb == 0) {
                uint32_t r0[16], r1;
                ld16(wcol, r0);
                ld1(wcol + 16, r1);
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 16; k++) acc1[k] += __uint_as_float(r0[k]);
                acc1[16] += __uint_as_float(r1);
            } else {
                uint32_t r0[16], r1[2];
                ld16(wcol + 16, r0);
                ld2(wcol + 32, r1);
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 15; k++) acc1[k] += __uint_as_float(r0[k + 1]);
                acc1[15] += __uint_as_float(r1[0]);
                acc1[16] += __uint_as_float(r1[1]);
            }
        };
        float dsum = 0.f, loss = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        // The two row blocks are independent pipelines (own named barrier; they meet
        // only at dh_ready, two tiles of slack behind the triple-buffered forward).
        // Row block 1 starts half a tile late -- after row block 0's MUFU-bound pass 1
        // of tile 0 -- so one block's sigmoid pass overlaps the other's shuffle / FMA
        // phases instead of both contending for the MUFU pipe at once.
#if GLX_BTC_OFFSET
        if (rb == 1) bar_sync(kEpiBar + 3, NEW * 32);
#endif
        for (int64_t lt = 0; lt < nt; lt++) {
            const int cs = (int)(lt % kXS), zb = (int)(lt % kZB);
            const int64_t row0 = (blockIdx.x + lt * gridDim.x) * kR;
            BTT(0);
            mbar_wait(&z_full[zb], (uint32_t)(lt / kZB) & 1);
            mbar_wait(&xc_full[cs], (uint32_t)(lt / kXS) & 1);  // orders the converters' tgt writes
            tc_fence_after();
            BTT(1);
            const uint32_t zcol = tmem + lanebase + kColZ + 128 * zb + 64 * hf + 32 * rb;
            float h[32];
            {
                uint32_t r0[32];
                ld32(zcol, r0);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; i++) h[i] = __uint_as_float(r0[i]);
            }
            // pass 1: h = sigmoid(z) (z prescaled by -log2 e)
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
#if GLX_BTC_EXP == 1
                h[i] = h[i] * 0.01f + 0.5f;
                h[i + 1] = h[i + 1] * 0.01f + 0.5f;
#else
                const float2 e2 = ((i >> 1) % GLX_BTC_POLY_DEN < GLX_BTC_POLY) ? exp2_poly2(make_float2(h[i], h[i + 1]))
                                                                 : make_float2(ex2_approx(h[i]), ex2_approx(h[i + 1]));
                const float2 den = __fadd2_rn(e2, bcast2(1.0f));
                h[i] = rcp_approx(den.x);
                h[i + 1] = rcp_approx(den.y);
#endif
            }
            // output partials w2s_j h_j reduce-scattered over the warp's 32 units: lane l
            // ends with row 32 rb + l
            {
                float p[32];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float2 pp = __fmul2_rn(bcast2(w2s), make_float2(h[i], h[i + 1]));
                    p[i] = pp.x;
                    p[i + 1] = pp.y;
                }
#pragma unroll
                for (int st = 0; st < 5; st++) {
                    const int half = 16 >> st;
                    const bool up = (lane >> (4 - st)) & 1;
#pragma unroll
                    for (int i = 0; i < half; i++) {
                        const float send = up ? p[i] : p[i + half];
                        const float keep = up ? p[i + half] : p[i];
                        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
                    }
                }
                opart[(int)(lt & 1) * NEW * 32 + ew * 32 + lane] = p[0];
            }
            BTT(2);
#if GLX_BTC_OFFSET
            if (lt == 0 && rb == 0) bar_arrive(kEpiBar + 3, NEW * 32);
#endif
            bar_sync(kEpiBar + rb, NEW * 16);  // the warps of this row block (they cover all units of its rows)
            BTT(3);
            {  // per row of this warp's block (lane = row 32 rb + l): o, delta_o (kernels.py:352-375);
               // every warp computes its own rows' delta_o, one warp per block keeps the statistics
                const int r = 32 * rb + lane;
                const float* op = opart + (int)(lt & 1) * NEW * 32 + rb * (4 * NH * 32) + lane;
                float z0 = 0.f, z1 = 0.f;
#pragma unroll
                for (int w = 0; w < 4 * NH; w += 2) {
                    z0 += op[w * 32];
                    z1 += op[(w + 1) * 32];
                }
                const float zo = z0 + z1;
                float d = 0.f;
                if (row0 + r < a.N) {
                    const float o = sigmoid_scaled(zo + b2s);
                    const float tt = tgt[cs * kR + r];
                    d = (o - tt) * o * (1.0f - o);
                    if (hf == 0 && quad == 0) {
                        loss = fmaf(0.5f * (tt - o), (tt - o), loss);
                        const bool pred = o >= 0.5f, pos = tt >= 0.5f;
                        c0 += (pred && pos) ? 1.f : 0.f;
                        c1 += (!pred && !pos) ? 1.f : 0.f;
                        c2 += (pred && !pos) ? 1.f : 0.f;
                        c3 += (!pred && pos) ? 1.f : 0.f;
                        dsum += d;
                    }
                }
                dob[ew * 32 + lane] = d;
                __syncwarp();
            }
            BTT(4);
            // the backward of tile lt restarts the dW1 accumulator every kDrain tiles: add the
            // finished partial (through the backward of tile lt - 1) into registers first
            if constexpr (FULL) {  // the backward of the previous tile still reads the dh lo buffer
                if (lt >= 1) {
                    mbar_wait(bwd_done, (uint32_t)(lt - 1) & 1);
                    tc_fence_after();
                }
            }
            if (lt >= 1 && lt % kDrain == 0) {
                mbar_wait(drain_bar, (uint32_t)((lt / kDrain) - 1) & 1);
                tc_fence_after();
                BTT(5);
                drain();
            }
            BTT(6);
            // pass 2: dh = delta_o h (1 - h) -> TMEM (tf32 hi in place of Z, FULL: + lo);
            // dW2 += delta_o h
            const uint32_t locol = tmem + lanebase + kColLo + 64 * hf + 32 * rb;
#pragma unroll
            for (int c = 0; c < 2; c++) {
                uint32_t rh[16], rl[16];
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    const int r = 16 * c + i;
                    const float2 d2 = *reinterpret_cast<const float2*>(dob + ew * 32 + r);
                    const float2 hp = make_float2(h[r], h[r + 1]);
                    const float2 v = __fmul2_rn(d2, hp);
                    acc2 = __fadd2_rn(acc2, v);
                    const float2 s2 = ffma2(make_float2(-v.x, -v.y), hp, v);
                    rh[i] = tf32_rn(s2.x);
                    rh[i + 1] = tf32_rn(s2.y);
                    if constexpr (FULL) {
                        const float2 lo2 =
                            __fadd2_rn(s2, make_float2(-__uint_as_float(rh[i]), -__uint_as_float(rh[i + 1])));
                        rl[i] = __float_as_uint(lo2.x);
                        rl[i + 1] = __float_as_uint(lo2.y);
                    }
                }
                st16(zcol + 16 * c, rh);
                if constexpr (FULL) st16(locol + 16 * c, rl);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dh_ready);
            BTT(7);
        }
        // ---------------------------------------------- per-CTA partial record
        mbar_wait(fin_bar, 0);
        tc_fence_after();
        drain();  // tiles since the last drain (>= 1)
        {
            float* o1 = out + (int64_t)j * (D + 1) + kDH * rb;
#pragma unroll
            for (int k = 0; k < kDH; k++)
                if (kDH * rb + k <= D) o1[k] = acc1[k];
        }
        bar_sync(kEpiBar + 2, NEW * 32);  // opart is free: exchange the dW2 partials of the two row blocks
        if (rb == 1) opart[j] = acc2.x + acc2.y;
        float* stat = opart + 2 * NEW * 32 - kR * 6;  // behind the dW2 exchange slots (H <= 256 floats)
        if (hf == 0 && quad == 0) {  // the statistics warps: rows 32 rb + lane
            const int r = 32 * rb + lane;
            stat[r * 6 + 0] = loss;
            stat[r * 6 + 1] = c0;
            stat[r * 6 + 2] = c1;
            stat[r * 6 + 3] = c2;
            stat[r * 6 + 4] = c3;
            stat[r * 6 + 5] = dsum;
        }
        bar_sync(kEpiBar + 2, NEW * 32);
        if (rb == 0) out[a.P1 + j] = (acc2.x + acc2.y) + opart[j];
        if (et < 6) {
            float s = 0.f;
            for (int r = 0; r < kR; r++) s += stat[r * 6 + et];
            if (et == 5) out[a.P1 + a.H] = s;
            else out[a.P1 + a.H + 1 + et] = s;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

int a4(int x) { return (x + 3) / 4 * 4; }

// row count from which the FAST precision runs (GLX_BTC_PREC=full / fast override it,
// read per launch for A/B tests)
int64_t btc_full_rows() {
    const char* e = getenv("GLX_BTC_PREC");
    if (e && e[0] == 'f' && e[1] == 'u') return INT64_MAX;
    if (e && e[0] == 'f' && e[1] == 'a') return 0;
    return (int64_t)1 << 17;
}
#ifdef GLX_BTC_TIMING
}  // namespace
}  // namespace glx
extern "C" void glx_btc_timing_dump(void) {
    unsigned long long h[4096];
    cudaMemcpyFromSymbol(h, glx::g_btc_dbg, sizeof(h));
    // per tile lt (8..23): epilogue slots 0-7 (warp 4), MMA slots 8-13 (warp 1; lt of the backward for 8-10)
    for (int t = 0; t < 16; t++) {
        const unsigned long long* e = h + t * 32;
        printf("lt %2d epi: wait_z %6lld pass1 %6lld bar1 %6lld rows+bar2 %6lld wait_bwd %6lld drain %6lld pass2 %6lld | "
               "mma: wait_dh %6lld bwd_issue %6lld wait_xf %6lld fwd_issue %6lld | t0 %lld\n",
               t + 8, (long long)(e[2] - e[0]), (long long)(e[4] - e[2]), (long long)(e[6] - e[4]),
               (long long)(e[8] - e[6]), (long long)(e[10] - e[8]), (long long)(e[12] - e[10]),
               (long long)(e[14] - e[12]), (long long)(e[19] - e[17]), (long long)(e[21] - e[19]),
               (long long)(e[25] - e[23]), (long long)(e[27] - e[25]), (long long)(e[0] - h[0]));
    }
}
namespace glx {
namespace {
#endif

}  // namespace

bool batchtc_geometry(int64_t N, int D, int H, int n_sms, BatchGeom* out) {
    if (N < 1 || D < 1 || D > 33 || (H != 128 && H != 256)) return false;
    BatchGeom g{};
    g.D = D;
    g.H = H;
    g.N = N;
    g.DP = D + 1 <= 8 ? 8 : D + 1 <= 16 ? 16 : 34;
    g.LD = a4(std::max(D + 2, g.DP));
    if (g.LD > kMaxLD) return false;
    g.HP = H;
    g.P1 = H * (D + 1);
    g.PS = a4(g.P1 + H + 6);
    g.WKS = a4(H * g.DP + 2 * H + 1);
    g.R = kR;
    g.ntiles = (N + kR - 1) / kR;
    g.grid = (int)std::min<int64_t>(g.ntiles, n_sms);
    // FAST above btc_full_rows() rows (tests/test_gpu_batch.py: FULL keeps small row
    // counts within 1e-5 of the oracle, where FAST's rounding has too few rows to average)
    g.MT = N < btc_full_rows() ? 1 : 0;  // 1: FULL precision
    g.smem = (size_t)(g.MT ? btc_smem<true>(H / 128).total : btc_smem<false>(H / 128).total);
    *out = g;
    return true;
}

template <int NH, bool FULL>
static cudaError_t launch_btc(const BatchGeom& g, const BtcArgs& a, cudaStream_t st) {
    auto k = batchtc_kernel<NH, FULL>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) {
        fprintf(stderr, "glx: batchtc_kernel<%d> smem=%zu: %s\n", NH, g.smem, cudaGetErrorString(e));
        return e;
    }
    k<<<g.grid, btc_threads(NH), g.smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "glx: batchtc_kernel<%d> launch: %s\n", NH, cudaGetErrorString(e));
    return e;
}

cudaError_t launch_batchtc_epoch(const BatchGeom& g, const float* Xp, const float* Wk, float* part, cudaStream_t st) {
    BtcArgs a;
    a.Xp = Xp;
    a.Wk = Wk;
    a.part = part;
    a.N = g.N;
    a.ntiles = g.ntiles;
    a.D = g.D;
    a.DP = g.DP;
    a.LD = g.LD;
    a.H = g.H;
    a.P1 = g.P1;
    a.PS = g.PS;
    if (g.MT) return g.H == 256 ? launch_btc<2, true>(g, a, st) : launch_btc<1, true>(g, a, st);
    return g.H == 256 ? launch_btc<2, false>(g, a, st) : launch_btc<1, false>(g, a, st);
}

}  // namespace glx
