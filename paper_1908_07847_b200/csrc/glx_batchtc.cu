// glx_batchtc.cu -- full-batch gradient-descent epoch (configs 2 and 4:
// D <= 33 inputs -> 24 <= H <= 256 sigmoid units -> 1 output) on the
// 5th-generation tensor cores (tcgen05 kind::tf32).
//
// Same contract as batch3_kernel (glx_batch3.cu): one persistent CTA per SM
// walks row tiles and writes one per-CTA partial record
//   [dW1acc (H*(D+1)) | dW2acc (H) | dsum | loss | c0 c1 c2 c3]
// that batch_update_kernel reduces in f64 and applies (kernels.py:264-295
// batch semantics).
//
// Both GEMMs of the epoch run with the hidden units on the TMEM lanes (M = 128
// units per half; units past H are zero-weight padding):
//   forward   Z^T[j][r]  = W1s[j][:] . x_r            (SS: A = W1s, B = x tile)
//   backward  dW1[j][k] += sum_r dh[j][r] x_r[k]       (TS: A = dh^T from TMEM, B = x^T tile)
// so the delta of every hidden unit stays in TMEM between the two MMAs. The rows
// arrive as per-tile MMA operands built once per training call (btc_pack_kernel:
// tf32-rounded forward and transposed copies, K-major no-swizzle core matrices);
// warp 0 bulk-copies them, warp 1 issues the MMAs (converged, one elect.sync
// lane). Precision (M4b): FULL = 3xTF32 below 2^17 rows,
// FAST = x and the deltas rounded once to tf32 (round to nearest) above.
//
// Per 64-row tile, the epilogue warps (4 TMEM lane quadrants x NH unit halves x 2
// row blocks; thread = hidden unit, 32 rows; two such groups on alternate tiles
// when NH = 1) read Z^T from TMEM, apply the sigmoid (MUFU ex2, one reciprocal
// per element pair), reduce the output partials w2s_j h_j with a warp
// reduce-scatter plus one shared-memory pass per row block, compute delta_o for
// their own rows, and write dh = delta_o h (1 - h) back over Z^T for the backward
// MMA. Z^T has 3-4 buffers (the forward runs ahead of the epilogue); the two row
// blocks are independent pipelines whose sigmoid passes alternate through a
// named-barrier token. DESIGN.md section 4 has the measured path and the per-phase
// timeline (GLX_BTC_TIMING builds, tools/btc_timeline.py).
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

namespace glx {

namespace {

constexpr int kR = 64;    // rows per tile (forward MMA N)
constexpr int kFC = 10;   // 4-feature chunks of the forward operands (K = 40)
constexpr int kFCS = 9;   // chunks stored per tile (k < 36; chunk 9 is zero: LD <= 36)
constexpr int kNB = 48;   // features in the backward (MMA N, multiple of 16)
constexpr int kNBS = 40;  // feature rows stored per tile (k < 40; block 5 is zero)
// Per 64-row tile the epoch reads the rows pre-laid-out for the MMAs (glx_tile_pack,
// once per training call) -- tf32-rounded, no conversion inside the epoch:
//   forward operand  [k/4][r/8][r%8][k%4]  (K-major core matrices, LBO 1024 B, SBO 128 B)
//   backward operand [k/8][r/4][k%8][r%4]  (x transposed: K = rows; LBO 128 B, SBO 2048 B)
// FAST stores the hi (tf32) copies, FULL also the lo copies. The target of row r
// travels as feature D + 1 (a zero weight column), read back from the backward copy.
constexpr int kXF = kFC * kR / 8 * 128;        // smem bytes, forward operand (10 KB)
constexpr int kXT = kNB / 8 * kR / 4 * 128;    // smem bytes, backward operand (12 KB)
constexpr int kXFG = kFCS * kR / 8 * 128;      // global bytes, forward operand (9 KB)
constexpr int kXTG = kNBS / 8 * kR / 4 * 128;  // global bytes, backward operand (10 KB)
constexpr int kWT = 16 * kFC * 128;            // bytes per 128-unit weight copy (hi or lo)
// Two precisions (template FULL): FAST (large N) uses tf32(x) only, forward
// hi(W) tf32(x) + lo(W) tf32(x), backward tf32(dh) tf32(x); FULL (small N, where
// too few rows average the operand rounding out) is 3xTF32 on both GEMMs (x and dh
// split into hi + lo as well), which needs the lo copies of x and a dh lo TMEM
// buffer. Stage counts per precision (shared memory, TMEM):
#ifndef GLX_BTC_S
#define GLX_BTC_S 6  // FAST tile-ring stages
#endif
template <bool FULL>
struct Pipe {
    static constexpr int NX = FULL ? 2 : 1;                       // x operand copies: hi (+ lo)
    static constexpr int STAGE = NX * (kXF + kXT);                 // smem bytes per tile stage
    static constexpr int GTILE = NX * (kXFG + kXTG);               // global bytes per tile
    static constexpr int S = FULL ? 3 : GLX_BTC_S;                 // tile stages (free after the backward)
    static constexpr int ZB = FULL ? 2 : 3;                        // Z^T buffers: the forward runs ZB tiles ahead
};
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
#ifndef GLX_BTC_ZB
#define GLX_BTC_ZB 2  // FAST, two unit halves: Z^T buffers (the forward runs this many tiles ahead; 2 frees the
                      // TMEM columns of the drain sums: 0.234 -> 0.224 ms per 1M rows at H = 256, 3 without: 0.234)
#endif
#ifndef GLX_BTC_ACC_TMEM
#define GLX_BTC_ACC_TMEM 1  // FAST dW1 drain sums in TMEM instead of 17 registers per thread (0: registers)
#endif
constexpr int kColA1 = 256;  // FAST: dW1 drain sums (needs the Z buffers below column 256)
#ifndef GLX_BTC_RCP2
#define GLX_BTC_RCP2 1  // 1: one MUFU reciprocal per element pair (0: one per element)
#endif
#ifndef GLX_BTC_RN2
#define GLX_BTC_RN2 0  // 1: tf32 rounding of the hidden deltas on the FMA pipe (pairs)
#endif
#ifndef GLX_BTC_TOKEN
#define GLX_BTC_TOKEN 1  // 0: the two row blocks' sigmoid passes are not interleaved
#endif
#ifndef GLX_BTC_EXP
#define GLX_BTC_EXP 0  // diagnostic builds only: 1 no MUFU sigmoid, 2 no backward MMAs, 3 no forward MMAs
#endif

#ifdef GLX_BTC_TIMING
// per-phase clock64 timeline of CTA 0 (diagnostic builds: tools/btc_timeline.py):
// tiles 8..23, 16 slots per tile, for warp 4 (row block 0), warp 1 (MMA), warp 12
// (row block 1 when NH = 2) and warp 0 (producer)
__device__ unsigned long long g_btc_dbg[4096];
#define BTT(slot)                                                                                           \
    do {                                                                                                    \
        const int wi_ = warp == 4 ? 0 : warp == 1 ? 1 : warp == 12 ? 2 : warp == 0 ? 3 : -1;                \
        if (blockIdx.x == 0 && lane == 0 && wi_ >= 0 && lt >= 8 && lt < 24)                                 \
            g_btc_dbg[((lt - 8) * 16 + (slot)) * 4 + wi_] = clock64();                                      \
    } while (0)
#else
#define BTT(slot) \
    do {          \
    } while (0)
#endif

struct BtcArgs {
    const unsigned char* tiles;  // glx_tile_pack output: ntiles x Pipe<FULL>::GTILE bytes
    const float* Wk;
    float* part;
    int64_t N, ntiles;
    int D, DP, H, P1, PS;
    int* dbg;  // pipeline checker (debug runs, else nullptr): see dbg_expect
};

// ---------------------------------------------------------------- pipeline checker
// Debug runs (GLX_FLAG_DEBUG / glx_set_debug) pass a.dbg: every hand-off of a tile
// between the roles carries a stamp (tile index + 1) that the producing role writes
// before its barrier arrive and the consuming role checks after its wait -- the
// device analogue of the reference's generation-stamped forward_pair_debug
// (backend.py:237-284): a role that passes a barrier on the wrong phase (the hazard
// of a counter shared by tiles that run ahead of each other) reads another tile's
// stamp. The roles also count the tiles they handled, the analogue of the
// reference's write-once shadow counts (backend.py:122-133): the host requires one
// forward issue and one dh hand-off per row group for every tile of the epoch.
// Layout (ints): [0] violations, [1] first check id, [2] its CTA, [3] expected
// stamp, [4] seen stamp; [kDbgHdr, + T) forward issues per tile, [+ T, + 2T) dh
// hand-offs per tile; then kDbgCta stamp slots per CTA. Stamps are global words:
// mbarrier arrive / wait order them (release / acquire at CTA scope); the arrives
// made by tcgen05.commit fire when the MMAs complete, long after the issuing
// thread's stamp store, which a CTA fence orders first.
#ifndef GLX_PIPELINE_CHECK
#define GLX_PIPELINE_CHECK 1  // 0 compiles the checker out (A/B timing of its cost)
#endif
#define GLX_DBG_ON(a) (GLX_PIPELINE_CHECK && (a).dbg != nullptr)
constexpr int kDbgHdr = 16, kDbgCta = 64;
struct DbgView {
    int* base;
    int* vf;
    int* vb;
    int* st;
};
__device__ __forceinline__ DbgView dbg_view(int* p, int64_t ntiles) {
    DbgView d;
    d.base = p;
    d.vf = p ? p + kDbgHdr : nullptr;
    d.vb = p ? p + kDbgHdr + ntiles : nullptr;
    d.st = p ? p + kDbgHdr + 2 * ntiles + (int64_t)blockIdx.x * kDbgCta : nullptr;
    return d;
}
__device__ __forceinline__ void dbg_put(const DbgView& d, int slot, int64_t lt) {
    reinterpret_cast<volatile int*>(d.st)[slot] = (int)(lt + 1);
    __threadfence_block();
}
// the producer's stamp of a loaded stage; header word 6 = 1 + a tile index makes
// that tile's stamp wrong (fault injection: tests prove the checker fires)
__device__ __forceinline__ void dbg_put_load(const DbgView& d, int slot, int64_t lt) {
    const int64_t tile = blockIdx.x + lt * gridDim.x;
    const int bad = d.base[6] == (int)(tile + 1);
    reinterpret_cast<volatile int*>(d.st)[slot] = (int)(lt + 1) + bad;
    __threadfence_block();
}
__device__ __forceinline__ void dbg_expect(const DbgView& d, int id, int slot, int64_t lt) {
    const int seen = reinterpret_cast<volatile int*>(d.st)[slot];
    if (seen != (int)(lt + 1) && atomicAdd(d.base, 1) == 0) {
        d.base[1] = id;
        d.base[2] = blockIdx.x;
        d.base[3] = (int)(lt + 1);
        d.base[4] = seen;
    }
}

struct BtcSmem {  // byte offsets
    int w, x, opart, dob, stat, bars;
    int total;
};

// warp 0 producer, warp 1 MMA, warps 2 .. 2 + 8 NH - 1 epilogue
// epilogue groups: with one 128-unit half (NH = 1) the FAST kernel runs two groups of 8
// warps on alternate tiles (the per-tile chain of a row block, not throughput, bounds
// the narrow layer); NH = 2 and FULL run one group
__host__ __device__ constexpr int btc_groups(int NH, bool FULL) { return (NH == 1 && !FULL) ? 2 : 1; }
__host__ __device__ constexpr int btc_threads(int NH, bool FULL) { return (2 + 8 * NH * btc_groups(NH, FULL)) * 32; }

template <bool FULL>
__host__ __device__ constexpr BtcSmem btc_smem(int NH) {
    using P = Pipe<FULL>;
    BtcSmem s{};
    s.w = 0;
    s.x = s.w + 2 * NH * kWT;          // stage i at x + i * STAGE: [xf hi | xt hi (| xf lo | xt lo)]
    s.opart = s.x + P::S * P::STAGE;
    const int nw = 8 * NH * btc_groups(NH, FULL);  // epilogue warps
    s.dob = s.opart + 2 * nw * 32 * 4;  // output partials, double-buffered by tile parity
    s.stat = s.dob + nw * 32 * 4;       // dob: one 32-row slot per epilogue warp
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

__device__ __forceinline__ void st1(uint32_t taddr, const uint32_t (&r)[1]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(r[0]) : "memory");
}
__device__ __forceinline__ void st2(uint32_t taddr, const uint32_t (&r)[2]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(r[0]), "r"(r[1]) : "memory");
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
#ifndef GLX_BTC_CVT
#define GLX_BTC_CVT 0  // 1: cvt.rn.satfinite.tf32.f32 (one F2FP: measured slower), 0: integer round-half-away
#endif
__device__ __forceinline__ uint32_t tf32_rn(float v) {
#if GLX_BTC_CVT
    uint32_t r;
    asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return r;
#else
    return (__float_as_uint(v) + 0x1000u) & kTf32Mask;
#endif
}
// the same rounding for a pair on the FMA pipe (Veltkamp split: t = v (2^13 + 1),
// hi = t - (t - v) keeps the leading 11 significant bits, round to nearest even;
// |v| < 2^114 so t cannot overflow)
__device__ __forceinline__ float2 tf32_rn2(float2 v) {
    const float2 t = __fmul2_rn(v, bcast2(8193.0f));
    return __fadd2_rn(t, make_float2(-(t.x - v.x), -(t.y - v.y)));
}

// 2^x for a pair on the FMA/ALU pipes (pass 1 is MUFU-bound): round-to-nearest by
// the 1.5 * 2^23 magic add, degree-5 polynomial on [-1/2, 1/2] (max rel. error 2.3e-7
// in fp32 Horner, on par with ex2.approx), exponent inserted with an integer add;
// |x| clamped to 125 (1 + 2^-125 == 1 and 1 / (1 + 2^125) ~ 0 in fp32 either way)
#ifndef GLX_BTC_POLY
#define GLX_BTC_POLY 0  // element pairs per GLX_BTC_POLY_DEN that take the polynomial (0: all MUFU)
#endif
#ifndef GLX_BTC_POLY_DEN
#define GLX_BTC_POLY_DEN 8
#endif
__device__ __forceinline__ float2 fminf2(float2 a, float2 b) { return make_float2(fminf(a.x, b.x), fminf(a.y, b.y)); }

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

// CHK: the pipeline-checker instantiation (debug runs only: the checks cost the
// production kernel ~10 % through code layout even when switched off at run time)
template <int NH, bool FULL, bool PAD, bool CHK>
__global__ void __launch_bounds__(btc_threads(NH, FULL), 1) batchtc_kernel(const BtcArgs a) {
    constexpr int G = btc_groups(NH, FULL);  // epilogue groups, on alternate tiles
    constexpr int NEWG = 8 * NH;             // warps per group: 4 lane quadrants x NH unit halves x 2 row blocks
    constexpr int NEW = NEWG * G;            // epilogue warps
    using P = Pipe<FULL>;
    constexpr BtcSmem L = btc_smem<FULL>(NH);
    constexpr int kS = P::S;
    constexpr int kZB = FULL ? 2 : (G == 2 ? 4 : GLX_BTC_ZB);  // Z^T buffers (64 NH columns each)
    // FAST: the dW1 drain sums in TMEM columns kColA1 .. (17 per unit half and row block),
    // free when the Z buffers end below them
    constexpr bool kAccT = GLX_BTC_ACC_TMEM && !FULL && 64 * NH * kZB <= kColA1;
    static_assert(kDrain % G == 0, "the drained tiles must all belong to group 0");
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* x_full = bars;                // tile stage loaded (bulk-copy bytes)
    uint64_t* x_empty = x_full + kS;        // tile stage free (its backward completed)
    uint64_t* z_full = x_empty + kS;        // Z^T buffer written by the forward
    // dh_ready[rb * kZB + lt % kZB]: row block rb wrote dh of tile lt. Per row block:
    // the blocks run up to kZB tiles apart, and a counter shared by both would complete
    // a tile's phase on the leading block's arrivals for a later tile. Per Z buffer: a
    // block cannot arrive for tile lt + kZB before backward(lt) was issued (it needs
    // Z(lt + kZB)), so each barrier is at most one phase ahead of the MMA warp's wait.
    uint64_t* dh_ready = z_full + kZB;
    uint64_t* drain_bar = dh_ready + 2 * kZB;  // the backward of the last tile before a dW1 drain completed
    uint64_t* fin_bar = drain_bar + 1;      // the last backward completed
    uint64_t* bwd_done = fin_bar + 1;       // FULL: every backward completed (the dh lo buffer is free)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bwd_done + 1);
    float* opart = reinterpret_cast<float*>(sm + L.opart);
    float* dob = reinterpret_cast<float*>(sm + L.dob);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nt = (a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA (>= 1)
    const int D = a.D, DP = a.DP;
    // checker slots: x stage [0, kS), its release by the backward [8, 8 + kS), Z buffer
    // [16, 16 + kZB), dh per row block and Z buffer [24, 24 + 2 kZB)
    const DbgView dv = dbg_view(a.dbg, a.ntiles);
#define BTC_CHK (CHK && a.dbg != nullptr)

    if (threadIdx.x == 0) {
        for (int i = 0; i < kS; i++) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_empty[i], 1);
        }
        for (int b = 0; b < kZB; b++) mbar_init(&z_full[b], 1);
        for (int b = 0; b < 2 * kZB; b++) mbar_init(&dh_ready[b], NEWG / 2);
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
            v[i] = (k <= D && j < a.H) ? a.Wk[(int64_t)j * DP + k] : 0.f;  // units >= H: zero rows
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
    // the operand regions the bulk copies never write (forward chunk 9, backward
    // feature block 5) stay zero for the whole launch
    for (int i = threadIdx.x; i < kS * P::NX * (kXF - kXFG + kXT - kXTG) / 16; i += blockDim.x) {
        const int per = (kXF - kXFG + kXT - kXTG) / 16, c = i / per, w = i - (i / per) * per;
        const int st = c / P::NX, cp = c - st * P::NX;
        unsigned char* base = sm + L.x + st * P::STAGE + cp * (kXF + kXT);
        unsigned char* dst = w < (kXF - kXFG) / 16 ? base + kXFG + 16 * w : base + kXF + kXTG + 16 * (w - (kXF - kXFG) / 16);
        *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
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
                const int xs = (int)(lt % kS);
                if (lt >= kS) {
                    mbar_wait(&x_empty[xs], (uint32_t)((lt / kS) - 1) & 1);
                    if (BTC_CHK) dbg_expect(dv, 1, 8 + xs, lt - kS);
                }
                BTT(14);
                const unsigned char* src = a.tiles + (blockIdx.x + lt * gridDim.x) * (int64_t)P::GTILE;
                unsigned char* dst = sm + L.x + xs * P::STAGE;
                if (BTC_CHK) dbg_put_load(dv, xs, lt);
                mbar_arrive_expect_tx(&x_full[xs], (uint32_t)P::GTILE);
#pragma unroll
                for (int cp = 0; cp < P::NX; cp++) {
                    bulk_g2s(dst + cp * (kXF + kXT), src + cp * (kXFG + kXTG), kXFG, &x_full[xs]);
                    bulk_g2s(dst + cp * (kXF + kXT) + kXF, src + cp * (kXFG + kXTG) + kXFG, kXTG, &x_full[xs]);
                }
                BTT(15);
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
            const uint64_t dx0 = desc_ns(smem_u32(sm + L.x), kR / 8 * 128, 128);
            const uint64_t dt0 = desc_ns(smem_u32(sm + L.x + kXF), 128, kR / 4 * 128);
            // backward of tile lt: dW1[j][k] += sum_r dh[j][r] x_r[k] (FAST: one tf32 product,
            // the rounding of dh and x averages out over the rows, tools/tf32_split_error.py)
            auto backward = [&](int64_t lt) {
                const int xs = (int)(lt % kS), zb = (int)(lt % kZB);
                BTT(8);
                mbar_wait(&dh_ready[zb], (uint32_t)(lt / kZB) & 1);
                mbar_wait(&dh_ready[kZB + zb], (uint32_t)(lt / kZB) & 1);
                tc_fence_after();
                if (BTC_CHK && el) {
                    dbg_expect(dv, 3, 24 + zb, lt);
                    dbg_expect(dv, 4, 24 + kZB + zb, lt);
                    dbg_put(dv, 8 + xs, lt);  // read by the producer after x_empty
                }
                BTT(9);
                const uint64_t dth = dt0 + ((xs * P::STAGE) >> 4);
                const uint64_t dtl = dth + ((kXF + kXT) >> 4);  // FULL: the lo copies follow
#pragma unroll
                for (int hf = 0; hf < NH; hf++) {
                    const uint32_t d = tmem + kColW + 48 * hf;
                    const uint32_t ahi = tmem + kColZ + 64 * NH * zb + 64 * hf, alo = tmem + kColLo + 64 * hf;
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
                commit(&x_empty[xs], el);
                if constexpr (FULL) commit(bwd_done, el);
                if ((lt + 1) % kDrain == 0) commit(drain_bar, el);
                if (lt == nt - 1) commit(fin_bar, el);
                BTT(10);
            };
            // forward of tile lt: Z^T = W1s . x as hi(W) x + lo(W) x (the small term first;
            // FULL adds hi(W) lo(x))
            auto forward = [&](int64_t lt) {
                const int xs = (int)(lt % kS), zb = (int)(lt % kZB);
                BTT(11);
                mbar_wait(&x_full[xs], (uint32_t)(lt / kS) & 1);
                tc_fence_after();
                if (BTC_CHK && el) {
                    dbg_expect(dv, 2, xs, lt);
                    atomicAdd(&dv.vf[blockIdx.x + lt * gridDim.x], 1);
                    dbg_put(dv, 16 + zb, lt);  // read by the epilogue after z_full
                }
                BTT(12);
                const uint64_t dx = dx0 + ((xs * P::STAGE) >> 4);
                const uint64_t dxl = dx + ((kXF + kXT) >> 4);  // FULL: lo copy
#pragma unroll
                for (int hf = 0; hf < NH; hf++) {
                    const uint32_t d = tmem + kColZ + 64 * NH * zb + 64 * hf;
                    const uint64_t wh = dwh + (hf * kWT >> 4), wl = dwl + (hf * kWT >> 4);
#if GLX_BTC_EXP == 3
                    mma_ss(d, wh, dx, idf, 0, el);
                    if (false)
#endif
                    {
#pragma unroll
                        for (int s = 0; s < kFC / 2; s++) {
                            mma_ss(d, wl + (s * 256 >> 4), dx + (s * 2048 >> 4), idf, s != 0, el);
                            if constexpr (FULL) mma_ss(d, wh + (s * 256 >> 4), dxl + (s * 2048 >> 4), idf, 1, el);
                        }
#pragma unroll
                        for (int s = 0; s < kFC / 2; s++)
                            mma_ss(d, wh + (s * 256 >> 4), dx + (s * 2048 >> 4), idf, 1, el);
                    }
                }
                commit(&z_full[zb], el);
                BTT(13);
            };
            // kZB Z^T buffers: the forward runs kZB tiles ahead; forward(lt + kZB) reuses the
            // buffer of tile lt right after backward(lt) (the tensor pipe executes in order)
            for (int64_t lt = 0; lt < kZB && lt < nt; lt++) forward(lt);
            for (int64_t lt = 0; lt < nt; lt++) {
                backward(lt);
                if (lt + kZB < nt) forward(lt + kZB);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // warp ew: TMEM lane quadrant quad = warp % 4 -> units 32 quad .. + 31 of half hf;
        // row block rb -> rows 32 rb .. 32 rb + 31 of the tile
        // group gi takes tiles lt = gi, gi + G, ...
        const int ew = warp - 2, quad = warp & 3, gi = ew / NEWG, ewg = ew - gi * NEWG;
        const int hf = (ewg >> 2) % NH, rb = ewg / (4 * NH);
        const int j = hf * 128 + quad * 32 + lane;  // this thread's hidden unit
        const int et = ew * 32 + lane;              // epilogue thread index; < kR: also owns row et
        const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
        // H not a multiple of 128: the padded units have zero weights (Z = 0, w2 = 0);
        // a warp whose 32 units are all padding skips the arithmetic and only keeps the
        // barrier protocol (its output partial slots stay zero)
        const bool active = !PAD || hf * 128 + quad * 32 < a.H;  // PAD: H is not 128 NH
        const float w2s = j < a.H ? a.Wk[a.H * DP + j] : 0.f;
        if (!active) {
            opart[ew * 32 + lane] = 0.f;
            opart[NEW * 32 + ew * 32 + lane] = 0.f;
        }
        const float b2s = a.Wk[a.H * DP + a.H];
        // the target of row r: feature D + 1 of the backward operand copy
        const int tk = D + 1;
        const int toff = kXF + (tk >> 3) * (kR / 4 * 128) + (tk & 7) * 16;
        float2 acc2 = make_float2(0.f, 0.f);
        float* out = a.part + (int64_t)blockIdx.x * a.PS;
        const uint32_t wcol = tmem + lanebase + kColW + 48 * hf;
        constexpr int kDH = kD1 / 2;  // dW1 columns drained by each row block (0..16 | 17..33)
        const uint32_t acol1 = tmem + lanebase + kColA1 + kDH * (2 * hf + rb);
        if constexpr (kAccT) {
            if (gi == 0 && active) {
                uint32_t z[16] = {}, z1[1] = {0u};
                st16(acol1, z);
                st1(acol1 + 16, z1);
                tmem_st_wait();
            }
        }
        float acc1[kAccT ? 1 : kDH];
#pragma unroll
        for (int k = 0; k < (kAccT ? 1 : kDH); k++) acc1[k] = 0.f;
        auto drain = [&]() {  // dW1 TMEM partial (this thread's unit) -> registers
            if constexpr (kAccT) {  // ... -> the TMEM sums: add the partial to them
                uint32_t q0[16], q1, s0[16], s1;
                if (rb == 0) {
                    ld16(wcol, q0);
                    ld1(wcol + 16, q1);
                } else {
                    uint32_t t0[16], t1[2];
                    ld16(wcol + 16, t0);
                    ld2(wcol + 32, t1);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 15; k++) q0[k] = t0[k + 1];
                    q0[15] = t1[0];
                    q1 = t1[1];
                }
                ld16(acol1, s0);
                ld1(acol1 + 16, s1);
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 16; k++) s0[k] = __float_as_uint(__uint_as_float(s0[k]) + __uint_as_float(q0[k]));
                uint32_t s1a[1] = {__float_as_uint(__uint_as_float(s1) + __uint_as_float(q1))};
                st16(acol1, s0);
                st1(acol1 + 16, s1a);
                tmem_st_wait();
                return;
            }
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
        // only at dh_ready, kZB tiles of slack behind the forward). Their MUFU-bound
        // sigmoid passes take turns -- a token passed through two named barriers: block 0
        // does tile lt's pass 1, then block 1 does its own, then block 0 tile lt + 1 --
        // so each pass has the MUFU pipe to itself while the other block runs its
        // shuffle / FMA phases, instead of both contending at once.
        // named barriers of group gi: its two row blocks, then the token pair
        const int kBarRb = 1 + 4 * gi, kTok0 = kBarRb + 2, kTok1 = kBarRb + 3;  // token: block 1 -> 0, 0 -> 1
        constexpr int kBarAll = 1 + 4 * G;  // all epilogue warps (the final exchange)
        for (int64_t lt = gi; lt < nt; lt += G) {
            const int xs = (int)(lt % kS), zb = (int)(lt % kZB);
            const int par = (int)((lt / G) & 1);  // this group's tile parity (double-buffered output partials)
            const int64_t row0 = (blockIdx.x + lt * gridDim.x) * kR;
            BTT(0);
            mbar_wait(&z_full[zb], (uint32_t)(lt / kZB) & 1);
            tc_fence_after();
            if (BTC_CHK && lane == 0) dbg_expect(dv, 5, 16 + zb, lt);
            BTT(1);
            const uint32_t zcol = tmem + lanebase + kColZ + 64 * NH * zb + 64 * hf + 32 * rb;
            float h[32];
            if (active) {
                uint32_t r0[32];
                ld32(zcol, r0);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; i++) h[i] = __uint_as_float(r0[i]);
            }
#if GLX_BTC_TOKEN
            if (rb == 1) bar_sync(kTok1, NEWG * 32);          // block 0 finished its pass 1 of tile lt
            else if (lt >= G) bar_sync(kTok0, NEWG * 32);     // block 1 finished its pass 1 of tile lt - G
#endif
            BTT(5);
            // pass 1: h = sigmoid(z) (z prescaled by -log2 e)
            if (active) {
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
#if GLX_BTC_EXP == 1
                    h[i] = h[i] * 0.01f + 0.5f;
                    h[i + 1] = h[i + 1] * 0.01f + 0.5f;
#else
                    const float2 e2 = ((i >> 1) % GLX_BTC_POLY_DEN < GLX_BTC_POLY)
                                          ? exp2_poly2(make_float2(h[i], h[i + 1]))
                                          : make_float2(ex2_approx(h[i]), ex2_approx(h[i + 1]));
#if GLX_BTC_RCP2
                    // one MUFU reciprocal per pair: 1/a = b / (ab), 1/b = a / (ab); e clamped to
                    // 2^60 so ab stays finite (h < 2^-60 there either way)
                    const float2 den = __fadd2_rn(fminf2(e2, bcast2(1.152921504606847e18f)), bcast2(1.0f));
                    const float r = rcp_approx(den.x * den.y);
                    const float2 hh = __fmul2_rn(make_float2(den.y, den.x), bcast2(r));
                    h[i] = hh.x;
                    h[i + 1] = hh.y;
#else
                    const float2 den = __fadd2_rn(e2, bcast2(1.0f));
                    h[i] = rcp_approx(den.x);
                    h[i + 1] = rcp_approx(den.y);
#endif
#endif
                }
            }
            BTT(6);
#if GLX_BTC_TOKEN
            bar_arrive(rb == 0 ? kTok1 : kTok0, NEWG * 32);  // the other block's turn on the MUFU pipe
#endif
            // output partials w2s_j h_j reduce-scattered over the warp's 32 units: lane l
            // ends with row 32 rb + l
            if (active) {
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
                opart[par * NEW * 32 + ew * 32 + lane] = p[0];
            }
            BTT(2);
            bar_sync(kBarRb + rb, NEWG * 16);  // the warps of this row block (they cover all units of its rows)
            BTT(3);
            if (active) {  // per row of this warp's block (lane = row 32 rb + l): o, delta_o (kernels.py:352-375);
               // every warp computes its own rows' delta_o, one warp per block keeps the statistics
                const int r = 32 * rb + lane;
                const float* op = opart + par * NEW * 32 + (gi * NEWG + rb * 4 * NH) * 32 + lane;
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
                    const float tt = *reinterpret_cast<const float*>(sm + L.x + xs * P::STAGE + toff +
                                                                     (r >> 2) * 128 + (r & 3) * 4);
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
            if constexpr (FULL) {  // the backward of the previous tile still reads the dh lo buffer
                if (lt >= 1 && active) {
                    mbar_wait(bwd_done, (uint32_t)(lt - 1) & 1);
                    tc_fence_after();
                }
            }
            // pass 2: dh = delta_o h (1 - h) -> TMEM (tf32 hi in place of Z, FULL: + lo);
            // dW2 += delta_o h
            const uint32_t locol = tmem + lanebase + kColLo + 64 * hf + 32 * rb;
            if (active) {
#pragma unroll
            for (int c = 0; c < 2; c++) {
                uint32_t rh[16], rl[16];
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const int r = 16 * c + i;
                    const float4 d4 = *reinterpret_cast<const float4*>(dob + ew * 32 + r);
#pragma unroll
                    for (int u = 0; u < 4; u += 2) {
                        const float2 d2 = u ? make_float2(d4.z, d4.w) : make_float2(d4.x, d4.y);
                        const float2 hp = make_float2(h[r + u], h[r + u + 1]);
                        const float2 v = __fmul2_rn(d2, hp);
                        acc2 = __fadd2_rn(acc2, v);
                        const float2 s2 = ffma2(make_float2(-v.x, -v.y), hp, v);
#if GLX_BTC_RN2
                        const float2 r2 = tf32_rn2(s2);
                        rh[i + u] = __float_as_uint(r2.x);
                        rh[i + u + 1] = __float_as_uint(r2.y);
#else
                        rh[i + u] = tf32_rn(s2.x);
                        rh[i + u + 1] = tf32_rn(s2.y);
#endif
                        if constexpr (FULL) {
                            const float2 lo2 = __fadd2_rn(
                                s2, make_float2(-__uint_as_float(rh[i + u]), -__uint_as_float(rh[i + u + 1])));
                            rl[i + u] = __float_as_uint(lo2.x);
                            rl[i + u + 1] = __float_as_uint(lo2.y);
                        }
                    }
                }
                st16(zcol + 16 * c, rh);
                if constexpr (FULL) st16(locol + 16 * c, rl);
            }
            }
            // the backward of tile lt restarts the dW1 accumulator every kDrain tiles: add the
            // finished partial (through the backward of tile lt - 1, issued a tile ago) into
            // registers before this tile's dh_ready releases that backward
            if (lt >= 1 && lt % kDrain == 0 && active) {
                mbar_wait(drain_bar, (uint32_t)((lt / kDrain) - 1) & 1);
                tc_fence_after();
                drain();
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (BTC_CHK && lane == 0) {
                dbg_put(dv, 24 + rb * kZB + zb, lt);
                if (ewg % (4 * NH) == 0) atomicAdd(&dv.vb[blockIdx.x + lt * gridDim.x], 1);  // one per row block
            }
            if (lane == 0) mbar_arrive(&dh_ready[rb * kZB + zb]);
            BTT(7);
        }
        // ---------------------------------------------- per-CTA partial record
#if GLX_BTC_TOKEN
        if (rb == 0 && gi < nt) bar_sync(kTok0, NEWG * 32);  // block 1's last token
#endif
        // dW1: the TMEM accumulator sums every tile's backward; group 0 drains it (the
        // drained tiles are all group 0's) and owns the dW1 partials
        if (gi == 0) {
            mbar_wait(fin_bar, 0);
            tc_fence_after();
            if (active) drain();  // tiles since the last drain (>= 1)
            if constexpr (kAccT) {
                if (active) {
                    uint32_t s0[16], s1;
                    ld16(acol1, s0);
                    ld1(acol1 + 16, s1);
                    tmem_ld_wait();
                    if (j < a.H) {
                        float* o1 = out + (int64_t)j * (D + 1) + kDH * rb;
#pragma unroll
                        for (int k = 0; k < kDH; k++)
                            if (kDH * rb + k <= D) o1[k] = __uint_as_float(k < 16 ? s0[k] : s1);
                    }
                }
            } else if (j < a.H) {
                float* o1 = out + (int64_t)j * (D + 1) + kDH * rb;
#pragma unroll
                for (int k = 0; k < kDH; k++)
                    if (kDH * rb + k <= D) o1[k] = acc1[k];
            }
        }
        // dW2 and the row statistics: one slot per (group, row block), summed in fixed order
        bar_sync(kBarAll, NEW * 32);  // opart is free
        if (j < a.H) opart[(gi * 2 + rb) * 256 + j] = acc2.x + acc2.y;
        bar_sync(kBarAll, NEW * 32);
        if (gi == 0 && rb == 0 && j < a.H) {
            float s2 = 0.f;
            for (int q = 0; q < 2 * G; q++) s2 += opart[q * 256 + j];
            out[a.P1 + j] = s2;
        }
        bar_sync(kBarAll, NEW * 32);
        float* stat = opart;  // [G][64 rows][6]
        if (hf == 0 && quad == 0) {  // the statistics warps: rows 32 rb + lane of this group's tiles
            const int r = gi * kR + 32 * rb + lane;
            stat[r * 6 + 0] = loss;
            stat[r * 6 + 1] = c0;
            stat[r * 6 + 2] = c1;
            stat[r * 6 + 3] = c2;
            stat[r * 6 + 4] = c3;
            stat[r * 6 + 5] = dsum;
        }
        bar_sync(kBarAll, NEW * 32);
        if (et < 6) {
            float s = 0.f;
            for (int r = 0; r < G * kR; r++) s += stat[r * 6 + et];
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

#undef BTC_CHK

// rows -> the per-tile operand layouts (see kXF / kXT), tf32 round to nearest; FULL
// also writes the lo remainders. One block per 64-row tile, the tile staged through
// shared memory so both the row reads and the tile writes are coalesced.
template <bool FULL>
__global__ void __launch_bounds__(256) btc_pack_kernel(const float* __restrict__ Xp, int64_t N, int LD,
                                                       unsigned char* __restrict__ tiles) {
    using P = Pipe<FULL>;
    __shared__ float t[kR * 37];
    const int64_t tile = blockIdx.x;
    const int64_t row0 = tile * kR;
    const int nr = (int)((N - row0) < kR ? (N - row0) : kR);
    for (int e = threadIdx.x; e < kR * 36; e += blockDim.x) {
        const int r = e / 36, k = e - (e / 36) * 36;
        t[r * 37 + k] = (r < nr && k < LD) ? Xp[(row0 + r) * LD + k] : 0.f;
    }
    __syncthreads();
    uint32_t* out = reinterpret_cast<uint32_t*>(tiles + tile * (int64_t)P::GTILE);
    // forward operand: word w = ((q * 8 + r / 8) * 8 + r % 8) * 4 + k % 4, k = 4 q + k % 4
    for (int w = threadIdx.x; w < kXFG / 4; w += blockDim.x) {
        const int e = w & 3, r8 = (w >> 2) & 7, ro = (w >> 5) & 7, q = w >> 8;
        const float v = t[(ro * 8 + r8) * 37 + 4 * q + e];
        const uint32_t hi = tf32_rn(v);
        out[w] = hi;
        if constexpr (FULL) out[(kXFG + kXTG) / 4 + w] = __float_as_uint(v - __uint_as_float(hi));
    }
    // backward operand: word w = ((kb * 16 + r / 4) * 8 + k % 8) * 4 + r % 4, k = 8 kb + k % 8
    for (int w = threadIdx.x; w < kXTG / 4; w += blockDim.x) {
        const int r4 = w & 3, k8 = (w >> 2) & 7, rq = (w >> 5) & 15, kb = w >> 9;
        const int k = kb * 8 + k8;
        const float v = k < 36 ? t[(rq * 4 + r4) * 37 + k] : 0.f;
        const uint32_t hi = tf32_rn(v);
        out[kXFG / 4 + w] = hi;
        if constexpr (FULL) out[(kXFG + kXTG + kXFG) / 4 + w] = __float_as_uint(v - __uint_as_float(hi));
    }
}

// =================================================== narrow layers: rows on the lanes
// For H <= 64 (the reference's default width is 33) the unit-on-lanes kernel above
// leaves most of its epilogue idle and pays a cross-lane reduction per row. Here the
// forward puts the ROWS on the TMEM lanes (M = 128 rows, N = HP units), so each
// epilogue thread owns one row: the output dot, delta_o and the statistics are
// per-thread sums. The backward contracts over rows, so the hidden deltas go to
// shared memory as the K-major A operand dh^T [128 units][128 rows] (128-byte
// swizzle: a warp's 32 rows of one unit are one conflict-free 128-byte row) and
//   dW1[j][k] += sum_r dh[j][r] x_r[k]      (SS: A = dh^T, B = x^T tile, M = 128 units)
// accumulates in TMEM, drained every kRDrain tiles into the per-CTA record.
// FAST precision only (x and dh rounded once to tf32, forward hi(W) x + lo(W) x);
// rows arrive as 128-row tiles built once per call by btr_pack_kernel:
//   forward A  [k/4][r/8][r%8][k%4]   (LBO 2048 B, SBO 128 B; 9 chunks stored, 18 KB)
//   backward B [f/8][r/4][f%8][r%4]   (LBO 128 B, SBO 4096 B; features < 40, 20 KB)
constexpr int kRR = 128;                      // rows per tile (forward M)
constexpr int kRXF = kFC * kRR / 8 * 128;     // smem bytes, forward operand (20 KB)
constexpr int kRXT = kNB / 8 * kRR / 4 * 128;  // smem bytes, backward operand (24 KB)
constexpr int kRXFG = kFCS * kRR / 8 * 128;   // global bytes, forward operand (18 KB)
constexpr int kRXTG = kNBS / 8 * kRR / 4 * 128;  // global bytes, backward operand (20 KB)
constexpr int kRGT = kRXFG + kRXTG;           // global bytes per tile
#ifndef GLX_BTR_RS
#define GLX_BTR_RS 2  // operand ring stages (3: 0.112 ms per 1M rows at H = 33, 2: 0.106)
#endif
#ifndef GLX_BTR_NB
#define GLX_BTR_NB 2  // dh^T buffers (tile lt uses buffer lt % NB and waits for backward(lt - NB))
#endif
constexpr int kRNB = GLX_BTR_NB;
constexpr int kRS = GLX_BTR_RS;                        // stages of each ring: forward operands (freed by the
                                              // forward MMA) and backward operands (freed by the backward)
constexpr int kRZB = 3;                       // Z buffers (forward kRZB tiles ahead)
// epilogue groups of 4 warps on alternate tiles: 3 (registers: h and the dW2 partials
// are 2 HP per thread), 2 for HP = 64
__host__ __device__ constexpr int btr_groups(int HP) { return HP <= 48 ? 3 : 2; }
// dW1 drain period (a multiple of the group count: group 0's tiles); a drain holds up the
// dh^T hand-off chain for its global read-modify-write, so it is rare: 48 tiles = 6144
// rows per TMEM fp32 partial
constexpr int kRDrain = 48;
constexpr int kRColW = 256;                   // dW1 accumulator columns (48)
constexpr int kRColA = 304;                   // dW2 partials, HP columns per epilogue group
#ifndef GLX_BTR_ACC_TMEM
#define GLX_BTR_ACC_TMEM 1
#endif
__host__ __device__ constexpr int btr_threads(int HP) { return (2 + 4 * btr_groups(HP)) * 32; }

template <int HP>
struct BtrSmem {  // byte offsets
    static constexpr int wt = HP / 8 * kFC * 128;       // one W1 copy (hi or lo): [j/8][k/4][j%8][k%4]
    static constexpr int w = 0;
    static constexpr int x = 1024 * ((2 * wt + 1023) / 1024);
    // dh^T, two buffers of 4 planes x 64 unit-rows x 128 B (1024-aligned swizzle atoms). The
    // backward MMA reads M = 128 unit-rows per plane; rows >= 64 fall in the next plane /
    // buffer / the backward ring (valid shared memory; their D rows are units >= HP, which
    // the drain never reads)
    static constexpr int dh = x + kRS * kRXF;
    static constexpr int xt = dh + kRNB * 4 * 8192;     // backward-operand ring
    static constexpr int w2 = xt + kRS * kRXT;          // w2s (HP floats), b2s
    static constexpr int red = w2 + (HP + 4) * 4;        // final reductions: [warps][HP + 8]
    static constexpr int bars = red + 4 * btr_groups(HP) * (HP + 8) * 4;
    static constexpr int total = bars + 256;
};

#ifdef GLX_BTR_TIMING
__device__ unsigned long long g_btr_dbg[4096];
// clock64 timeline of CTA 0, tiles 6..37: slot s of tile t at [(t - 6) * 8 + s] (per-tile
// slots: 0 epilogue start, 1 Z loaded, 2 deltas computed, 3 dh buffer free, 4 dh_ready
// arrived (warp 2); 5 MMA saw dh_ready, 6 backward issued (warp 1); 7 tile loaded (warp 0))
#define BTR_T(slot, lt)                                                                                     \
    do {                                                                                                    \
        if (blockIdx.x == 0 && lane == 0 && (lt) >= 6 && (lt) < 38) g_btr_dbg[((lt) - 6) * 8 + (slot)] = clock64(); \
    } while (0)
#else
#define BTR_T(slot, lt) \
    do {                \
    } while (0)
#endif
#ifdef GLX_BTR_DEBUG
// diagnostic builds: a bounded wait that reports which barrier never completed
__device__ __forceinline__ void btr_wait(uint64_t* bar, uint32_t parity, int tag, int64_t lt) {
    uint32_t ok = 0;
    const long long t0 = clock64();
    while (!ok && clock64() - t0 < 4000000000ll)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (!ok) {
        printf("btr hang: block %d warp %d lane %d tag %d lt %lld parity %u\n", blockIdx.x, threadIdx.x / 32,
               threadIdx.x % 32, tag, (long long)lt, parity);
        __trap();
    }
}
#define BTR_WAIT(bar, par, tag, lt) btr_wait(bar, par, tag, lt)
#else
#define BTR_WAIT(bar, par, tag, lt) mbar_wait(bar, par)
#endif

// HE: units the epilogue computes (H rounded up to even; HP = H padded to the MMA's N
// granularity of 16). The padded units HE .. HP - 1 have zero weights: their dh^T rows
// stay zero and their dW2 partials are never formed.
template <int HP, int HE = HP>
__global__ void __launch_bounds__(btr_threads(HP), 1) batchrt_kernel(const BtcArgs a) {
    static_assert(HE % 2 == 0 && HE <= HP && (HE % 16 == 0 || HE % 16 == 2), "epilogue width");
    using L = BtrSmem<HP>;
    constexpr int kRG = btr_groups(HP);
    static_assert(kRDrain % kRG == 0, "the drained tiles must all belong to group 0");
    static_assert(kRNB <= kRG, "dh_free slots alias beyond one dh buffer per group (hangs at HP = 64 with 3 buffers)");
    static_assert(kRColA + HP * kRG <= (int)kTmemCols, "dW2 partial columns");
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::bars);
    uint64_t* x_full = bars;            // forward operand of a tile loaded
    uint64_t* x_empty = x_full + kRS;   // forward-operand stage free (its forward completed)
    uint64_t* t_full = x_empty + kRS;   // backward operand of a tile loaded
    uint64_t* t_empty = t_full + kRS;   // backward-operand stage free (its backward completed)
    uint64_t* z_full = t_empty + kRS;   // Z buffer written by the forward
    uint64_t* z_free = z_full + kRZB;   // Z buffer read by the epilogue
    // dh_ready[lt % 2]: tile lt's dh^T is in buffer lt % 2 (4 warps); per buffer, since the
    // next tile's group may arrive before the MMA warp consumed this tile's phase
    uint64_t* dh_ready = z_free + kRZB;
    // dh_free[k % kRG]: backward(k) completed. Tile lt waits for backward(lt - 2) (the last
    // reader of its buffer); its group knows backward(lt - 2 - kRG) completed (its own
    // previous tile waited for it), so with kRG slots the barrier is never two phases behind
    uint64_t* dh_free = dh_ready + kRNB;
    uint64_t* fin_bar = dh_free + kRG;  // the last backward completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin_bar + 1);
    float* w2s = reinterpret_cast<float*>(sm + L::w2);
    float* red = reinterpret_cast<float*>(sm + L::red);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nt = (a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int D = a.D, DP = a.DP, H = a.H;
    float* out = a.part + (int64_t)blockIdx.x * a.PS;
    // checker slots: forward stage [0, kRS) and its release [4, 4 + kRS), backward stage
    // [8, 8 + kRS) and its release [12, 12 + kRS), Z buffer [16, 16 + kRZB) and its
    // release [20, 20 + kRZB), dh^T buffer [24, 26), backward completion [28, 28 + kRG)
    const DbgView dv = dbg_view(a.dbg, a.ntiles);
#ifdef GLX_BTR_DEBUG
    if (blockIdx.x == 0 && threadIdx.x == 0) printf("btr start: nt %lld N %lld D %d H %d HP %d\n", (long long)nt, (long long)a.N, D, H, HP);
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < kRS; i++) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_empty[i], 1);
            mbar_init(&t_full[i], 1);
            mbar_init(&t_empty[i], 1);
        }
        for (int b = 0; b < kRZB; b++) {
            mbar_init(&z_full[b], 1);
            mbar_init(&z_free[b], 4);
        }
        for (int b = 0; b < kRNB; b++) mbar_init(&dh_ready[b], 4);
        for (int b = 0; b < kRG; b++) mbar_init(&dh_free[b], 1);
        mbar_init(fin_bar, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // W1 (B operand of the forward: N = HP units, K = 40) as tf32 hi + lo; units >= H zero
    for (int e = threadIdx.x; e < HP * kFC; e += blockDim.x) {
        const int j = e / kFC, q = e - (e / kFC) * kFC;
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int k = 4 * q + i;
            v[i] = (k <= D && j < H) ? a.Wk[(int64_t)j * DP + k] : 0.f;
        }
        const int off = (j >> 3) * (kFC * 128) + q * 128 + (j & 7) * 16;
        uint4 hi, lo;
        hi.x = tf32_rn(v[0]);
        hi.y = tf32_rn(v[1]);
        hi.z = tf32_rn(v[2]);
        hi.w = tf32_rn(v[3]);
        lo.x = __float_as_uint(v[0] - __uint_as_float(hi.x));
        lo.y = __float_as_uint(v[1] - __uint_as_float(hi.y));
        lo.z = __float_as_uint(v[2] - __uint_as_float(hi.z));
        lo.w = __float_as_uint(v[3] - __uint_as_float(hi.w));
        *reinterpret_cast<uint4*>(sm + L::w + off) = hi;
        *reinterpret_cast<uint4*>(sm + L::w + L::wt + off) = lo;
    }
    for (int j = threadIdx.x; j < HP + 4; j += blockDim.x)
        w2s[j] = j < H ? a.Wk[(int64_t)H * DP + j] : (j == HP ? a.Wk[(int64_t)H * DP + H] : 0.f);
    // zero: the padding regions of every stage, the dh^T operand (units >= HP stay zero),
    // and this CTA's dW1 record (the drains accumulate into it)
    for (int i = threadIdx.x; i < kRS * (kRXF - kRXFG + kRXT - kRXTG) / 16; i += blockDim.x) {
        const int per = (kRXF - kRXFG + kRXT - kRXTG) / 16, st = i / per, w = i - (i / per) * per;
        unsigned char* dst = w < (kRXF - kRXFG) / 16 ? sm + L::x + st * kRXF + kRXFG + 16 * w
                                                      : sm + L::xt + st * kRXT + kRXTG + 16 * (w - (kRXF - kRXFG) / 16);
        *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
    }
    for (int i = threadIdx.x; i < kRNB * 4 * 8192 / 16; i += blockDim.x)  // units HP..63 stay zero
        reinterpret_cast<uint4*>(sm + L::dh)[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = threadIdx.x; i < a.P1; i += blockDim.x) out[i] = 0.f;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        // the forward operand of tile lt as soon as its stage frees (forward(lt - kRS) done);
        // the backward operand of tile lt - 2 behind it (needed a few tiles later, by
        // backward(lt - 2); its stage freed by backward(lt - 2 - kRS), long done)
        if (lane == 0) {
            auto load_t = [&](int64_t k) {
                const int ts = (int)(k % kRS);
                if (k >= kRS) {
                    BTR_WAIT(&t_empty[ts], (uint32_t)((k / kRS) - 1) & 1, 8, k);
                    if (GLX_DBG_ON(a)) dbg_expect(dv, 11, 12 + ts, k - kRS);
                }
                const unsigned char* src = a.tiles + (blockIdx.x + k * gridDim.x) * (int64_t)kRGT + kRXFG;
                if (GLX_DBG_ON(a)) dbg_put(dv, 8 + ts, k);
                mbar_arrive_expect_tx(&t_full[ts], (uint32_t)kRXTG);
                bulk_g2s(sm + L::xt + ts * kRXT, src, kRXTG, &t_full[ts]);
            };
            for (int64_t lt = 0; lt < nt; lt++) {
                const int xs = (int)(lt % kRS);
                if (lt >= kRS) {
                    BTR_WAIT(&x_empty[xs], (uint32_t)((lt / kRS) - 1) & 1, 1, lt);
                    if (GLX_DBG_ON(a)) dbg_expect(dv, 12, 4 + xs, lt - kRS);
                }
                const unsigned char* src = a.tiles + (blockIdx.x + lt * gridDim.x) * (int64_t)kRGT;
                if (GLX_DBG_ON(a)) dbg_put_load(dv, xs, lt);
                mbar_arrive_expect_tx(&x_full[xs], (uint32_t)kRXFG);
                bulk_g2s(sm + L::x + xs * kRXF, src, kRXFG, &x_full[xs]);
                BTR_T(7, lt);
                if (lt >= 2) load_t(lt - 2);
            }
            for (int64_t k = nt >= 2 ? nt - 2 : 0; k < nt; k++) load_t(k);
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t el = elect_one();
        constexpr uint32_t idf = idesc_tf32(HP, false);   // M = 128 rows, N = HP units
        constexpr uint32_t idb = idesc_tf32(kNB, false);  // M = 128 units, N = 48 features
        const uint64_t dwh = desc_ns(smem_u32(sm + L::w), 128, kFC * 128);
        const uint64_t dwl = desc_ns(smem_u32(sm + L::w + L::wt), 128, kFC * 128);
        const uint64_t dx0 = desc_ns(smem_u32(sm + L::x), kRR / 8 * 128, 128);
        const uint64_t dt0 = desc_ns(smem_u32(sm + L::xt), 128, kRR / 4 * 128);
        // dh^T: 128-byte-swizzled K-major (4 planes of 32 rows x 128 units, atoms 1 KB)
        const uint64_t dd0 = (uint64_t)((smem_u32(sm + L::dh) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
                             ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        auto forward = [&](int64_t lt) {
            const int xs = (int)(lt % kRS), zb = (int)(lt % kRZB);
            BTR_WAIT(&x_full[xs], (uint32_t)(lt / kRS) & 1, 2, lt);
            tc_fence_after();
            if (GLX_DBG_ON(a) && el) {
                dbg_expect(dv, 13, xs, lt);
                atomicAdd(&dv.vf[blockIdx.x + lt * gridDim.x], 1);
                dbg_put(dv, 4 + xs, lt);
                dbg_put(dv, 16 + zb, lt);
            }
            const uint32_t d = tmem + HP * zb;
            const uint64_t dx = dx0 + ((xs * kRXF) >> 4);
#pragma unroll
            for (int s = 0; s < kFC / 2; s++) mma_ss(d, dx + (s * 4096 >> 4), dwl + (s * 256 >> 4), idf, s != 0, el);
#pragma unroll
            for (int s = 0; s < kFC / 2; s++) mma_ss(d, dx + (s * 4096 >> 4), dwh + (s * 256 >> 4), idf, 1, el);
            commit(&x_empty[xs], el);
            commit(&z_full[zb], el);
        };
        auto backward = [&](int64_t lt) {
            const int ts = (int)(lt % kRS);
            BTR_WAIT(&dh_ready[lt % kRNB], (uint32_t)(lt / kRNB) & 1, 3, lt);
            BTR_WAIT(&t_full[ts], (uint32_t)(lt / kRS) & 1, 9, lt);
            tc_fence_after();
            if (GLX_DBG_ON(a) && el) {
                dbg_expect(dv, 14, 24 + (int)(lt % kRNB), lt);
                dbg_expect(dv, 15, 8 + ts, lt);
                dbg_put(dv, 12 + ts, lt);
                dbg_put(dv, 28 + (int)(lt % kRG), lt);
            }
            BTR_T(5, lt);
            const uint64_t dt = dt0 + ((ts * kRXT) >> 4);
#pragma unroll
            for (int c = 0; c < 4; c++) {
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    const uint32_t acc = (lt % kRDrain) != 0 || c != 0 || kk != 0;
                    mma_ss(tmem + kRColW, dd0 + (((int)(lt % kRNB) * 32768 + c * 8192 + kk * 32) >> 4),
                           dt + (((4 * c + kk) * 256) >> 4), idb, acc, el);
                }
            }
            commit(&t_empty[ts], el);
            commit(&dh_free[lt % kRG], el);
            if (lt == nt - 1) commit(fin_bar, el);
            BTR_T(6, lt);
        };
        for (int64_t lt = 0; lt < kRZB && lt < nt; lt++) forward(lt);
        for (int64_t lt = 0; lt < nt; lt++) {
            backward(lt);
            if (lt + kRZB < nt) {
                BTR_WAIT(&z_free[lt % kRZB], (uint32_t)(lt / kRZB) & 1, 4, lt);  // the epilogue read Z(lt)
                if (GLX_DBG_ON(a) && el) dbg_expect(dv, 16, 20 + (int)(lt % kRZB), lt);
                forward(lt + kRZB);
            }
        }
#ifdef GLX_BTR_DEBUG
        if (blockIdx.x == 0 && lane == 0) printf("btr mma: all %lld backwards issued\n", (long long)nt);
#endif
    } else {
        // ------------------------------------------------------------ epilogue
        // group gi (4 warps) takes tiles gi, gi + kRG, ...; warp quadrant q -> rows 32 q ..
        const int ew = warp - 2, gi = ew / 4, quad = warp & 3;
        const int r = quad * 32 + lane;  // this thread's row within the tile
        const uint32_t lanebase = (uint32_t)(quad * 32) << 16;
        const int tk = D + 1;            // the target travels as feature D + 1
        // its word in the tile's forward operand in global memory: [k/4][r/8][r%8][k%4]
        const int twd = (((tk >> 2) * 16 + (r >> 3)) * 8 + (r & 7)) * 4 + (tk & 3);
        const float b2s = w2s[HP];
#if GLX_BTR_ACC_TMEM
        // dW2 partials of this thread's row slot in TMEM (columns kRColA + HP gi ..), not
        // registers: held across the whole tile loop they pushed the row statistics and
        // themselves into local memory
        const uint32_t acol = tmem + lanebase + kRColA + HP * gi;
        {
            uint32_t z[16];
#pragma unroll
            for (int i = 0; i < 16; i++) z[i] = 0u;
#pragma unroll
            for (int c = 0; c < HP; c += 16) st16(acol + c, z);
            tmem_st_wait();
        }
#else
        float acc2[HP];
#pragma unroll
        for (int j = 0; j < HP; j++) acc2[j] = 0.f;
#endif
        float dsum = 0.f, loss = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        // dW1 drain: the TMEM accumulator (lanes = units) added into the per-CTA record by
        // the warps whose quadrant holds units (unit j = lane of quadrant j / 32)
        auto drain = [&]() {
            const int j = quad * 32 + lane;
            if (quad * 32 < HP) {
                uint32_t v0[32], v1[2];
                ld32(tmem + lanebase + kRColW, v0);
                ld2(tmem + lanebase + kRColW + 32, v1);
                tmem_ld_wait();
                if (j < H) {
                    float* o1 = out + (int64_t)j * (D + 1);
                    float cur[34];
#pragma unroll
                    for (int k = 0; k < 34; k++) cur[k] = k <= D ? o1[k] : 0.f;  // all loads in flight
#pragma unroll
                    for (int k = 0; k < 34; k++)
                        if (k <= D) o1[k] = cur[k] + __uint_as_float(k < 32 ? v0[k] : v1[k - 32]);
                }
            }
        };
        for (int64_t lt = gi; lt < nt; lt += kRG) {
            const int zb = (int)(lt % kRZB);
            const int64_t row = (blockIdx.x + lt * gridDim.x) * kRR + r;
            // the target, read early from global memory (the tile's smem stages are freed
            // by the MMAs before this epilogue needs it)
            const float tt = __ldg(reinterpret_cast<const float*>(a.tiles + (blockIdx.x + lt * gridDim.x) * (int64_t)kRGT) + twd);
            if (quad == 2) BTR_T(0, lt);
            BTR_WAIT(&z_full[zb], (uint32_t)(lt / kRZB) & 1, 5, lt);
            tc_fence_after();
            if (GLX_DBG_ON(a) && lane == 0) dbg_expect(dv, 17, 16 + zb, lt);
            float h[HE];
            {
                uint32_t v[32];
#pragma unroll
                for (int c = 0; c < HE; c += 32) {
                    if (HE - c >= 32) {
                        ld32(tmem + lanebase + HP * zb + c, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; i++) h[c + i] = __uint_as_float(v[i]);
                    } else if (HE - c >= 16) {
                        uint32_t v16[16];
                        ld16(tmem + lanebase + HP * zb + c, v16);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; i++) h[c + i] = __uint_as_float(v16[i]);
                    } else {
                        uint32_t v2[2];
                        ld2(tmem + lanebase + HP * zb + c, v2);
                        tmem_ld_wait();
                        h[c] = __uint_as_float(v2[0]);
                        h[c + 1] = __uint_as_float(v2[1]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (GLX_DBG_ON(a) && lane == 0) dbg_put(dv, 20 + zb, lt);
            if (lane == 0) mbar_arrive(&z_free[zb]);
            if (quad == 2) BTR_T(1, lt);
            // h = sigmoid(z) (z prescaled by -log2 e), one reciprocal per pair
#pragma unroll
            for (int i = 0; i < HE; i += 2) {
                const float2 e2 = make_float2(ex2_approx(h[i]), ex2_approx(h[i + 1]));
                const float2 den = __fadd2_rn(fminf2(e2, bcast2(1.152921504606847e18f)), bcast2(1.0f));
                const float rc = rcp_approx(den.x * den.y);
                const float2 hh = __fmul2_rn(make_float2(den.y, den.x), bcast2(rc));
                h[i] = hh.x;
                h[i + 1] = hh.y;
            }
            // the output neuron: a per-thread dot (w2s prescaled by -log2 e)
            float2 zo2 = make_float2(0.f, 0.f);
            if constexpr (HE % 4 == 0) {
#pragma unroll
                for (int i = 0; i < HE; i += 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(w2s + i);
                    zo2 = ffma2(make_float2(w4.x, w4.y), make_float2(h[i], h[i + 1]), zo2);
                    zo2 = ffma2(make_float2(w4.z, w4.w), make_float2(h[i + 2], h[i + 3]), zo2);
                }
            } else {
#pragma unroll
                for (int i = 0; i < HE; i += 2)
                    zo2 = ffma2(*reinterpret_cast<const float2*>(w2s + i), make_float2(h[i], h[i + 1]), zo2);
            }
            float d = 0.f;
            if (row < a.N) {
                const float o = sigmoid_scaled(zo2.x + zo2.y + b2s);
                d = (o - tt) * o * (1.0f - o);
                loss = fmaf(0.5f * (tt - o), tt - o, loss);
                const bool pred = o >= 0.5f, pos = tt >= 0.5f;
                c0 += (pred && pos) ? 1.f : 0.f;
                c1 += (!pred && !pos) ? 1.f : 0.f;
                c2 += (pred && !pos) ? 1.f : 0.f;
                c3 += (!pred && pos) ? 1.f : 0.f;
                dsum += d;
            }
            // dW2 += delta_o h; dh = delta_o h (1 - h) -> tf32 (h reused as dh)
#if GLX_BTR_ACC_TMEM
#pragma unroll
            for (int c = 0; c < HE; c += 16) {
                uint32_t av[16];
                if (HE - c >= 16) ld16(acol + c, av);
                else ld2(acol + c, reinterpret_cast<uint32_t(&)[2]>(av));
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < (HE - c >= 16 ? 16 : HE - c); i += 2) {
                    const float2 hp = make_float2(h[c + i], h[c + i + 1]);
                    const float2 v = __fmul2_rn(bcast2(d), hp);
                    const float2 a2 = __fadd2_rn(make_float2(__uint_as_float(av[i]), __uint_as_float(av[i + 1])), v);
                    av[i] = __float_as_uint(a2.x);
                    av[i + 1] = __float_as_uint(a2.y);
                    const float2 s2 = ffma2(make_float2(-v.x, -v.y), hp, v);
                    h[c + i] = __uint_as_float(tf32_rn(s2.x));
                    h[c + i + 1] = __uint_as_float(tf32_rn(s2.y));
                }
                if (HE - c >= 16) st16(acol + c, av);
                else st2(acol + c, reinterpret_cast<const uint32_t(&)[2]>(av));
            }
            tmem_st_wait();  // the next tile's loads of these columns follow the stores
#else
#pragma unroll
            for (int i = 0; i < HP; i += 2) {
                const float2 hp = make_float2(h[i], h[i + 1]);
                const float2 v = __fmul2_rn(bcast2(d), hp);
                const float2 a2 = __fadd2_rn(make_float2(acc2[i], acc2[i + 1]), v);
                acc2[i] = a2.x;
                acc2[i + 1] = a2.y;
                const float2 s2 = ffma2(make_float2(-v.x, -v.y), hp, v);
                h[i] = __uint_as_float(tf32_rn(s2.x));
                h[i + 1] = __uint_as_float(tf32_rn(s2.y));
            }
#endif
            if (quad == 2) BTR_T(2, lt);
            // dh^T buffer lt % 2: backward(lt - 2) read it last. A drain tile also needs
            // backward(lt - 1) (the end of the accumulation it takes)
            if (lt >= kRNB) {
                BTR_WAIT(&dh_free[(lt - kRNB) % kRG], (uint32_t)((lt - kRNB) / kRG) & 1, 6, lt);
                tc_fence_after();
                if (GLX_DBG_ON(a) && lane == 0) dbg_expect(dv, 18, 28 + (int)((lt - kRNB) % kRG), lt - kRNB);
            }
            if (quad == 2) BTR_T(3, lt);
            if (lt >= 1 && lt % kRDrain == 0) {  // group 0's tile: the backward of lt restarts
                BTR_WAIT(&dh_free[(lt - 1) % kRG], (uint32_t)((lt - 1) / kRG) & 1, 6, lt);
                tc_fence_after();
                drain();
            }
            {
                unsigned char* plane = sm + L::dh + (int)(lt % kRNB) * 32768 + quad * 8192;
#pragma unroll
                for (int j = 0; j < HE; j++)
                    *reinterpret_cast<float*>(plane + (j >> 3) * 1024 + (j & 7) * 128 +
                                              ((((lane >> 2) ^ (j & 7))) << 4) + (lane & 3) * 4) = h[j];
            }
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (GLX_DBG_ON(a) && lane == 0) {
                dbg_put(dv, 24 + (int)(lt % kRNB), lt);
                atomicAdd(&dv.vb[blockIdx.x + lt * gridDim.x], 1);  // one per row quadrant
            }
            if (lane == 0) mbar_arrive(&dh_ready[lt % kRNB]);
            if (quad == 2) BTR_T(4, lt);
        }
        // ---------------------------------------------- per-CTA partial record
        if (gi == 0) {
#ifdef GLX_BTR_DEBUG
            BTR_WAIT(&dh_free[(nt - 1) % kRG], (uint32_t)((nt - 1) / kRG) & 1, 8, nt);
#endif
            BTR_WAIT(fin_bar, 0, 7, nt);
            tc_fence_after();
            drain();  // tiles since the last drain
        }
        // dW2 and the statistics: warp sums, then a fixed-order sum over the warps
        float* slot = red + ew * (HP + 8);
#if GLX_BTR_ACC_TMEM
        float acc2[HP];
#pragma unroll
        for (int c = 0; c < HP; c += 16) {
            uint32_t av[16];
            ld16(acol + c, av);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; i++) acc2[c + i] = __uint_as_float(av[i]);
        }
#endif
#pragma unroll
        for (int j = 0; j < HP; j++) {
            float v = acc2[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) slot[j] = v;
        }
        float st[6] = {loss, c0, c1, c2, c3, dsum};
#pragma unroll
        for (int q = 0; q < 6; q++) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) st[q] += __shfl_xor_sync(0xffffffffu, st[q], o);
            if (lane == 0) slot[HP + q] = st[q];
        }
        bar_sync(kEpiBar, 4 * kRG * 32);
        const int et = ew * 32 + lane;
        if (et < HP + 6) {
            float sum = 0.f;
            for (int w = 0; w < 4 * kRG; w++) sum += red[w * (HP + 8) + et];
            if (et < H) out[a.P1 + et] = sum;
            else if (et == HP + 5) out[a.P1 + H] = sum;                   // dsum
            else if (et >= HP && et < HP + 5) out[a.P1 + H + 1 + (et - HP)] = sum;  // loss, counts
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// rows -> 128-row tiles in the two operand layouts of batchrt_kernel (tf32, round to nearest)
__global__ void __launch_bounds__(256) btr_pack_kernel(const float* __restrict__ Xp, int64_t N, int LD,
                                                       unsigned char* __restrict__ tiles) {
    __shared__ float t[kRR * 37];
    const int64_t tile = blockIdx.x;
    const int64_t row0 = tile * kRR;
    const int nr = (int)((N - row0) < kRR ? (N - row0) : kRR);
    for (int e = threadIdx.x; e < kRR * 36; e += blockDim.x) {
        const int rr = e / 36, k = e - (e / 36) * 36;
        t[rr * 37 + k] = (rr < nr && k < LD) ? Xp[(row0 + rr) * LD + k] : 0.f;
    }
    __syncthreads();
    uint32_t* out = reinterpret_cast<uint32_t*>(tiles + tile * (int64_t)kRGT);
    // forward: word w = ((q * 16 + r / 8) * 8 + r % 8) * 4 + k % 4, k = 4 q + k % 4
    for (int w = threadIdx.x; w < kRXFG / 4; w += blockDim.x) {
        const int e = w & 3, ro = (w >> 2) & 7, r8 = (w >> 5) & 15, q = w >> 9;
        out[w] = tf32_rn(t[(r8 * 8 + ro) * 37 + 4 * q + e]);
    }
    // backward: word w = ((fb * 32 + r / 4) * 8 + f % 8) * 4 + r % 4, f = 8 fb + f % 8
    for (int w = threadIdx.x; w < kRXTG / 4; w += blockDim.x) {
        const int r4 = w & 3, f8 = (w >> 2) & 7, rq = (w >> 5) & 31, fb = w >> 10;
        const int f = fb * 8 + f8;
        out[kRXFG / 4 + w] = tf32_rn(f < 36 ? t[(rq * 4 + r4) * 37 + f] : 0.f);
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
#ifdef GLX_BTR_TIMING
}  // namespace
}  // namespace glx
extern "C" void glx_btr_timing_dump(void) {
    unsigned long long h[4096];
    cudaMemcpyFromSymbol(h, glx::g_btr_dbg, sizeof(h));
    auto at = [&](int t, int s) { return (long long)h[t * 8 + s]; };
    const long long t0 = at(0, 0);
    for (int t = 0; t < 32; t++)
        printf("lt %2d epi @%7lld z %5lld sig %5lld free %5lld dhw %5lld | mma ready @%7lld issue %4lld | load @%7lld\n",
               t + 6, at(t, 0) - t0, at(t, 1) - at(t, 0), at(t, 2) - at(t, 1), at(t, 3) - at(t, 2), at(t, 4) - at(t, 3),
               at(t, 5) - t0, at(t, 6) - at(t, 5), at(t, 7) - t0);
}
namespace glx {
namespace {
#endif
#ifdef GLX_BTC_TIMING
}  // namespace
}  // namespace glx
extern "C" void glx_btc_timing_dump(void) {
    unsigned long long h[4096];
    cudaMemcpyFromSymbol(h, glx::g_btc_dbg, sizeof(h));
    auto at = [&](int t, int slot, int w) { return (long long)h[((t * 16) + slot) * 4 + w]; };
    const long long t0 = at(0, 0, 0);
    // epilogue slots 0-7 (rb0: warp 4, rb1: warp 12), MMA slots 8-13 (8-10 backward of tile
    // t, 11-13 forward of tile t), producer slots 14-15; times relative to tile 8's start
    for (int t = 0; t < 16; t++) {
        printf("lt %2d", t + 8);
        for (int w : {0, 2}) {
            printf(" | rb%d @%7lld z %4lld tok %4lld sig %4lld red %4lld bar %4lld rows %4lld p2 %4lld", w / 2,
                   at(t, 0, w) - t0, at(t, 1, w) - at(t, 0, w), at(t, 5, w) - at(t, 1, w), at(t, 6, w) - at(t, 5, w),
                   at(t, 2, w) - at(t, 6, w), at(t, 3, w) - at(t, 2, w), at(t, 4, w) - at(t, 3, w),
                   at(t, 7, w) - at(t, 4, w));
        }
        printf(" | mma bwd: wait %5lld @%7lld issue %4lld | fwd: wait %5lld @%7lld issue %4lld | load @%7lld %5lld\n",
               at(t, 9, 1) - at(t, 8, 1), at(t, 9, 1) - t0, at(t, 10, 1) - at(t, 9, 1), at(t, 12, 1) - at(t, 11, 1),
               at(t, 12, 1) - t0, at(t, 13, 1) - at(t, 12, 1), at(t, 14, 3) - t0, at(t, 15, 3) - at(t, 14, 3));
    }
}
namespace glx {
namespace {
#endif

}  // namespace

bool batchtc_geometry(int64_t N, int D, int H, int n_sms, BatchGeom* out) {
    if (N < 1 || D < 1 || D > 33 || H < 1 || H > 256) return false;
    BatchGeom g{};
    g.D = D;
    g.H = H;
    g.N = N;
    g.DP = D + 1 <= 8 ? 8 : D + 1 <= 16 ? 16 : 34;
    g.LD = a4(std::max(D + 2, g.DP));
    if (g.LD > 36) return false;
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
    const int nh = (H + 127) / 128;
    g.smem = (size_t)(g.MT ? btc_smem<true>(nh).total : btc_smem<false>(nh).total);
    *out = g;
    return true;
}

// narrow layers (rows on the lanes): FAST precision, D <= 33, H <= 64
bool batchrt_geometry(int64_t N, int D, int H, int n_sms, BatchGeom* out) {
    if (N < btc_full_rows() || N < 1 || D < 1 || D > 33 || H < 1 || H > 64) return false;
    BatchGeom g{};
    g.D = D;
    g.H = H;
    g.N = N;
    g.DP = D + 1 <= 8 ? 8 : D + 1 <= 16 ? 16 : 34;
    g.LD = a4(std::max(D + 2, g.DP));
    if (g.LD > 36) return false;
    g.HP = H <= 32 ? 32 : H <= 48 ? 48 : 64;
    g.P1 = H * (D + 1);
    g.PS = a4(g.P1 + H + 6);
    g.WKS = a4(H * g.DP + 2 * H + 1);
    g.R = kRR;
    g.ntiles = (N + kRR - 1) / kRR;
    g.grid = (int)std::min<int64_t>(g.ntiles, n_sms);
    g.MT = 0;
    g.smem = g.HP == 32 ? BtrSmem<32>::total : g.HP == 48 ? BtrSmem<48>::total : BtrSmem<64>::total;
    *out = g;
    return true;
}

size_t batchrt_tile_bytes(const BatchGeom& g) { return (size_t)g.ntiles * kRGT; }

cudaError_t launch_batchrt_pack(const BatchGeom& g, const float* Xp, void* tiles, cudaStream_t st) {
    btr_pack_kernel<<<(unsigned)g.ntiles, 256, 0, st>>>(Xp, g.N, g.LD, (unsigned char*)tiles);
    return cudaGetLastError();
}

#ifndef GLX_BTR_NARROW34
#define GLX_BTR_NARROW34 1  // H <= 34 at HP = 48 (the reference's default H = 33): a 34-unit epilogue
#endif
template <int HP>
static cudaError_t launch_btr(const BatchGeom& g, const BtcArgs& a, cudaStream_t st) {
    auto k = (HP == 48 && GLX_BTR_NARROW34 && g.H <= 34) ? batchrt_kernel<HP, (HP == 48 ? 34 : HP)> : batchrt_kernel<HP>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) {
        fprintf(stderr, "glx: batchrt_kernel<%d> smem=%zu: %s\n", HP, g.smem, cudaGetErrorString(e));
        return e;
    }
    k<<<g.grid, btr_threads(HP), g.smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_batchrt_epoch(const BatchGeom& g, const void* tiles, const float* Wk, float* part,
                                 cudaStream_t st, int* dbg) {
    BtcArgs a;
    a.dbg = dbg;
    a.tiles = (const unsigned char*)tiles;
    a.Wk = Wk;
    a.part = part;
    a.N = g.N;
    a.ntiles = g.ntiles;
    a.D = g.D;
    a.DP = g.DP;
    a.H = g.H;
    a.P1 = g.P1;
    a.PS = g.PS;
    return g.HP == 32 ? launch_btr<32>(g, a, st) : g.HP == 48 ? launch_btr<48>(g, a, st) : launch_btr<64>(g, a, st);
}

template <int NH, bool FULL>
static cudaError_t launch_btc(const BatchGeom& g, const BtcArgs& a, cudaStream_t st) {
    auto k = a.dbg ? (g.H % 128 ? batchtc_kernel<NH, FULL, true, true> : batchtc_kernel<NH, FULL, false, true>)
                   : (g.H % 128 ? batchtc_kernel<NH, FULL, true, false> : batchtc_kernel<NH, FULL, false, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) {
        fprintf(stderr, "glx: batchtc_kernel<%d> smem=%zu: %s\n", NH, g.smem, cudaGetErrorString(e));
        return e;
    }
    k<<<g.grid, btc_threads(NH, FULL), g.smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "glx: batchtc_kernel<%d> launch: %s\n", NH, cudaGetErrorString(e));
    return e;
}

size_t pipeline_check_ints(const BatchGeom& g) { return kDbgHdr + 2 * (size_t)g.ntiles + (size_t)g.grid * kDbgCta; }

size_t batchtc_tile_bytes(const BatchGeom& g) {
    return (size_t)g.ntiles * (g.MT ? Pipe<true>::GTILE : Pipe<false>::GTILE);
}

cudaError_t launch_batchtc_pack(const BatchGeom& g, const float* Xp, void* tiles, cudaStream_t st) {
    if (g.MT) btc_pack_kernel<true><<<(unsigned)g.ntiles, 256, 0, st>>>(Xp, g.N, g.LD, (unsigned char*)tiles);
    else btc_pack_kernel<false><<<(unsigned)g.ntiles, 256, 0, st>>>(Xp, g.N, g.LD, (unsigned char*)tiles);
    return cudaGetLastError();
}

cudaError_t launch_batchtc_epoch(const BatchGeom& g, const void* tiles, const float* Wk, float* part, cudaStream_t st,
                                 int* dbg) {
    BtcArgs a;
    a.dbg = dbg;
    a.tiles = (const unsigned char*)tiles;
    a.Wk = Wk;
    a.part = part;
    a.N = g.N;
    a.ntiles = g.ntiles;
    a.D = g.D;
    a.DP = g.DP;
    a.H = g.H;
    a.P1 = g.P1;
    a.PS = g.PS;
    if (g.MT) return g.H > 128 ? launch_btc<2, true>(g, a, st) : launch_btc<1, true>(g, a, st);
    return g.H > 128 ? launch_btc<2, false>(g, a, st) : launch_btc<1, false>(g, a, st);
}

}  // namespace glx
