// glx_data.cu -- the data format on the input side of the training path:
// per-column min-max normalisation fitted on the training rows and applied to
// any split (reference dataset.py:369-398).
//
//   fit:   col_min[c] = min_r X[r][c], col_max[c] = max_r X[r][c]      (f32, exact)
//   apply: y = span != 0 ? clamp(f32(f32(x - min) / span), -0.5, 1.5) : 0,
//          span = f32(max - min)                                      (IEEE f32 ops)
//
// Both are single HBM passes (fit: 4 B read per element; apply: 4 B read +
// 4 B written). The main kernels are persistent (2 CTAs per SM) and stream the
// row-major matrix in contiguous row tiles of ~32 KB: 1-D bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a 3-stage shared ring, threads
// mapped to (column, row phase) so a warp reads consecutive shared words, and
// for apply a bulk store (cp.async.bulk shared -> global) of the transformed
// tile. The fit folds per-thread min/max over phases in shared memory and then
// across CTAs with integer atomics on an order-preserving float encoding (min
// and max are exact, so the result does not depend on the order). The ragged
// tail (< one tile) and unaligned inputs use plain loads. The apply step is
// also fused into the batch row packing (pack_rows_kernel, glx_batch.cu).
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>

namespace glx {

constexpr int kFitCols = 256;  // columns per grid.y slice (8 per thread)

// order-preserving int encoding of an f32 (its own inverse)
__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); }

__global__ void minmax_init_kernel(int* __restrict__ omin, int* __restrict__ omax, int D) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < D) {
        omin[c] = 0x7FFFFFFF;
        omax[c] = (int)0x80000000;
    }
}

__global__ void __launch_bounds__(256) minmax_fit_kernel(const float* __restrict__ X, int64_t N, int D,
                                                         int* __restrict__ omin, int* __restrict__ omax) {
    __shared__ float smn[8][kFitCols], smx[8][kFitCols];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c0 = blockIdx.y * kFitCols;
    float mn[8], mx[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        mn[k] = __int_as_float(0x7F800000);   // +inf
        mx[k] = __int_as_float((int)0xFF800000);  // -inf
    }
    for (int64_t r = (int64_t)blockIdx.x * 8 + ty; r < N; r += (int64_t)gridDim.x * 8) {
        const float* row = X + r * D;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const int c = c0 + tx + 32 * k;
            if (c < D) {
                const float v = __ldcs(row + c);
                mn[k] = fminf(mn[k], v);
                mx[k] = fmaxf(mx[k], v);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
        smn[ty][tx + 32 * k] = mn[k];
        smx[ty][tx + 32 * k] = mx[k];
    }
    __syncthreads();
    const int t = ty * 32 + tx;  // one thread per column of the slice
    const int c = c0 + t;
    if (c < D) {
        float a = smn[0][t], b = smx[0][t];
#pragma unroll
        for (int y = 1; y < 8; y++) {
            a = fminf(a, smn[y][t]);
            b = fmaxf(b, smx[y][t]);
        }
        atomicMin(omin + c, f2ord(a));
        atomicMax(omax + c, f2ord(b));
    }
}

__global__ void minmax_finish_kernel(const int* __restrict__ omin, const int* __restrict__ omax, int D,
                                     float* __restrict__ col_min, float* __restrict__ col_max) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < D) {
        col_min[c] = ord2f(omin[c]);
        col_max[c] = ord2f(omax[c]);
    }
}

// Y may alias X (in-place): each element is read and written by the same thread
__global__ void __launch_bounds__(256) minmax_apply_kernel(const float* X, int64_t N, int D,
                                                           const float* __restrict__ col_min,
                                                           const float* __restrict__ col_max, float* Y) {
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int64_t r = (int64_t)blockIdx.x * 8 + ty; r < N; r += (int64_t)gridDim.x * 8) {
        for (int c = tx; c < D; c += 32) Y[r * D + c] = minmax_norm(X[r * D + c], col_min[c], col_max[c]);
    }
}

constexpr int kNormStages = 3;
constexpr int kNormTileFloats = 8192;  // ~32 KB per tile
constexpr int kNormMaxColsPerThread = 8;  // tiled fit handles D <= 2048

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// rows per tile: a multiple of 4 so every tile starts 16-byte aligned
__host__ __device__ inline int norm_tile_rows(int D) {
    const int r = (kNormTileFloats / D) & ~3;
    return r < 4 ? 4 : r;
}

// thread -> (first column, row phase, phase count); D < 256: P = 256 / D phases
// of D threads (a warp reads consecutive words), else one phase with columns
// t, t + 256, ...
struct ColMap {
    int c, ph, P;
    bool active;
    __device__ ColMap(int t, int D) {
        if (D < 256) {
            P = 256 / D;
            active = t < P * D;
            c = t % D;
            ph = t / D;
        } else {
            P = 1;
            active = t < D;
            c = t;
            ph = 0;
        }
    }
};

template <bool APPLY>
__global__ void __launch_bounds__(256) minmax_tiled_kernel(const float* X, float* Y, int64_t N, int D,
                                                           const float* __restrict__ col_min,
                                                           const float* __restrict__ col_max, int* __restrict__ omin,
                                                           int* __restrict__ omax) {
    extern __shared__ __align__(128) unsigned char nsm[];
    const int R = norm_tile_rows(D);
    const int tile_floats = R * D;
    float* ring = reinterpret_cast<float*>(nsm);
    uint64_t* full = reinterpret_cast<uint64_t*>(nsm + (size_t)kNormStages * tile_floats * 4);
    const int t = threadIdx.x;
    const ColMap cm(t, D);
    const int64_t n_tiles = N / R;  // full tiles; the tail is done with plain loads
    if (t == 0) {
        for (int s = 0; s < kNormStages; s++) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    float mn[kNormMaxColsPerThread], mx[kNormMaxColsPerThread], lo[kNormMaxColsPerThread],
        hi[kNormMaxColsPerThread];
#pragma unroll
    for (int k = 0; k < kNormMaxColsPerThread; k++) {
        mn[k] = __int_as_float(0x7F800000);
        mx[k] = __int_as_float((int)0xFF800000);
        const int c = cm.c + 256 * k;
        if (APPLY && cm.active && c < D) {
            lo[k] = col_min[c];
            hi[k] = col_max[c];
        }
    }
    auto issue = [&](int64_t tile, int s) {
        const uint32_t bytes = (uint32_t)tile_floats * 4;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * tile_floats, X + tile * tile_floats, bytes, &full[s]);
    };
    if (t == 0) {
        int s = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles && s < kNormStages; tile += gridDim.x, s++) issue(tile, s);
    }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, it++) {
        const int s = it % kNormStages;
        mbar_wait(&full[s], (it / kNormStages) & 1);
        float* tp = ring + (size_t)s * tile_floats;
        if (cm.active && D < 256) {  // one column per thread: independent rows, unrolled
            float* e = tp + cm.ph * D + cm.c;
            const int stride = cm.P * D;
            const int nr = (R - cm.ph + cm.P - 1) / cm.P;
            int i = 0;
            for (; i + 4 <= nr; i += 4, e += 4 * stride) {
                float v0 = e[0], v1 = e[stride], v2 = e[2 * stride], v3 = e[3 * stride];
                if (APPLY) {
                    e[0] = minmax_norm(v0, lo[0], hi[0]);
                    e[stride] = minmax_norm(v1, lo[0], hi[0]);
                    e[2 * stride] = minmax_norm(v2, lo[0], hi[0]);
                    e[3 * stride] = minmax_norm(v3, lo[0], hi[0]);
                } else {
                    mn[0] = fminf(mn[0], fminf(fminf(v0, v1), fminf(v2, v3)));
                    mx[0] = fmaxf(mx[0], fmaxf(fmaxf(v0, v1), fmaxf(v2, v3)));
                }
            }
            for (; i < nr; i++, e += stride) {
                if (APPLY) {
                    *e = minmax_norm(*e, lo[0], hi[0]);
                } else {
                    mn[0] = fminf(mn[0], *e);
                    mx[0] = fmaxf(mx[0], *e);
                }
            }
        } else if (cm.active) {
            for (int r = cm.ph; r < R; r += cm.P) {
#pragma unroll
                for (int k = 0; k < kNormMaxColsPerThread; k++) {
                    const int c = cm.c + 256 * k;
                    if (c >= D) break;
                    float* e = tp + r * D + c;
                    if (APPLY) {
                        *e = minmax_norm(*e, lo[k], hi[k]);
                    } else {
                        mn[k] = fminf(mn[k], *e);
                        mx[k] = fmaxf(mx[k], *e);
                    }
                }
            }
        }
        if (APPLY) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            if (APPLY) {
                bulk_s2g(Y + tile * tile_floats, tp, (uint32_t)tile_floats * 4);
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot s is free again
            }
            const int64_t nxt = tile + (int64_t)kNormStages * gridDim.x;
            if (nxt < n_tiles) issue(nxt, s);
        }
    }
    // ragged tail (< R rows): the last CTA, straight from global memory
    if (blockIdx.x == gridDim.x - 1 && cm.active) {
        for (int64_t r = n_tiles * R + cm.ph; r < N; r += cm.P) {
#pragma unroll
            for (int k = 0; k < kNormMaxColsPerThread; k++) {
                const int c = cm.c + 256 * k;
                if (c >= D) break;
                const float v = X[r * D + c];
                if (APPLY) {
                    Y[r * D + c] = minmax_norm(v, lo[k], hi[k]);
                } else {
                    mn[k] = fminf(mn[k], v);
                    mx[k] = fmaxf(mx[k], v);
                }
            }
        }
    }
    if (APPLY) {
        if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    // fold the row phases in shared memory (the ring is free now), then across CTAs
    __syncthreads();
    float* smn = ring;
    float* smx = ring + 256 * kNormMaxColsPerThread;
    if (cm.active) {
#pragma unroll
        for (int k = 0; k < kNormMaxColsPerThread; k++) {
            smn[k * 256 + t] = mn[k];
            smx[k * 256 + t] = mx[k];
        }
    }
    __syncthreads();
    if (t < D && t < 256) {
        const int P = cm.P;
        for (int k = 0; k < kNormMaxColsPerThread && t + 256 * k < D; k++) {
            // thread (c, ph) stored at index ph * D + c for D < 256, else at c
            float a = smn[k * 256 + t], b = smx[k * 256 + t];
            for (int ph = 1; ph < P; ph++) {
                a = fminf(a, smn[k * 256 + ph * D + t]);
                b = fmaxf(b, smx[k * 256 + ph * D + t]);
            }
            atomicMin(omin + t + 256 * k, f2ord(a));
            atomicMax(omax + t + 256 * k, f2ord(b));
        }
    }
}

// rows per packing tile: ~32 KB of input + output per stage, a multiple of 16
// so the u8 label slice of a tile stays 16-byte aligned
__host__ __device__ inline int pack_tile_rows(int D, int LD) {
    const int r = (kNormTileFloats / (D + LD + 1)) & ~15;
    return r < 16 ? 16 : r;
}

// Batch row packing (glx_batch.cu layout [x_0..x_{D-1}, 1, target, 0..] of LD
// floats), optionally min-max normalising x: feature tiles arrive by bulk copy,
// the packed tile is built in shared memory by (packed column, row phase)
// threads and leaves by bulk store. Targets come from T (f32) or labels (u8).
__global__ void __launch_bounds__(256) pack_tiled_kernel(const float* __restrict__ X, const float* __restrict__ T,
                                                         const uint8_t* __restrict__ labels, int64_t N, int D, int LD,
                                                         const float* __restrict__ col_min,
                                                         const float* __restrict__ col_max, float* __restrict__ Xp) {
    extern __shared__ __align__(128) unsigned char nsm[];
    const int R = pack_tile_rows(D, LD);
    float* in_ring = reinterpret_cast<float*>(nsm);
    float* out_ring = in_ring + (size_t)kNormStages * R * D;
    float* tgt_ring = out_ring + (size_t)kNormStages * R * LD;  // R floats or R label bytes per stage
    uint64_t* full = reinterpret_cast<uint64_t*>(tgt_ring + (size_t)kNormStages * R);
    const int t = threadIdx.x;
    const ColMap cm(t, LD);
    const int64_t n_tiles = N / R;
    if (t == 0) {
        for (int s = 0; s < kNormStages; s++) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int i = cm.c;  // packed column of this thread (LD < 256 always: D <= 250)
    float lo = 0.f, hi = 0.f;
    if (col_min && cm.active && i < D) {
        lo = col_min[i];
        hi = col_max[i];
    }
    // the tile's features and its slice of targets (f32) or labels (u8) arrive on one barrier
    const uint32_t tbytes = T ? (uint32_t)R * 4 : labels ? (uint32_t)R : 0u;
    auto issue = [&](int64_t tile, int s) {
        const uint32_t bytes = (uint32_t)R * D * 4;
        mbar_arrive_expect_tx(&full[s], bytes + tbytes);
        bulk_g2s(in_ring + (size_t)s * R * D, X + tile * R * D, bytes, &full[s]);
        if (T) bulk_g2s(tgt_ring + (size_t)s * R, T + tile * R, tbytes, &full[s]);
        else if (labels) bulk_g2s(tgt_ring + (size_t)s * R, labels + tile * R, tbytes, &full[s]);
    };
    auto target = [&](const float* tg, int64_t r_local, int64_t r) -> float {  // tg: staged slice or null
        if (T) return tg ? tg[r_local] : T[r];
        if (labels) return tg ? (float)reinterpret_cast<const uint8_t*>(tg)[r_local] : (float)labels[r];
        return 0.0f;
    };
    auto value = [&](const float* xrow, const float* tg, int64_t r_local, int64_t r) -> float {
        if (i < D) return col_min ? minmax_norm(xrow[i], lo, hi) : xrow[i];
        if (i == D) return 1.0f;
        if (i == D + 1) return target(tg, r_local, r);
        return 0.0f;
    };
    if (t == 0) {
        int s = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles && s < kNormStages; tile += gridDim.x, s++) issue(tile, s);
    }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, it++) {
        const int s = it % kNormStages;
        mbar_wait(&full[s], (it / kNormStages) & 1);
        const float* ip = in_ring + (size_t)s * R * D;
        const float* tg = tgt_ring + (size_t)s * R;
        float* op = out_ring + (size_t)s * R * LD;
        if (cm.active) {
#pragma unroll 4
            for (int r = cm.ph; r < R; r += cm.P) op[r * LD + i] = value(ip + r * D, tg, r, tile * R + r);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // tile consumed: in slot s may be refilled, out slot s is complete
        if (t == 0) {
            bulk_s2g(Xp + tile * R * LD, op, (uint32_t)R * LD * 4);
            const int64_t nxt = tile + (int64_t)kNormStages * gridDim.x;
            if (nxt < n_tiles) issue(nxt, s);
            // the out slot written in iteration it + 2 is the one stored at it + 2 - S:
            // leave at most S - 2 stores pending, so it is free; the next
            // iteration's __syncthreads orders this wait before those writes
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kNormStages - 2) : "memory");
        }
    }
    if (blockIdx.x == gridDim.x - 1 && cm.active) {  // ragged tail from global memory
        for (int64_t r = n_tiles * R + cm.ph; r < N; r += cm.P) Xp[r * LD + i] = value(X + r * D, nullptr, 0, r);
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static size_t pack_smem(int D, int LD) {
    return (size_t)kNormStages * pack_tile_rows(D, LD) * (D + LD + 1) * 4 + 64;
}

bool pack_tiled_ok(const void* X, const void* T, const void* labels, const void* Xp, int D, int LD) {
    return LD < 256 && pack_smem(D, LD) <= 113 * 1024 && ((uintptr_t)X & 15) == 0 && ((uintptr_t)Xp & 15) == 0 &&
           ((uintptr_t)T & 15) == 0 && ((uintptr_t)labels & 15) == 0;
}

cudaError_t launch_pack_tiled(const float* X, const float* T, const uint8_t* labels, int64_t N, int D, int LD,
                              const float* col_min, const float* col_max, float* Xp, cudaStream_t st) {
    const size_t smem = pack_smem(D, LD);
    cudaError_t e = cudaFuncSetAttribute(pack_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = N / pack_tile_rows(D, LD);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * sms));
    pack_tiled_kernel<<<grid, 256, smem, st>>>(X, T, labels, N, D, LD, col_min, col_max, Xp);
    return cudaGetLastError();
}

static size_t norm_smem(int D) {
    const size_t ring = (size_t)kNormStages * norm_tile_rows(D) * D * 4;
    const size_t red = (size_t)2 * 256 * kNormMaxColsPerThread * 4;
    return (ring > red ? ring : red) + 64;
}

static int row_blocks(int64_t N) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (N + 7) / 8;
    return (int)std::min<int64_t>(need, (int64_t)sms * 8);  // 8 resident 256-thread blocks per SM
}

static bool tiled_ok(const void* X, const void* Y, int D) {
    const size_t smem = norm_smem(D);
    return D <= 256 * kNormMaxColsPerThread && smem <= 113 * 1024 && ((uintptr_t)X & 15) == 0 &&
           ((uintptr_t)Y & 15) == 0;
}

template <bool APPLY>
static cudaError_t launch_tiled(const float* X, float* Y, int64_t N, int D, const float* cmin, const float* cmax,
                                int* omin, int* omax, cudaStream_t st) {
    const size_t smem = norm_smem(D);
    auto k = minmax_tiled_kernel<APPLY>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = N / norm_tile_rows(D);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * sms));
    k<<<grid, 256, smem, st>>>(X, Y, N, D, cmin, cmax, omin, omax);
    return cudaGetLastError();
}

cudaError_t launch_minmax_fit(const float* X, int64_t N, int D, int* work, float* col_min, float* col_max,
                              cudaStream_t st) {
    int* omin = work;
    int* omax = work + D;
    minmax_init_kernel<<<(D + 255) / 256, 256, 0, st>>>(omin, omax, D);
    if (tiled_ok(X, X, D)) {
        cudaError_t e = launch_tiled<false>(X, nullptr, N, D, nullptr, nullptr, omin, omax, st);
        if (e != cudaSuccess) return e;
    } else {
        dim3 grid(row_blocks(N), (D + kFitCols - 1) / kFitCols);
        minmax_fit_kernel<<<grid, dim3(32, 8), 0, st>>>(X, N, D, omin, omax);
    }
    minmax_finish_kernel<<<(D + 255) / 256, 256, 0, st>>>(omin, omax, D, col_min, col_max);
    return cudaGetLastError();
}

cudaError_t launch_minmax_apply(const float* X, int64_t N, int D, const float* col_min, const float* col_max,
                                float* Y, cudaStream_t st) {
    if (tiled_ok(X, Y, D)) return launch_tiled<true>(X, Y, N, D, col_min, col_max, nullptr, nullptr, st);
    minmax_apply_kernel<<<row_blocks(N), dim3(32, 8), 0, st>>>(X, N, D, col_min, col_max, Y);
    return cudaGetLastError();
}


// ============================================================ synthetic rows
// numpy's Generator(PCG64(seed)) on the device (reference dataset.py:260-289):
// a 128-bit LCG s <- s * M + inc whose 64-bit outputs are XSL-RR(s) of the
// state after each step; float32 draws use the low then the high 32 bits of one
// output as (u >> 8) * 2^-24, float64 draws use (u >> 11) * 2^-53. Jump-ahead
// (s_{k+n} = A_n s_k + C_n) lets thread t produce outputs t, t + T, t + 2T, ...,
// so a warp's stores are coalesced and the bytes equal numpy's sequential draws.
namespace pcg {
typedef unsigned __int128 u128;
__host__ __device__ inline u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }
__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
// (A, C) of n steps of s <- s * m + c
__device__ inline void jump(u128 m, u128 c, uint64_t n, u128& A, u128& C) {
    A = 1;
    C = 0;
    while (n) {
        if (n & 1) {
            A *= m;
            C = C * m + c;
        }
        c = (m + 1) * c;
        m *= m;
        n >>= 1;
    }
}
constexpr uint64_t kMultHi = 0x2360ed051fc65da4ULL, kMultLo = 0x4385df649fccf645ULL;
}  // namespace pcg

// out[i] for i < n_floats, float i = half (i & 1) of output first + i / 2
__global__ void pcg64_f32_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first,
                                 int64_t n_floats, float2* __restrict__ out2, float* __restrict__ out_tail) {
    using namespace pcg;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_out = (n_floats + 1) / 2;
    if (t >= n_out) return;
    u128 A, C;
    jump(mk(kMultHi, kMultLo), mk(inc_hi, inc_lo), (uint64_t)(first + t + 1), A, C);
    u128 s = A * mk(s_hi, s_lo) + C;
    u128 aT, cT;  // T steps at once (thread stride)
    jump(mk(kMultHi, kMultLo), mk(inc_hi, inc_lo), (uint64_t)T, aT, cT);
    for (int64_t k = t; k < n_out; k += T) {
        const uint64_t v = xsl_rr(s);
        const float f0 = (float)((uint32_t)v >> 8) * (1.0f / 16777216.0f);
        const float f1 = (float)((uint32_t)(v >> 32) >> 8) * (1.0f / 16777216.0f);
        if (2 * k + 1 < n_floats) out2[k] = make_float2(f0, f1);
        else out_tail[0] = f0;  // odd count: the last output's low half only
        s = aT * s + cT;
    }
}

// labels[r] = (float64 draw of output first + r) < 0.5, i.e. the output's top bit is 0
__global__ void pcg64_coin_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t first,
                                  int64_t n, uint8_t* __restrict__ labels) {
    using namespace pcg;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    u128 A, C;
    jump(mk(kMultHi, kMultLo), mk(inc_hi, inc_lo), (uint64_t)(first + t + 1), A, C);
    u128 s = A * mk(s_hi, s_lo) + C;
    u128 aT, cT;  // T steps at once (thread stride)
    jump(mk(kMultHi, kMultLo), mk(inc_hi, inc_lo), (uint64_t)T, aT, cT);
    for (int64_t k = t; k < n; k += T) {
        labels[k] = (xsl_rr(s) >> 63) == 0 ? 1 : 0;
        s = aT * s + cT;
    }
}

// planted-linear score: f64 sum over the picked columns, in pick order
__global__ void planted_score_kernel(const float* __restrict__ X, int64_t N, int D, const int* __restrict__ pick,
                                     const double* __restrict__ coef, int k, double* __restrict__ score) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= N) return;
    double s = 0.0;
    for (int q = 0; q < k; q++) s = __dadd_rn(s, __dmul_rn((double)X[r * D + pick[q]], coef[q]));
    score[r] = s;
}

__global__ void label_ge_kernel(const double* __restrict__ score, int64_t N, const double* __restrict__ thr,
                                uint8_t* __restrict__ labels) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < N) labels[r] = score[r] >= *thr ? 1 : 0;
}

static int pcg_grid(int64_t n) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
}

cudaError_t launch_pcg64_f32(const uint64_t* st4, int64_t first, int64_t n_floats, float* out, cudaStream_t st) {
    if (n_floats <= 0) return cudaSuccess;
    const int64_t n_out = (n_floats + 1) / 2;
    pcg64_f32_kernel<<<pcg_grid(n_out), 256, 0, st>>>(st4[0], st4[1], st4[2], st4[3], first, n_floats,
                                                      reinterpret_cast<float2*>(out), out + (n_floats - 1));
    return cudaGetLastError();
}

cudaError_t launch_pcg64_coin(const uint64_t* st4, int64_t first, int64_t n, uint8_t* labels, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    pcg64_coin_kernel<<<pcg_grid(n), 256, 0, st>>>(st4[0], st4[1], st4[2], st4[3], first, n, labels);
    return cudaGetLastError();
}

cudaError_t launch_planted_score(const float* X, int64_t N, int D, const int* pick, const double* coef, int k,
                                 double* score, cudaStream_t st) {
    planted_score_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(X, N, D, pick, coef, k, score);
    return cudaGetLastError();
}

cudaError_t launch_label_ge(const double* score, int64_t N, const double* thr, uint8_t* labels, cudaStream_t st) {
    label_ge_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(score, N, thr, labels);
    return cudaGetLastError();
}

}  // namespace glx
