// glx_generic.cu -- any-shape engines for the widths the specialised kernels do
// not instantiate: online SGD with D > 63 or H > 512 (glx_online.cu keeps a
// weight row per thread in registers) and the full-batch epoch with D > 127 or
// H > 512 (glx_batch*.cu keep [W1 | b1] rows of at most 128 floats). The
// reference engines take any input/hidden width (kernels.py:264-349); these
// keep that contract at reduced speed.
//
// online_generic_kernel: one CTA per network, the weights in global memory
// (each hidden row owned by one thread, so its update is race free), the
// training row and the hidden activations in shared memory, four block
// barriers per row. Numerics as glx_online.cu: "ref64" keeps the reference's
// exact op order (16-wide f64 blocks in index order, bias last, f64 sigmoid,
// unfused w - step*x with one f32 rounding per store; kernels.py:102-139),
// "fp32" the same order in float.
//
// The full-batch epoch (FP32) runs per chunk of C rows as
// three tiled FP32 GEMM-shaped kernels plus two reductions:
//   gen_fwd_kernel:  Z = [x,1] W1^T (64 x 64 tiles), h = sigmoid(Z) stored,
//                    per-tile partials of w2 . h per row
//   gen_out_kernel:  o, delta_o = (o - t) o (1 - o), loss / confusion partials
//   gen_dw1_kernel:  dW1 += dH^T [x,1] with dH = delta_o w2 h (1 - h) formed on
//                    load, split over rows; dW2 += delta_o h on the way
//   gen_reduce_kernel: the split partials summed in fixed order into the f64
//                    gradient (accumulated over chunks; deterministic)
// The gradient uses the layout of glx_batch_grad (dW1 sums with the w2 factor
// folded in, dW2, sum delta_o, loss, tp, tn, fp, fn), so the same apply /
// all-reduce / update code serves every shape.
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>

namespace glx {

constexpr int kGenBlk = 16;  // kernels.py:31 BLOCK
constexpr int kGenOnlineThreads = 256;

template <typename Real>
__device__ __forceinline__ Real gen_sigmoid(Real z);
template <>
__device__ __forceinline__ double gen_sigmoid<double>(double z) {
    return 1.0 / (1.0 + exp(-z));
}
template <>
__device__ __forceinline__ float gen_sigmoid<float>(float z) {
    return 1.0f / (1.0f + expf(-z));
}
// separately rounded products / differences: the reference's w - step * x is
// unfused (kernels.py:132-139), so no FMA contraction in the update
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }

// ------------------------------------------------------------- online SGD
template <typename Real>
__global__ void __launch_bounds__(kGenOnlineThreads) online_generic_kernel(const GenNet* __restrict__ nets,
                                                                          const float* __restrict__ X,
                                                                          const float* __restrict__ T, int64_t N,
                                                                          int D, int64_t epochs, double lr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const GenNet net = nets[blockIdx.x];
    const int H = net.H;
    const int nb = (H + kGenBlk - 1) / kGenBlk;
    Real* parts = reinterpret_cast<Real*>(smem_raw);  // nb output block partials
    Real* bc = parts + nb;                            // delta_o, lr * delta_o
    float* xs = reinterpret_cast<float*>(bc + 2);     // two row buffers (row parity)
    float* hs = xs + 2 * D;                           // H activations
    float* w_ih = net.w_ih;
    float* w_ho = net.w_ho;
    const int tid = threadIdx.x, nt = blockDim.x;
    const Real rlr = (Real)lr;
    int64_t step = 0;  // rows trained so far: consecutive rows alternate buffers across epochs too
    for (int64_t ep = 0; ep < epochs; ep++) {
        for (int64_t r = 0; r < N; r++, step++) {
            // the row buffer of this step's parity: its last readers (the updates two
            // steps back) finished before the previous step's barriers
            float* x = xs + (step & 1) * D;
            for (int i = tid; i < D; i += nt) x[i] = X[r * D + i];
            __syncthreads();
            for (int j = tid; j < H; j += nt) {  // kernels.py:118-122, 270-276
                const float* w = w_ih + (int64_t)j * (D + 1);
                Real acc = 0;
                for (int b0 = 0; b0 < D; b0 += kGenBlk) {
                    const int b1 = min(b0 + kGenBlk, D);
                    Real part = 0;
                    for (int i = b0; i < b1; i++) part += (Real)w[i] * (Real)x[i];
                    acc += part;
                }
                hs[j] = (float)gen_sigmoid<Real>(acc + (Real)w[D]);
            }
            __syncthreads();
            for (int b = tid; b < nb; b += nt) {  // output block partials (kernels.py:277-287)
                const int j1 = min(b * kGenBlk + kGenBlk, H);
                Real part = 0;
                for (int j = b * kGenBlk; j < j1; j++) part += (Real)w_ho[j] * (Real)hs[j];
                parts[b] = part;
            }
            __syncthreads();
            if (tid == 0) {
                Real acc = 0;
                for (int b = 0; b < nb; b++) acc += parts[b];
                const float o = (float)gen_sigmoid<Real>(acc + (Real)w_ho[H]);
                const Real od = (Real)o;
                const Real d_o = (od - (Real)T[r]) * od * ((Real)1 - od);  // kernels.py:125-129
                bc[0] = d_o;
                bc[1] = rlr * d_o;
            }
            __syncthreads();
            const Real d_o = bc[0], step_o = bc[1];
            for (int j = tid; j < H; j += nt) {  // hidden first, from the pre-update w_ho (kernels.py:290-292)
                float* w = w_ih + (int64_t)j * (D + 1);
                const Real hd = (Real)hs[j];
                const Real s = rlr * ((Real)w_ho[j] * d_o * hd * ((Real)1 - hd));
                for (int i = 0; i < D; i++) w[i] = (float)sub_rn((Real)w[i], mul_rn(s, (Real)x[i]));  // kernels.py:132-139
                w[D] = (float)sub_rn((Real)w[D], s);
                w_ho[j] = (float)sub_rn((Real)w_ho[j], mul_rn(step_o, hd));
            }
            if (tid == 0) w_ho[H] = (float)sub_rn((Real)w_ho[H], step_o);
        }
    }
}

size_t online_generic_smem(int D, int H) {
    const int nb = (H + kGenBlk - 1) / kGenBlk;
    return (size_t)(nb + 2) * 8 + (size_t)2 * D * 4 + (size_t)H * 4;
}

cudaError_t launch_online_generic(const GenNet* nets, int n_nets, int max_h, const float* X, const float* T, int64_t N,
                                  int D, int64_t epochs, double lr, bool ref64, cudaStream_t st) {
    const size_t smem = online_generic_smem(D, max_h);
    if (smem > kGenMaxSmem) return cudaErrorInvalidValue;
    const int threads = std::min(kGenOnlineThreads, std::max(32, (std::max(max_h, D) + 31) / 32 * 32));
    cudaError_t e;
    if (ref64) {
        e = cudaFuncSetAttribute(online_generic_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        online_generic_kernel<double><<<n_nets, threads, smem, st>>>(nets, X, T, N, D, epochs, lr);
    } else {
        e = cudaFuncSetAttribute(online_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        online_generic_kernel<float><<<n_nets, threads, smem, st>>>(nets, X, T, N, D, epochs, lr);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------- full-batch epoch
constexpr int kGT = 64;   // tile edge (rows x units, units x inputs)
constexpr int kGK = 16;   // contraction step
constexpr int kGPad = 4;  // smem row padding (floats)

// Z tile [64 rows][64 units] = [x,1] (packed rows, LD floats per row) . W1^T;
// h = sigmoid(Z) -> Hs (chunk rows x Hld), per-row partial of w2 . h over the
// tile's units -> opart[unit tile][row]
__global__ void __launch_bounds__(256) gen_fwd_kernel(const float* __restrict__ Xp, int LD, int C, int D, int H,
                                                      const float* __restrict__ W1, const float* __restrict__ W2,
                                                      float* __restrict__ Hs, int Hld, float* __restrict__ opart) {
    __shared__ __align__(16) float As[kGK][kGT + kGPad];  // [k][row]
    __shared__ __align__(16) float Bs[kGK][kGT + kGPad];  // [k][unit]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int row0 = blockIdx.x * kGT, unit0 = blockIdx.y * kGT;
    const int K1 = D + 1;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K1; k0 += kGK) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int e = tid + 256 * q, m = e >> 4, k = e & 15;
            const int r = row0 + m, u = unit0 + m, kk = k0 + k;
            As[k][m] = (r < C && kk < K1) ? Xp[(int64_t)r * LD + kk] : 0.f;
            Bs[k][m] = (u < H && kk < K1) ? W1[(int64_t)u * K1 + kk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kGK; k++) {
            const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    float w2[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int u = unit0 + tx * 4 + j;
        w2[j] = u < H ? W2[u] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int r = row0 + ty * 4 + i;
        float p = 0.f;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int u = unit0 + tx * 4 + j;
            const float h = gen_sigmoid<float>(acc[i][j]);
            if (r < C && u < H) Hs[(int64_t)r * Hld + u] = h;
            p = fmaf(w2[j], h, p);
        }
        // the 16 threads of this row group (one half warp) sum their units
#pragma unroll
        for (int s = 8; s >= 1; s >>= 1) p += __shfl_xor_sync(0xffffffffu, p, s);
        if (tx == 0 && r < C) opart[(int64_t)blockIdx.y * C + r] = p;
    }
}

// per row: o, delta_o (kernels.py:352-375 forward; the batch restatement of
// oracle train_batch), loss and confusion partials per block (fixed-order tree)
__global__ void __launch_bounds__(256) gen_out_kernel(const float* __restrict__ Xp, int LD, int C, int D, int H,
                                                      int nut, const float* __restrict__ opart,
                                                      const float* __restrict__ W2, float* __restrict__ dvec,
                                                      double* __restrict__ statpart) {
    __shared__ double red[6][256];
    const int r = blockIdx.x * 256 + threadIdx.x;
    const float b2 = W2[H];
    double v[6] = {0, 0, 0, 0, 0, 0};  // dsum, loss, tp, tn, fp, fn
    if (r < C) {
        float z = 0.f;
        for (int u = 0; u < nut; u++) z += opart[(int64_t)u * C + r];
        const float o = gen_sigmoid<float>(z + b2);
        const float t = Xp[(int64_t)r * LD + D + 1];
        const float d = (o - t) * o * (1.0f - o);
        dvec[r] = d;
        const bool pred = o >= 0.5f, pos = t >= 0.5f;
        v[0] = d;
        v[1] = 0.5 * (double)(t - o) * (double)(t - o);
        v[2] = pred && pos;
        v[3] = !pred && !pos;
        v[4] = pred && !pos;
        v[5] = !pred && pos;
    }
#pragma unroll
    for (int q = 0; q < 6; q++) red[q][threadIdx.x] = v[q];
    __syncthreads();
    for (int s = 128; s >= 1; s >>= 1) {
        if (threadIdx.x < s)
#pragma unroll
            for (int q = 0; q < 6; q++) red[q][threadIdx.x] += red[q][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 6) statpart[(int64_t)blockIdx.x * 6 + threadIdx.x] = red[threadIdx.x][0];
}

// dW1 tile [64 units][64 inputs of [x,1]] over rows [split * rps, ...) of the
// chunk: A[row][unit] = delta_o w2 h (1 - h), B[row][input] = packed row.
// Tiles of the first input column also sum dW2 = delta_o h per unit.
__global__ void __launch_bounds__(256) gen_dw1_kernel(const float* __restrict__ Xp, int LD, int C, int D, int H,
                                                      const float* __restrict__ W2, const float* __restrict__ Hs,
                                                      int Hld, const float* __restrict__ dvec, int rps,
                                                      float* __restrict__ p1, float* __restrict__ p2) {
    __shared__ __align__(16) float As[kGK][kGT + kGPad];  // [row][unit]
    __shared__ __align__(16) float Bs[kGK][kGT + kGPad];  // [row][input]
    __shared__ float g2s[4][kGT];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int in0 = blockIdx.x * kGT, unit0 = blockIdx.y * kGT, split = blockIdx.z;
    const int K1 = D + 1;
    const int r0 = split * rps, r1 = min(C, r0 + rps);
    const int lu = tid & 63, lr = tid >> 6;  // loader: unit / input column lu, rows lr + 4 q
    const int u = unit0 + lu, ii = in0 + lu;
    const float w2 = u < H ? W2[u] : 0.f;
    float g2 = 0.f;
    float acc[4][4] = {};
    for (int k0 = r0; k0 < r1; k0 += kGK) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int k = lr + 4 * q, r = k0 + k;
            float a = 0.f, b = 0.f;
            if (r < r1) {
                if (u < H) {
                    const float h = Hs[(int64_t)r * Hld + u];
                    const float d = dvec[r];
                    a = d * w2 * h * (1.0f - h);
                    g2 = fmaf(d, h, g2);
                }
                if (ii < K1) b = Xp[(int64_t)r * LD + ii];
            }
            As[k][lu] = a;
            Bs[k][lu] = b;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kGK; k++) {
            const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* out = p1 + (int64_t)split * H * K1;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int uu = unit0 + ty * 4 + i;
        if (uu >= H) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = in0 + tx * 4 + j;
            if (c < K1) out[(int64_t)uu * K1 + c] = acc[i][j];
        }
    }
    if (blockIdx.x == 0) {  // dW2 of this split: the 4 loader rows of each unit, in fixed order
        g2s[lr][lu] = g2;
        __syncthreads();
        if (tid < kGT && unit0 + tid < H)
            p2[(int64_t)split * H + unit0 + tid] = ((g2s[0][tid] + g2s[1][tid]) + g2s[2][tid]) + g2s[3][tid];
    }
}

// grad (f64, glx_batch_grad layout) = / += the chunk's split partials, summed in
// split order; the statistics from the per-block partials in block order
__global__ void __launch_bounds__(256) gen_reduce_kernel(const float* __restrict__ p1, const float* __restrict__ p2,
                                                         int splits, const double* __restrict__ statpart, int nsb,
                                                         int D, int H, int first, double* __restrict__ grad) {
    const int64_t P1 = (int64_t)H * (D + 1);
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P1 + H + 6) return;
    double s = 0.0;
    if (idx < P1) {
        for (int z = 0; z < splits; z++) s += (double)p1[(int64_t)z * P1 + idx];
    } else if (idx < P1 + H) {
        for (int z = 0; z < splits; z++) s += (double)p2[(int64_t)z * H + (idx - P1)];
    } else {
        const int q = (int)(idx - P1 - H);  // 0: sum delta_o, 1: loss, 2..5: tp, tn, fp, fn
        for (int b = 0; b < nsb; b++) s += statpart[(int64_t)b * 6 + q];
    }
    grad[idx] = first ? s : grad[idx] + s;
}

size_t generic_chunk_rows(int64_t N, int H) {
    const int64_t hbytes = (int64_t)((H + 3) / 4 * 4) * 4;
    int64_t c = std::min<int64_t>(65536, (N + kGT - 1) / kGT * kGT);
    while (c > kGT && c * hbytes > ((int64_t)512 << 20)) c /= 2;
    return (size_t)std::max<int64_t>(kGT, c / kGT * kGT);
}

static int generic_splits(int D, int H, int C) {
    const int tiles = ((D + 1 + kGT - 1) / kGT) * ((H + kGT - 1) / kGT);
    int s = (2 * 148 + tiles - 1) / tiles;
    return std::max(1, std::min(s, C / kGT));
}

size_t generic_work_bytes(int64_t N, int D, int H) {
    const int C = (int)generic_chunk_rows(N, H);
    const int Hld = (H + 3) / 4 * 4;
    const int nut = (H + kGT - 1) / kGT;
    const int S = generic_splits(D, H, C);
    const int nsb = (C + 255) / 256;
    size_t b = 0;
    b += (size_t)C * Hld * 4;                 // Hs
    b += (size_t)nut * C * 4;                 // opart
    b += (size_t)C * 4;                       // dvec
    b += (size_t)S * H * (D + 1) * 4;         // p1
    b += (size_t)S * H * 4;                   // p2
    b = (b + 15) / 16 * 16 + (size_t)nsb * 6 * 8;  // statpart
    return b + 64;
}

cudaError_t generic_batch_grad(const float* W1, const float* W2, const float* Xp, int64_t N, int D, int H, int LD,
                               void* work, double* grad, cudaStream_t st) {
    const int C = (int)generic_chunk_rows(N, H);
    const int Hld = (H + 3) / 4 * 4;
    const int nut = (H + kGT - 1) / kGT;
    const int S = generic_splits(D, H, C);
    const int nsb = (C + 255) / 256;
    unsigned char* p = reinterpret_cast<unsigned char*>(work);
    float* Hs = reinterpret_cast<float*>(p);
    p += (size_t)C * Hld * 4;
    float* opart = reinterpret_cast<float*>(p);
    p += (size_t)nut * C * 4;
    float* dvec = reinterpret_cast<float*>(p);
    p += (size_t)C * 4;
    float* p1 = reinterpret_cast<float*>(p);
    p += (size_t)S * H * (D + 1) * 4;
    float* p2 = reinterpret_cast<float*>(p);
    p += (size_t)S * H * 4;
    p = reinterpret_cast<unsigned char*>(((uintptr_t)p + 15) / 16 * 16);
    double* statpart = reinterpret_cast<double*>(p);
    const int64_t glen = (int64_t)H * (D + 1) + H + 6;
    for (int64_t c0 = 0; c0 < N; c0 += C) {
        const int Cc = (int)std::min<int64_t>(C, N - c0);
        const float* X = Xp + c0 * LD;
        gen_fwd_kernel<<<dim3((Cc + kGT - 1) / kGT, nut), 256, 0, st>>>(X, LD, Cc, D, H, W1, W2, Hs, Hld, opart);
        gen_out_kernel<<<(Cc + 255) / 256, 256, 0, st>>>(X, LD, Cc, D, H, nut, opart, W2, dvec, statpart);
        const int Sc = std::max(1, std::min(S, (Cc + kGT - 1) / kGT));
        const int rps = ((Cc + Sc - 1) / Sc + kGK - 1) / kGK * kGK;
        const int Sr = (Cc + rps - 1) / rps;
        gen_dw1_kernel<<<dim3((D + 1 + kGT - 1) / kGT, nut, Sr), 256, 0, st>>>(X, LD, Cc, D, H, W2, Hs, Hld, dvec, rps,
                                                                               p1, p2);
        gen_reduce_kernel<<<(unsigned)((glen + 255) / 256), 256, 0, st>>>(p1, p2, Sr, statpart, (Cc + 255) / 256, D,
                                                                          H, c0 == 0, grad);
    }
    return cudaGetLastError();
}

}  // namespace glx
