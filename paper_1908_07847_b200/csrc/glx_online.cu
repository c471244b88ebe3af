// glx_online.cu -- per-instance online SGD (the reference's training semantics).
//
// Replaces kernels.train_segment_seq / train_segment_par
// (/root/reference/pkg/src/glycemlp/kernels.py:264-349). The reference's
// "neuron-parallel" engine gives each worker a block of hidden neurons and
// meets at a spin barrier twice per training row; here each hidden neuron is
// one CUDA thread that keeps its weight row in REGISTERS, the training rows
// sit in shared memory, and the network's warps meet at one named barrier
// per row (fp32) or two (ref64). Several independent networks (hidden-width x
// seed sweeps) are packed into one CTA, each on its own
// warp range and named barrier, sharing the CTA's copy of the rows.
//
// Numerics (template Real):
//   double -- "ref64": the reference's exact op order: f64 products of f32
//             operands accumulated over 16-wide blocks in index order, bias
//             last, f64 sigmoid, unfused w - step*x, one f32 rounding per
//             store (kernels.py:102-139). Differs from the CPU only where
//             CUDA's f64 exp and glibc's differ in the last ulp.
//   float  -- "fp32": FFMA2 (packed f32x2) dot and update, MUFU sigmoid,
//             tree reduction. Within the 1e-4 max(1,|w|) tolerance.
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <type_traits>

#ifndef GLX_ONLINE_LANE_SUM
#define GLX_ONLINE_LANE_SUM 1  // sweep output partials: lane-parallel shuffle sum (1; 2% faster) or predicated loop (0)
#endif
#ifndef GLX_ONLINE_LA
// lookahead forward: z_{r+1} = W^(r) x_{r+1} + ns_r (x_r . x_{r+1}) lets the next
// row's dot product run alongside this row's output reduction (fp32 only)
#define GLX_ONLINE_LA 1
#endif

namespace glx {

template <typename Real, int DP, bool XS>
__device__ __forceinline__ void load_row(float (&x)[DP], const float* __restrict__ xs, const float* __restrict__ X,
                                         int64_t r, int D) {
    if (XS) {  // shared: rows pre-padded to DP floats as [x_0..x_{D-1}, 1, 0...]
        const float2* p = reinterpret_cast<const float2*>(xs + r * DP);
#pragma unroll
        for (int q = 0; q < DP / 2; q++) {
            float2 v = p[q];
            x[2 * q] = v.x;
            x[2 * q + 1] = v.y;
        }
    } else {  // global, caller layout (N, D)
        const float* p = X + r * D;
#pragma unroll
        for (int i = 0; i < DP; i++) x[i] = i < D ? __ldg(p + i) : (i == D ? 1.0f : 0.0f);
    }
}

template <typename Real, int DP, bool XS>
__global__ void __launch_bounds__(512) online_sgd_kernel(const OnlineNetDesc* __restrict__ nets,
                                                          const int2* __restrict__ cta_nets, const float* __restrict__ X,
                                                          const float* __restrict__ T, int64_t N, int D,
                                                          int64_t epochs, double lr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* xs = reinterpret_cast<float*>(smem_raw);  // N x DP (if XS)
    float* ts = xs + (XS ? N * DP : 0);              // N targets (if XS)
    float* gd = ts + (XS ? N : 0);                   // N lookahead dots x_r . x_{r+1} (if XS, fp32)
    constexpr bool kLA = XS && GLX_ONLINE_LA && sizeof(Real) == 4;

    const int2 cn = cta_nets[blockIdx.x];
    const int warp = threadIdx.x >> 5;

    // stage the training rows once per CTA (shared by every packed network)
    if (XS) {
        for (int64_t e = threadIdx.x; e < N * DP; e += blockDim.x) {
            int64_t r = e / DP;
            int i = (int)(e - r * DP);
            xs[e] = i < D ? X[r * D + i] : (i == D ? 1.0f : 0.0f);
        }
        for (int64_t r = threadIdx.x; r < N; r += blockDim.x) ts[r] = T[r];
        __syncthreads();
        if (kLA) {
            for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
                const float* a0 = xs + r * DP;
                const float* a1 = xs + (r + 1 == N ? 0 : r + 1) * DP;
                float s = 0.f;
                for (int i = 0; i < DP; i++) s = fmaf(a0[i], a1[i], s);
                gd[r] = s;
            }
            __syncthreads();
        }
    }

    // find my network
    int my = -1;
    for (int k = 0; k < cn.y; k++) {
        const OnlineNetDesc& nd = nets[cn.x + k];
        if (warp >= nd.warp0 && warp < nd.warp0 + nd.nwarps) my = cn.x + k;
    }
    if (my < 0) return;
    const OnlineNetDesc nd = nets[my];
    const int H = nd.H;
    const int nthr = nd.nwarps * 32;
    const int j = threadIdx.x - nd.warp0 * 32;
    const bool active = j < H;
    float* w_ih = nd.w_ih;
    float* w_ho = nd.w_ho;
    unsigned char* scratch = smem_raw + nd.scratch_off;

    // weight row j in registers; slot D is the bias (x_D == 1)
    float w[DP];
#pragma unroll
    for (int i = 0; i < DP; i++) w[i] = (active && i <= D) ? w_ih[(int64_t)j * (D + 1) + i] : 0.0f;
    float w2 = active ? w_ho[j] : 0.0f;
    float b2 = w_ho[H];  // only thread j == 0 updates / writes it back

    float x[DP];
    float bw = 0.0f;  // ref64: the bias weight (see below); fp32 keeps it in w[D]
    if constexpr (sizeof(Real) == 4) {
        // ---------------------------------------------------------------- fp32
        float* red = reinterpret_cast<float*>(scratch);  // [2][16] warp partials
        const float kScale = (float)(-GLX_LOG2E);
        int buf = 0;
        if constexpr (kLA) {
            // lookahead schedule of online_sgd_mt_kernel, one unit per thread
            const float2* x0 = reinterpret_cast<const float2*>(xs);
            float2 p0 = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < DP / 2; q++) p0 = ffma2(make_float2(w[2 * q], w[2 * q + 1]), x0[q], p0);
            float zc = p0.x + p0.y, nsp = 0.f;
            int64_t rp = 0;
            for (int64_t ep = 0; ep < epochs; ep++) {
                if (ep > 0) {  // epoch start: as a fresh call (see online_sgd_mt_kernel)
                    const float2* xl2 = reinterpret_cast<const float2*>(xs + rp * DP);
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) {
                        const float2 wq = ffma2(bcast2(nsp), xl2[q], make_float2(w[2 * q], w[2 * q + 1]));
                        w[2 * q] = wq.x;
                        w[2 * q + 1] = wq.y;
                    }
                    nsp = 0.f;
                    float2 pz = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) pz = ffma2(make_float2(w[2 * q], w[2 * q + 1]), x0[q], pz);
                    zc = pz.x + pz.y;
                }
                for (int64_t r = 0; r < N; r++) {
                    const int64_t rn = r + 1 == N ? 0 : r + 1;
                    const float2* xp2 = reinterpret_cast<const float2*>(xs + rp * DP);
                    const float2* xn2 = reinterpret_cast<const float2*>(xs + rn * DP);
                    float2 p = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) {
                        const float2 wq = ffma2(bcast2(nsp), xp2[q], make_float2(w[2 * q], w[2 * q + 1]));
                        w[2 * q] = wq.x;
                        w[2 * q + 1] = wq.y;
                        p = ffma2(wq, xn2[q], p);
                    }
                    const float zpre = p.x + p.y;
                    const float t = ts[r];
                    const float h = active ? sigmoid_scaled(kScale * zc) : 0.0f;
                    float prod = active ? w2 * h : 0.0f;
                    if (j == 0) prod += b2;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
                    if ((threadIdx.x & 31) == 0) red[buf * 16 + (j >> 5)] = prod;
                    bar_sync(nd.bar_id, nthr);
                    float zo = 0.0f;
                    for (int k = 0; k < nd.nwarps; k++) zo += red[buf * 16 + k];
                    buf ^= 1;
                    const float o = sigmoid_scaled(kScale * zo);
                    const float d_o = (o - t) * o * (1.0f - o);
                    const float step_o = (float)lr * d_o;
                    const float ns = active ? -(float)lr * (w2 * d_o * h * (1.0f - h)) : 0.0f;
                    if (active) w2 = fmaf(-step_o, h, w2);
                    if (j == 0) b2 -= step_o;
                    zc = fmaf(ns, gd[r], zpre);
                    nsp = ns;
                    rp = r;
                }
            }
            const float2* xp2 = reinterpret_cast<const float2*>(xs + rp * DP);
#pragma unroll
            for (int q = 0; q < DP / 2; q++) {
                const float2 wq = ffma2(bcast2(nsp), xp2[q], make_float2(w[2 * q], w[2 * q + 1]));
                w[2 * q] = wq.x;
                w[2 * q + 1] = wq.y;
            }
        } else {
        for (int64_t ep = 0; ep < epochs; ep++) {
            for (int64_t r = 0; r < N; r++) {
                load_row<Real, DP, XS>(x, xs, X, r, D);
                const float t = XS ? ts[r] : __ldg(T + r);
                float2 p = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < DP / 2; q++)
                    p = ffma2(make_float2(w[2 * q], w[2 * q + 1]), make_float2(x[2 * q], x[2 * q + 1]), p);
                const float h = active ? sigmoid_scaled(kScale * (p.x + p.y)) : 0.0f;
                float prod = active ? w2 * h : 0.0f;
                if (j == 0) prod += b2;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
                if ((threadIdx.x & 31) == 0) red[buf * 16 + (j >> 5)] = prod;
                bar_sync(nd.bar_id, nthr);
                float zo = 0.0f;
                for (int k = 0; k < nd.nwarps; k++) zo += red[buf * 16 + k];
                buf ^= 1;
                const float o = sigmoid_scaled(kScale * zo);
                const float d_o = (o - t) * o * (1.0f - o);
                const float step_o = (float)lr * d_o;
                if (active) {
                    const float d_h = w2 * d_o * h * (1.0f - h);
                    const float ns = -(float)lr * d_h;
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) {
                        float2 wp = ffma2(bcast2(ns), make_float2(x[2 * q], x[2 * q + 1]),
                                          make_float2(w[2 * q], w[2 * q + 1]));
                        w[2 * q] = wp.x;
                        w[2 * q + 1] = wp.y;
                    }
                    w2 = fmaf(-step_o, h, w2);
                }
                if (j == 0) b2 -= step_o;
            }
        }
        }
    } else {
        // ---------------------------------------------------------------- ref64
        const int nb = (H + 15) >> 4;
        // the bias weight w[D] lives in its own register here: any runtime index into
        // w (NVVM even rebuilds one from a predicated select) moves the row to local memory
        bw = active ? w_ih[(int64_t)j * (D + 1) + D] : 0.0f;
        double* prods = reinterpret_cast<double*>(scratch);  // nb blocks x 17 (padded against bank conflicts)
        double* bc = prods + nb * 17;                        // [0] = d_o, [1] = step_o
        for (int64_t ep = 0; ep < epochs; ep++) {
            for (int64_t r = 0; r < N; r++) {
                // the row stays in registers: reading it from shared memory inside the
                // f64 chains measured 2.4x slower (the kernel then drops to 64 registers)
                load_row<Real, DP, XS>(x, xs, X, r, D);
                auto xd = [&](int i) -> double { return (double)x[i]; };
                float h = 0.0f;
                if (active) {
                    // kernels.py:102-122: blocked f64 dot, bias last, f64 sigmoid, f32 round
                    double acc = 0.0;
#pragma unroll
                    for (int b0 = 0; b0 < DP; b0 += 16) {
                        double part = 0.0;
#pragma unroll
                        for (int k = 0; k < 16; k++) {  // constant trip count: w stays in registers
                            const int i = b0 + k;
                            if (i < DP && i < D) part = fma((double)w[i < DP ? i : 0], xd(i < DP ? i : 0), part);
                        }
                        if (b0 < D) acc = __dadd_rn(acc, part);
                    }
                    double z = __dadd_rn(acc, (double)bw);
                    h = __double2float_rn(1.0 / (1.0 + exp(-z)));
                    prods[(j >> 4) * 17 + (j & 15)] = (double)w2 * (double)h;  // exact product
                }
                bar_sync(nd.bar_id, nthr);
                if (j < 32) {  // leader warp: the output neuron (kernels.py:277-289)
                    double part = 0.0;
                    if (j < nb) {
                        const int jn = min(16, H - j * 16);
                        double pv[16];  // loads ahead of the sequential adds (see the small kernel)
#pragma unroll
                        for (int k = 0; k < 16; k++) pv[k] = k < jn ? prods[j * 17 + k] : 0.0;
#pragma unroll
                        for (int k = 0; k < 16; k++)
                            if (k < jn) part = __dadd_rn(part, pv[k]);
                    }
                    double z = 0.0;
                    for (int b = 0; b < nb; b++) z = __dadd_rn(z, __shfl_sync(0xffffffffu, part, b));
                    if (j == 0) {
                        z = __dadd_rn(z, (double)b2);
                        const float o = __double2float_rn(1.0 / (1.0 + exp(-z)));
                        const double od = (double)o;
                        const double td = (double)(XS ? ts[r] : __ldg(T + r));
                        const double d_o = __dmul_rn(__dmul_rn(__dsub_rn(od, td), od), __dsub_rn(1.0, od));
                        bc[0] = d_o;
                        bc[1] = __dmul_rn(lr, d_o);
                    }
                }
                bar_sync(nd.bar_id, nthr);
                const double d_o = bc[0], step_o = bc[1];
                if (active) {
                    // hidden first, from the pre-update w_ho (kernels.py:290-292)
                    const double hd = (double)h;
                    const double d_h = __dmul_rn(__dmul_rn(__dmul_rn((double)w2, d_o), hd), __dsub_rn(1.0, hd));
                    const double s = __dmul_rn(lr, d_h);
#pragma unroll
                    for (int i = 0; i < DP; i++)
                        if (i < D) w[i] = __double2float_rn(__dsub_rn((double)w[i], __dmul_rn(s, xd(i))));
                    bw = __double2float_rn(__dsub_rn((double)bw, s));  // bias (x_D = 1)
                    w2 = __double2float_rn(__dsub_rn((double)w2, __dmul_rn(step_o, hd)));
                }
                if (j == 0) b2 = __double2float_rn(__dsub_rn((double)b2, step_o));
            }
        }
    }
    if (active) {
#pragma unroll
        for (int i = 0; i < DP; i++)
            if (sizeof(Real) == 4 ? i <= D : i < D) w_ih[(int64_t)j * (D + 1) + i] = w[i];
        if constexpr (sizeof(Real) == 8) w_ih[(int64_t)j * (D + 1) + D] = bw;
        w_ho[j] = w2;
    }
    if (j == 0) w_ho[H] = b2;
}


// fp32 online SGD with an MT-unit register tile per thread (sweeps): the
// per-row reduction, barrier and output-neuron work are paid once per MT
// hidden units instead of once per unit.
#ifndef GLX_ONLINE_XSMEM
#define GLX_ONLINE_XSMEM 1  // x pairs from shared memory (frees 34 registers for occupancy)
#endif
#ifndef GLX_ONLINE_MT2_CTAS
#define GLX_ONLINE_MT2_CTAS 2  // resident 256-thread CTAs per SM for the 2-unit tile (<= 128 registers)
#endif
// ONEW: every network of the launch is one warp (H <= 32 MT): the warp-shuffle
// reduction already gives every lane the output sum, no shared-memory exchange
// or named barrier (a separate instantiation: a runtime branch cost the sweep)
template <int DP, int MT, bool XS, bool ONEW = false>
#ifndef GLX_ONLINE_ONEW_CTAS
#define GLX_ONLINE_ONEW_CTAS GLX_ONLINE_MT2_CTAS
#endif
__global__ void __launch_bounds__(256, MT == 2 ? (ONEW ? GLX_ONLINE_ONEW_CTAS : GLX_ONLINE_MT2_CTAS) : 1) online_sgd_mt_kernel(const OnlineNetDesc* __restrict__ nets,
                                                             const int2* __restrict__ cta_nets,
                                                             const float* __restrict__ X, const float* __restrict__ T,
                                                             int64_t N, int D, int64_t epochs, double lr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // staged rows are padded to SP floats (16-byte aligned): x is read as float4
    constexpr int SP = (DP + 3) & ~3;
    float* xs = reinterpret_cast<float*>(smem_raw);
    float* ts = xs + (XS ? N * SP : 0);
    float* gd = ts + (XS ? N : 0);  // gd[r] = x_r . x_{(r+1) mod N} (lookahead correction)
    const int2 cn = cta_nets[blockIdx.x];
    const int warp = threadIdx.x >> 5;
    if (XS) {
        for (int64_t e = threadIdx.x; e < N * SP; e += blockDim.x) {
            int64_t r = e / SP;
            int i = (int)(e - r * SP);
            xs[e] = i < D ? X[r * D + i] : (i == D ? 1.0f : 0.0f);
        }
        for (int64_t r = threadIdx.x; r < N; r += blockDim.x) ts[r] = T[r];
        __syncthreads();
        if (GLX_ONLINE_LA) {
            for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
                const float* a0 = xs + r * SP;
                const float* a1 = xs + (r + 1 == N ? 0 : r + 1) * SP;
                float s = 0.f;
                for (int i = 0; i < DP; i++) s = fmaf(a0[i], a1[i], s);
                gd[r] = s;
            }
            __syncthreads();
        }
    }
    int my = -1;
    for (int k = 0; k < cn.y; k++) {
        const OnlineNetDesc& nd = nets[cn.x + k];
        if (warp >= nd.warp0 && warp < nd.warp0 + nd.nwarps) my = cn.x + k;
    }
    if (my < 0) return;
    const OnlineNetDesc nd = nets[my];
    const int H = nd.H;
    const int nthr = nd.nwarps * 32;
    const int t = threadIdx.x - nd.warp0 * 32;
    float* w_ih = nd.w_ih;
    float* w_ho = nd.w_ho;
    float* red = reinterpret_cast<float*>(smem_raw + nd.scratch_off);  // [2][16]
    float2 w[MT][DP / 2];
    float w2[MT];
    bool act[MT];
#pragma unroll
    for (int u = 0; u < MT; u++) {
        const int j = t * MT + u;
        act[u] = j < H;
#pragma unroll
        for (int q = 0; q < DP / 2; q++) {
            const int i0 = 2 * q, i1 = 2 * q + 1;
            w[u][q] = make_float2((act[u] && i0 <= D) ? w_ih[(int64_t)j * (D + 1) + i0] : 0.f,
                                  (act[u] && i1 <= D) ? w_ih[(int64_t)j * (D + 1) + i1] : 0.f);
        }
        w2[u] = act[u] ? w_ho[j] : 0.f;
    }
    float b2 = w_ho[H];
    const float kScale = (float)(-GLX_LOG2E);
    const float flr = (float)lr;
    int buf = 0;
    float x[DP];
    // GLX_ONLINE_XSMEM: with the rows staged in shared memory, read x pairs from
    // there in both loops instead of holding the row in 34 registers
    constexpr bool kXs = XS && GLX_ONLINE_XSMEM;
    if constexpr (kXs && GLX_ONLINE_LA) {
        // Lookahead schedule. At row r the thread holds z_r (this row's dots) and
        // the pending update (ns of row r-1, applied lazily). Off the critical
        // path: apply that update (W becomes W^(r)) and form W^(r) x_{r+1}. On it:
        // sigmoid, output reduction, delta_o, ns_r, then z_{r+1} = that dot +
        // ns_r * gd[r]. Same arithmetic as the reference order up to f32 rounding.
        const float2* x0 = reinterpret_cast<const float2*>(xs);
        float zc[MT], nsp[MT];
#pragma unroll
        for (int u = 0; u < MT; u++) {
            float2 p = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < DP / 2; q++) p = ffma2(w[u][q], x0[q], p);
            zc[u] = p.x + p.y;
            nsp[u] = 0.f;
        }
        // rows are staged in shared memory (<= 160 KB), so 32-bit row indices and
        // byte offsets suffice: the row loop's integer work stays 32-bit
        // (the one-warp instantiation measured faster with 64-bit indices: 175 vs 199 ns/row)
        using RowT = typename std::conditional<ONEW, int64_t, int>::type;
        const RowT n_rows = (RowT)N;
        RowT rp = 0;  // row of the pending update (nsp = 0 before the first row)
        for (int64_t ep = 0; ep < epochs; ep++) {
            if (ep > 0) {
                // epoch start: settle the pending update and form z_0 directly, exactly
                // as a fresh call does, so results do not depend on how the epochs are
                // split into calls (checkpoint segments)
                const float2* xl2 = reinterpret_cast<const float2*>(xs + rp * SP);
#pragma unroll
                for (int u = 0; u < MT; u++) {
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) w[u][q] = ffma2(bcast2(nsp[u]), xl2[q], w[u][q]);
                    nsp[u] = 0.f;
                }
#pragma unroll
                for (int u = 0; u < MT; u++) {
                    float2 p = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < DP / 2; q++) p = ffma2(w[u][q], x0[q], p);
                    zc[u] = p.x + p.y;
                }
            }
            for (RowT r = 0; r < n_rows; r++) {
                const RowT rn = r + 1 == n_rows ? 0 : r + 1;
                const float4* xp4 = reinterpret_cast<const float4*>(xs + rp * SP);
                const float4* xn4 = reinterpret_cast<const float4*>(xs + rn * SP);
                // (B) off the critical path: one float4 of each row feeds every unit
                float2 pz[MT];
#pragma unroll
                for (int u = 0; u < MT; u++) pz[u] = make_float2(0.f, 0.f);
#pragma unroll
                for (int q4 = 0; q4 < (DP + 3) / 4; q4++) {
                    const float4 a = xp4[q4], c = xn4[q4];
#pragma unroll
                    for (int u = 0; u < MT; u++) {
                        w[u][2 * q4] = ffma2(bcast2(nsp[u]), make_float2(a.x, a.y), w[u][2 * q4]);
                        pz[u] = ffma2(w[u][2 * q4], make_float2(c.x, c.y), pz[u]);
                        if (2 * q4 + 1 < DP / 2) {
                            w[u][2 * q4 + 1] = ffma2(bcast2(nsp[u]), make_float2(a.z, a.w), w[u][2 * q4 + 1]);
                            pz[u] = ffma2(w[u][2 * q4 + 1], make_float2(c.z, c.w), pz[u]);
                        }
                    }
                }
                float zpre[MT];
#pragma unroll
                for (int u = 0; u < MT; u++) zpre[u] = pz[u].x + pz[u].y;  // (pairs: see below)
                // (A) the row's critical chain; unit pairs use packed FMUL2/FADD2/FFMA2
                // (per lane the same IEEE ops as the scalar form)
                const float tt = ts[r];
                float h[MT];
                float prod = (t == 0) ? b2 : 0.f;
                if constexpr (MT % 2 == 0) {
#pragma unroll
                    for (int p = 0; p < MT / 2; p++) {
                        const float2 zz = __fmul2_rn(make_float2(zc[2 * p], zc[2 * p + 1]), bcast2(kScale));
                        const float2 den =
                            __fadd2_rn(make_float2(ex2_approx(zz.x), ex2_approx(zz.y)), bcast2(1.0f));
                        h[2 * p] = act[2 * p] ? rcp_approx(den.x) : 0.f;
                        h[2 * p + 1] = act[2 * p + 1] ? rcp_approx(den.y) : 0.f;
                        prod = fmaf(w2[2 * p], h[2 * p], prod);
                        prod = fmaf(w2[2 * p + 1], h[2 * p + 1], prod);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < MT; u++) {
                        h[u] = act[u] ? sigmoid_scaled(kScale * zc[u]) : 0.f;
                        prod = fmaf(w2[u], h[u], prod);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
                float zo = prod;
                if constexpr (!ONEW) {
                    if ((threadIdx.x & 31) == 0) red[buf * 16 + (t >> 5)] = prod;
                    bar_sync(nd.bar_id, nthr);
#if GLX_ONLINE_LANE_SUM
                    // each group of 8 lanes holds the <= 8 warp partials, 3 xor shuffles
                    const int kk = threadIdx.x & 7;
                    zo = kk < nd.nwarps ? red[buf * 16 + kk] : 0.f;
                    zo += __shfl_xor_sync(0xffffffffu, zo, 4);
                    zo += __shfl_xor_sync(0xffffffffu, zo, 2);
                    zo += __shfl_xor_sync(0xffffffffu, zo, 1);
#else
                    zo = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; k++)  // <= 8 warps per CTA: predicated, no loop
                        if (k < nd.nwarps) zo += red[buf * 16 + k];
#endif
                    buf ^= 1;
                }
                const float o = sigmoid_scaled(kScale * zo);
                const float d_o = (o - tt) * o * (1.0f - o);
                const float step_o = flr * d_o;
                const float g = gd[r];
                if constexpr (MT % 2 == 0) {
#pragma unroll
                    for (int p = 0; p < MT / 2; p++) {
                        const float2 hp = make_float2(h[2 * p], h[2 * p + 1]);
                        const float2 omh = ffma2(hp, bcast2(-1.0f), bcast2(1.0f));  // 1 - h, one rounding
                        const float2 w2p = make_float2(w2[2 * p], w2[2 * p + 1]);
                        const float2 ns =
                            __fmul2_rn(__fmul2_rn(__fmul2_rn(__fmul2_rn(w2p, bcast2(d_o)), hp), omh), bcast2(-flr));
                        const float2 w2n = ffma2(bcast2(-step_o), hp, w2p);
                        const float2 zn = ffma2(ns, bcast2(g), make_float2(zpre[2 * p], zpre[2 * p + 1]));
                        w2[2 * p] = w2n.x;
                        w2[2 * p + 1] = w2n.y;
                        zc[2 * p] = zn.x;
                        zc[2 * p + 1] = zn.y;
                        nsp[2 * p] = ns.x;
                        nsp[2 * p + 1] = ns.y;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < MT; u++) {
                        const float ns = -flr * (w2[u] * d_o * h[u] * (1.0f - h[u]));
                        w2[u] = fmaf(-step_o, h[u], w2[u]);
                        zc[u] = fmaf(ns, g, zpre[u]);
                        nsp[u] = ns;
                    }
                }
                if (t == 0) b2 -= step_o;
                rp = r;
            }
        }
        const float2* xp2 = reinterpret_cast<const float2*>(xs + rp * SP);
#pragma unroll
        for (int u = 0; u < MT; u++)
#pragma unroll
            for (int q = 0; q < DP / 2; q++) w[u][q] = ffma2(bcast2(nsp[u]), xp2[q], w[u][q]);
    } else {  // (braced: an unbraced discarded `else` swallowed the pragma'd write-back loop below)
    for (int64_t ep = 0; ep < epochs; ep++) {
        for (int64_t r = 0; r < N; r++) {
            const float2* xr2 = reinterpret_cast<const float2*>(xs + (XS ? r * SP : 0));
            if constexpr (!kXs) load_row<float, DP, XS>(x, xs, X, r, D);
            auto xp = [&](int q) { return kXs ? xr2[q] : make_float2(x[2 * q], x[2 * q + 1]); };
            const float tt = XS ? ts[r] : __ldg(T + r);
            float h[MT];
            float prod = (t == 0) ? b2 : 0.f;
#pragma unroll
            for (int u = 0; u < MT; u++) {
                float2 p = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < DP / 2; q++) p = ffma2(w[u][q], xp(q), p);
                h[u] = act[u] ? sigmoid_scaled(kScale * (p.x + p.y)) : 0.f;
                prod = fmaf(w2[u], h[u], prod);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
            if ((threadIdx.x & 31) == 0) red[buf * 16 + (t >> 5)] = prod;
            bar_sync(nd.bar_id, nthr);
            float zo = 0.f;
            for (int k = 0; k < nd.nwarps; k++) zo += red[buf * 16 + k];
            buf ^= 1;
            const float o = sigmoid_scaled(kScale * zo);
            const float d_o = (o - tt) * o * (1.0f - o);
            const float step_o = flr * d_o;
#pragma unroll
            for (int u = 0; u < MT; u++) {
                const float ns = -flr * (w2[u] * d_o * h[u] * (1.0f - h[u]));
#pragma unroll
                for (int q = 0; q < DP / 2; q++) w[u][q] = ffma2(bcast2(ns), xp(q), w[u][q]);
                w2[u] = fmaf(-step_o, h[u], w2[u]);
            }
            if (t == 0) b2 -= step_o;
        }
    }
    }
#pragma unroll
    for (int u = 0; u < MT; u++) {
        const int j = t * MT + u;
        if (!act[u]) continue;
#pragma unroll
        for (int q = 0; q < DP / 2; q++) {
            if (2 * q <= D) w_ih[(int64_t)j * (D + 1) + 2 * q] = w[u][q].x;
            if (2 * q + 1 <= D) w_ih[(int64_t)j * (D + 1) + 2 * q + 1] = w[u][q].y;
        }
        w_ho[j] = w2[u];
    }
    if (t == 0) w_ho[H] = b2;
}

// ref64 online SGD for ONE network of <= 64 hidden units (configs 1/cohorts with
// sequential()): the same operation order as online_sgd_kernel<double> (the
// reference's kernels.py:264-295), with the rows staged once as f64 and the weight
// row held as f64 registers that always carry f32-representable values. Per row
// that removes the f32 -> f64 conversions of x and w from the dot and the update
// (the 512-thread kernel is capped at 128 registers and cannot hold both).
template <int DP>
__global__ void __launch_bounds__(64) online_ref64_small_kernel(float* __restrict__ w_ih, float* __restrict__ w_ho,
                                                               int H, const float* __restrict__ X,
                                                               const float* __restrict__ T, int64_t N, int D,
                                                               int64_t epochs, double lr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* x64 = reinterpret_cast<double*>(smem_raw);  // N x DP, [x, 1, 0...]
    double* t64 = x64 + N * DP;                         // N
    double* prods = t64 + N;                            // 4 blocks x 17
    double* bc = prods + 4 * 17;                        // d_o, step_o
    for (int64_t e = threadIdx.x; e < N * DP; e += blockDim.x) {
        const int64_t r = e / DP;
        const int i = (int)(e - r * DP);
        x64[e] = i < D ? (double)X[r * D + i] : (i == D ? 1.0 : 0.0);
    }
    for (int64_t r = threadIdx.x; r < N; r += blockDim.x) t64[r] = (double)T[r];
    __syncthreads();
    const int j = threadIdx.x;
    const bool active = j < H;
    double w[DP];
#pragma unroll
    for (int i = 0; i < DP; i++) w[i] = (active && i < D) ? (double)w_ih[(int64_t)j * (D + 1) + i] : 0.0;
    double bw = active ? (double)w_ih[(int64_t)j * (D + 1) + D] : 0.0;
    double w2 = active ? (double)w_ho[j] : 0.0;
    double b2 = (double)w_ho[H];
    const int nb = (H + 15) >> 4;
    for (int64_t ep = 0; ep < epochs; ep++) {
        for (int64_t r = 0; r < N; r++) {
            const double* xr = x64 + r * DP;
            float h = 0.0f;
            if (active) {
                double acc = 0.0;
#pragma unroll
                for (int b0 = 0; b0 < DP; b0 += 16) {
                    double part = 0.0;
#pragma unroll
                    for (int k = 0; k < 16; k++) {
                        const int i = b0 + k;
                        if (i < DP && i < D) part = fma(w[i < DP ? i : 0], xr[i < DP ? i : 0], part);
                    }
                    if (b0 < D) acc = __dadd_rn(acc, part);
                }
                const double z = __dadd_rn(acc, bw);
                h = __double2float_rn(1.0 / (1.0 + exp(-z)));
                prods[(j >> 4) * 17 + (j & 15)] = w2 * (double)h;  // exact product
            }
            __syncthreads();
            if (j < 32) {  // the output neuron (kernels.py:277-289)
                double part = 0.0;
                if (j < nb) {
                    const int jn = min(16, H - j * 16);
                    // unrolled and predicated: the 16 loads issue ahead of the dependent
                    // sequential adds (the reference's in-block order is kept)
                    double pv[16];
#pragma unroll
                    for (int k = 0; k < 16; k++) pv[k] = k < jn ? prods[j * 17 + k] : 0.0;
#pragma unroll
                    for (int k = 0; k < 16; k++)
                        if (k < jn) part = __dadd_rn(part, pv[k]);
                }
                double z = 0.0;
                for (int b = 0; b < nb; b++) z = __dadd_rn(z, __shfl_sync(0xffffffffu, part, b));
                if (j == 0) {
                    z = __dadd_rn(z, b2);
                    const double od = (double)__double2float_rn(1.0 / (1.0 + exp(-z)));
                    const double d_o = __dmul_rn(__dmul_rn(__dsub_rn(od, t64[r]), od), __dsub_rn(1.0, od));
                    bc[0] = d_o;
                    bc[1] = __dmul_rn(lr, d_o);
                }
            }
            __syncthreads();
            const double d_o = bc[0], step_o = bc[1];
            if (active) {  // hidden first, from the pre-update w_ho (kernels.py:290-292)
                const double hd = (double)h;
                const double d_h = __dmul_rn(__dmul_rn(__dmul_rn(w2, d_o), hd), __dsub_rn(1.0, hd));
                const double s = __dmul_rn(lr, d_h);
#pragma unroll
                for (int i = 0; i < DP; i++)
                    if (i < D) w[i] = (double)__double2float_rn(__dsub_rn(w[i], __dmul_rn(s, xr[i])));
                bw = (double)__double2float_rn(__dsub_rn(bw, s));
                w2 = (double)__double2float_rn(__dsub_rn(w2, __dmul_rn(step_o, hd)));
            }
            if (j == 0) b2 = (double)__double2float_rn(__dsub_rn(b2, step_o));
        }
    }
    if (active) {
#pragma unroll
        for (int i = 0; i < DP; i++)
            if (i < D) w_ih[(int64_t)j * (D + 1) + i] = (float)w[i];
        w_ih[(int64_t)j * (D + 1) + D] = (float)bw;
        w_ho[j] = (float)w2;
    }
    if (j == 0) w_ho[H] = (float)b2;
}

size_t online_ref64_small_smem(int64_t N, int D) {
    const int dp = online_dp_for(D);
    return (size_t)N * dp * 8 + (size_t)N * 8 + 4 * 17 * 8 + 16;
}

cudaError_t launch_online_ref64_small(float* w_ih, float* w_ho, int H, const float* X, const float* T, int64_t N,
                                      int D, int64_t epochs, double lr, cudaStream_t st) {
    const size_t smem = online_ref64_small_smem(N, D);
    const int threads = H <= 32 ? 32 : 64;
    const int dp = online_dp_for(D);
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kernel) {
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) kernel<<<1, threads, smem, st>>>(w_ih, w_ho, H, X, T, N, D, epochs, lr);
    };
    switch (dp) {
        case 8: go(online_ref64_small_kernel<8>); break;
        case 16: go(online_ref64_small_kernel<16>); break;
        case 34: go(online_ref64_small_kernel<34>); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ launcher
template <int DP, int MT>
static cudaError_t launch_online_mt(const OnlineLaunch& L, cudaStream_t st) {
    const size_t smem = L.smem_bytes;
    auto k = L.x_in_smem ? (L.one_warp && MT == 2 ? online_sgd_mt_kernel<DP, MT, true, true>
                                                  : online_sgd_mt_kernel<DP, MT, true>)
                         : online_sgd_mt_kernel<DP, MT, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<L.n_ctas, L.threads, smem, st>>>(L.nets, L.cta_nets, L.X, L.T, L.N, L.D, L.epochs, L.lr);
    return cudaGetLastError();
}

template <typename Real, int DP>
static cudaError_t launch_online_dp(const OnlineLaunch& L, cudaStream_t st) {
    if constexpr (sizeof(Real) == 4) {
        if (L.mt == 2) return launch_online_mt<DP, 2>(L, st);
        if (L.mt == 4) return launch_online_mt<DP, 4>(L, st);
    }
    const size_t smem = L.smem_bytes;
    if (L.x_in_smem) {
        auto k = online_sgd_kernel<Real, DP, true>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<L.n_ctas, L.threads, smem, st>>>(L.nets, L.cta_nets, L.X, L.T, L.N, L.D, L.epochs, L.lr);
    } else {
        auto k = online_sgd_kernel<Real, DP, false>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<L.n_ctas, L.threads, smem, st>>>(L.nets, L.cta_nets, L.X, L.T, L.N, L.D, L.epochs, L.lr);
    }
    return cudaGetLastError();
}

int online_dp_for(int D) {
    if (D + 1 <= 8) return 8;
    if (D + 1 <= 16) return 16;
    if (D + 1 <= 34) return 34;
    if (D + 1 <= 64) return 64;
    return -1;
}

cudaError_t launch_online(const OnlineLaunch& L, cudaStream_t st) {
    const int dp = online_dp_for(L.D);
    if (L.ref64) {
        switch (dp) {
            case 8: return launch_online_dp<double, 8>(L, st);
            case 16: return launch_online_dp<double, 16>(L, st);
            case 34: return launch_online_dp<double, 34>(L, st);
            case 64: return launch_online_dp<double, 64>(L, st);
        }
    } else {
        switch (dp) {
            case 8: return launch_online_dp<float, 8>(L, st);
            case 16: return launch_online_dp<float, 16>(L, st);
            case 34: return launch_online_dp<float, 34>(L, st);
            case 64: return launch_online_dp<float, 64>(L, st);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace glx
