// glx_batch.cu -- full-batch gradient descent epoch for the 1-hidden-layer
// sigmoid MLP (configs 2 and 4), plus the fused
// accuracy/loss evaluation pass (kernels.py:352-375 eval_counts).
//
// One persistent CTA per SM streams row tiles of the packed sample matrix
// (HBM row layout [x_0..x_{D-1}, 1, t, 0..], LD floats) into a
// 3-stage shared-memory ring with 1-D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx). The CTA is warp-specialised:
//
//   warps 0-3  FORWARD   each thread owns MT hidden units of a row group and
//                        holds their W1 rows (pre-scaled by -log2 e, bias in
//                        slot D) in registers; z = W1 x as FFMA2 (packed
//                        f32x2) chains, h = 1/(1+2^z) (MUFU ex2 + rcp), the
//                        per-thread output partial sum_j w2_j h_j to smem,
//                        h to the H tile; then per row o, delta_o, loss,
//                        confusion counts.
//   warps 4-7  BACKWARD  each thread owns the dW1 accumulators of MT hidden
//                        units (MT x DP registers) and folds every row in:
//                        v = delta_o*h, s = v - v*h (= delta_o h(1-h)),
//                        acc[u][:] += s * [x,1] as FFMA2 with a broadcast
//                        scalar, acc2[u] += v. Because K = 1 and W2 is fixed
//                        within an epoch, dW1[j][:] = w2_j * acc[j][:] is
//                        applied once per epoch in the update kernel.
//   thread 0 of the forward warps doubles as the TMA producer: it keeps two
//   tiles in flight ahead of the forward pass in a 4-stage ring (8 warps per
//   CTA = 2 per SM sub-partition, so each thread may use up to 255 registers).
//
// Forward and backward warps hand tiles over through double-buffered H /
// delta_o tiles and named barriers (bar.arrive / bar.sync pairs), so the two
// halves of every row's work overlap on the FMA pipe. Per-CTA gradient
// partials are reduced deterministically (fixed CTA order, f64) by
// batch_update_kernel, which also applies W <- f32(f64(W) - lr/N * grad).
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>
#include <cstdio>

namespace glx {

#ifndef GLX_NW
#define GLX_NW 4
#endif
#ifndef GLX_FROWS
#define GLX_FROWS 2
#endif
#ifndef GLX_BROWS
#define GLX_BROWS 2
#endif
#ifndef GLX_PACK_SCALARS
#define GLX_PACK_SCALARS 0  // packed f32x2 for the per-unit scalar math (runs on fmaheavy like FFMA2)
#endif
#ifndef GLX_MAXMT
#define GLX_MAXMT 4  // max hidden units per thread (register tile)
#endif
#ifndef GLX_TILE_ROWS
#define GLX_TILE_ROWS 256  // target rows per tile (shared memory permitting)
#endif
constexpr int kNF = GLX_NW;  // forward warps
constexpr int kNB = GLX_NW;  // backward warps
constexpr int kNX = 4;  // x tile stages
constexpr int kFT = kNF * 32;
constexpr int kBT = kNB * 32;
constexpr int kBarF = 1, kBarHFull = 2, kBarHEmpty = 4, kBarEpi = 6;

struct BatchArgs {
    const float* Xp;
    const float* Wk;
    float* part;
    int64_t N, ntiles;
    int D, LD, H, HP, TPG, G, R, RPG, P1, PS;
};

template <int DP, int MT, bool TRAIN>
__global__ void __launch_bounds__(kFT + (TRAIN ? kBT : 0), 1) batch_epoch_kernel(const BatchArgs a) {
    constexpr int NBT = TRAIN ? kBT : 0;
    constexpr int NTH = kFT + NBT;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* xfull = reinterpret_cast<uint64_t*>(sm);
    uint64_t* xempty = xfull + kNX;
    float* stat = reinterpret_cast<float*>(sm + 128);  // kFT x 5 (loss, tp, tn, fp, fn)
    float* xbuf = stat + kFT * 5;                      // ring; reused as the epilogue area
    float* hbuf = xbuf + kNX * a.R * a.LD;
    float* dobuf = hbuf + (TRAIN ? 2 * a.R * a.HP : 0);
    float* opart = dobuf + (TRAIN ? 2 * a.R : 0);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t bx = blockIdx.x;
    const int nk = bx < a.ntiles ? (int)((a.ntiles - bx + gridDim.x - 1) / gridDim.x) : 0;

    if (tid == 0) {
        for (int s = 0; s < kNX; s++) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], TRAIN ? kNB : kNF);
        }
        fence_mbar_init();
    }
    // zero the x ring so the unfilled tail rows of the last tile stay finite
    for (int e = tid; e < kNX * a.R * a.LD; e += NTH) xbuf[e] = 0.0f;
    fence_proxy_async();
    __syncthreads();

    const float* Wk = a.Wk;
    // TMA producer (forward thread 0): tile k -> ring slot k % kNX
    auto issue = [&](int k) {
        const int s = k % kNX;
        if (k >= kNX) mbar_wait(&xempty[s], ((k / kNX) - 1) & 1);
        const int64_t t = bx + (int64_t)k * gridDim.x;
        const int64_t rows = min((int64_t)a.R, a.N - t * a.R);
        const uint32_t bytes = (uint32_t)(rows * a.LD * 4);
        mbar_arrive_expect_tx(&xfull[s], bytes);
        bulk_g2s(xbuf + s * a.R * a.LD, a.Xp + t * a.R * a.LD, bytes, &xfull[s]);
    };
    if (warp < kNF) {
        // ------------------------------------------------------------- forward
        const int f = tid;
        const int g = f / a.TPG, jq = f - (f / a.TPG) * a.TPG;
        const bool fv = g < a.G;
        float2 w[MT][DP / 2];
        float w2s[MT];
#pragma unroll
        for (int u = 0; u < MT; u++) {
            const int j = fv ? jq * MT + u : 0;
            const float2* src = reinterpret_cast<const float2*>(Wk + (int64_t)j * DP);
#pragma unroll
            for (int q = 0; q < DP / 2; q++) w[u][q] = fv ? src[q] : make_float2(0.f, 0.f);
            w2s[u] = fv ? Wk[a.H * DP + j] : 0.f;
        }
        const float b2s = Wk[a.H * DP + a.H];
        float loss = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        if (tid == 0)
            for (int k = 0; k < 3 && k < nk; k++) issue(k);
        for (int k = 0; k < nk; k++) {
            const int s = k % kNX, hb = k & 1;
            const int64_t t = bx + (int64_t)k * gridDim.x;
            if (TRAIN && k >= 2) bar_sync(kBarHEmpty + hb, kFT + NBT);
            // slot of tile k+2 last held tile k-2, which both consumers have released
            if (tid == 0 && k >= 1 && k + 2 < nk) issue(k + 2);
            mbar_wait(&xfull[s], (k / kNX) & 1);
            const float* xt = xbuf + s * a.R * a.LD;
            float* op = opart + hb * a.R * (a.TPG + 1);
            float* hrow = hbuf + hb * a.R * a.HP;
            if (fv) {
                // FR rows per step, software-pipelined: the FFMA2 chains of step i+1
                // are issued in the same basic block as the sigmoid / output-partial
                // tail of step i, so MUFU latency hides under FMA work
                constexpr int FR = GLX_FROWS;
                auto chains = [&](int rr, float2 (&p)[FR][MT]) {
                    const float* xr[FR];
#pragma unroll
                    for (int f2 = 0; f2 < FR; f2++) xr[f2] = xt + (g + (rr + f2) * a.G) * a.LD;
#pragma unroll
                    for (int f2 = 0; f2 < FR; f2++)
#pragma unroll
                        for (int u = 0; u < MT; u++) p[f2][u] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q4 = 0; q4 < DP / 4; q4++) {
                        float4 v[FR];
#pragma unroll
                        for (int f2 = 0; f2 < FR; f2++) v[f2] = reinterpret_cast<const float4*>(xr[f2])[q4];
#pragma unroll
                        for (int u = 0; u < MT; u++) {
#pragma unroll
                            for (int f2 = 0; f2 < FR; f2++)
                                p[f2][u] = ffma2(w[u][2 * q4], make_float2(v[f2].x, v[f2].y), p[f2][u]);
#pragma unroll
                            for (int f2 = 0; f2 < FR; f2++)
                                p[f2][u] = ffma2(w[u][2 * q4 + 1], make_float2(v[f2].z, v[f2].w), p[f2][u]);
                        }
                    }
                    if (DP % 4) {
#pragma unroll
                        for (int f2 = 0; f2 < FR; f2++) {
                            const float2 v = reinterpret_cast<const float2*>(xr[f2])[DP / 2 - 1];
#pragma unroll
                            for (int u = 0; u < MT; u++) p[f2][u] = ffma2(w[u][DP / 2 - 1], v, p[f2][u]);
                        }
                    }
                };
                auto finish = [&](int rr, const float2 (&p)[FR][MT]) {
#pragma unroll
                    for (int f2 = 0; f2 < FR; f2++) {
                        const int row = g + (rr + f2) * a.G;
                        float h[MT];
                        float osum;
                        if constexpr (MT % 2 == 0 && GLX_PACK_SCALARS) {
                            // unit pairs share packed f32x2 adds / FMAs
                            float2 os = make_float2(0.f, 0.f);
#pragma unroll
                            for (int u = 0; u < MT; u += 2) {
                                const float2 z = __fadd2_rn(make_float2(p[f2][u].x, p[f2][u + 1].x),
                                                            make_float2(p[f2][u].y, p[f2][u + 1].y));
#ifdef GLX_DEBUG_NOSIGMOID
                                h[u] = z.x;
                                h[u + 1] = z.y;
#else
                                const float2 e1 = __fadd2_rn(make_float2(ex2_approx(z.x), ex2_approx(z.y)),
                                                             make_float2(1.f, 1.f));
                                h[u] = rcp_approx(e1.x);
                                h[u + 1] = rcp_approx(e1.y);
#endif
                                os = ffma2(make_float2(w2s[u], w2s[u + 1]), make_float2(h[u], h[u + 1]), os);
                            }
                            osum = os.x + os.y;
                        } else {
                            osum = 0.f;
#pragma unroll
                            for (int u = 0; u < MT; u++) {
                                h[u] = sigmoid_scaled(p[f2][u].x + p[f2][u].y);
                                osum = fmaf(w2s[u], h[u], osum);
                            }
                        }
                        if (TRAIN) store_units<MT>(hrow + row * a.HP + jq * MT, h);
                        op[row * (a.TPG + 1) + jq] = osum;
                    }
                };
                // two accumulator sets alternate (no register copies between steps)
                float2 pA[FR][MT], pB[FR][MT];
                chains(0, pA);
                int rr = FR;
                for (; rr + FR < a.RPG; rr += 2 * FR) {
                    chains(rr, pB);
                    finish(rr - FR, pA);
                    chains(rr + FR, pA);
                    finish(rr, pB);
                }
                if (rr < a.RPG) {
                    chains(rr, pB);
                    finish(rr - FR, pA);
                    finish(rr, pB);
                } else {
                    finish(rr - FR, pA);
                }
            }
            bar_sync(kBarF, kFT);
            // per-row output neuron: o, delta_o, loss, confusion (kernels.py:352-375);
            // TPR threads per row split the partial sums, 4 accumulators each
            {
                const int tpr = (2 * a.R <= kFT) ? 2 : 1;
                const int part = f - (f / tpr) * tpr;
                for (int r = f / tpr; r - f / tpr < a.R; r += kFT / tpr) {  // warp-uniform trip count
                    const bool rv = r < a.R;
                    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
                    if (rv) {
                        const float* opr = op + r * (a.TPG + 1);
                        int q = part;
                        for (; q + 3 * tpr < a.TPG; q += 4 * tpr) {
                            z0 += opr[q];
                            z1 += opr[q + tpr];
                            z2 += opr[q + 2 * tpr];
                            z3 += opr[q + 3 * tpr];
                        }
                        for (; q < a.TPG; q += tpr) z0 += opr[q];
                    }
                    float zo = (z0 + z1) + (z2 + z3);
                    if (tpr == 2) zo += __shfl_xor_sync(0xffffffffu, zo, 1);
                    const int64_t grow = t * a.R + r;
                    if (rv && part == 0) {
                        float d = 0.f;
                        if (grow < a.N) {
                            const float o = sigmoid_scaled(zo + b2s);
                            const float tt = xt[r * a.LD + a.D + 1];
                            d = (o - tt) * o * (1.0f - o);
                            loss = fmaf(0.5f * (tt - o), (tt - o), loss);
                            const bool pred = o >= 0.5f, pos = tt >= 0.5f;
                            c0 += (pred && pos) ? 1.f : 0.f;    // tp
                            c1 += (!pred && !pos) ? 1.f : 0.f;  // tn
                            c2 += (pred && !pos) ? 1.f : 0.f;   // fp
                            c3 += (!pred && pos) ? 1.f : 0.f;   // fn
                        }
                        if (TRAIN) dobuf[hb * a.R + r] = d;
                    }
                }
            }
            if (TRAIN) {
                bar_arrive(kBarHFull + hb, kFT + NBT);
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&xempty[s]);
            }
        }
        if (TRAIN) {
            for (int k = (nk >= 2 ? nk - 2 : 0); k < nk; k++) bar_sync(kBarHEmpty + (k & 1), kFT + NBT);
        }
        stat[f * 5 + 0] = loss;
        stat[f * 5 + 1] = c0;
        stat[f * 5 + 2] = c1;
        stat[f * 5 + 3] = c2;
        stat[f * 5 + 4] = c3;
        bar_sync(kBarEpi, NTH);  // (A)
    } else if (TRAIN) {
        // ------------------------------------------------------------ backward
        const int b = tid - kFT;
        const int gb = b / a.TPG, jq = b - (b / a.TPG) * a.TPG;
        const bool bv = gb < a.G;
        float2 acc[MT][DP / 2];
        float acc2[MT];
#pragma unroll
        for (int u = 0; u < MT; u++) {
            acc2[u] = 0.f;
#pragma unroll
            for (int q = 0; q < DP / 2; q++) acc[u][q] = make_float2(0.f, 0.f);
        }
        float dsum = 0.f;
        for (int k = 0; k < nk; k++) {
            const int s = k % kNX, hb = k & 1;
            bar_sync(kBarHFull + hb, kFT + NBT);
            mbar_wait(&xfull[s], (k / kNX) & 1);
            const float* xt = xbuf + s * a.R * a.LD;
            const float* hrow = hbuf + hb * a.R * a.HP;
            const float* dr = dobuf + hb * a.R;
            if (bv) {
                // BR rows per iteration; the next rows' delta_o and h are prefetched
                constexpr int BR = GLX_BROWS;
                float dn[BR], hn[BR][MT];
#pragma unroll
                for (int b2 = 0; b2 < BR; b2++) {
                    dn[b2] = dr[gb + b2 * a.G];
                    load_units<MT>(hrow + (gb + b2 * a.G) * a.HP + jq * MT, hn[b2]);
                }
#ifdef GLX_DEBUG_NOB
                if (a.N > 0) {} else
#endif
                for (int rr = 0; rr < a.RPG; rr += BR) {
                    float sv[BR][MT];
                    const float* xr[BR];
#pragma unroll
                    for (int b2 = 0; b2 < BR; b2++) {
                        xr[b2] = xt + (gb + (rr + b2) * a.G) * a.LD;
                        const float d = dn[b2];
                        if constexpr (MT % 2 == 0 && GLX_PACK_SCALARS) {
#pragma unroll
                            for (int u = 0; u < MT; u += 2) {
                                const float2 hh = make_float2(hn[b2][u], hn[b2][u + 1]);
                                const float2 v = __fmul2_rn(bcast2(d), hh);
                                const float2 t = ffma2(make_float2(-v.x, -v.y), hh, v);
                                sv[b2][u] = t.x;
                                sv[b2][u + 1] = t.y;
                                const float2 a2 = __fadd2_rn(make_float2(acc2[u], acc2[u + 1]), v);
                                acc2[u] = a2.x;
                                acc2[u + 1] = a2.y;
                            }
                        } else {
#pragma unroll
                            for (int u = 0; u < MT; u++) {
                                const float v = d * hn[b2][u];
                                sv[b2][u] = fmaf(-v, hn[b2][u], v);
                                acc2[u] += v;
                            }
                        }
                        if (jq == 0) dsum += d;
                    }
                    if (rr + BR < a.RPG) {
#pragma unroll
                        for (int b2 = 0; b2 < BR; b2++) {
                            const int rn = gb + (rr + BR + b2) * a.G;
                            dn[b2] = dr[rn];
                            load_units<MT>(hrow + rn * a.HP + jq * MT, hn[b2]);
                        }
                    }
#pragma unroll
                    for (int q4 = 0; q4 < DP / 4; q4++) {
                        float4 v[BR];
#pragma unroll
                        for (int b2 = 0; b2 < BR; b2++) v[b2] = reinterpret_cast<const float4*>(xr[b2])[q4];
#pragma unroll
                        for (int u = 0; u < MT; u++) {
#pragma unroll
                            for (int b2 = 0; b2 < BR; b2++) {
                                acc[u][2 * q4] = ffma2(bcast2(sv[b2][u]), make_float2(v[b2].x, v[b2].y), acc[u][2 * q4]);
                                acc[u][2 * q4 + 1] =
                                    ffma2(bcast2(sv[b2][u]), make_float2(v[b2].z, v[b2].w), acc[u][2 * q4 + 1]);
                            }
                        }
                    }
                    if (DP % 4) {
#pragma unroll
                        for (int b2 = 0; b2 < BR; b2++) {
                            const float2 v = reinterpret_cast<const float2*>(xr[b2])[DP / 2 - 1];
#pragma unroll
                            for (int u = 0; u < MT; u++)
                                acc[u][DP / 2 - 1] = ffma2(bcast2(sv[b2][u]), v, acc[u][DP / 2 - 1]);
                        }
                    }
                }
            }
            bar_arrive(kBarHEmpty + hb, kFT + NBT);
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[s]);
        }
        bar_sync(kBarEpi, NTH);  // (A) every warp is past the tile loop: the ring is free
        float* epi = xbuf;  // [G][H][DP] | [G][H] | [G]
        float* epi2 = epi + a.G * a.H * DP;
        float* epi3 = epi2 + a.G * a.H;
        if (bv) {
#pragma unroll
            for (int u = 0; u < MT; u++) {
                float2* dst = reinterpret_cast<float2*>(epi + ((int64_t)gb * a.H + jq * MT + u) * DP);
#pragma unroll
                for (int q = 0; q < DP / 2; q++) dst[q] = acc[u][q];
                epi2[gb * a.H + jq * MT + u] = acc2[u];
            }
            if (jq == 0) epi3[gb] = dsum;
        }
    }
    bar_sync(kBarEpi, NTH);  // (B) epilogue staging complete

    // ----------------------------------------------------- epilogue: partials
    float* out = a.part + bx * (int64_t)a.PS;
    if (TRAIN) {
        const float* epi = xbuf;
        const float* epi2 = epi + a.G * a.H * DP;
        const float* epi3 = epi2 + a.G * a.H;
        const int D1 = a.D + 1;
        for (int e = tid; e < a.P1; e += NTH) {
            const int j = e / D1, i = e - (e / D1) * D1;
            float s = 0.f;
            for (int gg = 0; gg < a.G; gg++) s += epi[((int64_t)gg * a.H + j) * DP + i];
            out[e] = s;
        }
        for (int j = tid; j < a.H; j += NTH) {
            float s = 0.f;
            for (int gg = 0; gg < a.G; gg++) s += epi2[gg * a.H + j];
            out[a.P1 + j] = s;
        }
        if (tid == 0) {
            float s = 0.f;
            for (int gg = 0; gg < a.G; gg++) s += epi3[gg];
            out[a.P1 + a.H] = s;
        }
    }
    if (tid < 5) {
        float s = 0.f;
        for (int f = 0; f < kFT; f++) s += stat[f * 5 + tid];
        out[a.P1 + a.H + 1 + tid] = s;
    }
}

// ------------------------------------------------------------- update kernel
// f64 sum of one record slot over the per-CTA partial records: a block is
// kRedW warps x 32 consecutive slots (coalesced 128-byte rows), warp l takes
// records l, l+kRedW, ... (about ten independent loads per thread for 148
// records); the kRedW sums are added in a fixed order (deterministic)
constexpr int kRedW = 16;
__device__ __forceinline__ double reduce_partials(const float* __restrict__ part, int nparts, int PS, int idx,
                                                  int nidx, double* red) {
    const int l = threadIdx.x >> 5, i = threadIdx.x & 31;
    double s = 0.0;
    if (idx < nidx) {
#pragma unroll 10
        for (int c = l; c < nparts; c += kRedW) s += (double)part[(int64_t)c * PS + idx];
    }
    red[l * 32 + i] = s;
    __syncthreads();
    if (l != 0) return 0.0;
    double t = red[i];
#pragma unroll
    for (int k = 1; k < kRedW; k++) t += red[k * 32 + i];
    return t;
}

__global__ void batch_update_kernel(const float* __restrict__ part, int nparts, int PS, int D, int H, int DP,
                                    float* __restrict__ W1, float* __restrict__ W2, const float* __restrict__ Wk_cur,
                                    float* __restrict__ Wk_next, double lr_over_n, int train,
                                    double* __restrict__ stats, int* __restrict__ nonfinite) {
    __shared__ double red[kRedW * 32];
    const int P1 = H * (D + 1);
    const int nidx = P1 + H + 1 + 5;
    const int idx = blockIdx.x * 32 + (threadIdx.x & 31);
    const double s = reduce_partials(part, nparts, PS, idx, nidx, red);
    if ((threadIdx.x >> 5) != 0 || idx >= nidx) return;
    const float kScale = (float)(-GLX_LOG2E);
    if (idx >= P1 + H + 1) {
        if (stats) stats[idx - (P1 + H + 1)] = s;
        return;
    }
    if (!train) return;
    const float* w2r_cur = Wk_cur + H * DP + H + 1;
    float wnew;
    if (idx < P1) {
        const int j = idx / (D + 1), i = idx - (idx / (D + 1)) * (D + 1);
        const double grad = (double)w2r_cur[j] * s;
        wnew = __double2float_rn((double)W1[idx] - lr_over_n * grad);
        W1[idx] = wnew;
        Wk_next[j * DP + i] = kScale * wnew;
    } else if (idx < P1 + H) {
        const int j = idx - P1;
        wnew = __double2float_rn((double)W2[j] - lr_over_n * s);
        W2[j] = wnew;
        Wk_next[H * DP + j] = kScale * wnew;
        Wk_next[H * DP + H + 1 + j] = wnew;
    } else {
        wnew = __double2float_rn((double)W2[H] - lr_over_n * s);
        W2[H] = wnew;
        Wk_next[H * DP + H] = kScale * wnew;
    }
    if (!isfinite(wnew) && nonfinite) atomicOr(nonfinite, 1);
}

__global__ void batch_prep_kernel(const float* __restrict__ W1, const float* __restrict__ W2, float* __restrict__ Wk0,
                                  float* __restrict__ Wk1, int D, int H, int DP) {
    const float kScale = (float)(-GLX_LOG2E);
    const int n1 = H * DP;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n1 + 2 * H + 1; e += gridDim.x * blockDim.x) {
        float v;
        if (e < n1) {
            const int j = e / DP, i = e - (e / DP) * DP;
            v = i <= D ? kScale * W1[j * (D + 1) + i] : 0.0f;
            if (i > D) Wk1[e] = 0.0f;
        } else if (e < n1 + H + 1) {
            v = kScale * W2[e - n1];
        } else {
            v = W2[e - (n1 + H + 1)];
        }
        Wk0[e] = v;
    }
}

__global__ void pack_rows_kernel(const float* __restrict__ X, const float* __restrict__ T,
                                 const uint8_t* __restrict__ labels, int64_t N, int D, int LD, float* __restrict__ Xp,
                                 const float* __restrict__ col_min, const float* __restrict__ col_max) {
    const int64_t total = N * LD;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / LD;
        const int i = (int)(e - r * LD);
        float v;
        if (i < D) v = col_min ? minmax_norm(X[r * D + i], col_min[i], col_max[i]) : X[r * D + i];
        else if (i == D) v = 1.0f;
        else if (i == D + 1) v = T ? T[r] : (labels ? (float)labels[r] : 0.0f);
        else v = 0.0f;
        Xp[e] = v;
    }
}

// DP split (config 4): this rank's gradient SUM in f64 -> grad[], with the
// w2_j factor folded into the dW1 rows so that apply is a plain axpy.
__global__ void batch_grad_kernel(const float* __restrict__ part, int nparts, int PS, int D, int H, int DP,
                                  const float* __restrict__ Wk, double* __restrict__ grad) {
    __shared__ double red[kRedW * 32];
    const int P1 = H * (D + 1);
    const int nidx = P1 + H + 1 + 5;
    const int idx = blockIdx.x * 32 + (threadIdx.x & 31);
    double s = reduce_partials(part, nparts, PS, idx, nidx, red);
    if ((threadIdx.x >> 5) != 0 || idx >= nidx) return;
    if (idx < P1) {
        const int j = idx / (D + 1);
        s *= (double)Wk[H * DP + H + 1 + j];
    }
    grad[idx] = s;
}

__global__ void batch_apply_kernel(int D, int H, float* __restrict__ W1, float* __restrict__ W2,
                                   const double* __restrict__ grad, double lr_over_n, int* __restrict__ nonfinite) {
    const int P1 = H * (D + 1);
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P1 + H + 1) return;
    float* w = idx < P1 ? W1 + idx : W2 + (idx - P1);
    const float wnew = __double2float_rn((double)*w - lr_over_n * grad[idx]);
    *w = wnew;
    if (!isfinite(wnew) && nonfinite) atomicOr(nonfinite, 1);
}

// DP epoch tail (config 4, after the all-reduce of grad): the update of
// batch_apply_kernel plus the next epoch's pre-scaled weight copy (as
// batch_update_kernel writes it) and the epoch statistics into stats_slot.
__global__ void batch_dp_update_kernel(int D, int H, int DP, float* __restrict__ W1, float* __restrict__ W2,
                                       float* __restrict__ Wk_next, const double* __restrict__ grad, double lr_over_n,
                                       double* __restrict__ stats_slot, int* __restrict__ nonfinite) {
    const int P1 = H * (D + 1);
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const float kScale = (float)(-GLX_LOG2E);
    if (idx >= P1 + H + 1) {
        if (idx < P1 + H + 6 && stats_slot) stats_slot[idx - (P1 + H + 1)] = grad[idx];
        return;
    }
    float wnew;
    if (idx < P1) {
        const int j = idx / (D + 1), i = idx - j * (D + 1);
        wnew = __double2float_rn((double)W1[idx] - lr_over_n * grad[idx]);
        W1[idx] = wnew;
        Wk_next[j * DP + i] = kScale * wnew;
    } else if (idx < P1 + H) {
        const int j = idx - P1;
        wnew = __double2float_rn((double)W2[j] - lr_over_n * grad[idx]);
        W2[j] = wnew;
        Wk_next[H * DP + j] = kScale * wnew;
        Wk_next[H * DP + H + 1 + j] = wnew;
    } else {
        wnew = __double2float_rn((double)W2[H] - lr_over_n * grad[idx]);
        W2[H] = wnew;
        Wk_next[H * DP + H] = kScale * wnew;
    }
    if (!isfinite(wnew) && nonfinite) atomicOr(nonfinite, 1);
}

cudaError_t launch_batch_dp_update(const BatchGeom& g, float* W1, float* W2, float* Wk_next, const double* grad,
                                   double lr_over_n, double* stats_slot, int* nonfinite, cudaStream_t st) {
    const int n = g.P1 + g.H + 1 + 5;
    batch_dp_update_kernel<<<(n + 255) / 256, 256, 0, st>>>(g.D, g.H, g.DP, W1, W2, Wk_next, grad, lr_over_n,
                                                            stats_slot, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_batch_grad(const BatchGeom& g, const float* part, const float* Wk, double* grad, cudaStream_t st) {
    const int nidx = g.P1 + g.H + 1 + 5;
    batch_grad_kernel<<<(nidx + 31) / 32, kRedW * 32, 0, st>>>(part, g.grid, g.PS, g.D, g.H, g.DP, Wk, grad);
    return cudaGetLastError();
}

cudaError_t launch_batch_apply(int D, int H, float* W1, float* W2, const double* grad, double lr_over_n,
                               int* nonfinite, cudaStream_t st) {
    const int n = H * (D + 1) + H + 1;
    batch_apply_kernel<<<(n + 255) / 256, 256, 0, st>>>(D, H, W1, W2, grad, lr_over_n, nonfinite);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
// weight-row stride (the [W1 | b1] row in registers, float2 pairs): the kernels are
// instantiated for these widths; D + 1 <= 128 (kernels.py:264-295 takes any D)
int pick_dp(int D) {
    for (int dp : {8, 16, 34, 48, 64, 128})
        if (D + 1 <= dp) return dp;
    return -1;
}

static size_t batch_smem(const BatchGeom& g, bool train) {
    size_t f = 0;
    f += (size_t)kNX * g.R * g.LD;
    if (train) f += 2 * (size_t)g.R * g.HP + 2 * (size_t)g.R;
    f += 2 * (size_t)g.R * (g.TPG + 1);
    size_t epi = train ? ((size_t)g.G * g.H * g.DP + (size_t)g.G * g.H + g.G) : 0;
    return 128 + 4 * ((size_t)kFT * 5 + (f > epi ? f : epi));
}

bool batch_geometry(int64_t N, int D, int H, int n_sms, bool train, BatchGeom* g) {
    BatchGeom q{};
    q.D = D;
    q.H = H;
    q.N = N;
    q.DP = pick_dp(D);
    if (q.DP < 0 || H < 1 || N < 1) return false;
    q.LD = ((std::max(D + 2, q.DP)) + 3) / 4 * 4;
    q.MT = 0;
    for (int mt : {4, 3, 2, 1})
        if (mt <= GLX_MAXMT && (q.DP <= 34 || mt <= 2) && (q.DP < 128 || mt == 1) && H % mt == 0 &&
            H / mt <= kFT) {
            q.MT = mt;
            break;
        }
    if (!q.MT) return false;
    q.TPG = H / q.MT;
    q.G = std::min(kFT / q.TPG, kFT / 2);  // rows come in pairs, <= kFT rows per tile
    q.HP = (H + 3) / 4 * 4;
    q.P1 = H * (D + 1);
    q.PS = (q.P1 + H + 6 + 3) / 4 * 4;
    q.WKS = (H * q.DP + 2 * H + 1 + 3) / 4 * 4;
    // rows per tile: a multiple of G, <= 128 (one finalising thread per row), as
    // large as the shared-memory budget allows (target 64)
    int rpg = (GLX_TILE_ROWS + q.G - 1) / q.G;
    rpg += rpg & 1;  // the row loops take rows in pairs
    for (;; rpg -= 2) {
        if (rpg < 2) return false;
        q.RPG = rpg;
        q.R = q.G * rpg;
        if (q.R > 4 * kFT) continue;
        q.smem = batch_smem(q, train);
        if (q.smem <= 227 * 1024) break;
    }
    q.ntiles = (N + q.R - 1) / q.R;
    q.grid = (int)std::min<int64_t>(q.ntiles, n_sms);
    *g = q;
    return true;
}

template <int DP, int MT, bool TRAIN>
static cudaError_t launch_t(const BatchGeom& g, const BatchArgs& a, cudaStream_t st) {
    auto k = batch_epoch_kernel<DP, MT, TRAIN>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) {
        fprintf(stderr, "glx: batch_epoch_kernel<%d,%d,%d> cudaFuncSetAttribute(smem=%zu): %s\n", DP, MT,
                (int)TRAIN, g.smem, cudaGetErrorString(e));
        return e;
    }
    k<<<g.grid, kFT + (TRAIN ? kBT : 0), g.smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        fprintf(stderr, "glx: batch_epoch_kernel<%d,%d,%d> launch grid=%d smem=%zu: %s\n", DP, MT, (int)TRAIN,
                g.grid, g.smem, cudaGetErrorString(e));
    return e;
}

template <int DP, bool TRAIN>
static cudaError_t launch_mt(const BatchGeom& g, const BatchArgs& a, cudaStream_t st) {
    if constexpr (DP <= 34) {  // wide rows: at most 2 units per thread (register tile)
        switch (g.MT) {
            case 4: return launch_t<DP, 4, TRAIN>(g, a, st);
            case 3: return launch_t<DP, 3, TRAIN>(g, a, st);
        }
    }
    if constexpr (DP < 128)
        if (g.MT == 2) return launch_t<DP, 2, TRAIN>(g, a, st);
    if (g.MT == 1) return launch_t<DP, 1, TRAIN>(g, a, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_batch_epoch(const BatchGeom& g, const float* Xp, const float* Wk, float* part, bool train,
                               cudaStream_t st) {
    BatchArgs a;
    a.Xp = Xp;
    a.Wk = Wk;
    a.part = part;
    a.N = g.N;
    a.ntiles = g.ntiles;
    a.D = g.D;
    a.LD = g.LD;
    a.H = g.H;
    a.HP = g.HP;
    a.TPG = g.TPG;
    a.G = g.G;
    a.R = g.R;
    a.RPG = g.RPG;
    a.P1 = g.P1;
    a.PS = g.PS;
    if (train) {
        switch (g.DP) {
            case 8: return launch_mt<8, true>(g, a, st);
            case 16: return launch_mt<16, true>(g, a, st);
            case 34: return launch_mt<34, true>(g, a, st);
            case 48: return launch_mt<48, true>(g, a, st);
            case 64: return launch_mt<64, true>(g, a, st);
            case 128: return launch_mt<128, true>(g, a, st);
        }
    } else {
        switch (g.DP) {
            case 8: return launch_mt<8, false>(g, a, st);
            case 16: return launch_mt<16, false>(g, a, st);
            case 34: return launch_mt<34, false>(g, a, st);
            case 48: return launch_mt<48, false>(g, a, st);
            case 64: return launch_mt<64, false>(g, a, st);
            case 128: return launch_mt<128, false>(g, a, st);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_batch_update(const BatchGeom& g, const float* part, float* W1, float* W2, const float* Wk_cur,
                                float* Wk_next, double lr_over_n, bool train, double* stats, int* nonfinite,
                                cudaStream_t st) {
    const int nidx = g.P1 + g.H + 1 + 5;
    const int blocks = (nidx + 31) / 32;
    batch_update_kernel<<<blocks, kRedW * 32, 0, st>>>(part, g.grid, g.PS, g.D, g.H, g.DP, W1, W2, Wk_cur, Wk_next,
                                                lr_over_n, train ? 1 : 0, stats, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_batch_prep(const BatchGeom& g, const float* W1, const float* W2, float* Wk0, float* Wk1,
                              cudaStream_t st) {
    const int n = g.H * g.DP + 2 * g.H + 1;
    batch_prep_kernel<<<(n + 255) / 256, 256, 0, st>>>(W1, W2, Wk0, Wk1, g.D, g.H, g.DP);
    return cudaGetLastError();
}

cudaError_t launch_pack_rows(const float* X, const float* T, const uint8_t* labels, int64_t N, int D, int LD,
                             float* Xp, cudaStream_t st, const float* col_min, const float* col_max) {
    if (pack_tiled_ok(X, T, labels, Xp, D, LD)) return launch_pack_tiled(X, T, labels, N, D, LD, col_min, col_max, Xp, st);
    const int64_t total = N * LD;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (blocks < 1) blocks = 1;
    pack_rows_kernel<<<blocks, 256, 0, st>>>(X, T, labels, N, D, LD, Xp, col_min, col_max);
    return cudaGetLastError();
}

}  // namespace glx
