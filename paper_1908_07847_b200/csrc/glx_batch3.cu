// glx_batch3.cu -- full-batch epoch kernel with three warp-specialised roles.
//
// Same math and partial-record format as batch_epoch_kernel (glx_batch.cu;
// SURVEY.md 8(a) a13), re-split so that the two FFMA2 streams carry no
// scalar work (profiles/r01_summary.md: the forward warps' MUFU/scalar mix
// left the fmaheavy pipe ~35% idle):
//
//   warpgroup 0  FORWARD     z = W1s [x,1] for MT hidden units x 2 rows per
//                            step, W1s (pre-scaled by -log2 e) in registers,
//                            x as float4 broadcasts from the TMA ring; stores z.
//                            Thread 0 is also the TMA producer.
//   warpgroup 2  ACTIVATION  h = 1/(1+2^z) in place, output-neuron partials,
//                            per row o / delta_o / loss / confusion, then
//                            s = delta_o h(1-h) in place and dW2 += delta_o h.
//   warpgroup 1  BACKWARD    acc[u][:] += s * [x,1] (FFMA2, broadcast s).
//
// A tile of R rows flows F -> A -> B through a 3-deep buffer ring (z, then h,
// then s in the same slot), so F(k+2), A(k+1) and B(k) run concurrently.
// Registers move between roles with setmaxnreg: F and B hold 136-float
// register tiles, A needs few.
#include "glx_common.cuh"
#include "glx_kernels.h"

#include <algorithm>
#include <cstdio>

namespace glx {

constexpr int k3WG = 128;
constexpr int k3NT = 3 * k3WG;
#ifndef GLX3_NZ
#define GLX3_NZ 3  // z/h/s tile slots (F on k+2, A on k+1, B on k)
#endif
constexpr int k3NZ = GLX3_NZ;
constexpr int k3NX = k3NZ + 2;  // x ring stages: the z ring plus 2 prefetched
// named barriers: per-slot z-full, s-full, z-empty, then two CTA-wide ones (<= 16)
constexpr int k3ZFull = 1, k3SFull = 1 + k3NZ, k3ZEmpty = 1 + 2 * k3NZ, k3AInt = 1 + 3 * k3NZ, k3Epi = 2 + 3 * k3NZ;
static_assert(k3Epi < 16, "named barrier ids");
#ifndef GLX3_RS
#define GLX3_RS 4  // rows per step in the forward / backward streams (RPG must be a multiple)
#endif
#ifndef GLX3_FWD_BCAST
#define GLX3_FWD_BCAST 0  // forward FFMA2 in broadcast-scalar form (x_i * weight pair of two units)
#endif
#ifndef GLX3_REGS_F
#define GLX3_REGS_F 216
#endif
#ifndef GLX3_REGS_B
#define GLX3_REGS_B 200
#endif
#ifndef GLX3_REGS_A
#define GLX3_REGS_A 88  // F + B + A = 3 * 168: the launch allocation is redistributed exactly
#endif

struct Batch3Args {
    const float* Xp;
    const float* Wk;
    float* part;
    int64_t N, ntiles;
    int D, LD, H, HP;
    int TPG, G, R, RPG;  // forward / backward: MT units per thread, G row groups
    int QR, AG;          // activation: QR unit chunks per row, AG row groups
    int P1, PS;
    int off_dob, off_opart, off_z, off_x;  // float offsets from the stat base
    unsigned long long* dbg;                // GLX3_TIMING builds: per-role cycle counters
};

#ifdef GLX3_TIMING
__device__ unsigned long long g_glx3_dbg[8];
#define T_BEGIN(v) const long long v = clock64()
#define T_ADD(acc, v) acc += clock64() - v
#else
#define T_BEGIN(v)
#define T_ADD(acc, v)
#endif

__device__ __forceinline__ float2 ld_f2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ float4 ld_f4(const float* p) { return *reinterpret_cast<const float4*>(p); }

template <int DP, int MT, int UA>
__global__ void __launch_bounds__(k3NT, 1) batch3_kernel(const Batch3Args a) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* xfull = reinterpret_cast<uint64_t*>(sm);
    uint64_t* xempty = xfull + k3NX;
    float* stat = reinterpret_cast<float*>(sm + 128);  // k3WG x 5 (activation threads)
    float* dob = stat + a.off_dob;                      // R
    float* opart = stat + a.off_opart;                  // R x (QR + 1)
    float* zbuf = stat + a.off_z;                       // k3NZ x R x HP
    float* xbuf = stat + a.off_x;                       // k3NX x R x LD
    float* epi = zbuf;                                  // epilogue staging (after the tile loop)

    const int tid = threadIdx.x;
    const int role = tid / k3WG, rt = tid % k3WG, lane = tid & 31;
    const int64_t bx = blockIdx.x;
    const int nk = bx < a.ntiles ? (int)((a.ntiles - bx + gridDim.x - 1) / gridDim.x) : 0;
    const int RZ = a.R * a.HP;

    if (tid == 0) {
        for (int s = 0; s < k3NX; s++) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], 4);  // one arrival per backward warp
        }
        fence_mbar_init();
    }
    for (int e = tid; e < k3NX * a.R * a.LD; e += k3NT) xbuf[e] = 0.0f;
    fence_proxy_async();
    __syncthreads();

    const float* Wk = a.Wk;
    float* out = a.part + bx * (int64_t)a.PS;

    if (role == 0) {
        // =============================================================== FORWARD
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(GLX3_REGS_F));
        const int f = rt;
        const int g = f / a.TPG, jq = f - (f / a.TPG) * a.TPG;
        const bool fv = g < a.G;
        // broadcast form (MT even): wp[up][i] = (w_{2up,i}, w_{2up+1,i}); else pair-of-inputs form
        constexpr bool kBc = GLX3_FWD_BCAST && (MT % 2 == 0);
        float2 wp[kBc ? MT / 2 : 1][kBc ? DP : 1];
        float2 w[kBc ? 1 : MT][kBc ? 1 : DP / 2];
        if constexpr (kBc) {
#pragma unroll
            for (int up = 0; up < MT / 2; up++) {
                const float* r0 = Wk + (int64_t)(fv ? jq * MT + 2 * up : 0) * DP;
                const float* r1 = Wk + (int64_t)(fv ? jq * MT + 2 * up + 1 : 0) * DP;
#pragma unroll
                for (int i = 0; i < DP; i++) wp[up][i] = fv ? make_float2(r0[i], r1[i]) : make_float2(0.f, 0.f);
            }
        } else {
#pragma unroll
            for (int u = 0; u < MT; u++) {
                const float2* src = reinterpret_cast<const float2*>(Wk + (int64_t)(fv ? jq * MT + u : 0) * DP);
#pragma unroll
                for (int q = 0; q < DP / 2; q++) w[u][q] = fv ? src[q] : make_float2(0.f, 0.f);
            }
        }
#ifdef GLX3_TIMING
        long long t_comp = 0, t_wait = 0;
#endif
        auto issue = [&](int k) {
            const int s = k % k3NX;
            if (k >= k3NX) mbar_wait(&xempty[s], ((k / k3NX) - 1) & 1);
            const int64_t t = bx + (int64_t)k * gridDim.x;
            const int64_t rows = min((int64_t)a.R, a.N - t * a.R);
            const uint32_t bytes = (uint32_t)(rows * a.LD * 4);
            mbar_arrive_expect_tx(&xfull[s], bytes);
            bulk_g2s(xbuf + s * a.R * a.LD, a.Xp + t * a.R * a.LD, bytes, &xfull[s]);
        };
        if (f == 0)
            for (int k = 0; k < 3 && k < nk; k++) issue(k);
        for (int k = 0; k < nk; k++) {
            const int s = k % k3NX, zb = k % k3NZ;
            T_BEGIN(tw);
            if (k >= k3NZ) bar_sync(k3ZEmpty + zb, 2 * k3WG);  // backward is done with tile k-3
            if (f == 0 && k >= 1 && k + 2 < nk) issue(k + 2);  // its slot last held tile k-3
            mbar_wait(&xfull[s], (k / k3NX) & 1);
            T_ADD(t_wait, tw);
            T_BEGIN(tc);
            const float* xt = xbuf + s * a.R * a.LD;
            float* zt = zbuf + zb * RZ;
            if (fv) {
                // RS rows per step: RS*MT independent FFMA2 chains per load latency
                constexpr int RS = GLX3_RS;
                for (int rr = 0; rr < a.RPG; rr += RS) {
                    const float* xr[RS];
#pragma unroll
                    for (int q = 0; q < RS; q++) xr[q] = xt + (g + (rr + q) * a.G) * a.LD;
                    if constexpr (kBc) {
                    float2 zp[RS][MT / 2];
#pragma unroll
                    for (int q = 0; q < RS; q++)
#pragma unroll
                        for (int up = 0; up < MT / 2; up++) zp[q][up] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q4 = 0; q4 < DP / 4; q4++) {
                        float4 v[RS];
#pragma unroll
                        for (int q = 0; q < RS; q++) v[q] = ld_f4(xr[q] + 4 * q4);
#pragma unroll
                        for (int e = 0; e < 4; e++)
#pragma unroll
                            for (int up = 0; up < MT / 2; up++)
#pragma unroll
                                for (int q = 0; q < RS; q++) {
                                    const float xs = e == 0 ? v[q].x : e == 1 ? v[q].y : e == 2 ? v[q].z : v[q].w;
                                    zp[q][up] = ffma2(bcast2(xs), wp[up][(4 * q4 + e) % DP], zp[q][up]);
                                }
                    }
                    if (DP % 4) {
#pragma unroll
                        for (int q = 0; q < RS; q++) {
                            const float2 v = ld_f2(xr[q] + DP - 2);
#pragma unroll
                            for (int up = 0; up < MT / 2; up++) {
                                zp[q][up] = ffma2(bcast2(v.x), wp[up][(DP - 2) % DP], zp[q][up]);
                                zp[q][up] = ffma2(bcast2(v.y), wp[up][(DP - 1) % DP], zp[q][up]);
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < RS; q++) {
                        float z[MT];
#pragma unroll
                        for (int up = 0; up < MT / 2; up++) {
                            z[2 * up] = zp[q][up].x;
                            z[2 * up + 1] = zp[q][up].y;
                        }
                        store_units<MT>(zt + (g + (rr + q) * a.G) * a.HP + jq * MT, z);
                    }
                    } else {
                    float2 p[RS][MT];
#pragma unroll
                    for (int q = 0; q < RS; q++)
#pragma unroll
                        for (int u = 0; u < MT; u++) p[q][u] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q4 = 0; q4 < DP / 4; q4++) {
                        float4 v[RS];
#pragma unroll
                        for (int q = 0; q < RS; q++) v[q] = ld_f4(xr[q] + 4 * q4);
#pragma unroll
                        for (int u = 0; u < MT; u++) {
#pragma unroll
                            for (int q = 0; q < RS; q++) p[q][u] = ffma2(w[u % (kBc ? 1 : MT)][(2 * q4) % (kBc ? 1 : DP / 2)], make_float2(v[q].x, v[q].y), p[q][u]);
#pragma unroll
                            for (int q = 0; q < RS; q++)
                                p[q][u] = ffma2(w[u][2 * q4 + 1], make_float2(v[q].z, v[q].w), p[q][u]);
                        }
                    }
                    if (DP % 4) {
#pragma unroll
                        for (int q = 0; q < RS; q++) {
                            const float2 v = ld_f2(xr[q] + DP - 2);
#pragma unroll
                            for (int u = 0; u < MT; u++) p[q][u] = ffma2(w[u][DP / 2 - 1], v, p[q][u]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < RS; q++) {
                        float z[MT];
#pragma unroll
                        for (int u = 0; u < MT; u++) z[u] = p[q][u].x + p[q][u].y;
                        store_units<MT>(zt + (g + (rr + q) * a.G) * a.HP + jq * MT, z);
                    }
                    }
                }
            }
            bar_arrive(k3ZFull + zb, 2 * k3WG);
        }
        for (int k = (nk >= k3NZ ? nk - k3NZ : 0); k < nk; k++) bar_sync(k3ZEmpty + (k % k3NZ), 2 * k3WG);
#ifdef GLX3_TIMING
        if ((f & 31) == 0 && a.dbg) { atomicAdd(a.dbg + 0, (unsigned long long)t_comp); atomicAdd(a.dbg + 1, (unsigned long long)t_wait); }
#endif
        bar_sync(k3Epi, k3NT);  // (A)
        bar_sync(k3Epi, k3NT);  // (B)
    } else if (role == 2) {
        // ============================================================ ACTIVATION
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(GLX3_REGS_A));
        const int ai = rt;
        const int qa = ai % a.QR, ga = ai / a.QR;
        const bool av = ga < a.AG;
        const int j0 = qa * UA;
        float w2s[UA], acc2[UA];
#pragma unroll
        for (int u = 0; u < UA; u++) {
            w2s[u] = av ? Wk[a.H * DP + j0 + u] : 0.f;
            acc2[u] = 0.f;
        }
        const float b2s = Wk[a.H * DP + a.H];
        float dsum = 0.f, loss = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        const int tpr = (2 * a.R <= k3WG) ? 2 : 1;
#ifdef GLX3_TIMING
        long long t_comp = 0, t_wait = 0;
#endif
        for (int k = 0; k < nk; k++) {
            const int s = k % k3NX, zb = k % k3NZ;
            const int64_t t = bx + (int64_t)k * gridDim.x;
            float* zt = zbuf + zb * RZ;
            const float* xt = xbuf + s * a.R * a.LD;
            T_BEGIN(tw);
            bar_sync(k3ZFull + zb, 2 * k3WG);
            mbar_wait(&xfull[s], (k / k3NX) & 1);
            T_ADD(t_wait, tw);
            T_BEGIN(tc);
            // pass 1: h = sigmoid(z) in place, output-neuron partials
            if (av) {
                for (int r = ga; r < a.R; r += a.AG) {
                    float* zp = zt + r * a.HP + j0;
                    float hv[UA];
                    load_units<UA>(zp, hv);
                    float os = 0.f;
                    if constexpr (UA % 2 == 0) {  // unit pairs in packed FADD2 / FFMA2
                        float2 os2 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int p = 0; p < UA / 2; p++) {
                            const float2 den =
                                __fadd2_rn(make_float2(ex2_approx(hv[2 * p]), ex2_approx(hv[2 * p + 1])), bcast2(1.0f));
                            hv[2 * p] = rcp_approx(den.x);
                            hv[2 * p + 1] = rcp_approx(den.y);
                            os2 = ffma2(make_float2(w2s[2 * p], w2s[2 * p + 1]), make_float2(hv[2 * p], hv[2 * p + 1]),
                                        os2);
                        }
                        os = os2.x + os2.y;
                    } else {
#pragma unroll
                        for (int u = 0; u < UA; u++) {
                            hv[u] = sigmoid_scaled(hv[u]);
                            os = fmaf(w2s[u], hv[u], os);
                        }
                    }
                    store_units<UA>(zp, hv);
                    opart[r * (a.QR + 1) + qa] = os;
                }
            }
            bar_sync(k3AInt, k3WG);
            // per row: o, delta_o, loss, confusion (kernels.py:352-375)
            {
                const int part = ai - (ai / tpr) * tpr;
                for (int r = ai / tpr; r - ai / tpr < a.R; r += k3WG / tpr) {
                    const bool rv = r < a.R;
                    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
                    if (rv) {
                        const float* opr = opart + r * (a.QR + 1);
                        int q = part;
                        for (; q + 3 * tpr < a.QR; q += 4 * tpr) {
                            z0 += opr[q];
                            z1 += opr[q + tpr];
                            z2 += opr[q + 2 * tpr];
                            z3 += opr[q + 3 * tpr];
                        }
                        for (; q < a.QR; q += tpr) z0 += opr[q];
                    }
                    float zo = (z0 + z1) + (z2 + z3);
                    if (tpr == 2) zo += __shfl_xor_sync(0xffffffffu, zo, 1);
                    if (rv && part == 0) {
                        float d = 0.f;
                        if (t * a.R + r < a.N) {
                            const float o = sigmoid_scaled(zo + b2s);
                            const float tt = xt[r * a.LD + a.D + 1];
                            d = (o - tt) * o * (1.0f - o);
                            loss = fmaf(0.5f * (tt - o), (tt - o), loss);
                            const bool pred = o >= 0.5f, pos = tt >= 0.5f;
                            c0 += (pred && pos) ? 1.f : 0.f;
                            c1 += (!pred && !pos) ? 1.f : 0.f;
                            c2 += (pred && !pos) ? 1.f : 0.f;
                            c3 += (!pred && pos) ? 1.f : 0.f;
                        }
                        dob[r] = d;
                    }
                }
            }
            bar_sync(k3AInt, k3WG);
            // pass 2: s = delta_o h (1 - h) in place; dW2 += delta_o h
            if (av) {
                for (int r = ga; r < a.R; r += a.AG) {
                    float* zp = zt + r * a.HP + j0;
                    const float d = dob[r];
                    float hv[UA];
                    load_units<UA>(zp, hv);
                    if constexpr (UA % 2 == 0) {  // same IEEE ops per lane, packed
#pragma unroll
                        for (int p = 0; p < UA / 2; p++) {
                            const float2 hp = make_float2(hv[2 * p], hv[2 * p + 1]);
                            const float2 v = __fmul2_rn(bcast2(d), hp);
                            const float2 ac = __fadd2_rn(make_float2(acc2[2 * p], acc2[2 * p + 1]), v);
                            acc2[2 * p] = ac.x;
                            acc2[2 * p + 1] = ac.y;
                            const float2 s2 = ffma2(make_float2(-v.x, -v.y), hp, v);
                            hv[2 * p] = s2.x;
                            hv[2 * p + 1] = s2.y;
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < UA; u++) {
                            const float v = d * hv[u];
                            acc2[u] += v;
                            hv[u] = fmaf(-v, hv[u], v);
                        }
                    }
                    store_units<UA>(zp, hv);
                    if (qa == 0) dsum += d;
                }
            }
            T_ADD(t_comp, tc);
            bar_arrive(k3SFull + zb, 2 * k3WG);
        }
#ifdef GLX3_TIMING
        if ((ai & 31) == 0 && a.dbg) { atomicAdd(a.dbg + 2, (unsigned long long)t_comp); atomicAdd(a.dbg + 3, (unsigned long long)t_wait); }
#endif
        stat[ai * 5 + 0] = loss;
        stat[ai * 5 + 1] = c0;
        stat[ai * 5 + 2] = c1;
        stat[ai * 5 + 3] = c2;
        stat[ai * 5 + 4] = c3;
        bar_sync(k3Epi, k3NT);  // (A): tile buffers are free
        float* epi2 = epi + a.G * a.H * DP;  // [AG][H]
        float* epi3 = epi2 + a.AG * a.H;     // [AG]
        if (av) {
#pragma unroll
            for (int u = 0; u < UA; u++) epi2[ga * a.H + j0 + u] = acc2[u];
            if (qa == 0) epi3[ga] = dsum;
        }
        bar_sync(k3Epi, k3NT);  // (B)
    } else {
        // ============================================================== BACKWARD
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(GLX3_REGS_B));
        const int b = rt;
        const int gb = b / a.TPG, jq = b - (b / a.TPG) * a.TPG;
        const bool bv = gb < a.G;
        float2 acc[MT][DP / 2];
#pragma unroll
        for (int u = 0; u < MT; u++)
#pragma unroll
            for (int q = 0; q < DP / 2; q++) acc[u][q] = make_float2(0.f, 0.f);
#ifdef GLX3_TIMING
        long long t_comp = 0, t_wait = 0;
#endif
        for (int k = 0; k < nk; k++) {
            const int s = k % k3NX, zb = k % k3NZ;
            const float* xt = xbuf + s * a.R * a.LD;
            const float* st = zbuf + zb * RZ;
            T_BEGIN(tw);
            bar_sync(k3SFull + zb, 2 * k3WG);
            mbar_wait(&xfull[s], (k / k3NX) & 1);
            T_ADD(t_wait, tw);
            T_BEGIN(tc);
            if (bv) {
                constexpr int RS = GLX3_RS;
                for (int rr = 0; rr < a.RPG; rr += RS) {
                    float sv[RS][MT];
                    const float* xr[RS];
#pragma unroll
                    for (int q = 0; q < RS; q++) {
                        const int r = gb + (rr + q) * a.G;
                        load_units<MT>(st + r * a.HP + jq * MT, sv[q]);
                        xr[q] = xt + r * a.LD;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < DP / 4; q4++) {
                        float4 v[RS];
#pragma unroll
                        for (int q = 0; q < RS; q++) v[q] = ld_f4(xr[q] + 4 * q4);
#pragma unroll
                        for (int q = 0; q < RS; q++) {
#pragma unroll
                            for (int u = 0; u < MT; u++) {
                                acc[u][2 * q4] = ffma2(bcast2(sv[q][u]), make_float2(v[q].x, v[q].y), acc[u][2 * q4]);
                                acc[u][2 * q4 + 1] =
                                    ffma2(bcast2(sv[q][u]), make_float2(v[q].z, v[q].w), acc[u][2 * q4 + 1]);
                            }
                        }
                    }
                    if (DP % 4) {
#pragma unroll
                        for (int q = 0; q < RS; q++) {
                            const float2 v = ld_f2(xr[q] + DP - 2);
#pragma unroll
                            for (int u = 0; u < MT; u++) acc[u][DP / 2 - 1] = ffma2(bcast2(sv[q][u]), v, acc[u][DP / 2 - 1]);
                        }
                    }
                }
            }
            T_ADD(t_comp, tc);
            bar_arrive(k3ZEmpty + zb, 2 * k3WG);
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[s]);
        }
#ifdef GLX3_TIMING
        if ((b & 31) == 0 && a.dbg) { atomicAdd(a.dbg + 4, (unsigned long long)t_comp); atomicAdd(a.dbg + 5, (unsigned long long)t_wait); }
#endif
        bar_sync(k3Epi, k3NT);  // (A)
        if (bv) {
#pragma unroll
            for (int u = 0; u < MT; u++) {
                float2* dst = reinterpret_cast<float2*>(epi + ((int64_t)gb * a.H + jq * MT + u) * DP);
#pragma unroll
                for (int q = 0; q < DP / 2; q++) dst[q] = acc[u][q];
            }
        }
        bar_sync(k3Epi, k3NT);  // (B)
    }

    // ------------------------------------------ per-CTA partial record
    {
        const float* epi2 = epi + a.G * a.H * DP;
        const float* epi3 = epi2 + a.AG * a.H;
        const int D1 = a.D + 1;
        for (int e = tid; e < a.P1; e += k3NT) {
            const int j = e / D1, i = e - (e / D1) * D1;
            float s = 0.f;
            for (int gg = 0; gg < a.G; gg++) s += epi[((int64_t)gg * a.H + j) * DP + i];
            out[e] = s;
        }
        for (int j = tid; j < a.H; j += k3NT) {
            float s = 0.f;
            for (int gg = 0; gg < a.AG; gg++) s += epi2[gg * a.H + j];
            out[a.P1 + j] = s;
        }
        if (tid == 0) {
            float s = 0.f;
            for (int gg = 0; gg < a.AG; gg++) s += epi3[gg];
            out[a.P1 + a.H] = s;
        }
        if (tid < 5) {
            float s = 0.f;
            for (int q = 0; q < k3WG; q++) s += stat[q * 5 + tid];
            out[a.P1 + a.H + 1 + tid] = s;
        }
    }
}

// ------------------------------------------------------------------ host side
static int a4(int x) { return (x + 3) / 4 * 4; }

bool batch3_geometry(int64_t N, int D, int H, int n_sms, Batch3Geom* out) {
    Batch3Geom g{};
    g.D = D;
    g.H = H;
    g.N = N;
    g.DP = D + 1 <= 8 ? 8 : D + 1 <= 16 ? 16 : D + 1 <= 34 ? 34 : -1;
    if (g.DP < 0 || H < 1 || N < 1) return false;
    g.LD = a4(std::max(D + 2, g.DP));
    g.MT = 0;
    for (int mt : {4, 3, 2, 1})
        if (H % mt == 0 && H / mt <= k3WG) {
            g.MT = mt;
            break;
        }
    g.UA = 0;
    for (int ua : {4, 2, 1})
        if (H % ua == 0 && H / ua <= k3WG) {
            g.UA = ua;
            break;
        }
    if (!g.MT || !g.UA) return false;
    g.TPG = H / g.MT;
    g.G = std::min(k3WG / g.TPG, k3WG / 2);
    g.QR = H / g.UA;
    g.AG = k3WG / g.QR;
    g.HP = a4(H);
    g.P1 = H * (D + 1);
    g.PS = a4(g.P1 + H + 6);
    g.WKS = a4(H * g.DP + 2 * H + 1);
    int rpg = (GLX3_TILE_ROWS + g.G - 1) / g.G;
    rpg = (rpg + GLX3_RS - 1) / GLX3_RS * GLX3_RS;
    for (;; rpg -= GLX3_RS) {
        if (rpg < GLX3_RS) return false;
        g.RPG = rpg;
        g.R = g.G * rpg;
        g.off_dob = a4(k3WG * 5);
        g.off_opart = g.off_dob + a4(g.R);
        g.off_z = g.off_opart + a4(g.R * (g.QR + 1));
        g.off_x = g.off_z + k3NZ * g.R * g.HP;
        const size_t end = (size_t)g.off_x + (size_t)k3NX * g.R * g.LD;
        const size_t epi = (size_t)g.off_z + (size_t)g.G * H * g.DP + (size_t)g.AG * H + g.AG;
        g.smem = 128 + 4 * std::max(end, epi);
        if (g.smem <= 227 * 1024) break;
    }
    g.ntiles = (N + g.R - 1) / g.R;
    g.grid = (int)std::min<int64_t>(g.ntiles, n_sms);
    *out = g;
    return true;
}

template <int DP, int MT, int UA>
static cudaError_t launch3_t(const Batch3Geom& g, const Batch3Args& a, cudaStream_t st) {
    auto k = batch3_kernel<DP, MT, UA>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) {
        fprintf(stderr, "glx: batch3_kernel<%d,%d,%d> smem=%zu: %s\n", DP, MT, UA, g.smem, cudaGetErrorString(e));
        return e;
    }
    k<<<g.grid, k3NT, g.smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        fprintf(stderr, "glx: batch3_kernel<%d,%d,%d> launch: %s\n", DP, MT, UA, cudaGetErrorString(e));
    return e;
}

template <int DP, int MT>
static cudaError_t launch3_ua(const Batch3Geom& g, const Batch3Args& a, cudaStream_t st) {
    switch (g.UA) {
        case 4: return launch3_t<DP, MT, 4>(g, a, st);
        case 2: return launch3_t<DP, MT, 2>(g, a, st);
        case 1: return launch3_t<DP, MT, 1>(g, a, st);
    }
    return cudaErrorInvalidValue;
}

template <int DP>
static cudaError_t launch3_mt(const Batch3Geom& g, const Batch3Args& a, cudaStream_t st) {
    switch (g.MT) {
        case 4: return launch3_ua<DP, 4>(g, a, st);
        case 3: return launch3_ua<DP, 3>(g, a, st);
        case 2: return launch3_ua<DP, 2>(g, a, st);
        case 1: return launch3_ua<DP, 1>(g, a, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_batch3_epoch(const Batch3Geom& g, const float* Xp, const float* Wk, float* part, cudaStream_t st) {
    Batch3Args a;
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
    a.QR = g.QR;
    a.AG = g.AG;
    a.P1 = g.P1;
    a.PS = g.PS;
    a.off_dob = g.off_dob;
    a.off_opart = g.off_opart;
    a.off_z = g.off_z;
    a.off_x = g.off_x;
    a.dbg = nullptr;
#ifdef GLX3_TIMING
    void* dbg = nullptr;
    cudaGetSymbolAddress(&dbg, g_glx3_dbg);
    a.dbg = reinterpret_cast<unsigned long long*>(dbg);
#endif
    switch (g.DP) {
        case 8: return launch3_mt<8>(g, a, st);
        case 16: return launch3_mt<16>(g, a, st);
        case 34: return launch3_mt<34>(g, a, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace glx

#ifdef GLX3_TIMING
// diagnostic builds only: per-role cycles (F comp, F wait, A comp, A wait, B comp, B wait), summed over warps
extern "C" void glx3_timing_dump(void) {
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, glx::g_glx3_dbg, sizeof(h));
    fprintf(stderr, "GLX3_TIMING F comp %llu wait %llu | A comp %llu wait %llu | B comp %llu wait %llu\n", h[0], h[1],
            h[2], h[3], h[4], h[5]);
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(glx::g_glx3_dbg, z, sizeof(z));
}
#endif
