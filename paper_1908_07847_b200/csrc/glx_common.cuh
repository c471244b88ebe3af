// glx_common.cuh -- shared device helpers for the glycemlp B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef GLX_LOG2E
#define GLX_LOG2E 1.4426950408889634
#endif

namespace glx {

// ---------------------------------------------------------------- fp32 math
// sigmoid from a pre-scaled argument: zs = -log2(e) * z  ->  1 / (1 + 2^zs).
// MUFU.EX2 + FADD + MUFU.RCP; saturates to 0 / 1 exactly like the f64 form.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sigmoid_scaled(float zs) { return rcp_approx(1.0f + ex2_approx(zs)); }

// reference normalize_apply (dataset.py:383-392): every op a separately
// rounded f32 op (no contraction), constant columns -> 0, clamp [-0.5, 1.5]
__device__ __forceinline__ float minmax_norm(float x, float mn, float mx) {
    const float span = __fsub_rn(mx, mn);
    if (span == 0.0f) return 0.0f;
    const float y = __fdiv_rn(__fsub_rn(x, mn), span);
    return fminf(fmaxf(y, -0.5f), 1.5f);
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 bcast2(float s) { return make_float2(s, s); }

// ------------------------------------------------------------ named barriers
// non-.aligned forms: safe when the calling warp may be diverged
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
    asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ----------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine, completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// MT consecutive floats <-> registers (vectorised when MT is 2 or 4)
template <int MT>
__device__ __forceinline__ void store_units(float* p, const float (&v)[MT]) {
    if constexpr (MT == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (MT == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
#pragma unroll
        for (int u = 0; u < MT; u++) p[u] = v[u];
    }
}

template <int MT>
__device__ __forceinline__ void load_units(const float* p, float (&v)[MT]) {
    if constexpr (MT == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    } else if constexpr (MT == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
#pragma unroll
        for (int u = 0; u < MT; u++) v[u] = p[u];
    }
}


}  // namespace glx
