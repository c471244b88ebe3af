// Microbenchmark: FFMA2 throughput at 2 warps/SMSP (256 threads, 1 CTA/SM) with a
// controllable mix of broadcast LDS.128 and MUFU per FFMA2 block. Tuning aid only.
#include <cstdio>
#include <cuda_runtime.h>
template <int NLDS, int NMUFU, bool BCAST>
__global__ void __launch_bounds__(256, 1) mix(float* out, int iters) {
    extern __shared__ float4 sm[];
    if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(threadIdx.x, 1, 2, 3);
    __syncthreads();
    float2 acc[16];
    float2 w[17];
    for (int k = 0; k < 16; k++) acc[k] = make_float2(k, -k);
    for (int q = 0; q < 17; q++) w[q] = make_float2(1e-3f * q, 2e-3f * q);
    float m = threadIdx.x * 1e-3f;
    for (int it = 0; it < iters; it++) {
        float4 v[NLDS > 0 ? NLDS : 1];
#pragma unroll
        for (int l = 0; l < NLDS; l++) v[l] = sm[(it + l) & 63];
#pragma unroll
        for (int q = 0; q < 8; q++) {
#pragma unroll
            for (int k = 0; k < 16; k++) {
                float2 x = NLDS > 0 ? make_float2(v[(q + k) % (NLDS > 0 ? NLDS : 1)].x, v[(q + k) % (NLDS > 0 ? NLDS : 1)].y) : w[k];
                if (BCAST) acc[k] = __ffma2_rn(make_float2(w[q].x, w[q].x), x, acc[k]);
                else acc[k] = __ffma2_rn(w[q + (k & 1)], x, acc[k]);
            }
        }
#pragma unroll
        for (int u = 0; u < NMUFU; u++) { float e; asm volatile("ex2.approx.ftz.f32 %0,%1;" : "=f"(e) : "f"(m + u)); m += e * 1e-9f; }
    }
    float s = m;
    for (int k = 0; k < 16; k++) s += acc[k].x + acc[k].y;
    if (s == 1.234f) out[threadIdx.x] = s;
}
template <int A, int B, bool C> void run(const char* name) {
    float* out; cudaMalloc(&out, 4096);
    auto k = mix<A, B, C>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int iters = 20000;
    k<<<148, 256, 200 * 1024>>>(out, 100);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<<<148, 256, 200 * 1024>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * 256 * iters * 128 * 4;
    printf("%-28s %7.2f TFLOP/s (FFMA2 only count)  err=%s\n", name, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<0, 0, false>("pure ffma2 vec");
    run<0, 0, true>("pure ffma2 bcast");
    run<4, 0, false>("4 lds / 128 ffma2");
    run<8, 0, false>("8 lds / 128 ffma2");
    run<0, 8, false>("8 mufu / 128 ffma2");
    run<8, 8, false>("8 lds + 8 mufu / 128");
    run<16, 16, false>("16 lds + 16 mufu / 128");
}
