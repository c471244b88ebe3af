// umma_probe.cu -- standalone check of tcgen05 kind::tf32 operand forms (no-swizzle
// canonical layouts) used by glx_batchtc.cu. Prints the max error per configuration.
// nvcc -gencode arch=compute_100a,code=sm_100a -o umma_probe tools/umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_ns(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc(int N, bool bmn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((bmn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
struct Cfg { int bmode; int lbo; int sbo; int ts; int N; int layout; };
// A: 128 x 8 (M x K); B: 8 x N (K x N); D = A.B
// bmode 0: B K-major  [n/8][k/4][n%8][k%4]  (core matrix 8 n-rows x 16 B of k)
// bmode 1: B MN-major [k/8][n/4][k%8][n%4]  (core matrix 8 k-rows x 16 B of n), chunk stride 128
// bmode 2: B MN-major [n/4][k/8][k%8][n%4]  (n-chunks outermost)
__global__ void probe(const float* A, const float* B, float* D, Cfg c) {
    __shared__ __align__(1024) unsigned char sm[128 * 8 * 4 + 2048 + 64];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    unsigned char* sa = sm;
    unsigned char* sb = sm + 128 * 8 * 4;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, N = c.N;
    for (int e = t; e < 128 * 8; e += blockDim.x) {
        int m = e / 8, k = e % 8;
        *(float*)(sa + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) = A[e];
    }
    for (int e = t; e < 8 * N; e += blockDim.x) {
        int k = e / N, n = e % N, off;
        if (c.bmode == 0) off = (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
        else if (c.bmode == 1) off = (k / 8) * (N / 4 * 128) + (n / 4) * 128 + (k % 8) * 16 + (n % 4) * 4;
        else if (c.bmode == 2) off = (n / 4) * 128 + (k % 8) * 16 + (n % 4) * 4;
        else off = (n / 32) * 1024 + k * 128 + ((((n % 32) / 4) ^ (k % 8)) * 16) + (n % 4) * 4;  // MN-major SW128
        *(float*)(sb + off) = B[e];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    {   // A into TMEM cols [128, 136) and poison D cols
        uint32_t r[8];
        for (int k = 0; k < 8; k++) r[k] = __float_as_uint(A[(warp * 32 + lane) * 8 + k]);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + 128 + ((uint32_t)(warp * 32) << 16)),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        const uint32_t pz = __float_as_uint(-12345.f);
        for (int c0 = 0; c0 < 64; c0 += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tm + c0 + ((uint32_t)(warp * 32) << 16)), "r"(pz) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (t == 0) {
        const uint64_t db = desc_ns(su32(sb), c.lbo, c.sbo, c.layout);
        const uint32_t id = idesc(N, c.bmode != 0);
        if (!c.ts) {
            const uint64_t da = desc_ns(su32(sa), 128, 256);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(0) : "memory");
        } else {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 128), "l"(db), "r"(id), "r"(0) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    {
        uint32_t a = su32(&bar), done = 0;
        while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(a), "r"(0) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r[16];
    for (int c0 = 0; c0 < N; c0 += 16) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tm + c0 + ((uint32_t)(warp * 32) << 16)) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; i++) D[(warp * 32 + lane) * N + c0 + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory");
}

int main() {
    std::vector<float> A(128 * 8), B(8 * 64), D(128 * 64);
    for (int i = 0; i < 128 * 8; i++) A[i] = (float)((i * 37) % 17 - 8);
    for (int i = 0; i < 8 * 64; i++) B[i] = (float)((i * 13) % 11 - 5);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    Cfg cfgs[] = {
        {0, 128, 256, 0, 48, 0}, {0, 128, 256, 1, 48, 0},   // K-major B (control), SS / TS
        {3, 1024, 1024, 0, 48, 2}, {3, 1024, 1024, 1, 48, 2}, // MN-major SW128, LBO = N-atom stride
        {3, 1024, 128, 1, 48, 2}, {3, 128, 1024, 1, 48, 2},
        {3, 1024, 1024, 1, 64, 2},
    };
    for (auto c : cfgs) {
        std::vector<float> B2 = B;
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128>>>(dA, dB, dD, c);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, 128 * c.N * 4, cudaMemcpyDeviceToHost);
        double err = 0; int poison = 0;
        for (int m = 0; m < 128; m++) for (int n = 0; n < c.N; n++) {
            double ref = 0; for (int k = 0; k < 8; k++) ref += (double)A[m * 8 + k] * B[k * c.N + n];
            err = fmax(err, fabs(ref - D[m * c.N + n])); poison += D[m * c.N + n] == -12345.f;
        }
        printf("bmode %d layout %d lbo %4d sbo %4d ts %d N %d: %s max err %g poisoned %d  D[0][0..3] %g %g %g %g\n", c.bmode, c.layout, c.lbo, c.sbo, c.ts, c.N,
               cudaGetErrorString(e), err, poison, D[0], D[1], D[2], D[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
