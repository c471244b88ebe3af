// Probe of the tcgen05.ld 16x256b / 16x64b register layouts (tools only):
// one warp writes v = 1000 * lane + column into its 32 TMEM lanes (32x32b.x32),
// reads the same region back with 16x256b.x1 / 16x64b.x1 and prints, per thread,
// which (lane, column) each register holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_shape_probe tools/tmem_shape_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(int* out) {
    __shared__ uint32_t slot;
    const int lane = threadIdx.x;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    uint32_t v[32];
    for (int c = 0; c < 32; c++) v[c] = 1000 * lane + c;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t a0, a1, a2, a3;
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(tmem) : "memory");
    uint32_t b0;
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(b0) : "r"(tmem) : "memory");
    uint32_t c0, c1;
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(c0), "=r"(c1) : "r"(tmem) : "memory");
    uint32_t d0, d1, d2, d3, d4, d5, d6, d7;
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(d4), "=r"(d5), "=r"(d6), "=r"(d7) : "r"(tmem)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int* o = out + lane * 16;
    o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3; o[4] = b0; o[5] = c0; o[6] = c1;
    o[7] = d0; o[8] = d1; o[9] = d2; o[10] = d3; o[11] = d4; o[12] = d5; o[13] = d6; o[14] = d7;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
    int* d;
    cudaMalloc(&d, 32 * 16 * sizeof(int));
    probe<<<1, 32>>>(d);
    int h[32 * 16];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    printf("thread: 16x256b.x1 (lane,col)x4 | 16x64b.x1 | 16x128b.x1 x2 | 16x256b.x2 x8\n");
    for (int t = 0; t < 32; t++) {
        printf("%2d:", t);
        for (int k = 0; k < 15; k++) printf(" (%d,%d)", h[t * 16 + k] / 1000, h[t * 16 + k] % 1000);
        printf("\n");
    }
    return 0;
}
