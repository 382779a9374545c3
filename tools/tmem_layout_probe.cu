// tmem_layout_probe.cu -- prints which (TMEM lane, column) each thread's registers hold after
// tcgen05.ld.16x256b.x2 (tool; decides the fragment mapping the helper's mma path relies on).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(unsigned* out) {
    __shared__ std::uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(
            static_cast<unsigned>(__cvta_generic_to_shared(&tbase))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const std::uint32_t t = tbase;
    const unsigned row = 32 * warp + lane;   // this thread's TMEM lane under 32x32b
    unsigned v[16];
    for (int c = 0; c < 16; ++c) v[c] = row * 100 + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(t + ((32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                 "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                 "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    for (int m = 0; m < 2; ++m) {
        unsigned r[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(t + ((32 * warp + 16 * m) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int i = 0; i < 8; ++i) out[((warp * 2 + m) * 32 + lane) * 8 + i] = r[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(t));
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 4 * 2 * 32 * 8 * 4);
    cudaMemset(d, 0xff, 4 * 2 * 32 * 8 * 4);
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    unsigned h[4 * 2 * 32 * 8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    for (int w = 0; w < 4; w += 3)
        for (int m = 0; m < 2; ++m)
            for (int l = 0; l < 32; l += (l < 8 ? 1 : 9)) {
                printf("warp %d m %d thread %2d:", w, m, l);
                for (int i = 0; i < 8; ++i) {
                    const unsigned x = h[((w * 2 + m) * 32 + l) * 8 + i];
                    printf(" (%u,%u)", x / 100, x % 100);
                }
                printf("\n");
            }
    return 0;
}
