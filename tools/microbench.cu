// microbench.cu -- latency probes behind the sparse kernel's per-level cost (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mb tools/microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1907_05124_b200/csrc/umma.cuh"

using namespace marsb200;

__device__ __forceinline__ double trial(double phi, double t) { return -tanh(__ddiv_rn(phi, t)); }

__global__ void chain_tanh(double* out, long long* cyc, int iters, double t) {
    double x = 0.3 + threadIdx.x * 1e-3;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) x = trial(x * 3.0 + 0.1, t);
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

__global__ void chain_dadd(double* out, long long* cyc, int iters) {
    double x = threadIdx.x * 1e-3, y = 1.0000001;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = __dadd_rn(x, y);
        x = __dadd_rn(x, -y * 0.5);
        x = __dadd_rn(x, y);
        x = __dadd_rn(x, -y * 0.5);
    }
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

__global__ void bar_lat(long long* cyc, int iters) {
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

__global__ void tma_lat(const int* src, long long* cyc, int iters, int bytes) {
    __shared__ __align__(16) unsigned char buf[8192];
    __shared__ __align__(8) std::uint64_t bar;
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_mbar_init();
    }
    __syncthreads();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) {
            umma::mbar_arrive_expect_tx(&bar, bytes);
            umma::bulk_load(buf, src + (i % 64) * 2048, bytes, &bar);
        }
        umma::mbar_wait(&bar, i & 1);
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0 + buf[5];
}

__global__ void ldg_lat(const int* src, long long* cyc, int iters) {
    int p = threadIdx.x;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) p = src[p];
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0 + p;
}

int main() {
    double* out;
    long long* cyc;
    int* src;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 1 << 16);
    cudaMalloc(&src, 64 << 20);
    // pointer chase with a stride that defeats L1 but stays in L2 (16 MB)
    {
        const int N = 4 << 20;
        int* h = new int[N];
        for (int i = 0; i < N; ++i) h[i] = (i + 40013 * 32) % N;
        cudaMemcpy(src, h, N * 4, cudaMemcpyHostToDevice);
        delete[] h;
    }
    static long long h[8192];
    auto report = [&](const char* name, int blocks, double per) {
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int b = 0; b < blocks; ++b) s += h[b];
        std::printf("%-44s %8.1f cycles\n", name, s / blocks / per);
    };
    const int it = 2000;
    chain_tanh<<<1, 32>>>(out, cyc, it, 2.5);
    report("tanh(phi/T) fp64 dependent chain, 1 warp", 1, it);
    chain_tanh<<<148, 32>>>(out, cyc, it, 2.5);
    report("tanh(phi/T) fp64 chain, 1 warp/SM x148", 148, it);
    chain_tanh<<<148 * 16, 32>>>(out, cyc, it, 2.5);
    report("tanh(phi/T) fp64 chain, 16 warps/SM", 148 * 16, it);
    chain_dadd<<<1, 32>>>(out, cyc, it);
    report("DADD dependent latency", 1, 4.0 * it);
    for (int w : {1, 2, 4, 8, 16}) {
        bar_lat<<<1, 32 * w>>>(cyc, it);
        char nm[64];
        std::snprintf(nm, sizeof nm, "__syncthreads, %d warps", w);
        report(nm, 1, it);
    }
    for (int b : {512, 2048, 8192}) {
        tma_lat<<<1, 32>>>(src, cyc, 200, b);
        char nm[64];
        std::snprintf(nm, sizeof nm, "cp.async.bulk %d B issue->complete", b);
        report(nm, 1, 200);
    }
    ldg_lat<<<1, 32>>>(src, cyc, it);
    report("LDG dependent (L2 hit)", 1, it);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
