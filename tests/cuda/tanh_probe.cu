// tanh_probe.cu -- TEST ONLY: the device restatement of the reference's tanh/expm1
// (csrc/ref_tanh.cuh) evaluated on an array, for tests/test_gpu_parity.py.
#include <cuda_runtime.h>

#include "../../paper_1907_05124_b200/csrc/ref_tanh.cuh"

__global__ void probe_kernel(const double* x, double* t, double* e, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        t[i] = marsb200::ref_tanh(x[i]);
        e[i] = marsb200::ref_expm1(x[i]);
    }
}

extern "C" int tanh_probe(const double* x, double* t, double* e, long long n) {
    double *dx, *dt, *de;
    if (cudaMalloc(&dx, n * 8) || cudaMalloc(&dt, n * 8) || cudaMalloc(&de, n * 8)) return 1;
    cudaMemcpy(dx, x, n * 8, cudaMemcpyHostToDevice);
    probe_kernel<<<static_cast<unsigned>((n + 255) / 256), 256>>>(dx, dt, de, n);
    cudaMemcpy(t, dt, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(e, de, n * 8, cudaMemcpyDeviceToHost);
    const cudaError_t err = cudaDeviceSynchronize();
    cudaFree(dx);
    cudaFree(dt);
    cudaFree(de);
    return err == cudaSuccess ? 0 : 2;
}
