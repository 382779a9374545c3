// umma_probe.cu -- TEST-ONLY probe of the product's tcgen05/TMA layer (csrc/umma.cuh,
// csrc/tma_host.hpp): D[128 x N] = A[128 x K] * B[N x K]^T in fp16 -> fp32, one CTA.
// Built by tests/test_umma_probe.py; compared against torch.matmul.
#include <cuda_fp16.h>

#include "../../paper_1907_05124_b200/csrc/tma_host.hpp"
#include "../../paper_1907_05124_b200/csrc/umma.cuh"

using namespace marsb200;
using namespace marsb200::umma;

template <int N>
__global__ void __launch_bounds__(128, 1) probe_kernel(const __grid_constant__ CUtensorMap ta,
                                                        const __grid_constant__ CUtensorMap tb,
                                                        float* D, int K) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
    unsigned char* sA = base;                 // 128 rows x 128 B = 16 KB
    unsigned char* sB = base + 16384;         // N rows x 128 B
    __shared__ __align__(8) std::uint64_t bar_full, bar_mma;
    __shared__ std::uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar_full, 1);
        mbar_init(&bar_mma, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, N < 32 ? 32 : N);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tb0 = tmem_base;
    const std::uint32_t idesc = idesc_f16(128, N, 0);
    std::uint32_t phase = 0;
    for (int kc = 0; kc < K / 64; ++kc) {
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&bar_full, 16384 + N * 128);
            tma_load_2d(sA, &ta, &bar_full, kc * 64, 0);
            tma_load_2d(sB, &tb, &bar_full, kc * 64, 0);
        }
        mbar_wait(&bar_full, phase);
        tc_fence_after();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_f16_ss(tb0, desc_k_sw128(smem_u32(sA) + kk * 32), desc_k_sw128(smem_u32(sB) + kk * 32),
                           idesc, (kc | kk) != 0);
            mma_commit(&bar_mma);
        }
        mbar_wait(&bar_mma, phase);
        tc_fence_after();
        phase ^= 1;
        __syncthreads();
    }
    // thread (warp w, lane l) owns TMEM lane 32w + l = output row
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; c += 32) {
        float v[32];
        tmem_ld32(tb0 + (static_cast<std::uint32_t>(warp * 32) << 16) + c, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[row * N + c + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb0, N < 32 ? 32 : N);
}

// A from TMEM ("ts"): thread t of warp w writes row 32w+t's K values, 2 fp16 per column
template <int N>
__global__ void __launch_bounds__(128, 1) probe_ts_kernel(const __half* A, const __grid_constant__ CUtensorMap tb,
                                                           float* D, int K) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sB = smem_raw;
    __shared__ __align__(8) std::uint64_t bar_full, bar_mma;
    __shared__ std::uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar_full, 1);
        mbar_init(&bar_mma, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tb0 = tmem_base;                // D at columns [0, N), A at [256, 288)
    const std::uint32_t ta = tb0 + 256;
    const std::uint32_t idesc = idesc_f16(128, N, 0);
    const int row = warp * 32 + lane;
    std::uint32_t phase = 0;
    for (int kc = 0; kc < K / 64; ++kc) {
        // this thread's row, 64 K values -> 32 TMEM columns
        std::uint32_t v[16];
        for (int half = 0; half < 2; ++half) {
            for (int j = 0; j < 16; ++j) {
                const __half2 h2 = __halves2half2(A[row * K + kc * 64 + half * 32 + 2 * j],
                                                  A[row * K + kc * 64 + half * 32 + 2 * j + 1]);
                v[j] = *reinterpret_cast<const std::uint32_t*>(&h2);
            }
            tmem_st16(ta + (static_cast<std::uint32_t>(warp * 32) << 16) + half * 16, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&bar_full, N * 128);
            tma_load_2d(sB, &tb, &bar_full, kc * 64, 0);
        }
        mbar_wait(&bar_full, phase);
        tc_fence_after();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_f16_ts(tb0, ta + kk * 8, desc_k_sw128(smem_u32(sB) + kk * 32), idesc, (kc | kk) != 0);
            mma_commit(&bar_mma);
        }
        mbar_wait(&bar_mma, phase);
        tc_fence_after();
        phase ^= 1;
        __syncthreads();
    }
    for (int c = 0; c < N; c += 32) {
        float out[32];
        tmem_ld32(tb0 + (static_cast<std::uint32_t>(warp * 32) << 16) + c, out);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[row * N + c + j] = out[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb0, 512);
}

extern "C" int umma_probe_ts(const void* dA, const void* dB, float* dD, int K, int N) {
    CUtensorMap tb;
    if (!make_tmap_f16_sw128(&tb, dB, N, K, 64, N)) return 2;
    const int smem = 256 * 128 + 1024;
    if (N == 128) {
        cudaFuncSetAttribute(probe_ts_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_ts_kernel<128><<<1, 128, smem>>>(static_cast<const __half*>(dA), tb, dD, K);
    } else if (N == 256) {
        cudaFuncSetAttribute(probe_ts_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_ts_kernel<256><<<1, 128, smem>>>(static_cast<const __half*>(dA), tb, dD, K);
    } else {
        return 3;
    }
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 100 + static_cast<int>(e);
}

extern "C" int umma_probe(const void* dA, const void* dB, float* dD, int K, int N) {
    CUtensorMap ta, tb;
    if (!make_tmap_f16_sw128(&ta, dA, 128, K, 64, 128)) return 1;
    if (!make_tmap_f16_sw128(&tb, dB, N, K, 64, N)) return 2;
    const int smem = 16384 + 256 * 128 + 1024;
    cudaError_t e;
    if (N == 128) {
        cudaFuncSetAttribute(probe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_kernel<128><<<1, 128, smem>>>(ta, tb, dD, K);
    } else if (N == 256) {
        cudaFuncSetAttribute(probe_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_kernel<256><<<1, 128, smem>>>(ta, tb, dD, K);
    } else {
        return 3;
    }
    e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 100 + static_cast<int>(e);
}
