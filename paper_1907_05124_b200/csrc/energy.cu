// energy.cu -- exact Ising energy / cut of the rounded spins, and the best-of-R reduction.
//
// energy_kernel restates, per run, in the reference's exact fp64 operation order:
//   row_dot_spins   model.cpp:153-163   acc += J_ij * s_j, j ascending (or CSR order)
//   coupling_term   model.cpp:203-218   total += s_i * row_i, i ascending
//   energy          model.cpp:220-225   + h_i * s_i, i ascending
//   cut_value       model.cpp:227-229   0.25 * (coupling_sum - coupling_term)
// Because s_j = +-1 every product is exact, so FMA contraction cannot change a rounding:
// the device energies are bit-identical to the reference's for ANY coupling values.
//
// best_kernel: "first strict minimum" over completed runs (runner.cpp:147-150) as a
// warp-shuffle / shared-memory / two-pass grid reduction on (energy, run index).
#include <cuda_runtime.h>

#include <cfloat>

#include "kernels.cuh"

namespace marsb200 {
namespace {

__global__ void __launch_bounds__(128) energy_kernel(EnergyArgs a) {
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.count || a.status[r] == 1) return;   // Skipped slots carry no spins
    const int n = a.n;
    const std::int8_t* s = a.spins + static_cast<size_t>(r) * n;
    double total = 0.0;
    if (a.J64) {
        for (int i = 0; i < n; ++i) {
            const double* Jr = a.J64 + static_cast<size_t>(i) * n;
            double row = 0.0;
            for (int j = 0; j < n; ++j) row += __ldg(Jr + j) * static_cast<double>(s[j]);
            total += static_cast<double>(s[i]) * row;
        }
    } else {
        for (int i = 0; i < n; ++i) {
            double row = 0.0;
            for (int k = __ldg(a.off + i), e = __ldg(a.off + i + 1); k < e; ++k)
                row += __ldg(a.w64 + k) * static_cast<double>(s[__ldg(a.idx + k)]);
            total += static_cast<double>(s[i]) * row;
        }
    }
    double e = total;
    if (a.h64)
        for (int i = 0; i < n; ++i) e += __ldg(a.h64 + i) * static_cast<double>(s[i]);
    a.energy[r] = e;
    a.cut[r] = 0.25 * (a.coupling_sum - total);
}

struct Best {
    double e;
    long long i;
};

__device__ __forceinline__ Best better(Best x, Best y) {
    if (y.i < 0) return x;
    if (x.i < 0) return y;
    if (y.e < x.e || (y.e == x.e && y.i < x.i)) return y;
    return x;
}

__device__ __forceinline__ Best block_best(Best v) {
    __shared__ double se[32];
    __shared__ long long si[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Best w{__shfl_xor_sync(0xffffffffu, v.e, o), __shfl_xor_sync(0xffffffffu, v.i, o)};
        v = better(v, w);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        se[warp] = v.e;
        si[warp] = v.i;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        v = lane < nw ? Best{se[lane], si[lane]} : Best{DBL_MAX, -1};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            Best w{__shfl_xor_sync(0xffffffffu, v.e, o), __shfl_xor_sync(0xffffffffu, v.i, o)};
            v = better(v, w);
        }
    }
    return v;
}

__global__ void __launch_bounds__(256) best_partial_kernel(BestArgs a) {
    Best v{DBL_MAX, -1};
    for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < a.count;
         r += static_cast<long long>(gridDim.x) * blockDim.x)
        if (a.status[r] == 0) v = better(v, Best{a.energy[r], r});
    v = block_best(v);
    if (threadIdx.x == 0) {
        a.part_energy[blockIdx.x] = v.e;
        a.part_index[blockIdx.x] = v.i;
    }
}

__global__ void __launch_bounds__(256) best_final_kernel(BestArgs a, int parts) {
    Best v{DBL_MAX, -1};
    for (int p = threadIdx.x; p < parts; p += blockDim.x) v = better(v, Best{a.part_energy[p], a.part_index[p]});
    v = block_best(v);
    if (threadIdx.x == 0) *a.best_index = v.i;
}

}  // namespace

cudaError_t launch_energy(const EnergyArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((a.count + 127) / 128);
    energy_kernel<<<grid, 128, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_best(const BestArgs& a, int grid, cudaStream_t st) {
    best_partial_kernel<<<grid, 256, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    best_final_kernel<<<1, 256, 0, st>>>(a, grid);
    return cudaGetLastError();
}

}  // namespace marsb200
