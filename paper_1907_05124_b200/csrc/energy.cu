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

#include <algorithm>
#include <cfloat>
#include <cstdint>

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

// progress: the same exact-order energy for a list of finished runs, compact outputs
__global__ void __launch_bounds__(128) energy_list_kernel(EnergyArgs a, const int* list, double* out_e,
                                                           std::uint8_t* out_st) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= a.count) return;
    const int r = list[k];
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
            for (int q = __ldg(a.off + i), e = __ldg(a.off + i + 1); q < e; ++q)
                row += __ldg(a.w64 + q) * static_cast<double>(s[__ldg(a.idx + q)]);
            total += static_cast<double>(s[i]) * row;
        }
    }
    double e = total;
    if (a.h64)
        for (int i = 0; i < n; ++i) e += __ldg(a.h64 + i) * static_cast<double>(s[i]);
    out_e[k] = e;
    out_st[k] = *reinterpret_cast<volatile const std::uint8_t*>(a.status + r);
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

// Dense couplings: the same exact operation order, with J rows streamed through shared
// memory (cp.async, double buffered, shared by every run of the CTA) and each run's spins
// bit-packed in shared memory.  acc += J_ij * s_j with s_j = +-1 is acc + (J_ij with its sign
// bit flipped when s_j = -1): bit-identical to the reference's multiply-add, one DADD per term.
constexpr int EJ = 512;        // J entries per staged chunk (4 KB)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}

__global__ void __launch_bounds__(256) energy_dense_kernel(EnergyArgs a, int runs_per_cta, int words) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* jbuf = reinterpret_cast<double*>(sm);                            // [2][EJ]
    unsigned* bits = reinterpret_cast<unsigned*>(sm + 2 * EJ * sizeof(double));   // [words][runs]
    const int t = threadIdx.x;
    const int n = a.n;
    const long long r = static_cast<long long>(blockIdx.x) * runs_per_cta + t;
    const bool mine = t < runs_per_cta && r < a.count && a.status[r] != 1;  // Skipped: no spins
    // pack this run's spins: bit j of word w set when s_(32w+j) = -1
    if (t < runs_per_cta) {
        const std::int8_t* s = a.spins + static_cast<size_t>(mine ? r : 0) * n;
        for (int w = 0; w < words; ++w) {
            unsigned v = 0;
            if (mine)
                for (int j = 0; j < 32 && 32 * w + j < n; ++j) v |= (s[32 * w + j] < 0 ? 1u : 0u) << j;
            bits[w * runs_per_cta + t] = v;
        }
    }
    const int chunks = (n + EJ - 1) / EJ;
    auto stage = [&](int i, int c, int buf) {
        const double* src = a.J64 + static_cast<size_t>(i) * n + c * EJ;
        const int len = min(EJ, n - c * EJ);
        // rows of J64 are n doubles long: 16-byte cp.async needs an even start and length
        for (int k = 2 * t; k < len; k += 2 * blockDim.x) {
            if (k + 1 < len && ((reinterpret_cast<std::uintptr_t>(src + k) & 15u) == 0)) {
                cp_async16(jbuf + buf * EJ + k, src + k);
            } else {
                jbuf[buf * EJ + k] = src[k];
                if (k + 1 < len) jbuf[buf * EJ + k + 1] = src[k + 1];
            }
        }
    };
    double total = 0.0;
    int it = 0;
    stage(0, 0, 0);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    for (int i = 0; i < n; ++i) {
        double row = 0.0;
        for (int c = 0; c < chunks; ++c, ++it) {
            // prefetch the next chunk (of this row or the next) into the other buffer
            const int ni = c + 1 < chunks ? i : i + 1, nc = c + 1 < chunks ? c + 1 : 0;
            if (ni < n) stage(ni, nc, (it + 1) & 1);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            __syncthreads();
            if (mine) {
                const double* jb = jbuf + (it & 1) * EJ;
                const int j0 = c * EJ, len = min(EJ, n - j0);
                for (int w = 0; w < len / 32; ++w) {
                    const unsigned sb = bits[((j0 >> 5) + w) * runs_per_cta + t];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        const unsigned long long jv = __double_as_longlong(jb[32 * w + jj]);
                        row += __longlong_as_double(jv ^ (static_cast<unsigned long long>((sb >> jj) & 1u) << 63));
                    }
                }
                for (int j = (len / 32) * 32; j < len; ++j) {
                    const unsigned sb = bits[((j0 + j) >> 5) * runs_per_cta + t];
                    const unsigned long long jv = __double_as_longlong(jb[j]);
                    row += __longlong_as_double(jv ^ (static_cast<unsigned long long>((sb >> ((j0 + j) & 31)) & 1u) << 63));
                }
            }
            __syncthreads();
        }
        if (mine) {
            const unsigned si = (bits[(i >> 5) * runs_per_cta + t] >> (i & 31)) & 1u;
            total += si ? -row : row;                           // total += s_i * row
        }
    }
    if (!mine) return;
    double e = total;
    if (a.h64) {
        for (int i = 0; i < n; ++i) {
            const unsigned si = (bits[(i >> 5) * runs_per_cta + t] >> (i & 31)) & 1u;
            e += si ? -__ldg(a.h64 + i) : __ldg(a.h64 + i);     // + h_i * s_i
        }
    }
    a.energy[r] = e;
    a.cut[r] = 0.25 * (a.coupling_sum - total);
}

cudaError_t launch_energy(const EnergyArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (a.J64) {
        const int words = (a.n + 31) / 32;
        int runs = static_cast<int>(std::min<long long>(256, (96 * 1024) / (words * 4)) / 32 * 32);
        runs = std::max(runs, 32);
        const std::size_t smem = 2 * EJ * sizeof(double) + static_cast<std::size_t>(words) * runs * 4;
        cudaError_t e = cudaFuncSetAttribute(energy_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned grid = static_cast<unsigned>((a.count + runs - 1) / runs);
        energy_dense_kernel<<<grid, std::max(runs, 32), smem, st>>>(a, runs, words);
        return cudaGetLastError();
    }
    const unsigned grid = static_cast<unsigned>((a.count + 127) / 128);
    energy_kernel<<<grid, 128, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_energy_list(const EnergyArgs& a, const int* list, double* out_e, std::uint8_t* out_st,
                               cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    energy_list_kernel<<<static_cast<unsigned>((a.count + 127) / 128), 128, 0, st>>>(a, list, out_e, out_st);
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
