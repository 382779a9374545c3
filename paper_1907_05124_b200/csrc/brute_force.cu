// brute_force.cu -- exhaustive ground state for small instances.
//
// Replaces brute_force_ground_state (model.cpp:265-324): a Gray-code walk over all 2^n spin
// configurations (n <= 26), energy updated by one flip_delta per step (model.cpp:237-242:
// -2 s_i (2 row_i + h_i), row_i = sum_j J_ij s_j in ascending j), best by energy with ties
// broken toward the lexicographically smallest configuration (-1 before +1, position 0
// first).  Here the walk is cut into one contiguous Gray range per thread (the reference's
// own OpenMP path does the same with fewer chunks: each chunk starts from the exact energy of
// its first configuration), J and h sit in shared memory, spins in a bitmask, and the
// per-thread bests are reduced by (energy, bit-reversed mask) -- bit-reversal turns the
// lexicographic order into integer order.  For integer couplings every energy is an exact
// integer, so the result is the reference's exactly; the reported energy is recomputed in the
// reference's order (model.cpp:220-225) by the exact energy kernel.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "kernels.cuh"

namespace marsb200 {
namespace {

constexpr int kMaxN = 26;
constexpr int kThreads = 256;

struct BestPair {
    double e;
    unsigned key;   // bit-reversed mask: integer order == lexicographic spin order
};

__device__ __forceinline__ bool better(BestPair a, BestPair b) {   // a better than b
    return a.e < b.e || (a.e == b.e && a.key < b.key);
}

__global__ void __launch_bounds__(kThreads) brute_kernel(const double* J, const double* h, int n,
                                                         unsigned long long per_thread, double* out_e,
                                                         unsigned* out_key) {
    __shared__ double sJ[kMaxN * kMaxN];
    __shared__ double sh[kMaxN];
    __shared__ double re[kThreads];
    __shared__ unsigned rk[kThreads];
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) sJ[i] = J[i];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = h ? h[i] : 0.0;
    __syncthreads();
    const unsigned long long total = 1ull << n;
    const unsigned long long tid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long first = tid * per_thread;
    const unsigned long long last = min(total, first + per_thread);
    BestPair best{DBL_MAX, 0xffffffffu};
    if (first < last) {
        // Gray code g(c) = c ^ (c >> 1); spin i = +1 when bit i of g is set
        unsigned mask = static_cast<unsigned>(first ^ (first >> 1));
        // exact energy of the first configuration (energy(), model.cpp:203-225 order)
        double coupling = 0.0;
        for (int i = 0; i < n; ++i) {
            double row = 0.0;
            for (int j = 0; j < n; ++j) row += sJ[i * n + j] * (((mask >> j) & 1u) ? 1.0 : -1.0);
            coupling += (((mask >> i) & 1u) ? 1.0 : -1.0) * row;
        }
        double e = coupling;
        for (int i = 0; i < n; ++i) e += sh[i] * (((mask >> i) & 1u) ? 1.0 : -1.0);
        best = {e, __brev(mask) >> (32 - n)};
        for (unsigned long long c = first + 1; c < last; ++c) {
            const int bit = __ffsll(static_cast<long long>(c)) - 1;           // countr_zero(c)
            double row = 0.0;                                                 // row_dot_spins
            for (int j = 0; j < n; ++j) row += sJ[bit * n + j] * (((mask >> j) & 1u) ? 1.0 : -1.0);
            const double si = ((mask >> bit) & 1u) ? 1.0 : -1.0;
            e += -2.0 * si * (2.0 * row + sh[bit]);                           // flip_delta
            mask ^= 1u << bit;
            const BestPair cand{e, __brev(mask) >> (32 - n)};
            if (better(cand, best)) best = cand;
        }
    }
    re[threadIdx.x] = best.e;
    rk[threadIdx.x] = best.key;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const BestPair o{re[threadIdx.x + s], rk[threadIdx.x + s]};
            if (better(o, BestPair{re[threadIdx.x], rk[threadIdx.x]})) {
                re[threadIdx.x] = o.e;
                rk[threadIdx.x] = o.key;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out_e[blockIdx.x] = re[0];
        out_key[blockIdx.x] = rk[0];
    }
}

}  // namespace

int brute_force_max_n() { return kMaxN; }

// Best (energy, bit-reversed mask) over all 2^n configurations; host reduces the per-block
// results.  J: dense n*n on the device, h: n or nullptr.
cudaError_t launch_brute_force(const double* J, const double* h, int n, double* part_e, unsigned* part_key,
                               int blocks, cudaStream_t st) {
    const unsigned long long total = 1ull << n;
    const unsigned long long threads = static_cast<unsigned long long>(blocks) * kThreads;
    const unsigned long long per = (total + threads - 1) / threads;
    brute_kernel<<<blocks, kThreads, 0, st>>>(J, h, n, per, part_e, part_key);
    return cudaGetLastError();
}

}  // namespace marsb200
