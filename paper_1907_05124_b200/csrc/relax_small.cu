// relax_small.cu -- small dense instances with integer couplings (N <= 256), default for
// batches up to 4 x 16 warps x SMs runs (beyond that the tcgen05 kernel is full and faster);
// MARS_DENSE_SMALL=1/0 forces it on/off.  cfg1 (1024 runs, N=256): 16.0K descents/s vs 12.5K
// for the tensor-core kernel.
//
// Replaces, like relax_dense_umma.cu (fp32 state, same tolerance bar):
//   mars_relax_sweep        solvers.cpp:150-161   (Gauss-Seidel in index order)
//   IsingProblem::row_dot   model.cpp:141-151
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// When a batch is too small to fill the tensor-core kernel (cfg1: 1024 runs = 8 CTAs of 128)
// its descents are tail-bound by per-sweep latency, and with n <= 256 that latency is set by
// the TMA/GEMM round trip per spin block, not by arithmetic.  Here one warp owns one run and
// everything stays on chip: J (fp16, exact for integer couplings) in shared memory, shared by
// the CTA's warps; lane l holds the spin pairs k = 64p + 2l + {0, 1} and their fields in
// registers as float2 (one half2 load and one FFMA2 per pair and spin step).  A
// sweep refreshes every field from scratch (phi_k = sum_j J_kj s_j + h_k, j ascending), then
// walks i = 0..n-1: the owner lane evaluates tanh_trial, the change is broadcast with a shuffle
// and every lane adds J_ik * delta to the fields it owns (J symmetric: row i, consecutive k).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

constexpr int kSmallMaxN = 256;
constexpr int kSmallWarps = 16;

template <int P>
__global__ void __launch_bounds__(kSmallWarps * 32, 1) relax_small_kernel(RelaxArgs a, const __half* J) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NP = 64 * P;                                         // padded spins
    __half* sJ = reinterpret_cast<__half*>(smem_raw);                  // [NP][NP]
    float* sS = reinterpret_cast<float*>(smem_raw + sizeof(__half) * NP * NP);   // [warps][NP]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = a.n, ldj = a.np;                                     // J rows in global: a.np halves
    for (int idx = threadIdx.x; idx < NP * NP; idx += blockDim.x) {
        const int r = idx / NP, c = idx % NP;
        sJ[idx] = (r < n && c < n) ? J[static_cast<std::size_t>(r) * ldj + c] : __float2half(0.0f);
    }
    __syncthreads();
    float* myS = sS + warp * NP;
    // lane l owns the spin pairs k = 64p + 2l + {0, 1}: one half2 load and one FFMA2 per pair
    float2 h[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int k = 64 * p + 2 * lane;
        h[p] = make_float2((a.h32 && k < n) ? a.h32[k] : 0.0f, (a.h32 && k + 1 < n) ? a.h32[k + 1] : 0.0f);
    }
    for (;;) {
        int run = lane == 0 ? claim_run(a) : 0;
        run = __shfl_sync(0xffffffffu, run, 0);
        if (run < 0) return;
        Slot slot;
        slot_start(slot, run, a);
        const float* s0 = a.s0 + static_cast<std::size_t>(run) * n;
        float2 s[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int k = 64 * p + 2 * lane;
            s[p] = make_float2(k < n ? s0[k] : 0.0f, k + 1 < n ? s0[k + 1] : 0.0f);
        }
        int code;
        do {
            const float T = static_cast<float>(slot.T);
            const bool quench = slot_quench(slot);
            const float rT = quench ? 0.0f : recip_for_div(T);
            // exact refresh: phi_k = sum_j J_kj s_j, j ascending (row_dot's order); J is
            // symmetric, so J_kj is read as row j, columns 2l, 2l+1 (consecutive lanes,
            // consecutive words: conflict-free), s_j a shared-memory broadcast
#pragma unroll
            for (int p = 0; p < P; ++p) *reinterpret_cast<float2*>(myS + 64 * p + 2 * lane) = s[p];
            __syncwarp();
            float2 phi[P];
#pragma unroll
            for (int p = 0; p < P; ++p) phi[p] = make_float2(0.0f, 0.0f);
#pragma unroll 4
            for (int j = 0; j < n; ++j) {
                const float sj = myS[j];
                const __half2* row = reinterpret_cast<const __half2*>(sJ + j * NP) + lane;
#pragma unroll
                for (int p = 0; p < P; ++p)
                    phi[p] = __ffma2_rn(__half22float2(row[32 * p]), make_float2(sj, sj), phi[p]);
            }
#pragma unroll
            for (int p = 0; p < P; ++p) phi[p] = make_float2(phi[p].x + h[p].x, phi[p].y + h[p].y);
            __syncwarp();
            float dmax = 0.0f;
#pragma unroll
            for (int pi = 0; pi < P; ++pi) {
                for (int o = 0; o < 32; ++o) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i = 64 * pi + 2 * o + e;
                        if (i >= n) break;                              // uniform
                        // every lane evaluates its own field (no divergent owner branch); the
                        // owner's change is the one broadcast
                        const float f = e ? phi[pi].y : phi[pi].x;
                        const float cur = e ? s[pi].y : s[pi].x;
                        const float trial = tanh_trial_r(f, T, rT, quench);
                        const float mine = trial - cur;
                        const float delta = __shfl_sync(0xffffffffu, mine, o);
                        if (lane == o) {
                            dmax = fmaxf(dmax, fabsf(mine));
                            if (e) s[pi].y = trial; else s[pi].x = trial;
                        }
                        const __half2* row = reinterpret_cast<const __half2*>(sJ + i * NP) + lane;   // J_ki = J_ik
                        const float2 d2 = make_float2(delta, delta);
#pragma unroll
                        for (int p = 0; p < P; ++p) phi[p] = __ffma2_rn(__half22float2(row[32 * p]), d2, phi[p]);
                    }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            code = slot_after_sweep(slot, static_cast<double>(dmax), a);
        } while (code == kSlotContinue);
        if (lane == 0) slot_finish(slot, code, a);
        std::int8_t* out = a.spins + static_cast<std::size_t>(run) * n;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int k = 64 * p + 2 * lane;
            if (k < n) out[k] = s[p].x < 0.0f ? -1 : 1;
            if (k + 1 < n) out[k + 1] = s[p].y < 0.0f ? -1 : 1;
            if (a.state_out) {
                float* so = a.state_out + static_cast<std::size_t>(run) * n;
                if (k < n) so[k] = s[p].x;
                if (k + 1 < n) so[k + 1] = s[p].y;
            }
        }
        __syncwarp();
        if (lane == 0) log_retired(a, run);
    }
}

template <int P>
cudaError_t launch_t(const RelaxArgs& a, const __half* J, int grid, int warps, cudaStream_t st) {
    const std::size_t bytes = sizeof(__half) * (64 * P) * (64 * P) + sizeof(float) * warps * 64 * P;
    cudaError_t e = cudaFuncSetAttribute(relax_small_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    relax_small_kernel<P><<<grid, warps * 32, bytes, st>>>(a, J);
    return cudaGetLastError();
}

}  // namespace

int relax_small_max_n() { return kSmallMaxN; }
int relax_small_slots_per_cta() { return kSmallWarps; }

cudaError_t launch_relax_small(const RelaxArgs& a, const __half* J, int grid, int warps, cudaStream_t st) {
    const int pairs = (a.n + 63) / 64;
    if (warps < 1 || warps > kSmallWarps) return cudaErrorInvalidValue;
    switch (pairs) {
        case 1: return launch_t<1>(a, J, grid, warps, st);
        case 2: return launch_t<2>(a, J, grid, warps, st);
        case 3: return launch_t<3>(a, J, grid, warps, st);
        case 4: return launch_t<4>(a, J, grid, warps, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace marsb200
