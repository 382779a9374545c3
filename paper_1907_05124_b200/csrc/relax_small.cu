// relax_small.cu -- small dense instances with integer couplings (opt-in: MARS_DENSE_SMALL=1;
// measured slower than the tensor-core kernel on cfg1, 9.7K vs 12.4K descents/s).
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
// the CTA's warps; lane l holds spins k = l + 32q (q < NQ) and their fields in registers.  A
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

template <int NQ>
__global__ void __launch_bounds__(kSmallWarps * 32, 1) relax_small_kernel(RelaxArgs a, const __half* J) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __half* sJ = reinterpret_cast<__half*>(smem_raw);                 // [np][np], np = 32 * NQ
    float* sS = reinterpret_cast<float*>(smem_raw + sizeof(__half) * 32 * NQ * 32 * NQ);   // [warps][np]
    constexpr int NP = 32 * NQ;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = a.n, ldj = a.np;                                    // J rows in global: a.np halves
    for (int idx = threadIdx.x; idx < NP * NP; idx += blockDim.x) {
        const int r = idx / NP, c = idx % NP;
        sJ[idx] = (r < n && c < n) ? J[static_cast<std::size_t>(r) * ldj + c] : __float2half(0.0f);
    }
    __syncthreads();
    float* myS = sS + warp * NP;
    float h[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int k = lane + 32 * q;
        h[q] = (a.h32 && k < n) ? a.h32[k] : 0.0f;
    }
    for (;;) {
        int run = lane == 0 ? claim_run(a) : 0;
        run = __shfl_sync(0xffffffffu, run, 0);
        if (run < 0) return;
        Slot slot;
        slot_start(slot, run, a);
        float s[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int k = lane + 32 * q;
            s[q] = k < n ? a.s0[static_cast<std::size_t>(run) * n + k] : 0.0f;
        }
        int code;
        do {
            const float T = static_cast<float>(slot.T);
            const bool quench = slot_quench(slot);
            // exact refresh of every field owned by this lane
#pragma unroll
            for (int q = 0; q < NQ; ++q) myS[lane + 32 * q] = s[q];
            __syncwarp();
            float phi[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const __half* row = sJ + (lane + 32 * q) * NP;
                float acc = 0.0f;
                for (int j = 0; j < n; ++j) acc = fmaf(__half2float(row[j]), myS[j], acc);
                phi[q] = acc + h[q];
            }
            __syncwarp();
            float dmax = 0.0f;
#pragma unroll
            for (int qi = 0; qi < NQ; ++qi) {
                for (int o = 0; o < 32; ++o) {
                    const int i = 32 * qi + o;
                    if (i >= n) break;                                 // uniform
                    // every lane evaluates its own field (no divergent owner branch); the
                    // owner's change is the one broadcast
                    const float trial = tanh_trial(phi[qi], T, quench);
                    const float mine = trial - s[qi];
                    const float delta = __shfl_sync(0xffffffffu, mine, o);
                    if (lane == o) {
                        dmax = fmaxf(dmax, fabsf(mine));
                        s[qi] = trial;
                    }
                    const __half* row = sJ + i * NP;                   // J symmetric: J_ki = J_ik
#pragma unroll
                    for (int q = 0; q < NQ; ++q) phi[q] = fmaf(__half2float(row[lane + 32 * q]), delta, phi[q]);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
            code = slot_after_sweep(slot, static_cast<double>(dmax), a);
        } while (code == kSlotContinue);
        if (lane == 0) slot_finish(slot, code, a);
        std::int8_t* out = a.spins + static_cast<std::size_t>(run) * n;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int k = lane + 32 * q;
            if (k < n) out[k] = s[q] < 0.0f ? -1 : 1;
        }
    }
}

template <int NQ>
cudaError_t launch_t(const RelaxArgs& a, const __half* J, int grid, cudaStream_t st) {
    const std::size_t bytes = sizeof(__half) * (32 * NQ) * (32 * NQ) + sizeof(float) * kSmallWarps * 32 * NQ;
    cudaError_t e = cudaFuncSetAttribute(relax_small_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    relax_small_kernel<NQ><<<grid, kSmallWarps * 32, bytes, st>>>(a, J);
    return cudaGetLastError();
}

}  // namespace

int relax_small_max_n() { return kSmallMaxN; }
int relax_small_slots_per_cta() { return kSmallWarps; }

cudaError_t launch_relax_small(const RelaxArgs& a, const __half* J, int grid, cudaStream_t st) {
    const int nq = (a.n + 31) / 32;
    switch (nq) {
        case 1: return launch_t<1>(a, J, grid, st);
        case 2: return launch_t<2>(a, J, grid, st);
        case 3: return launch_t<3>(a, J, grid, st);
        case 4: return launch_t<4>(a, J, grid, st);
        case 5: return launch_t<5>(a, J, grid, st);
        case 6: return launch_t<6>(a, J, grid, st);
        case 7: return launch_t<7>(a, J, grid, st);
        case 8: return launch_t<8>(a, J, grid, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace marsb200
