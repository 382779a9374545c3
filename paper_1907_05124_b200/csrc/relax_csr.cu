// relax_csr.cu -- persistent thread-per-run MARS relaxation for CSR (sparse) couplings.
//
// Replaces, for sparse storage (edge density < 5%, model.cpp:91):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:147-148   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// One thread owns one run slot and sweeps its spins in ascending order, summing each
// neighbour list in the reference's (sorted) order -- the exact Gauss-Seidel order and the
// exact summation order, in fp32.  The CSR arrays are read uniformly by a warp (broadcast);
// the state lives in a per-CTA workspace W[n][TM] (runs contiguous) so each neighbour
// gather is one coalesced 128-byte row per warp.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

constexpr int TM = 128;  // slots (threads) per CTA

__global__ void __launch_bounds__(TM) relax_csr_kernel(RelaxArgs a) {
    const int tid = threadIdx.x;
    const int n = a.n;
    float* W = a.work + static_cast<size_t>(blockIdx.x) * a.np * TM + tid;

    Slot slot;
    slot.run = -1;
    {
        const int r = claim_run(a);
        if (r >= 0) {
            slot_start(slot, r, a);
            const float* src = a.s0 + static_cast<size_t>(r) * n;
            for (int i = 0; i < n; ++i) W[static_cast<size_t>(i) * TM] = src[i];
        }
    }
    while (__syncthreads_or(slot.run >= 0)) {
        if (slot.run < 0) continue;
        const bool quench = slot_quench(slot);
        const float Tf = static_cast<float>(slot.T);
        float dmax = 0.0f;
        int k = __ldg(a.off);
        for (int i = 0; i < n; ++i) {
            const int kend = __ldg(a.off + i + 1);
            float phi = 0.0f;
            for (; k < kend; ++k)
                phi = fmaf(__ldg(a.w32 + k), W[static_cast<size_t>(__ldg(a.idx + k)) * TM], phi);
            if (a.h32) phi += __ldg(a.h32 + i);
            const float trial = tanh_trial(phi, Tf, quench);
            float* wp = W + static_cast<size_t>(i) * TM;
            dmax = fmaxf(dmax, fabsf(trial - *wp));
            *wp = trial;
        }
        const int code = slot_after_sweep(slot, dmax, a);
        if (code != kSlotContinue) {
            slot_finish(slot, code, a);
            std::int8_t* out = a.spins + static_cast<size_t>(slot.run) * n;
            for (int i = 0; i < n; ++i) out[i] = W[static_cast<size_t>(i) * TM] < 0.0f ? -1 : 1;
            const int r = claim_run(a);
            if (r >= 0) {
                slot_start(slot, r, a);
                const float* src = a.s0 + static_cast<size_t>(r) * n;
                for (int i = 0; i < n; ++i) W[static_cast<size_t>(i) * TM] = src[i];
            } else {
                slot.run = -1;
            }
        }
    }
}

}  // namespace

int relax_csr_slots_per_cta() { return TM; }
std::size_t relax_csr_work_floats(int np) { return static_cast<std::size_t>(np) * TM; }

cudaError_t launch_relax_csr(const RelaxArgs& a, int grid, cudaStream_t st) {
    relax_csr_kernel<<<grid, TM, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace marsb200
