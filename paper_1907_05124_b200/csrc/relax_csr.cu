// relax_csr.cu -- persistent thread-per-run MARS relaxation for sparse couplings, fp64.
//
// Replaces, for sparse instances (CSR storage, model.cpp:91, or dense storage whose
// nonzeros are below kCsrDensity -- see mars_host.cpp):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:141-151   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// One thread owns one run slot and sweeps its spins in ascending order, summing each
// neighbour list in the reference's (sorted) order with the reference's fp64 operations,
// unfused (__dmul_rn/__dadd_rn), so a sweep differs from mars_relax_sweep only where the
// device tanh and libm tanh round differently.  fp64 matters here: on integer lattices the
// quench's phi == 0 ties are decided by ~1e-12 residuals that fp32 state cannot hold
// (measured: an fp32 replay of the reference keeps only 75% of EA 16x16 final states).
// The CSR arrays are read uniformly by a warp (broadcast); the state lives in a per-CTA
// workspace W[n][TM] (runs contiguous) so each neighbour gather is one coalesced row.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

constexpr int TM = 128;  // slots (threads) per CTA

__device__ __forceinline__ double tanh_trial64(double phi, double t) {
    if (t < kTempFloor) return phi > 0.0 ? -1.0 : (phi < 0.0 ? 1.0 : 0.0);
    return -tanh(__ddiv_rn(phi, t));
}

__device__ __forceinline__ void load_initial(double* W, const double* src, int n) {
    for (int i = 0; i < n; ++i) W[static_cast<size_t>(i) * TM] = src[i];
}

__global__ void __launch_bounds__(TM) relax_csr_kernel(RelaxArgs a) {
    const int tid = threadIdx.x;
    const int n = a.n;
    double* W = reinterpret_cast<double*>(a.work) + static_cast<size_t>(blockIdx.x) * a.np * TM + tid;
    const double* s0 = static_cast<const double*>(a.s0_64);

    Slot slot;
    slot.run = -1;
    {
        const int r = claim_run(a);
        if (r >= 0) {
            slot_start(slot, r, a);
            load_initial(W, s0 + static_cast<size_t>(r) * n, n);
        }
    }
    while (__syncthreads_or(slot.run >= 0)) {
        if (slot.run < 0) continue;
        const double T = slot.T;
        double dmax = 0.0;
        int k = __ldg(a.off);
        for (int i = 0; i < n; ++i) {
            const int kend = __ldg(a.off + i + 1);
            double acc = 0.0;
            for (; k < kend; ++k)
                acc = __dadd_rn(acc, __dmul_rn(__ldg(a.w64 + k),
                                               W[static_cast<size_t>(__ldg(a.idx + k)) * TM]));
            const double phi = __dadd_rn(acc, a.h64 ? __ldg(a.h64 + i) : 0.0);
            const double trial = tanh_trial64(phi, T);
            double* wp = W + static_cast<size_t>(i) * TM;
            dmax = fmax(dmax, fabs(__dsub_rn(trial, *wp)));
            *wp = trial;
        }
        const int code = slot_after_sweep(slot, dmax, a);
        if (code != kSlotContinue) {
            slot_finish(slot, code, a);
            std::int8_t* out = a.spins + static_cast<size_t>(slot.run) * n;
            for (int i = 0; i < n; ++i) out[i] = W[static_cast<size_t>(i) * TM] < 0.0 ? -1 : 1;
            const int r = claim_run(a);
            if (r >= 0) {
                slot_start(slot, r, a);
                load_initial(W, s0 + static_cast<size_t>(r) * n, n);
            } else {
                slot.run = -1;
            }
        }
    }
}

}  // namespace

int relax_csr_slots_per_cta() { return TM; }
std::size_t relax_csr_work_bytes(int np) { return static_cast<std::size_t>(np) * TM * sizeof(double); }

cudaError_t launch_relax_csr(const RelaxArgs& a, int grid, cudaStream_t st) {
    relax_csr_kernel<<<grid, TM, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace marsb200
