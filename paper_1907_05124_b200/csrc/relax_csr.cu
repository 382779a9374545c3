// relax_csr.cu -- level-scheduled MARS relaxation for sparse couplings, fp64, exact order.
//
// Replaces, for sparse instances (CSR storage, model.cpp:91, or dense storage whose
// nonzeros are below kCsrDensity -- see mars_host.cpp):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:141-151   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// Gauss-Seidel in ascending spin order is a DAG: spin i reads the NEW value of every
// neighbour j < i and the OLD value of every neighbour j > i.  With
//     level(i) = 1 + max{ level(j) : j < i, J_ij != 0 }   (0 if none)
// a spin's lower neighbours sit in strictly earlier levels and its higher neighbours in
// strictly later ones (i is a lower neighbour of each of them), so no two spins of one
// level are coupled.  Updating a whole level at once, level after level, therefore reads
// exactly the values the sequential sweep reads: the result is bit-identical to the
// reference's sweep, with each spin's neighbour sum still taken in the reference's sorted
// order with unfused fp64 operations (__dmul_rn/__dadd_rn).  fp64 matters: on integer
// lattices the quench's phi == 0 ties are decided by ~1e-12 residuals.
//
// One CTA owns one run slot (persistent over the run queue).  Its fp64 state lives in
// shared memory when n doubles fit, else in an L2-resident global workspace row.  Levels
// are stored as 32-spin chunks (lane = spin); each chunk's neighbour lists are interleaved
// [k][32] so one load instruction fetches entry k for the 32 spins.  Lanes whose list is
// shorter than the chunk's longest read a padding slot st[n] == +0.0: acc never holds -0
// (it starts at +0 and exact cancellation rounds to +0), so adding +-0 leaves it unchanged
// bit for bit.  Unit couplings (every |J_ij| == 1, the +-J lattices and +-1 graphs) carry
// the sign in bit 31 of the index and skip the multiply: (+-1) * v is exact.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

__device__ __forceinline__ double tanh_trial64(double phi, double t) {
    if (t < kTempFloor) return phi > 0.0 ? -1.0 : (phi < 0.0 ? 1.0 : 0.0);
    return -tanh(__ddiv_rn(phi, t));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <bool SMEM_STATE, bool UNIT>
__global__ void __launch_bounds__(512) relax_levels_kernel(RelaxArgs a, SparseLevels g) {
    extern __shared__ double smem_state[];   // [n + 1] when SMEM_STATE
    __shared__ double red[32];
    __shared__ int s_run;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int n = a.n;
    double* st = SMEM_STATE ? smem_state
                            : reinterpret_cast<double*>(a.work) + static_cast<size_t>(blockIdx.x) * a.np;
    const double* s0 = static_cast<const double*>(a.s0_64);

    Slot slot;
    for (;;) {
        if (tid == 0) s_run = claim_run(a);
        __syncthreads();
        const int r = s_run;
        __syncthreads();
        if (r < 0) break;
        slot_start(slot, r, a);
        const double* src = s0 + static_cast<size_t>(r) * n;
        for (int i = tid; i < n; i += blockDim.x) st[i] = src[i];
        if (tid == 0) st[n] = 0.0;   // padding slot read by short neighbour lists
        __syncthreads();
        int code;
        do {
            const double T = slot.T;
            double dmax = 0.0;
            for (int L = 0; L < g.nlev; ++L) {
                const int c1 = __ldg(g.lvl_chunk + L + 1);
                for (int c = __ldg(g.lvl_chunk + L) + warp; c < c1; c += nwarps) {
                    const int base = __ldg(g.chunk_base + c);
                    const int md = __ldg(g.chunk_md + c);
                    const int sp = __ldg(g.spin + c * 32 + lane);
                    const int* ip = g.nidx + base + lane;
                    double acc = 0.0;
                    if (UNIT) {
#pragma unroll 4
                        for (int k = 0; k < md; ++k) {
                            const int e = __ldg(ip + 32 * k);
                            const unsigned long long v = __double_as_longlong(st[e & 0x7fffffff]);
                            // (+-1) * v == v with the sign bit flipped for -1: exact
                            acc = __dadd_rn(acc, __longlong_as_double(
                                                     v ^ (static_cast<unsigned long long>(static_cast<unsigned>(e) >> 31) << 63)));
                        }
                    } else {
                        const double* wp = g.nw + base + lane;
#pragma unroll 4
                        for (int k = 0; k < md; ++k)
                            acc = __dadd_rn(acc, __dmul_rn(__ldg(wp + 32 * k), st[__ldg(ip + 32 * k)]));
                    }
                    if (sp >= 0) {
                        const double phi = __dadd_rn(acc, a.h64 ? __ldg(a.h64 + sp) : 0.0);
                        const double trial = tanh_trial64(phi, T);
                        dmax = fmax(dmax, fabs(__dsub_rn(trial, st[sp])));
                        st[sp] = trial;
                    }
                }
                __syncthreads();
            }
            dmax = warp_max(dmax);
            if (lane == 0) red[warp] = dmax;
            __syncthreads();
            double d = red[0];
            for (int w = 1; w < nwarps; ++w) d = fmax(d, red[w]);
            // red is rewritten only after the next sweep's level barriers
            code = slot_after_sweep(slot, d, a);
        } while (code == kSlotContinue);
        if (tid == 0) slot_finish(slot, code, a);
        std::int8_t* out = a.spins + static_cast<size_t>(slot.run) * n;
        for (int i = tid; i < n; i += blockDim.x) out[i] = st[i] < 0.0 ? -1 : 1;
    }
}

template <bool SMEM_STATE, bool UNIT>
cudaError_t launch_t(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l, cudaStream_t st) {
    const std::size_t smem = SMEM_STATE ? static_cast<std::size_t>(a.n + 1) * sizeof(double) : 0;
    if (SMEM_STATE) {
        const cudaError_t e = cudaFuncSetAttribute(relax_levels_kernel<SMEM_STATE, UNIT>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    relax_levels_kernel<SMEM_STATE, UNIT><<<l.grid, l.warps * 32, smem, st>>>(a, g);
    return cudaGetLastError();
}

template <bool SMEM_STATE, bool UNIT>
int occupancy_t(int warps, int n) {
    const std::size_t smem = SMEM_STATE ? static_cast<std::size_t>(n + 1) * sizeof(double) : 0;
    if (SMEM_STATE &&
        cudaFuncSetAttribute(relax_levels_kernel<SMEM_STATE, UNIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
        return 0;
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, relax_levels_kernel<SMEM_STATE, UNIT>, warps * 32,
                                                      smem) != cudaSuccess)
        return 0;
    return blocks;
}

}  // namespace

int relax_sparse_occupancy(const SparseLaunch& l, bool unit, int n) {
    if (l.smem_state) return unit ? occupancy_t<true, true>(l.warps, n) : occupancy_t<true, false>(l.warps, n);
    return unit ? occupancy_t<false, true>(l.warps, n) : occupancy_t<false, false>(l.warps, n);
}

cudaError_t launch_relax_sparse(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l,
                                cudaStream_t st) {
    if (l.smem_state) return g.unit ? launch_t<true, true>(a, g, l, st) : launch_t<true, false>(a, g, l, st);
    return g.unit ? launch_t<false, true>(a, g, l, st) : launch_t<false, false>(a, g, l, st);
}

}  // namespace marsb200
