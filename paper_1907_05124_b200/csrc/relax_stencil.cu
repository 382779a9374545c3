// relax_stencil.cu -- MARS relaxation on periodic lattices (Edwards-Anderson +-J tori),
// fp64, exact reference order, no neighbour-index stream.
//
// Replaces, for adjacency instances the host recognises as an L^DIMS torus with unit
// couplings (site i = c0 + L*c1 + L^2*c2, bonds to c_d +- 1 mod L -- the gen_ea shape):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:141-151   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// On such a torus the Gauss-Seidel level of a site is its coordinate sum (its lower
// neighbours are c_d - 1, one level down, and the wrap bond of a c_d = L-1 site, further
// down), so level l is the diagonal sum(c) = l: DIMS*(L-1)+1 levels, each a set of
// uncoupled sites.  A CTA owns one run; each level's sites are spread over the threads,
// one barrier per level.  A thread computes its site's 2*DIMS neighbour indices from the
// coordinates, puts them in ascending order with a sorting network (the order of the
// reference's sorted adjacency row) and applies the row's signs from the site's sign bits
// (bit k = sign of the k-th smallest neighbour's coupling), packed with the coordinates in
// one word per site (L <= 256) and fetched a level ahead, so a level's critical path is the
// shared-memory gathers, the fp64 sum and the tanh.  The neighbour sum is the
// reference's: acc = 0, acc += (+-1) * s_j in ascending j, unfused fp64 -- (+-1) * v is a
// sign flip, exact -- then + h_i.  State: fp64 in shared memory when it fits, else an
// L2-resident global row per CTA.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "ref_tanh.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

// tanh_trial (solvers.cpp:145-148) with the reference's own tanh, bit for bit (ref_tanh.cuh)
__device__ __forceinline__ double tanh_trial64(double phi, double t) { return ref_tanh_trial(phi, t); }

__device__ __forceinline__ void cswap(int& a, int& b) {
    const int lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

template <int DIMS>
__device__ __forceinline__ void sort_nb(int (&v)[2 * DIMS]) {
    if constexpr (DIMS == 2) {   // optimal 4-input network
        cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[1], v[2]);
    } else {                     // optimal 6-input network (12 comparators)
        cswap(v[1], v[2]); cswap(v[0], v[2]); cswap(v[0], v[1]); cswap(v[4], v[5]); cswap(v[3], v[5]);
        cswap(v[3], v[4]); cswap(v[0], v[3]); cswap(v[1], v[4]); cswap(v[2], v[5]); cswap(v[2], v[4]);
        cswap(v[1], v[3]); cswap(v[2], v[3]);
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One site: its packed word is c0 | c1 << 8 | c2 << 16 | signs << 24.
template <int DIMS>
__device__ __forceinline__ void relax_site(unsigned cc, int L, int s1, int s2, double T, const double* __restrict__ h64,
                                           double* st, double& dmax) {
    const int c0 = cc & 255, c1 = (cc >> 8) & 255, c2 = (cc >> 16) & 255;
    const unsigned bits = cc >> 24;
    const int i = c0 + s1 * c1 + s2 * c2;
    int nb[2 * DIMS];
    nb[0] = c0 ? i - 1 : i + (L - 1);
    nb[1] = c0 < L - 1 ? i + 1 : i - (L - 1);
    nb[2] = c1 ? i - s1 : i + (L - 1) * s1;
    nb[3] = c1 < L - 1 ? i + s1 : i - (L - 1) * s1;
    if constexpr (DIMS == 3) {
        nb[4] = c2 ? i - s2 : i + (L - 1) * s2;
        nb[5] = c2 < L - 1 ? i + s2 : i - (L - 1) * s2;
    }
    sort_nb<DIMS>(nb);
    double v[2 * DIMS];
#pragma unroll
    for (int k = 0; k < 2 * DIMS; ++k) v[k] = st[nb[k]];
    const double old = st[i];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 2 * DIMS; ++k)
        acc = __dadd_rn(acc, __hiloint2double(__double2hiint(v[k]) ^ static_cast<int>(((bits >> k) & 1u) << 31),
                                              __double2loint(v[k])));
    const double phi = __dadd_rn(acc, h64 ? __ldg(h64 + i) : 0.0);
    const double trial = tanh_trial64(phi, T);
    dmax = fmax(dmax, fabs(__dsub_rn(trial, old)));
    st[i] = trial;
}

template <int DIMS, bool SMEM_STATE>
__global__ void __launch_bounds__(1024, 1) relax_stencil_kernel(RelaxArgs a, StencilArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    __shared__ int s_run;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int n = a.n, L = g.L, nlev = g.nlev;
    const std::size_t state_bytes = SMEM_STATE ? (static_cast<std::size_t>(n) * sizeof(double) + 15) / 16 * 16 : 0;
    double* st = SMEM_STATE ? reinterpret_cast<double*>(smem_raw)
                            : reinterpret_cast<double*>(a.work) + static_cast<std::size_t>(blockIdx.x) * a.np;
    int* lvl = reinterpret_cast<int*>(smem_raw + state_bytes);   // [nlev + 1] level offsets
    for (int i = tid; i <= nlev; i += blockDim.x) lvl[i] = g.lvl_off[i];
    const double* s0 = static_cast<const double*>(a.s0_64);
    const unsigned* __restrict__ words = g.coords;
    const int s1 = L, s2 = L * L;

    Slot slot;
    for (;;) {
        if (tid == 0) s_run = claim_run(a);
        __syncthreads();
        const int r = s_run;
        __syncthreads();
        if (r < 0) break;
        slot_start(slot, r, a);
        for (int i = tid; i < n; i += blockDim.x) st[i] = s0[static_cast<std::size_t>(r) * n + i];
        __syncthreads();
        int code;
        do {
            const double T = slot.T;
            double dmax = 0.0;
            // the first site word of each level is fetched one level ahead (off the chain)
            unsigned next = tid < lvl[1] ? __ldg(words + tid) : 0u;
            for (int lv = 0; lv < nlev; ++lv) {
                const int b = lvl[lv], e = lvl[lv + 1];
                const unsigned cur = next;
                if (lv + 1 < nlev && lvl[lv + 1] + tid < lvl[lv + 2]) next = __ldg(words + lvl[lv + 1] + tid);
                if (b + tid < e) relax_site<DIMS>(cur, L, s1, s2, T, a.h64, st, dmax);
                for (int p = b + tid + static_cast<int>(blockDim.x); p < e; p += blockDim.x)
                    relax_site<DIMS>(__ldg(words + p), L, s1, s2, T, a.h64, st, dmax);
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
        std::int8_t* out = a.spins + static_cast<std::size_t>(slot.run) * n;
        for (int i = tid; i < n; i += blockDim.x) out[i] = st[i] < 0.0 ? -1 : 1;
        if (a.retire_log) {
            __syncthreads();
            if (tid == 0) log_retired(a, slot.run);
        }
    }
}

template <int DIMS, bool SMEM_STATE>
std::size_t smem_t(int n, int nlev) {
    return (SMEM_STATE ? (static_cast<std::size_t>(n) * sizeof(double) + 15) / 16 * 16 : 0) +
           static_cast<std::size_t>(nlev + 2) * sizeof(int);
}

template <int DIMS, bool SMEM_STATE>
cudaError_t launch_t(const RelaxArgs& a, const StencilArgs& g, const StencilLaunch& l, cudaStream_t st) {
    const std::size_t bytes = smem_t<DIMS, SMEM_STATE>(a.n, g.nlev);
    cudaError_t e = cudaFuncSetAttribute(relax_stencil_kernel<DIMS, SMEM_STATE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    relax_stencil_kernel<DIMS, SMEM_STATE><<<l.grid, l.threads, bytes, st>>>(a, g);
    return cudaGetLastError();
}

}  // namespace

std::size_t relax_stencil_smem(int n, int nlev, bool smem_state) {
    return smem_state ? smem_t<2, true>(n, nlev) : smem_t<2, false>(n, nlev);
}

cudaError_t launch_relax_stencil(const RelaxArgs& a, const StencilArgs& g, const StencilLaunch& l, cudaStream_t st) {
    if (l.threads < 32 || l.threads > 1024 || l.threads % 32) return cudaErrorInvalidValue;
    if (g.dims == 2) return l.smem_state ? launch_t<2, true>(a, g, l, st) : launch_t<2, false>(a, g, l, st);
    if (g.dims == 3) return l.smem_state ? launch_t<3, true>(a, g, l, st) : launch_t<3, false>(a, g, l, st);
    return cudaErrorInvalidValue;
}

}  // namespace marsb200
