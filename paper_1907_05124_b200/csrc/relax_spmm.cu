// relax_spmm.cu -- warp-per-run MARS relaxation for sparse couplings whose fp64 state is
// small enough for several runs per SM (G-set-shape graphs), exact reference order.
//
// Replaces, like relax_csr.cu (same chunk layout, same exactness argument):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:141-151   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// SpMM shape: one CTA per SM holds RUNS = W*(32/CW) runs, each owned by a CW-lane group of
// one of W consumer warps, with its fp64 state row in shared memory.  Every consumer warp
// walks ALL chunks of the sweep in level order (a level's chunks are uncoupled; a chunk
// only reads rows written by earlier levels of the same group, so __syncwarp orders them)
// -- no CTA barrier inside a sweep.  A producer warp streams the chunk blocks through an
// S-slot shared-memory ring with the TMA engine (cp.async.bulk; `full` mbarrier per slot
// completes on the bytes, `empty` mbarrier collects one arrival per consumer warp), so each
// coupling block is read from L2 once per CTA per sweep and applied to all RUNS runs.
// One CTA barrier per sweep: finished runs are rounded, written out and refilled from the
// run queue by their own lane group; the CTA stops when no run is left.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

constexpr int kMaxConsumerWarps = 16;
constexpr int kMaxRing = 8;

__device__ __forceinline__ double tanh_trial64(double phi, double t) {
    if (t < kTempFloor) return phi > 0.0 ? -1.0 : (phi < 0.0 ? 1.0 : 0.0);
    return -tanh(__ddiv_rn(phi, t));
}

// Row e of a state array, with the coupling sign (bit 31 of the code) applied: (+-1) * v.
// The byte offset e << 3 drops the sign bit, so the address needs no mask.
__device__ __forceinline__ double signed_load(const double* st, int code) {
    const double v = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(st) + (static_cast<unsigned>(code) << 3));
    return __hiloint2double(__double2hiint(v) ^ (code & static_cast<int>(0x80000000u)), __double2loint(v));
}

template <int CW, bool UNIT>
__global__ void __launch_bounds__((kMaxConsumerWarps + 1) * 32, 1)
relax_spmm_kernel(RelaxArgs a, SparseLevels g, int nring) {
    constexpr int H = 32 / CW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) std::uint64_t full[kMaxRing], empty[kMaxRing];
    __shared__ Slot slots[kMaxConsumerWarps * H];
    __shared__ int s_active;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = (blockDim.x >> 5) - 1;          // consumer warps; warp W is the producer
    const int s = lane % CW, h = lane / CW;
    const int n = a.n, np = a.np;
    const int nch = g.nchunks;
    const std::uint32_t buf_bytes = g.buf_bytes;
    unsigned char* ring = smem_raw;
    double* st_all = reinterpret_cast<double*>(smem_raw + static_cast<std::size_t>(nring) * buf_bytes);
    const double* s0 = static_cast<const double*>(a.s0_64);

    if (tid == 0) {
        for (int i = 0; i < nring; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&empty[i], W);
        }
        umma::fence_mbar_init();
        s_active = 0;
    }
    __syncthreads();
    const int my = warp * H + h;                  // this lane group's run slot
    double* st = st_all + static_cast<std::size_t>(my) * np;
    if (warp < W) {
        if (s == 0) {
            const int run = claim_run(a);
            if (run >= 0) {
                slot_start(slots[my], run, a);
                atomicAdd(&s_active, 1);
            } else {
                slots[my].run = -1;
            }
        }
        __syncwarp();
        const int run = slots[my].run;
        if (run >= 0)
            for (int i = s; i < n; i += CW) st[i] = s0[static_cast<std::size_t>(run) * n + i];
        if (s == 0) st[n] = 0.0;                  // padding row read by short neighbour lists
    }
    __syncthreads();
    if (s_active == 0) return;

    unsigned q = 0;                               // chunks streamed so far (all warps agree)
    for (;;) {
        if (warp == W) {
            // ---------------- producer: one sweep of chunk blocks through the ring
            if (lane == 0) {
                for (int c = 0; c < nch; ++c) {
                    const unsigned k = q + c, slot = k % nring;
                    if (k >= static_cast<unsigned>(nring)) umma::mbar_wait(&empty[slot], ((k / nring) - 1) & 1);
                    const int4 d = __ldg(g.ctab + c);
                    const std::uint32_t ib = static_cast<std::uint32_t>(d.y) * 4u;
                    const std::uint32_t wb = UNIT ? 0u : static_cast<std::uint32_t>(d.w) * CW * 8u;
                    unsigned char* dst = ring + slot * buf_bytes;
                    umma::mbar_arrive_expect_tx(&full[slot], ib + wb);
                    umma::bulk_load(dst, g.blk + d.x, ib, &full[slot]);
                    if (!UNIT && wb) umma::bulk_load(dst + g.wbuf_off, g.wblk + d.z, wb, &full[slot]);
                }
            }
        } else {
            // ---------------- consumers: one Gauss-Seidel sweep of this group's run
            const bool act = slots[my].run >= 0;
            const double T = slots[my].T;
            double dmax = 0.0;
            for (int c = 0; c < nch; ++c) {
                const unsigned k = q + c, slot = k % nring;
                umma::mbar_wait(&full[slot], (k / nring) & 1);
                const int* blk = reinterpret_cast<const int*>(ring + slot * buf_bytes);
                if (act) {
                    const int md = blk[0];
                    const int sp = blk[4 + s];
                    const int* ip = blk + 4 + CW + s;
                    double acc = 0.0;
                    if (UNIT) {
#pragma unroll 8
                        for (int j = 0; j < md; ++j) acc = __dadd_rn(acc, signed_load(st, ip[CW * j]));
                    } else {
                        const double* wp = reinterpret_cast<const double*>(ring + slot * buf_bytes + g.wbuf_off) + s;
#pragma unroll 8
                        for (int j = 0; j < md; ++j) acc = __dadd_rn(acc, __dmul_rn(wp[CW * j], st[ip[CW * j]]));
                    }
                    if (sp >= 0) {
                        const double hf = a.h64 ? __ldg(a.h64 + sp) : 0.0;
                        const double trial = tanh_trial64(__dadd_rn(acc, hf), T);
                        dmax = fmax(dmax, fabs(__dsub_rn(trial, st[sp])));
                        st[sp] = trial;
                    }
                }
                __syncwarp();                     // block consumed; this level's writes visible
                if (lane == 0) umma::mbar_arrive(&empty[slot]);
            }
            // sweep end: the lane group's max change, state machine, refill
#pragma unroll
            for (int o = CW / 2; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            int code = kSlotContinue;
            if (act && s == 0) {
                code = slot_after_sweep(slots[my], dmax, a);
                if (code != kSlotContinue) slot_finish(slots[my], code, a);
            }
            code = __shfl_sync(0xffffffffu, code, h * CW);
            if (code != kSlotContinue) {               // uniform per lane group, not per warp
                const unsigned gmask = CW == 32 ? 0xffffffffu : (0xffffu << (h * CW));
                const int done = __shfl_sync(gmask, s == 0 ? slots[my].run : 0, h * CW);
                std::int8_t* out = a.spins + static_cast<std::size_t>(done) * n;
                for (int i = s; i < n; i += CW) out[i] = st[i] < 0.0 ? -1 : 1;
                int run = -1;
                if (s == 0) {
                    run = claim_run(a);
                    if (run >= 0) {
                        slot_start(slots[my], run, a);
                    } else {
                        slots[my].run = -1;
                        atomicSub(&s_active, 1);
                    }
                }
                run = __shfl_sync(gmask, run, h * CW);
                if (run >= 0)
                    for (int i = s; i < n; i += CW) st[i] = s0[static_cast<std::size_t>(run) * n + i];
            }
        }
        q += nch;
        __syncthreads();
        if (s_active == 0) return;                // every streamed block was consumed
    }
}

template <int CW, bool UNIT>
struct SpmmVariant {
    static std::size_t smem(int np, int warps, int nring, std::uint32_t buf_bytes) {
        return static_cast<std::size_t>(nring) * buf_bytes +
               static_cast<std::size_t>(warps) * (32 / CW) * np * sizeof(double);
    }
    static cudaError_t launch(const RelaxArgs& a, const SparseLevels& g, const SpmmLaunch& l, cudaStream_t st) {
        const std::size_t bytes = smem(a.np, l.warps, l.ring, g.buf_bytes);
        cudaError_t e = cudaFuncSetAttribute(relax_spmm_kernel<CW, UNIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bytes));
        if (e != cudaSuccess) return e;
        relax_spmm_kernel<CW, UNIT><<<l.grid, (l.warps + 1) * 32, bytes, st>>>(a, g, l.ring);
        return cudaGetLastError();
    }
};

}  // namespace

std::size_t relax_spmm_smem(int np, int cw, int warps, int ring, unsigned buf_bytes) {
    return static_cast<std::size_t>(ring) * buf_bytes + static_cast<std::size_t>(warps) * (32 / cw) * np * sizeof(double);
}
int relax_spmm_max_warps() { return kMaxConsumerWarps; }
int relax_spmm_max_ring() { return kMaxRing; }

cudaError_t launch_relax_spmm(const RelaxArgs& a, const SparseLevels& g, const SpmmLaunch& l, cudaStream_t st) {
    if (l.warps < 1 || l.warps > kMaxConsumerWarps || l.ring < 2 || l.ring > kMaxRing) return cudaErrorInvalidValue;
    if (l.cw == 32) return g.unit ? SpmmVariant<32, true>::launch(a, g, l, st) : SpmmVariant<32, false>::launch(a, g, l, st);
    if (l.cw == 16) return g.unit ? SpmmVariant<16, true>::launch(a, g, l, st) : SpmmVariant<16, false>::launch(a, g, l, st);
    return cudaErrorInvalidValue;
}

}  // namespace marsb200
