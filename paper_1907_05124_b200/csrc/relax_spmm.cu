// relax_spmm.cu -- warp-per-run MARS relaxation for sparse couplings whose fp64 state is
// small enough for several runs per SM (G-set-shape graphs), exact reference order.
//
// Replaces, like relax_csr.cu (same chunk layout, same exactness argument):
//   mars_relax_sweep        solvers.cpp:150-161
//   IsingProblem::row_dot   model.cpp:141-151   (sum over the sorted neighbour list)
//   tanh_trial / relax_to_fixed_point / mars_descent loop  (solvers.cpp:145-200)
//
// SpMM shape: one CTA holds RUNS = W*H runs, each owned by a 32/H-lane group of one of W
// consumer warps, with its fp64 state row in shared memory.  Every consumer warp walks ALL
// chunks of the sweep in level order (a level's spins are uncoupled; a chunk only reads
// rows written by earlier levels of the same group, so __syncwarp orders them) -- no CTA
// barrier inside a sweep.  A chunk is CWL = (32/H)*K spins wide: each lane owns K spins of
// it, i.e. K independent exact-order sums and tanh chains in flight per lane.  Neighbour
// lists are padded to a multiple of 4 with the +0.0 row, so the gather loop has no
// remainder (padding reads hit one address: a shared-memory broadcast).
//
// A producer warp streams the chunk blocks through a shared-memory byte ring with the TMA
// engine (cp.async.bulk): chunks are packed back to back at their own size (FIFO, wrapping
// to offset 0 when the tail does not fit), up to kMaxSlots in flight; per slot a `full`
// mbarrier completes on the bytes and an `empty` mbarrier collects one arrival per
// consumer warp, and the slot's ring offset is published in shared memory before the copy
// is armed.  Each coupling block is read from L2 once per CTA per sweep and applied to all
// RUNS runs.  One CTA barrier per sweep: finished runs are rounded, written out and
// refilled from the run queue by their own lane group; the CTA stops when no run is left.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "ref_tanh.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

constexpr int kMaxConsumerWarps = 16;
constexpr int kMaxSlots = 16;   // chunks in flight

// tanh_trial (solvers.cpp:145-148) with the reference's own tanh, bit for bit (ref_tanh.cuh)
__device__ __forceinline__ double tanh_trial64(double phi, double t) { return ref_tanh_trial(phi, t); }

// Row e of a state array, with the coupling sign (bit 31 of the code) applied: (+-1) * v.
// The byte offset e << 3 drops the sign bit, so the address needs no mask.
__device__ __forceinline__ double signed_load(const double* st, int code) {
    const double v = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(st) + (static_cast<unsigned>(code) << 3));
    return __hiloint2double(__double2hiint(v) ^ (code & static_cast<int>(0x80000000u)), __double2loint(v));
}

// Single-producer FIFO allocator over the byte ring (lane 0 of the producer warp).
struct RingAlloc {
    unsigned head, oldest, inflight;   // next free byte, oldest in-flight chunk index, count
};

template <int H, int K, int R, bool UNIT>
__global__ void __launch_bounds__((kMaxConsumerWarps + 1) * 32, 1)
relax_spmm_kernel(RelaxArgs a, SparseLevels g, int ring_bytes) {
    static_assert(R == 1 || (R == 2 && K == 1), "two runs per lane group only with one spin per lane");
    constexpr int CWR = 32 / H;        // lanes per lane group
    constexpr int CWL = CWR * K;       // spins per chunk (layout width)
    constexpr int nring = kMaxSlots;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) std::uint64_t full[kMaxSlots], empty[kMaxSlots];
    __shared__ unsigned offs[kMaxSlots];
    __shared__ Slot slots[kMaxConsumerWarps * H * R];
    __shared__ int s_active;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = (blockDim.x >> 5) - 1;          // consumer warps; warp W is the producer
    const int s = lane % CWR, h = lane / CWR;
    const unsigned gmask = H == 1 ? 0xffffffffu : (((1u << CWR) - 1u) << (h * CWR));
    const int n = a.n, np = a.np;
    const int nch = g.nchunks;
    unsigned char* ring = smem_raw;
    double* st_all = reinterpret_cast<double*>(smem_raw + ring_bytes);
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
    // lane group (warp, h) owns R run slots; their states are interleaved st[i][R]
    const int my = (warp * H + h) * R;            // first run slot of this lane group
    double* st = st_all + static_cast<std::size_t>(warp * H + h) * np * R;
    if (warp < W) {
        for (int r = 0; r < R; ++r) {
            if (s == 0) {
                const int run = claim_run(a);
                if (run >= 0) {
                    slot_start(slots[my + r], run, a);
                    atomicAdd(&s_active, 1);
                } else {
                    slots[my + r].run = -1;
                }
            }
            __syncwarp();
            const int run = slots[my + r].run;
            if (run >= 0)
                for (int i = s; i < n; i += CWR) st[static_cast<std::size_t>(i) * R + r] = s0[static_cast<std::size_t>(run) * n + i];
            if (s == 0) st[static_cast<std::size_t>(n) * R + r] = 0.0;   // padding row
        }
    }
    __syncthreads();
    if (s_active == 0) return;

    unsigned q = 0;                               // chunks streamed so far (all warps agree)
    RingAlloc ra{0, 0, 0};                        // producer lane 0 only
    for (;;) {
        if (warp == W) {
            // ---------------- producer: one sweep of chunk blocks through the ring
            if (lane == 0) {
                int4 d = __ldg(g.ctab);
                for (int c = 0; c < nch; ++c) {
                    const unsigned k = q + c, slot = k % nring;
                    const std::uint32_t ib = static_cast<std::uint32_t>(d.y) * 4u;
                    const std::uint32_t wb = UNIT ? 0u : static_cast<std::uint32_t>(d.w) * CWL * 8u;
                    const std::uint32_t sz = ib + wb;     // both multiples of 16
                    // FIFO space: release the oldest chunks until sz contiguous bytes are free
                    unsigned off;
                    for (;;) {
                        if (ra.inflight == 0) {
                            ra.head = 0;
                            off = 0;
                            break;
                        }
                        if (ra.inflight < static_cast<unsigned>(nring)) {
                            // occupied: [tail, head) or, wrapped, [tail, end) + [0, head);
                            // strict bounds keep head != tail while anything is in flight
                            const unsigned tail = offs[ra.oldest % nring];
                            if (tail > ra.head) {
                                if (ra.head + sz < tail) { off = ra.head; break; }
                            } else if (ra.head + sz <= static_cast<unsigned>(ring_bytes)) {
                                off = ra.head;
                                break;
                            } else if (sz < tail) {
                                off = 0;
                                break;
                            }
                        }
                        umma::mbar_wait(&empty[ra.oldest % nring], (ra.oldest / nring) & 1);
                        ++ra.oldest;
                        --ra.inflight;
                    }
                    ra.head = off + sz;
                    ++ra.inflight;
                    offs[slot] = off;
                    unsigned char* dst = ring + off;
                    umma::mbar_arrive_expect_tx(&full[slot], sz);
                    umma::bulk_load(dst, g.blk + d.x, ib, &full[slot]);
                    if (!UNIT && wb) umma::bulk_load(dst + ib, g.wblk + d.z, wb, &full[slot]);
                    if (c + 1 < nch) d = __ldg(g.ctab + c + 1);
                }
            }
        } else {
            // ---------------- consumers: one Gauss-Seidel sweep of this group's runs
            bool act[R];
            double T[R], dmax[R];
            bool any = false;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                act[r] = slots[my + r].run >= 0;
                T[r] = slots[my + r].T;
                dmax[r] = 0.0;
                any |= act[r];
            }
            long long t_wait = 0, t_sum = 0, t_trial = 0;
            for (int c = 0; c < nch; ++c) {
                const unsigned k = q + c, slot = k % nring;
                const long long t0 = a.prof ? clock64() : 0;
                umma::mbar_wait(&full[slot], (k / nring) & 1);
                const long long t1 = a.prof ? clock64() : 0;
                const unsigned char* cbase = ring + offs[slot];
                const int* blk = reinterpret_cast<const int*>(cbase);
                if (any) {
                    const int md = blk[0];                  // multiple of 4
                    int sp[K];
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) sp[kk] = blk[4 + s + CWR * kk];
                    const int* ip = blk + 4 + CWL + s;
                    double acc[K][R];
#pragma unroll
                    for (int kk = 0; kk < K; ++kk)
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[kk][r] = 0.0;
                    if (UNIT) {
                        for (int j = 0; j < md; j += 4) {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
#pragma unroll
                                for (int kk = 0; kk < K; ++kk) {
                                    const int code = ip[CWL * (j + u) + CWR * kk];
                                    if constexpr (R == 1) {
                                        acc[kk][0] = __dadd_rn(acc[kk][0], signed_load(st, code));
                                    } else {
                                        // both runs' values of row e: one 16-byte load (code << 4
                                        // drops the sign bit), (+-1) * v as a sign-bit flip
                                        const double2 v = *reinterpret_cast<const double2*>(
                                            reinterpret_cast<const char*>(st) + (static_cast<unsigned>(code) << 4));
                                        const int sg = code & static_cast<int>(0x80000000u);
                                        acc[kk][0] = __dadd_rn(acc[kk][0], __hiloint2double(__double2hiint(v.x) ^ sg, __double2loint(v.x)));
                                        acc[kk][1] = __dadd_rn(acc[kk][1], __hiloint2double(__double2hiint(v.y) ^ sg, __double2loint(v.y)));
                                    }
                                }
                        }
                    } else {
                        const double* wp = reinterpret_cast<const double*>(cbase + ((4 + CWL + md * CWL) * 4 + 15) / 16 * 16) + s;
                        for (int j = 0; j < md; j += 4) {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
#pragma unroll
                                for (int kk = 0; kk < K; ++kk) {
                                    const double wk = wp[CWL * (j + u) + CWR * kk];
                                    const int e = ip[CWL * (j + u) + CWR * kk];
#pragma unroll
                                    for (int r = 0; r < R; ++r)
                                        acc[kk][r] = __dadd_rn(acc[kk][r], __dmul_rn(wk, st[static_cast<std::size_t>(e) * R + r]));
                                }
                        }
                    }
                    if (a.prof) {
                        __syncwarp();
                        const long long t2 = clock64();
                        t_sum += t2 - t1;
                        t_wait += t1 - t0;
                        t_trial -= t2;
                    }
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        if (sp[kk] >= 0) {
                            const double hf = a.h64 ? __ldg(a.h64 + sp[kk]) : 0.0;
                            double* row = st + static_cast<std::size_t>(sp[kk]) * R;
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const double trial = tanh_trial64(__dadd_rn(acc[kk][r], hf), T[r]);
                                dmax[r] = fmax(dmax[r], fabs(__dsub_rn(trial, row[r])));
                                row[r] = trial;
                            }
                        }
                    }
                }
                __syncwarp();                     // block consumed; this level's writes visible
                if (a.prof && any) t_trial += clock64();
                if (lane == 0) umma::mbar_arrive(&empty[slot]);
            }
            if (a.prof && lane == 0 && any) {
                long long* pr = a.prof + static_cast<std::size_t>(blockIdx.x) * kProfSlots;
                atomicAdd(reinterpret_cast<unsigned long long*>(pr + 0), 1ull);                 // warp-sweeps
                atomicAdd(reinterpret_cast<unsigned long long*>(pr + 1), static_cast<unsigned long long>(t_wait));
                atomicAdd(reinterpret_cast<unsigned long long*>(pr + 2), static_cast<unsigned long long>(t_sum));
                atomicAdd(reinterpret_cast<unsigned long long*>(pr + 3), static_cast<unsigned long long>(t_trial));
            }
            // sweep end, per run: the lane group's max change, state machine, refill
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double d = dmax[r];
#pragma unroll
                for (int o = CWR / 2; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
                int code = kSlotContinue;
                if (act[r] && s == 0) {
                    code = slot_after_sweep(slots[my + r], d, a);
                    if (code != kSlotContinue) slot_finish(slots[my + r], code, a);
                }
                code = __shfl_sync(0xffffffffu, code, h * CWR);
                if (code != kSlotContinue) {               // uniform per lane group, not per warp
                    const int done = __shfl_sync(gmask, s == 0 ? slots[my + r].run : 0, h * CWR);
                    std::int8_t* out = a.spins + static_cast<std::size_t>(done) * n;
                    for (int i = s; i < n; i += CWR) out[i] = st[static_cast<std::size_t>(i) * R + r] < 0.0 ? -1 : 1;
                    __syncwarp(gmask);
                    if (s == 0) log_retired(a, done);
                    int run = -1;
                    if (s == 0) {
                        run = claim_run(a);
                        if (run >= 0) {
                            slot_start(slots[my + r], run, a);
                        } else {
                            slots[my + r].run = -1;
                            atomicSub(&s_active, 1);
                        }
                    }
                    run = __shfl_sync(gmask, run, h * CWR);
                    if (run >= 0)
                        for (int i = s; i < n; i += CWR)
                            st[static_cast<std::size_t>(i) * R + r] = s0[static_cast<std::size_t>(run) * n + i];
                }
            }
        }
        q += nch;
        __syncthreads();
        if (s_active == 0) return;                // every streamed block was consumed
    }
}

template <int H, int K, int R, bool UNIT>
cudaError_t launch_t(const RelaxArgs& a, const SparseLevels& g, const SpmmLaunch& l, cudaStream_t st) {
    const std::size_t bytes = relax_spmm_smem(a.np, H * R, l.warps, l.ring_bytes);
    cudaError_t e = cudaFuncSetAttribute(relax_spmm_kernel<H, K, R, UNIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    relax_spmm_kernel<H, K, R, UNIT><<<l.grid, (l.warps + 1) * 32, bytes, st>>>(a, g, l.ring_bytes);
    return cudaGetLastError();
}

}  // namespace

std::size_t relax_spmm_smem(int np, int runs_per_warp, int warps, int ring_bytes) {
    return static_cast<std::size_t>(ring_bytes) + static_cast<std::size_t>(warps) * runs_per_warp * np * sizeof(double);
}
int relax_spmm_max_warps() { return kMaxConsumerWarps; }

bool relax_spmm_shape_ok(int layout_width, int runs_per_warp) {
    const int k = layout_width * runs_per_warp / 32;
    return (runs_per_warp == 1 || runs_per_warp == 2) && (k == 1 || k == 2) && k * 32 == layout_width * runs_per_warp;
}

cudaError_t launch_relax_spmm(const RelaxArgs& a, const SparseLevels& g, const SpmmLaunch& l, cudaStream_t st) {
    // the ring must hold the largest chunk block
    if (l.warps < 1 || l.warps > kMaxConsumerWarps || l.ring_bytes < static_cast<int>(g.buf_bytes) || l.ring_bytes % 16 ||
        !relax_spmm_shape_ok(l.cw, l.h))
        return cudaErrorInvalidValue;
    const int k = l.cw * l.h / 32;
    if (l.r == 2) {
        if (k != 1) return cudaErrorInvalidValue;
        if (l.h == 1) return g.unit ? launch_t<1, 1, 2, true>(a, g, l, st) : launch_t<1, 1, 2, false>(a, g, l, st);
        return g.unit ? launch_t<2, 1, 2, true>(a, g, l, st) : launch_t<2, 1, 2, false>(a, g, l, st);
    }
    if (l.h == 1 && k == 1) return g.unit ? launch_t<1, 1, 1, true>(a, g, l, st) : launch_t<1, 1, 1, false>(a, g, l, st);
    if (l.h == 1 && k == 2) return g.unit ? launch_t<1, 2, 1, true>(a, g, l, st) : launch_t<1, 2, 1, false>(a, g, l, st);
    if (l.h == 2 && k == 1) return g.unit ? launch_t<2, 1, 1, true>(a, g, l, st) : launch_t<2, 1, 1, false>(a, g, l, st);
    return g.unit ? launch_t<2, 2, 1, true>(a, g, l, st) : launch_t<2, 2, 1, false>(a, g, l, st);
}

}  // namespace marsb200
