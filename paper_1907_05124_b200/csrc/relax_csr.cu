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
// Layout (SpMM-shaped): a CTA relaxes RUNS = (32/CW)*R run slots in lockstep -- they share
// the graph, so they share the level schedule.  Levels are cut into CW-spin chunks; lane
// (s, h) = (lane % CW, lane / CW) owns spin s of the chunk for the R runs of group h, so
// every neighbour index feeds R independent fp64 chains.  The state is interleaved
// st[i][RUNS] (the R values a lane gathers are one 16-byte vector load), in shared memory
// when it fits, else in an L2-resident global row per CTA.
//
// Graph stream: each chunk is one contiguous block [md,-,-,-][spin x CW][idx: md x CW]
// (+ an fp64 weight block [md x CW] for non-unit couplings).  Each warp walks its chunks
// (c = first + warp, step nwarps, level by level) and double-buffers them in shared memory
// with the TMA engine (cp.async.bulk on a per-warp mbarrier), one chunk ahead and across
// level and sweep boundaries (the graph is the same every sweep), so the inner loop reads
// only shared memory.  Lanes whose list is shorter than the chunk's longest read padding
// row n (all +0.0): acc never holds -0 (it starts at +0 and exact cancellation rounds to
// +0), so adding +-0 leaves it unchanged bit for bit.  Unit couplings (every |J_ij| == 1:
// the +-J lattices, +-1 graphs) carry the sign in bit 31 and skip the multiply, since
// (+-1) * v is exact.  Runs finish at different sweeps; a finished slot is refilled from
// the run queue at the sweep boundary while the others wait at the barrier.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "ref_tanh.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

// tanh_trial (solvers.cpp:145-148) with the reference's own tanh, bit for bit (ref_tanh.cuh)
__device__ __forceinline__ double tanh_trial64(double phi, double t) { return ref_tanh_trial(phi, t); }

__device__ __forceinline__ double flip(double v, unsigned long long sign) {
    return __longlong_as_double(__double_as_longlong(v) ^ sign);
}

// The R values of lane group h at state row e (R consecutive doubles, 16-byte aligned).
template <int R>
__device__ __forceinline__ void gather(const double* row, double (&v)[R]) {
    if constexpr (R == 1) {
        v[0] = row[0];
    } else {
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
            const double2 x = reinterpret_cast<const double2*>(row)[q];
            v[2 * q] = x.x;
            v[2 * q + 1] = x.y;
        }
    }
}

// Per-warp chunk iterator: chunks first(L) + warp + k*nwarps of each level, cycling through
// the levels (and into the next sweep).  Requires nwarps <= the widest level's chunk count,
// so every warp owns at least one chunk per sweep.
struct ChunkIter {
    int L, c, end;
    __device__ __forceinline__ void seek(const SparseLevels& g, int warp, int nwarps) {
        while (c >= end) {
            L = L + 1 == g.nlev ? 0 : L + 1;
            c = __ldg(g.lvl_chunk + L) + warp;
            end = __ldg(g.lvl_chunk + L + 1);
        }
    }
};

// Lane 0: stream the chunk described by `d` = {block offset (ints), block length (ints),
// weight offset (doubles), md} into buffer `slot & 1` of this warp, then advance the
// producer iterator and prefetch the next descriptor.
template <int CW, bool UNIT>
__device__ __forceinline__ void issue_chunk(const SparseLevels& g, int4& d, ChunkIter& it, unsigned char* wbuf,
                                            std::uint64_t (&bar)[2], unsigned slot, int warp, int nwarps) {
    unsigned char* dst = wbuf + (slot & 1) * g.buf_bytes;
    const std::uint32_t ib = static_cast<std::uint32_t>(d.y) * 4u;
    const std::uint32_t wb = UNIT ? 0u : static_cast<std::uint32_t>(d.w) * CW * 8u;
    umma::mbar_arrive_expect_tx(&bar[slot & 1], ib + wb);
    umma::bulk_load(dst, g.blk + d.x, ib, &bar[slot & 1]);
    if (!UNIT && wb) umma::bulk_load(dst + g.wbuf_off, g.wblk + d.z, wb, &bar[slot & 1]);
    it.c += nwarps;
    it.seek(g, warp, nwarps);
    d = __ldg(g.ctab + it.c);
}

template <int CW, int R, bool SMEM_STATE, bool UNIT>
__global__ void __launch_bounds__(512) relax_levels_kernel(RelaxArgs a, SparseLevels g) {
    constexpr int H = 32 / CW;
    constexpr int RUNS = H * R;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[16 * RUNS];        // per warp, per run (<= 16 warps)
    __shared__ Slot slots[RUNS];
    __shared__ int s_code[RUNS];
    __shared__ int s_active;
    __shared__ __align__(8) std::uint64_t bars[16][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = lane % CW, h = lane / CW;
    const int nwarps = blockDim.x >> 5;
    const int n = a.n;
    // dynamic smem: [state (n+1) x RUNS doubles, if SMEM_STATE][per warp: 2 x chunk buffer]
    const std::size_t state_bytes = SMEM_STATE ? (static_cast<std::size_t>(n + 1) * RUNS * sizeof(double) + 15) / 16 * 16 : 0;
    double* st = SMEM_STATE ? reinterpret_cast<double*>(smem_raw)
                            : reinterpret_cast<double*>(a.work) + static_cast<size_t>(blockIdx.x) * a.np * RUNS;
    const std::uint32_t buf_bytes = g.buf_bytes;
    unsigned char* wbuf = smem_raw + state_bytes + static_cast<std::size_t>(warp) * 2 * buf_bytes;
    const double* s0 = static_cast<const double*>(a.s0_64);

    if (lane == 0) {
        umma::mbar_init(&bars[warp][0], 1);
        umma::mbar_init(&bars[warp][1], 1);
        umma::fence_mbar_init();
    }
    for (int r = tid; r < RUNS; r += blockDim.x) st[static_cast<size_t>(n) * RUNS + r] = 0.0;   // padding row
    // fill every slot from the queue (highest start temperature first)
    for (int r = 0; r < RUNS; ++r) {
        if (tid == 0) {
            const int run = claim_run(a);
            if (run >= 0) slot_start(slots[r], run, a);
            else slots[r].run = -1;
        }
        __syncthreads();
        const int run = slots[r].run;
        if (run >= 0)
            for (int i = tid; i < n; i += blockDim.x)
                st[static_cast<size_t>(i) * RUNS + r] = s0[static_cast<size_t>(run) * n + i];
    }
    __syncthreads();
    if (slots[0].run < 0) return;   // queue empty before this CTA started (uniform)

    // producer side of the chunk stream (lane 0): issue chunk blocks one ahead of use
    ChunkIter prod{0, __ldg(g.lvl_chunk) + warp, __ldg(g.lvl_chunk + 1)};
    int4 pdesc = make_int4(0, 0, 0, 0);
    if (lane == 0) {
        prod.seek(g, warp, nwarps);
        pdesc = __ldg(g.ctab + prod.c);
    }
    unsigned item = 0;                   // chunks consumed by this warp
    if (lane == 0) issue_chunk<CW, UNIT>(g, pdesc, prod, wbuf, bars[warp], 0, warp, nwarps);

    for (;;) {
        double T[R], dmax[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T[r] = slots[h * R + r].T;
            dmax[r] = 0.0;
        }
        for (int L = 0; L < g.nlev; ++L) {
            const int c1 = __ldg(g.lvl_chunk + L + 1);
            for (int c = __ldg(g.lvl_chunk + L) + warp; c < c1; c += nwarps, ++item) {
                __syncwarp();             // the other buffer's previous chunk is fully consumed
                if (lane == 0) {
                    umma::fence_proxy_async_smem();
                    issue_chunk<CW, UNIT>(g, pdesc, prod, wbuf, bars[warp], item + 1, warp, nwarps);
                }
                umma::mbar_wait(&bars[warp][item & 1], (item >> 1) & 1);
                const int* blk = reinterpret_cast<const int*>(wbuf + (item & 1) * buf_bytes);
                const int md = blk[0];
                const int sp = blk[4 + s];
                const int* ip = blk + 4 + CW + s;
                double acc[R];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = 0.0;
                if (UNIT) {
#pragma unroll 8
                    for (int k = 0; k < md; ++k) {
                        const int e = ip[CW * k];
                        const unsigned long long sign = static_cast<unsigned long long>(static_cast<unsigned>(e) >> 31) << 63;
                        double v[R];
                        gather<R>(st + static_cast<size_t>(e & 0x7fffffff) * RUNS + h * R, v);
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], flip(v[r], sign));
                    }
                } else {
                    const double* wp = reinterpret_cast<const double*>(wbuf + (item & 1) * buf_bytes + g.wbuf_off) + s;
#pragma unroll 8
                    for (int k = 0; k < md; ++k) {
                        const int e = ip[CW * k];
                        const double wk = wp[CW * k];
                        double v[R];
                        gather<R>(st + static_cast<size_t>(e) * RUNS + h * R, v);
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(wk, v[r]));
                    }
                }
                if (sp >= 0) {
                    const double hf = a.h64 ? __ldg(a.h64 + sp) : 0.0;
                    double* row = st + static_cast<size_t>(sp) * RUNS + h * R;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double trial = tanh_trial64(__dadd_rn(acc[r], hf), T[r]);
                        dmax[r] = fmax(dmax[r], fabs(__dsub_rn(trial, row[r])));
                        row[r] = trial;
                    }
                }
            }
            __syncthreads();
        }
        // per-run max change over the CTA
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double v = dmax[r];
#pragma unroll
            for (int o = CW / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (s == 0) red[warp * RUNS + h * R + r] = v;
        }
        __syncthreads();
        if (tid < RUNS) {
            Slot& sl = slots[tid];
            int code = kSlotContinue;
            if (sl.run >= 0) {
                double d = red[tid];
                for (int w = 1; w < nwarps; ++w) d = fmax(d, red[w * RUNS + tid]);
                code = slot_after_sweep(sl, d, a);
                if (code != kSlotContinue) slot_finish(sl, code, a);
            }
            s_code[tid] = code;
        }
        __syncthreads();
        // round and store finished runs, refill their slots
        for (int r = 0; r < RUNS; ++r) {
            if (s_code[r] == kSlotContinue) continue;            // uniform
            std::int8_t* out = a.spins + static_cast<size_t>(slots[r].run) * n;
            for (int i = tid; i < n; i += blockDim.x) out[i] = st[static_cast<size_t>(i) * RUNS + r] < 0.0 ? -1 : 1;
            __syncthreads();
            if (tid == 0) {
                log_retired(a, slots[r].run);
                const int run = claim_run(a);
                if (run >= 0) slot_start(slots[r], run, a);
                else slots[r].run = -1;
            }
            __syncthreads();
            const int run = slots[r].run;
            if (run >= 0)
                for (int i = tid; i < n; i += blockDim.x)
                    st[static_cast<size_t>(i) * RUNS + r] = s0[static_cast<size_t>(run) * n + i];
        }
        if (tid == 0) {
            int act = 0;
            for (int r = 0; r < RUNS; ++r) act += slots[r].run >= 0;
            s_active = act;
        }
        __syncthreads();
        if (s_active == 0) break;
    }
    // drain the chunk block still in flight before the CTA's shared memory is released
    if (lane == 0) umma::mbar_wait(&bars[warp][item & 1], (item >> 1) & 1);
}

template <int CW, int R, bool SMEM_STATE, bool UNIT>
struct Variant {
    static constexpr int kRuns = (32 / CW) * R;
    static std::size_t smem(int n, int warps, std::uint32_t buf_bytes) {
        const std::size_t state = SMEM_STATE ? (static_cast<std::size_t>(n + 1) * kRuns * sizeof(double) + 15) / 16 * 16 : 0;
        return state + static_cast<std::size_t>(warps) * 2 * buf_bytes;
    }
    static cudaError_t prepare(std::size_t bytes) {
        return cudaFuncSetAttribute(relax_levels_kernel<CW, R, SMEM_STATE, UNIT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    }
    static cudaError_t launch(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l, cudaStream_t st) {
        const std::size_t bytes = smem(a.n, l.warps, g.buf_bytes);
        const cudaError_t e = prepare(bytes);
        if (e != cudaSuccess) return e;
        relax_levels_kernel<CW, R, SMEM_STATE, UNIT><<<l.grid, l.warps * 32, bytes, st>>>(a, g);
        return cudaGetLastError();
    }
    static int occupancy(int warps, int n, std::uint32_t buf_bytes) {
        const std::size_t bytes = smem(n, warps, buf_bytes);
        if (prepare(bytes) != cudaSuccess) return 0;
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, relax_levels_kernel<CW, R, SMEM_STATE, UNIT>,
                                                          warps * 32, bytes) != cudaSuccess)
            return 0;
        return blocks;
    }
};

// f(Variant<...>{}) for the launch's (cw, r, smem_state, unit).
template <class F>
auto dispatch(const SparseLaunch& l, bool unit, F&& f) {
#define MARS_SPARSE_CASE(CW, R)                                                                    \
    if (l.cw == CW && l.r == R) {                                                                  \
        if (l.smem_state) return unit ? f(Variant<CW, R, true, true>{}) : f(Variant<CW, R, true, false>{}); \
        return unit ? f(Variant<CW, R, false, true>{}) : f(Variant<CW, R, false, false>{});        \
    }
    MARS_SPARSE_CASE(32, 1)
    MARS_SPARSE_CASE(32, 2)
    MARS_SPARSE_CASE(32, 4)
    MARS_SPARSE_CASE(16, 1)
    MARS_SPARSE_CASE(16, 2)
    MARS_SPARSE_CASE(16, 4)
#undef MARS_SPARSE_CASE
    return f(Variant<32, 1, false, false>{});   // unreachable for validated shapes
}

}  // namespace

bool relax_sparse_shape_ok(int cw, int r) { return (cw == 32 || cw == 16) && (r == 1 || r == 2 || r == 4); }

int relax_sparse_occupancy(const SparseLaunch& l, const SparseLevels& g, int n) {
    if (!relax_sparse_shape_ok(l.cw, l.r)) return 0;
    return dispatch(l, g.unit, [&](auto v) { return decltype(v)::occupancy(l.warps, n, g.buf_bytes); });
}

cudaError_t launch_relax_sparse(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l,
                                cudaStream_t st) {
    if (!relax_sparse_shape_ok(l.cw, l.r)) return cudaErrorInvalidValue;
    return dispatch(l, g.unit, [&](auto v) { return decltype(v)::launch(a, g, l, st); });
}

}  // namespace marsb200
