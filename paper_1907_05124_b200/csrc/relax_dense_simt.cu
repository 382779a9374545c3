// relax_dense_simt.cu -- persistent blocked Gauss-Seidel MARS relaxation, dense J, CUDA cores.
//
// Replaces, for a tile of TM concurrent descents per CTA:
//   mars_relax_sweep        solvers.cpp:150-161  (in-place ascending-index Gauss-Seidel)
//   IsingProblem::row_dot   model.cpp:141-146    (dense row dot product)
//   tanh_trial              solvers.cpp:145-148
//   relax_to_fixed_point    solvers.cpp:163-176  and the mars_descent level loop 178-200
//   run_batch_with's queue  runner.cpp:95-115    (slots refill from an atomic run queue)
//
// Left-looking blocked Gauss-Seidel.  For spin block b = [b*TB, (b+1)*TB) the fields of the
// whole tile are one GEMM over all K = np spins of the *current* state (new values for
// j < b*TB, old values for j >= b*TB):  Phi[r][i] = sum_j S[r][j] J[j][b*TB+i].  One thread
// per run then walks the block in ascending order, adding the in-block corrections
// J[k][i] * (s_i_new - s_i_old) for k > i, so every spin sees exactly its predecessors'
// fresh values -- the reference's update order.  Only the summation order differs
// (fp32, blocked), so trajectories agree within fp tolerance, not bitwise.
//
// Layout: per-CTA workspace W[np][TM] fp32 (spin-major, runs contiguous) so the GEMM's
// state chunks and the correction's write-back are both coalesced 256-byte rows.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "slot.cuh"

namespace marsb200 {
namespace {

constexpr int TM = 64;   // runs (slots) per CTA
constexpr int TB = 64;   // spins per Gauss-Seidel block
constexpr int KC = 32;   // K chunk staged per pipeline step
constexpr int NT = 256;  // threads: 16 x 16 grid of 4x4 register tiles

struct __align__(16) Smem {
    float S[2][KC][TM];    // state chunk (double buffered); reused as the block state Sb[TB][TM]
    float Jc[2][KC][TB];   // coupling chunk J[k][b*TB .. b*TB+TB)
    float Jd[TB][TB];      // diagonal block J[b*TB+i][b*TB+k]
    float Phi[TM][TB + 1]; // block fields, padded against bank conflicts
    float h[TB];
    int refill[TM];
    int retire[TM];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void load_chunk(Smem& sm, int buf, const float* W, const float* J32,
                                           int np, int b, int c, int tid) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int f = tid + q * NT;         // 512 float4 per operand
        const int row = f >> 4, col = (f & 15) * 4;
        cp_async16(&sm.S[buf][row][col], W + static_cast<size_t>(c * KC + row) * TM + col);
        cp_async16(&sm.Jc[buf][row][col],
                   J32 + static_cast<size_t>(c * KC + row) * np + b * TB + col);
    }
}

__global__ void __launch_bounds__(NT, 1) relax_dense_simt_kernel(RelaxArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x;
    const int n = a.n, np = a.np;
    const int nb = np / TB, nk = np / KC;
    float* W = static_cast<float*>(a.work) + static_cast<size_t>(blockIdx.x) * np * TM;
    const int tx = tid & 15, ty = tid >> 4;
    const int warp = tid >> 5, lane = tid & 31;

    Slot slot;
    slot.run = -1;
    if (tid < TM) {
        sm.retire[tid] = -1;
        sm.refill[tid] = -1;
        const int r = claim_run(a);
        if (r >= 0) {
            slot_start(slot, r, a);
            sm.refill[tid] = r;
        }
    }
    __syncthreads();

    for (;;) {
        // ---- slot turnover: rounded spins out of retired runs, s0 into refilled slots
        for (int r = warp; r < TM; r += NT / 32) {
            const int old_run = sm.retire[r];
            if (old_run >= 0) {
                std::int8_t* out = a.spins + static_cast<size_t>(old_run) * n;
                for (int i = lane; i < n; i += 32)                  // round_spins, model.cpp:245
                    out[i] = W[static_cast<size_t>(i) * TM + r] < 0.0f ? -1 : 1;
                if (a.state_out)
                    for (int i = lane; i < n; i += 32)
                        a.state_out[static_cast<size_t>(old_run) * n + i] = W[static_cast<size_t>(i) * TM + r];
            }
            const int new_run = sm.refill[r];
            if (new_run >= 0) {
                const float* src = a.s0 + static_cast<size_t>(new_run) * n;
                for (int i = lane; i < n; i += 32) W[static_cast<size_t>(i) * TM + r] = src[i];
            }
        }
        __syncthreads();
        if (tid < TM) {
            if (sm.retire[tid] >= 0) log_retired(a, sm.retire[tid]);
            sm.retire[tid] = -1;
            sm.refill[tid] = -1;
        }
        if (!__syncthreads_or(tid < TM && slot.run >= 0)) break;

        // ---- one Gauss-Seidel sweep of every active slot
        const bool mine = tid < TM && slot.run >= 0;
        const bool quench = mine && slot_quench(slot);
        const float Tf = static_cast<float>(slot.T);
        float dmax = 0.0f;

        for (int b = 0; b < nb; ++b) {
            // diagonal block + field slice, then the pipelined K loop
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int f = tid + q * NT;
                const int row = f >> 4, col = (f & 15) * 4;
                cp_async16(&sm.Jd[row][col],
                           a.J32 + static_cast<size_t>(b * TB + row) * np + b * TB + col);
            }
            if (tid < TB) sm.h[tid] = (a.h32 && b * TB + tid < n) ? a.h32[b * TB + tid] : 0.0f;
            load_chunk(sm, 0, W, a.J32, np, b, 0, tid);
            cp_commit();

            float acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

            for (int c = 0; c < nk; ++c) {
                const int buf = c & 1;
                if (c + 1 < nk) {
                    load_chunk(sm, buf ^ 1, W, a.J32, np, b, c + 1, tid);
                    cp_commit();
                    cp_wait<1>();
                } else {
                    cp_wait<0>();
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    const float4 sv = *reinterpret_cast<const float4*>(&sm.S[buf][k][4 * ty]);
                    const float4 jv = *reinterpret_cast<const float4*>(&sm.Jc[buf][k][4 * tx]);
                    const float s4[4] = {sv.x, sv.y, sv.z, sv.w};
                    const float j4[4] = {jv.x, jv.y, jv.z, jv.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(s4[i], j4[j], acc[i][j]);
                }
                __syncthreads();
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) sm.Phi[4 * ty + i][4 * tx + j] = acc[i][j];

            // block state (old values) into smem: Sb[i][r] = W[b*TB+i][r]
            float* Sb = &sm.S[0][0][0];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int f = tid + q * NT;
                const int row = f >> 4, col = (f & 15) * 4;
                *reinterpret_cast<float4*>(Sb + row * TM + col) =
                    *reinterpret_cast<const float4*>(W + static_cast<size_t>(b * TB + row) * TM + col);
            }
            __syncthreads();

            // ---- in-block sequential correction: one thread per run, ascending spin order
            if (mine) {
                float phi[TB];
#pragma unroll
                for (int k = 0; k < TB; ++k) phi[k] = sm.Phi[tid][k];
                const int lim = min(TB, n - b * TB);
#pragma unroll
                for (int i = 0; i < TB; ++i) {
                    if (i < lim) {
                        const float trial = tanh_trial(phi[i] + sm.h[i], Tf, quench);
                        const float delta = trial - Sb[i * TM + tid];
                        dmax = fmaxf(dmax, fabsf(delta));
                        Sb[i * TM + tid] = trial;
#pragma unroll
                        for (int k = i + 1; k < TB; ++k) phi[k] = fmaf(sm.Jd[i][k], delta, phi[k]);
                    }
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int f = tid + q * NT;
                const int row = f >> 4, col = (f & 15) * 4;
                *reinterpret_cast<float4*>(W + static_cast<size_t>(b * TB + row) * TM + col) =
                    *reinterpret_cast<const float4*>(Sb + row * TM + col);
            }
            __syncthreads();
        }

        // ---- annealing state machine per slot
        if (mine) {
            const int code = slot_after_sweep(slot, dmax, a);
            if (code != kSlotContinue) {
                slot_finish(slot, code, a);
                sm.retire[tid] = slot.run;
                const int r = claim_run(a);
                if (r >= 0) {
                    slot_start(slot, r, a);
                    sm.refill[tid] = r;
                } else {
                    slot.run = -1;
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace

int relax_dense_simt_slots_per_cta() { return TM; }
int relax_dense_simt_block() { return TB; }
std::size_t relax_dense_simt_work_bytes(int np) { return static_cast<std::size_t>(np) * TM * sizeof(float); }

cudaError_t launch_relax_dense_simt(const RelaxArgs& a, int grid, cudaStream_t st) {
    const int smem = static_cast<int>(sizeof(Smem));
    cudaError_t e = cudaFuncSetAttribute(relax_dense_simt_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    relax_dense_simt_kernel<<<grid, NT, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace marsb200
