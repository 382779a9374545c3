// relax_dense_umma.cu -- persistent blocked Gauss-Seidel MARS relaxation on tcgen05 tensor
// cores (sm_100a): TMA-fed UMMA field GEMM into TMEM + fused Gauss-Seidel epilogue.
//
// Replaces, for a tile of TM = 128 concurrent descents per CTA (one TMEM lane per run):
//   mars_relax_sweep        solvers.cpp:150-161  (in-place ascending-index Gauss-Seidel)
//   IsingProblem::row_dot   model.cpp:141-146    (dense row dot product)
//   tanh_trial              solvers.cpp:145-148
//   relax_to_fixed_point    solvers.cpp:163-176  and the mars_descent level loop 178-200
//   run_batch_with's queue  runner.cpp:95-115    (slots refill from an atomic run queue)
//
// Algorithm (left-looking blocked Gauss-Seidel).  For spin block b (TB spins) the fields of
// all 128 runs are one GEMM over the whole current state,
//     Phi[r][i] = sum_j S[r][j] * J[j][b*TB + i]      (runs on TMEM lanes, spins on columns)
// where S holds this sweep's new values for j < b*TB and the previous sweep's for j >= b*TB.
// The epilogue (one thread per run) then walks the block in ascending order adding the
// in-block corrections J[k][i]*(s_i_new - s_i_old) for k > i -- exactly the reference's
// update order; only the summation order/precision differs.
//
// Precision ("fp32-accurate split"): the state is kept as an fp16 pair s = hi + lo (22-23
// significant bits) and J as J_hi + J_lo, and the field is J_hi*S_hi + J_hi*S_lo + J_lo*S_hi
// accumulated in fp32 (J_lo*S_lo < 2^-22 relative is dropped).  Integer couplings
// (|J| <= 2048) are exact in J_hi, so the J_lo product is skipped (JLO = false).
//
// Pipelining.  GEMM(b) consumes its K chunks starting at block b and ending with block
// b-1, so it runs concurrently with the epilogue of block b-1 and only its last TB/KC
// chunks wait for that epilogue's state write-back; two TMEM accumulators ping-pong.
// A finished slot is refilled without stalling the pipeline: for one "loading" sweep the
// epilogue streams the old run's final spins out and the new run's initial state in, block
// by block, in Gauss-Seidel order, so every GEMM always reads a consistent state.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2..9 = epilogue, two per TMEM lane quarter (warp w accesses lanes 32*(w%4) .. +31).
//
// Global layout: state planes S_hi/S_lo [grid*TM][np] fp16 (row per slot, K-major for
// UMMA), couplings J_hi/J_lo [np][np] fp16 (J symmetric, so row i of J is column i: the
// K-major B operand of block b is the row block J[b*TB .. b*TB+TB)[*]), J32 [np][np] fp32
// for the epilogue's diagonal block.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "kernels.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

using namespace umma;

constexpr int TM = 128;      // runs per CTA = TMEM lanes = UMMA M
constexpr int TB = 128;      // spins per Gauss-Seidel block = UMMA N
constexpr int KC = 64;       // K per pipeline stage (one 128-byte swizzle atom of fp16)
constexpr int CPB = TB / KC; // chunks per block
constexpr int STAGES = 2;
constexpr int NT = 320;             // 2 control warps + 8 epilogue warps
constexpr int EPI0 = 2;      // first epilogue warp
constexpr int NEPI = 256;    // epilogue threads
constexpr std::uint32_t TILE_A = TM * KC * 2;   // 16 KB
constexpr std::uint32_t TILE_J = TB * KC * 2;   // 16 KB
constexpr std::uint32_t STAGE_BYTES = 2 * TILE_A + 2 * TILE_J;

enum : int { kIdle = 0, kActive = 1, kLoading = 2, kDrain = 3 };

struct __align__(8) Ctl {
    std::uint64_t full[STAGES];
    std::uint64_t empty[STAGES];
    std::uint64_t tmem_full[2];
    std::uint64_t tmem_empty[2];
    std::uint64_t chunk_ready;
    std::uint64_t mma_done;
    std::uint32_t tmem_base;
    volatile std::uint32_t stop;
    volatile std::uint32_t poison_it;
};

// dynamic smem: [stages: A_hi A_lo J_hi J_lo] [Jtri: upper triangle of the diagonal block,
// fp32, row i stored from column (i+1) rounded down to a multiple of 4 so every row is
// float4-aligned] [Sdel: the block's Delta history, fp32 [TB][TM], one column per slot] [Ctl]
__host__ __device__ constexpr int tri_k0(int i) { return (i + 1) & ~3; }
__host__ __device__ constexpr int tri_row_off(int i) {
    int off = 0;
    for (int r = 0; r < i; ++r) off += TB - tri_k0(r);
    return off;
}
constexpr std::uint32_t SMEM_STAGES = STAGES * STAGE_BYTES;
constexpr std::uint32_t TRI = tri_row_off(TB);
constexpr std::uint32_t SMEM_TRI = ((TRI * 4 + 127) / 128) * 128;
constexpr std::uint32_t SMEM_SBLK = TB * TM * 4;
constexpr std::uint32_t SMEM_TOTAL = SMEM_STAGES + SMEM_TRI + SMEM_SBLK + sizeof(Ctl);
static_assert(SMEM_TOTAL <= 232448, "shared memory budget");

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

__device__ __forceinline__ bool epi_any(bool v) {
    std::uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "barrier.cta.red.or.pred q, 1, 256, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}\n"
        : "=r"(r)
        : "r"(static_cast<std::uint32_t>(v))
        : "memory");
    return r != 0;
}

struct UmmaParams {
    const __half* s_hi;      // state planes (generic pointers for the epilogue)
    __half* s_hi_w;
    __half* s_lo_w;
    int nb;                  // blocks per sweep = np / TB
    int l2hint;              // coupling tiles loaded with an L2 evict_last hint (shared by all CTAs)
};

__device__ __forceinline__ void split16(float v, __half& hi, __half& lo, float& back) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
    back = __half2float(hi) + __half2float(lo);
}

// runtime tri_row_off: i*TB - sum_{r<i} tri_k0(r), with sum_{m=1..i} floor(m/4) in closed form
__device__ __forceinline__ int tri_row_off_rt(int i) {
    const int q = i >> 2, rem = i & 3;
    return i * TB - 4 * (2 * q * (q - 1) + q * (rem + 1));
}

// ---- the in-block Gauss-Seidel walk.  Two levels: SB-spin sub-blocks walked with a fully
// unrolled body (fold expressions), inside a runtime loop over the block; before sub-block
// s walks, every earlier spin's Delta (kept in this thread's smem column) is applied to its
// fields.  Fields are fp32 pairs so the updates issue as FFMA2; J rows come from smem as
// 16-byte loads issued before the spin's trial so their latency hides under the tanh.  The
// compact loop keeps the hot code inside the instruction cache (a fully unrolled 128-spin
// triangle is ~220 KB of SASS, streamed from L2 by every SM).
constexpr int SB = 16;

struct SubCtx {
    const float* jtri;
    float* sdel;          // this slot's Delta column: sdel[i * TM]
    const float* h;       // field slice or nullptr
    float T;              // level temperature (fp32)
    float rT;             // recip_for_div(T), or 0 at the quench
    bool quench;
    int lim;
    float dmax;
};

__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
    return __ffma2_rn(a, make_float2(b, b), c);
}

template <int I, int G>
__device__ __forceinline__ void sub_update_group(float2 (&p)[SB / 2], const float4 j, float d) {
    // columns 4G .. 4G+3 of spin row I; only columns > I are updated
    constexpr int m = 4 * G;
    if constexpr (m > I) {
        p[m / 2] = ffma2(make_float2(j.x, j.y), d, p[m / 2]);
    } else if constexpr (m + 1 > I) {
        p[m / 2].y = fmaf(j.y, d, p[m / 2].y);
    }
    if constexpr (m + 2 > I) {
        p[m / 2 + 1] = ffma2(make_float2(j.z, j.w), d, p[m / 2 + 1]);
    } else if constexpr (m + 3 > I) {
        p[m / 2 + 1].y = fmaf(j.w, d, p[m / 2 + 1].y);
    }
}

template <int I, int... G>
__device__ __forceinline__ void sub_update(float2 (&p)[SB / 2], const float4 (&jr)[SB / 4], float d,
                                           std::integer_sequence<int, G...>) {
    (sub_update_group<I, ((I + 1) & ~3) / 4 + G>(p, jr[((I + 1) & ~3) / 4 + G], d), ...);
}

template <int I, bool FULL, bool HAS_H>
__device__ __forceinline__ void sub_step(float2 (&p)[SB / 2], const float (&old)[SB], float (&nv)[SB], int k0,
                                         SubCtx& c) {
    if (FULL || k0 + I < c.lim) {
        // J[k0+I][k0 + 4g ..] for the groups this spin updates, issued before the trial
        float4 jr[SB / 4];
        if constexpr (I + 1 < SB) {
            const int i = k0 + I;
            const float* row = c.jtri + tri_row_off_rt(i) - tri_k0(i) + k0;   // row[m] = J[i][k0+m]
#pragma unroll
            for (int g = ((I + 1) & ~3) / 4; g < SB / 4; ++g) jr[g] = *reinterpret_cast<const float4*>(row + 4 * g);
        }
        const float x = (I & 1 ? p[I / 2].y : p[I / 2].x) + (HAS_H ? __ldg(c.h + k0 + I) : 0.0f);
        // tanh_trial (solvers.cpp:145-148): -tanh(phi/t), or -sign(phi) at the quench
        const float sgn = x > 0.0f ? -1.0f : (x < 0.0f ? 1.0f : 0.0f);
        // phi / t rounded as div.rn does (quotient from the hoisted refined reciprocal plus
        // div.rn's two correction FMAs: bit-identical to __fdiv_rn for these operands)
        const float q0 = fmaf(c.rT, x, 0.0f);
        const float th = -tanhf(fmaf(fmaf(-c.T, q0, x), c.rT, q0));
        const float trial = c.quench ? sgn : th;
        const float delta = trial - old[I];
        c.sdel[(k0 + I) * TM] = delta;
        nv[I] = trial;
        c.dmax = fmaxf(c.dmax, fabsf(delta));
        if constexpr (I + 1 < SB)
            sub_update<I>(p, jr, delta, std::make_integer_sequence<int, SB / 4 - ((I + 1) & ~3) / 4>{});
    } else {
        nv[I] = old[I];
    }
}

template <bool FULL, bool HAS_H, int... I>
__device__ __forceinline__ void sub_walk(float2 (&p)[SB / 2], const float (&old)[SB], float (&nv)[SB], int k0,
                                         SubCtx& c, std::integer_sequence<int, I...>) {
    (sub_step<I, FULL, HAS_H>(p, old, nv, k0, c), ...);
}

template <bool HAS_H>
__device__ __forceinline__ void walk_dispatch(float2 (&p)[SB / 2], const float (&old)[SB], float (&nv)[SB],
                                              int k0, SubCtx& c) {
    if (k0 + SB <= c.lim)
        sub_walk<true, HAS_H>(p, old, nv, k0, c, std::make_integer_sequence<int, SB>{});
    else
        sub_walk<false, HAS_H>(p, old, nv, k0, c, std::make_integer_sequence<int, SB>{});
}

__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, float (&v)[16]) {
    std::uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void load_old16(const __half* hi, const __half* lo, float (&old)[SB]) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const uint4 hv = *reinterpret_cast<const uint4*>(hi + v * 8);
        const uint4 lv = *reinterpret_cast<const uint4*>(lo + v * 8);
        const __half* h8 = reinterpret_cast<const __half*>(&hv);
        const __half* l8 = reinterpret_cast<const __half*>(&lv);
#pragma unroll
        for (int e = 0; e < 8; ++e) old[v * 8 + e] = __half2float(h8[e]) + __half2float(l8[e]);
    }
}

__device__ __forceinline__ void store_new16(__half* hi, __half* lo, const float (&nv)[SB]) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        uint4 hv, lv;
        __half* h8 = reinterpret_cast<__half*>(&hv);
        __half* l8 = reinterpret_cast<__half*>(&lv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float back;
            split16(nv[v * 8 + e], h8[e], l8[e], back);
        }
        *reinterpret_cast<uint4*>(hi + v * 8) = hv;
        *reinterpret_cast<uint4*>(lo + v * 8) = lv;
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <bool JLO>
__global__ void __launch_bounds__(NT, 1)
relax_dense_umma_kernel(RelaxArgs a, UmmaParams up, const __grid_constant__ CUtensorMap tm_shi,
                        const __grid_constant__ CUtensorMap tm_slo,
                        const __grid_constant__ CUtensorMap tm_jhi,
                        const __grid_constant__ CUtensorMap tm_jlo) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw;   // SWIZZLE_128B tiles need 1024-byte alignment (checked)
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0) __trap();
    float* Jtri = reinterpret_cast<float*>(base + SMEM_STAGES);
    float* Sdel = reinterpret_cast<float*>(base + SMEM_STAGES + SMEM_TRI);
    Ctl& ctl = *reinterpret_cast<Ctl*>(base + SMEM_STAGES + SMEM_TRI + SMEM_SBLK);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int np = a.np, n = a.n, nb = up.nb, nk = np / KC;
    const int row0 = blockIdx.x * TM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&ctl.full[s], 1);
            mbar_init(&ctl.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.tmem_full[s], 1);
            mbar_init(&ctl.tmem_empty[s], NEPI);
        }
        mbar_init(&ctl.chunk_ready, NEPI);
        mbar_init(&ctl.mma_done, 1);
        ctl.stop = 0;
        ctl.poison_it = 0xFFFFFFFFu;
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&ctl.tmem_base, 2 * TB);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = ctl.tmem_base;

    if (warp == 0) {
        // ================================================================ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_shi);
            tma_prefetch_desc(&tm_slo);
            tma_prefetch_desc(&tm_jhi);
            if (JLO) tma_prefetch_desc(&tm_jlo);
            const std::uint64_t jpol = policy_evict_last();
            std::uint32_t g = 0, it = 0;
            long long w_ready = 0, w_empty = 0;
            for (;;) {
                for (int b = 0; b < nb; ++b, ++g) {
                    for (int j = 0; j < nk; ++j, ++it) {
                        if (j == nk - CPB && g > 0) {
                            // the last chunks of GEMM(b) are block b-1: wait for its update
                            const long long t0 = clock64();
                            mbar_wait(&ctl.chunk_ready, (g - 1) & 1);
                            w_ready += clock64() - t0;
                            if (ctl.stop) {
                                const int s = it % STAGES;
                                mbar_wait(&ctl.empty[s], ((it / STAGES) & 1) ^ 1);
                                ctl.poison_it = it;
                                mbar_arrive(&ctl.full[s]);
                                if (a.prof) {
                                    a.prof[blockIdx.x * kProfSlots + 8] = w_ready;
                                    a.prof[blockIdx.x * kProfSlots + 9] = w_empty;
                                }
                                goto producer_done;
                            }
                        }
                        const int s = it % STAGES;
                        const int c = (b * CPB + j) % nk;
                        const long long t1 = clock64();
                        mbar_wait(&ctl.empty[s], ((it / STAGES) & 1) ^ 1);
                        w_empty += clock64() - t1;
                        unsigned char* st = base + s * STAGE_BYTES;
                        mbar_arrive_expect_tx(&ctl.full[s], JLO ? STAGE_BYTES : STAGE_BYTES - TILE_J);
                        tma_load_2d(st, &tm_shi, &ctl.full[s], c * KC, row0);
                        tma_load_2d(st + TILE_A, &tm_slo, &ctl.full[s], c * KC, row0);
                        // the coupling tiles are read by every CTA every sweep: keep them in L2
                        // ahead of the per-CTA state planes (155 MB at 148 CTAs > L2)
                        if (up.l2hint) {
                            tma_load_2d_hint(st + 2 * TILE_A, &tm_jhi, &ctl.full[s], c * KC, b * TB, jpol);
                            if (JLO) tma_load_2d_hint(st + 2 * TILE_A + TILE_J, &tm_jlo, &ctl.full[s], c * KC, b * TB, jpol);
                        } else {
                            tma_load_2d(st + 2 * TILE_A, &tm_jhi, &ctl.full[s], c * KC, b * TB);
                            if (JLO) tma_load_2d(st + 2 * TILE_A + TILE_J, &tm_jlo, &ctl.full[s], c * KC, b * TB);
                        }
                    }
                }
            }
        producer_done:;
        }
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            constexpr std::uint32_t idesc = idesc_f16(TM, TB, 0);
            std::uint32_t g = 0, it = 0;
            long long w_full = 0, w_tmem = 0;
            for (;;) {
                for (int b = 0; b < nb; ++b, ++g) {
                    const int buf = g & 1;
                    const long long t0 = clock64();
                    mbar_wait(&ctl.tmem_empty[buf], ((g >> 1) & 1) ^ 1);
                    w_tmem += clock64() - t0;
                    tc_fence_after();
                    const std::uint32_t d = tmem + buf * TB;
                    for (int j = 0; j < nk; ++j, ++it) {
                        const int s = it % STAGES;
                        const long long t1 = clock64();
                        mbar_wait(&ctl.full[s], (it / STAGES) & 1);
                        w_full += clock64() - t1;
                        if (ctl.poison_it == it) {
                            if (a.prof) {
                                a.prof[blockIdx.x * kProfSlots + 10] = w_full;
                                a.prof[blockIdx.x * kProfSlots + 11] = w_tmem;
                            }
                            goto mma_done;
                        }
                        tc_fence_after();
                        const std::uint32_t st = smem_u32(base + s * STAGE_BYTES);
#pragma unroll
                        for (int kk = 0; kk < KC / 16; ++kk) {
                            const std::uint64_t ahi = desc_k_sw128(st + kk * 32);
                            const std::uint64_t alo = desc_k_sw128(st + TILE_A + kk * 32);
                            const std::uint64_t jhi = desc_k_sw128(st + 2 * TILE_A + kk * 32);
                            mma_f16_ss(d, ahi, jhi, idesc, (j | kk) != 0);
                            mma_f16_ss(d, alo, jhi, idesc, 1);
                            if (JLO) {
                                const std::uint64_t jlo = desc_k_sw128(st + 2 * TILE_A + TILE_J + kk * 32);
                                mma_f16_ss(d, ahi, jlo, idesc, 1);
                            }
                        }
                        mma_commit(&ctl.empty[s]);
                    }
                    mma_commit(&ctl.tmem_full[buf]);
                }
            }
        mma_done:
            mma_commit(&ctl.mma_done);
            mbar_wait(&ctl.mma_done, 0);
        }
        __syncwarp();
    } else {
        // ================================================================ epilogue
        // Eight warps, two per TMEM lane quarter: warp pair (w, w+4) owns slots
        // r = 32*(w%4) + lane and alternates the SB-spin sub-blocks of every block, so one warp
        // pre-applies the Delta history to its next sub-block while its partner walks the
        // current one; a pair-private named barrier hands each finished sub-block's Delta over.
        // Side 0 owns the slot state machine and publishes it to side 1 at sweep ends.
        const int q = warp & 3;                            // TMEM lane quarter
        const int side = warp >= EPI0 + 4 ? 1 : 0;
        const int r = q * 32 + lane;                       // slot = TMEM lane
        const int et = threadIdx.x - EPI0 * 32;            // 0..255 for cooperative loads
        // hand-off of sub-block h uses named barrier 2 + 2q + (h & 1): two IDs per pair, so a
        // producer running ahead can never complete the phase its partner has not reached
        const int pair_bar = 2 + 2 * q;
        __half* hi_row = up.s_hi_w + static_cast<size_t>(row0 + r) * np;
        __half* lo_row = up.s_lo_w + static_cast<size_t>(row0 + r) * np;
        // sweep-boundary exchange area (the Delta history is dead between blocks)
        int* x_mode = reinterpret_cast<int*>(Sdel);
        int* x_new = x_mode + TM;
        int* x_old = x_mode + 2 * TM;
        float* x_rT = reinterpret_cast<float*>(x_mode + 3 * TM);
        float* x_T = reinterpret_cast<float*>(x_mode + 6 * TM);
        int* x_quench = x_mode + 4 * TM;
        float* x_dmax = reinterpret_cast<float*>(x_mode + 5 * TM);

        Slot slot;
        slot.run = -1;
        int mode = kIdle, old_run = -1, new_run = -1;
        float rT = 1.0f, Tf = 1.0f;
        bool quench = false;
        if (side == 0) {
            new_run = claim_run(a);
            mode = new_run >= 0 ? kLoading : kIdle;
            x_mode[r] = mode;
            x_new[r] = new_run;
        }
        epi_sync();
        if (side == 1) {
            mode = x_mode[r];
            new_run = x_new[r];
        }
        std::uint32_t g = 0;
        long long c_loads = 0, c_wait = 0, c_corr = 0, c_wb = 0, n_sweeps = 0;
        long long c_walk = 0, c_pass0 = 0, c_hand = 0, c_pass1 = 0, n_walks = 0;
        const long long c_start = clock64();

        for (;;) {
            ++n_sweeps;
            const bool active = mode == kActive;
            float dmax = 0.0f;
            for (int b = 0; b < nb; ++b, ++g) {
                const int b0 = b * TB;
                const int lim = min(TB, n - b0);
                const int nsub = (lim + SB - 1) / SB;
                long long t0 = clock64();
                // diagonal block's upper triangle -> smem, overlapping the wait for GEMM(b)
                epi_sync();
                for (int f = et; f < TB * TB / 4; f += 2 * TM) {
                    const int i = f / (TB / 4), k = (f % (TB / 4)) * 4;
                    if (k >= tri_k0(i))
                        cp_async16(Jtri + tri_row_off_rt(i) + k - tri_k0(i),
                                   a.J32 + static_cast<size_t>(b0 + i) * np + b0 + k);
                }
                const int buf = g & 1;
                long long t1 = clock64();
                mbar_wait(&ctl.tmem_full[buf], (g >> 1) & 1);
                long long t2 = clock64();
                c_wait += t2 - t1;
                cp_async_wait_all();
                epi_sync();
                const long long t2b = clock64();
                c_loads += (t1 - t0) + (t2b - t2);
                t2 = t2b;
                tc_fence_after();
                const std::uint32_t tacc = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + buf * TB;

                if (__any_sync(0xffffffffu, active)) {
                    // ---- in-block Gauss-Seidel correction, ascending spin order (warp-uniform:
                    // tcgen05.ld is .sync.aligned; lanes of inactive slots compute, never store)
                    SubCtx ctx{Jtri, Sdel + r, a.h32 ? a.h32 + b0 : nullptr, Tf, rT, quench, lim, 0.0f};
                    const float* dcol = Sdel + r;
                    for (int s = side; s < nsub; s += 2) {
                        const int k0 = s * SB;
                        float old[SB];
                        load_old16(hi_row + b0 + k0, lo_row + b0 + k0, old);
                        float pv[SB];
                        tmem_ld16(tacc + k0, pv);
                        float2 pf[SB / 2];
#pragma unroll
                        for (int j = 0; j < SB / 2; ++j) pf[j] = make_float2(pv[2 * j], pv[2 * j + 1]);
                        // corrections J[j][k0..k0+SB) * Delta_j: first every Delta already final
                        // (sub-blocks < s-1), then -- after the partner hands it over -- s-1's
                        const int jpre = s > 0 ? k0 - SB : 0;
                        long long tp = clock64();
                        for (int pass = 0; pass < 2; ++pass) {
                            const int jb = pass == 0 ? 0 : jpre, je = pass == 0 ? jpre : k0;
                            if (pass == 1) {
                                if (s == 0) break;
                                const long long ta = clock64();
                                c_pass0 += ta - tp;
                                asm volatile("bar.sync %0, 64;\n" ::"r"(pair_bar + ((s - 1) & 1)) : "memory");
                                tp = clock64();
                                c_hand += tp - ta;
                            }
#pragma unroll 2
                            for (int j = jb; j < je; ++j) {
                                const float d = dcol[j * TM];
                                const float4* jr = reinterpret_cast<const float4*>(
                                    Jtri + tri_row_off_rt(j) + k0 - tri_k0(j));
#pragma unroll
                                for (int m = 0; m < SB / 4; ++m) {
                                    const float4 jv = jr[m];
                                    pf[2 * m] = ffma2(make_float2(jv.x, jv.y), d, pf[2 * m]);
                                    pf[2 * m + 1] = ffma2(make_float2(jv.z, jv.w), d, pf[2 * m + 1]);
                                }
                            }
                        }
                        float nv[SB];
                        const long long tw = clock64();
                        if (s > 0) c_pass1 += tw - tp; else c_pass0 += tw - tp;
                        if (ctx.h) walk_dispatch<true>(pf, old, nv, k0, ctx);
                        else walk_dispatch<false>(pf, old, nv, k0, ctx);
                        c_walk += clock64() - tw;
                        ++n_walks;
                        if (active) store_new16(hi_row + b0 + k0, lo_row + b0 + k0, nv);
                        if (s + 1 < nsub) asm volatile("bar.arrive %0, 64;\n" ::"r"(pair_bar + (s & 1)) : "memory");
                    }
                    dmax = fmaxf(dmax, ctx.dmax);
                }
                tc_fence_before();
                mbar_arrive(&ctl.tmem_empty[buf]);
                const long long t3 = clock64();
                c_corr += t3 - t2;
                t2 = t3;
                if (!active && (mode == kLoading || mode == kDrain)) {
                    // ---- slot turnover, block by block (each side one half of the columns):
                    // the old run's rounded spins out, the new run's initial state in
                    const int c0 = side * (TB / 2), c1 = c0 + TB / 2;
                    if (old_run >= 0) {
                        std::int8_t* out = a.spins + static_cast<size_t>(old_run) * n + b0;
                        for (int i = c0; i < c1 && i < lim; ++i) {        // round_spins (model.cpp:245)
                            const float s = __half2float(hi_row[b0 + i]) + __half2float(lo_row[b0 + i]);
                            out[i] = s < 0.0f ? -1 : 1;
                            if (a.state_out) a.state_out[static_cast<size_t>(old_run) * n + b0 + i] = s;
                        }
                    }
                    if (mode == kLoading) {
                        const float* src = a.s0 + static_cast<size_t>(new_run) * n + b0;
                        for (int v = c0 / 8; v < c1 / 8; ++v) {
                            uint4 hv, lv;
                            __half* h8 = reinterpret_cast<__half*>(&hv);
                            __half* l8 = reinterpret_cast<__half*>(&lv);
                            for (int e = 0; e < 8; ++e) {
                                const int i = v * 8 + e;
                                float back;
                                split16(i < lim ? src[i] : 0.0f, h8[e], l8[e], back);
                            }
                            *reinterpret_cast<uint4*>(hi_row + b0 + v * 8) = hv;
                            *reinterpret_cast<uint4*>(lo_row + b0 + v * 8) = lv;
                        }
                    }
                }
                c_wb += clock64() - t2;
                if (b == nb - 1) {
                    // ---- end of sweep: annealing state machine (solvers.cpp:178-200), side 0
                    epi_sync();                                   // walks done: Sdel is scratch
                    if (side == 1) x_dmax[r] = dmax;
                    epi_sync();
                    if (side == 0) {
                        dmax = fmaxf(dmax, x_dmax[r]);
                        if (active) {
                            const int code = slot_after_sweep(slot, dmax, a);
                            if (code != kSlotContinue) {
                                slot_finish(slot, code, a);
                                old_run = slot.run;
                                new_run = claim_run(a);
                                mode = new_run >= 0 ? kLoading : kDrain;
                            }
                        } else if (mode == kLoading) {
                            slot_start(slot, new_run, a);
                            mode = kActive;
                            old_run = -1;
                        } else if (mode == kDrain) {
                            mode = kIdle;
                            old_run = -1;
                        }
                        quench = mode == kActive && slot_quench(slot);
                        Tf = static_cast<float>(slot.T);
                        rT = quench ? 0.0f : recip_for_div(Tf);
                        x_mode[r] = mode;
                        x_new[r] = new_run;
                        x_old[r] = old_run;
                        x_rT[r] = rT;
                        x_T[r] = Tf;
                        x_quench[r] = quench;
                    }
                    const bool more = epi_any(side == 0 && mode != kIdle);
                    if (side == 1) {
                        mode = x_mode[r];
                        new_run = x_new[r];
                        old_run = x_old[r];
                        rT = x_rT[r];
                        Tf = x_T[r];
                        quench = x_quench[r] != 0;
                    }
                    if (!more && et == 0) ctl.stop = 1;
                    fence_proxy_async_global();
                    mbar_arrive(&ctl.chunk_ready);
                    if (!more) goto epilogue_done;
                } else {
                    fence_proxy_async_global();
                    mbar_arrive(&ctl.chunk_ready);
                }
            }
        }
    epilogue_done:
        if (a.prof && et == 0) {
            long long* pr = a.prof + blockIdx.x * kProfSlots;
            pr[0] = n_sweeps;
            pr[1] = clock64() - c_start;
            pr[2] = c_loads;
            pr[3] = c_wait;
            pr[4] = c_corr;
            pr[5] = c_wb;
            pr[6] = nb;
            pr[12] = c_walk;
            pr[13] = n_walks;
            pr[14] = c_pass0 + (c_pass1 << 0) * 0;
            pr[15] = c_hand;
            pr[7] = c_pass1;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 2 * TB);
}

}  // namespace

int relax_dense_umma_slots_per_cta() { return TM; }
int relax_dense_umma_block() { return TB; }
std::size_t relax_dense_umma_plane_rows(int grid) { return static_cast<std::size_t>(grid) * TM; }

cudaError_t launch_relax_dense_umma(const RelaxArgs& a, const UmmaLaunch& u, int grid, cudaStream_t st) {
    const char* hint = std::getenv("MARS_UMMA_L2HINT");
    UmmaParams up{u.s_hi, u.s_hi, u.s_lo, a.np / TB, hint ? std::atoi(hint) : 1};
    if (a.np % TB != 0) return cudaErrorInvalidValue;
    cudaError_t e;
    if (u.jlo) {
        e = cudaFuncSetAttribute(relax_dense_umma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
        if (e != cudaSuccess) return e;
        relax_dense_umma_kernel<true><<<grid, NT, SMEM_TOTAL, st>>>(a, up, u.tm_shi, u.tm_slo, u.tm_jhi, u.tm_jlo);
    } else {
        e = cudaFuncSetAttribute(relax_dense_umma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
        if (e != cudaSuccess) return e;
        relax_dense_umma_kernel<false><<<grid, NT, SMEM_TOTAL, st>>>(a, up, u.tm_shi, u.tm_slo, u.tm_jhi, u.tm_jlo);
    }
    return cudaGetLastError();
}

}  // namespace marsb200
