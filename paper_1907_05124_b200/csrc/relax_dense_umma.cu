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
// Pipelining.  GEMM(b) consumes its K chunks starting at block b and ending with block b-1.
// All but that last block come through a 3-stage TMA ring from the fp16 state planes in
// HBM; the last block's K range -- the state the epilogue of block b-1 is producing right
// now -- is read by the tensor core straight from TMEM (tcgen05.mma with A in TMEM), one
// 16-spin K step as soon as the epilogue has walked that sub-block.  The GEMM of the next
// block therefore finishes one K step after the epilogue of the current block.  Two TMEM
// accumulators ping-pong; a finished slot is refilled without stalling the pipeline: for
// one "loading" sweep the old run's spins stream out and the new run's initial state in,
// block by block, in Gauss-Seidel order, so every GEMM reads a consistent state.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2..9 = epilogue, two per TMEM lane quarter (warp w accesses lanes 32*(w%4) .. +31).
//
// TMEM (512 columns): [0,128) [128,256) accumulators; [256,384) tail A operand (16-spin
// K steps: hi at 256 + 8s, lo at 320 + 8s, two fp16 per column); [384,512) Delta history
// of the block being walked (fp32, column 384 + spin).
//
// Global layout: state planes S_hi/S_lo [grid*TM][np] fp16 (row per slot, K-major for
// UMMA), couplings J_hi/J_lo [np][np] fp16 (J symmetric, so row i of J is column i: the
// K-major B operand of block b is the row block J[b*TB .. b*TB+TB)[*]), J32 [np][np] fp32
// for the epilogue's diagonal block.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

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
constexpr int SB = 16;       // spins per sub-block = one UMMA K step
constexpr int NSB = TB / SB; // sub-blocks per block
constexpr int STAGES = 3;
constexpr int NT = 320;      // 2 control warps + 8 epilogue warps
constexpr int EPI0 = 2;      // first epilogue warp
constexpr int NEPI = 256;    // epilogue threads
constexpr std::uint32_t TILE_A = TM * KC * 2;   // 16 KB
constexpr std::uint32_t TILE_J = TB * KC * 2;   // 16 KB
constexpr std::uint32_t STAGE_BYTES = 2 * TILE_A + 2 * TILE_J;
constexpr std::uint32_t TM_ACC = 0, TM_AHI = 256, TM_ALO = 320, TM_DEL = 384, TM_COLS = 512;

enum : int { kIdle = 0, kActive = 1, kLoading = 2, kDrain = 3 };

struct __align__(8) Ctl {
    std::uint64_t full[STAGES];
    std::uint64_t empty[STAGES];
    std::uint64_t tmem_full[2];
    std::uint64_t tmem_empty[2];
    std::uint64_t chunk_ready[2];   // block g's planes written: barrier g & 1
    std::uint64_t asub[NSB];        // tail A sub-block s of the current block written to TMEM
    std::uint64_t mma_done;
    std::uint32_t tmem_base;
    volatile std::uint32_t stop;
    // sweep-boundary exchange between the two epilogue sides: side 1 posts its dmax in xa,
    // then side 0 publishes the slot state (xa = new run, xb = old run, xc = mode | quench<<2,
    // xd = 1/T as float bits)
    int xa[TM], xb[TM], xc[TM], xd[TM];
};

// dynamic smem: [stages: A_hi A_lo J_hi J_lo] [Jtri: upper triangle of the diagonal block,
// fp32, row i stored from column (i+1) rounded down to a multiple of 4 so every row is
// float4-aligned] [Ctl]
__host__ __device__ constexpr int tri_k0(int i) { return (i + 1) & ~3; }
__host__ __device__ constexpr int tri_row_off(int i) {
    int off = 0;
    for (int r = 0; r < i; ++r) off += TB - tri_k0(r);
    return off;
}
constexpr std::uint32_t SMEM_STAGES = STAGES * STAGE_BYTES;
constexpr std::uint32_t TRI = tri_row_off(TB);
constexpr std::uint32_t SMEM_TRI = ((TRI * 4 + 127) / 128) * 128;
constexpr std::uint32_t SMEM_TOTAL = SMEM_STAGES + SMEM_TRI + sizeof(Ctl);
static_assert(SMEM_TOTAL <= 232448, "shared memory budget");

// runtime tri_row_off: i*TB - sum_{r<i} tri_k0(r), with sum_{m=1..i} floor(m/4) in closed form
__device__ __forceinline__ int tri_row_off_rt(int i) {
    const int q = i >> 2, rem = i & 3;
    return i * TB - 4 * (2 * q * (q - 1) + q * (rem + 1));
}

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

// Wait for a barrier phase unless the CTA is shutting down; false = stop observed.
__device__ __forceinline__ bool mbar_wait_or_stop(std::uint64_t* bar, std::uint32_t parity,
                                                  const volatile std::uint32_t* stop) {
    for (;;) {
        if (mbar_try_wait(bar, parity)) return true;
        if (*stop) return false;
    }
}

struct UmmaParams {
    __half* s_hi;            // state planes (generic pointers for the epilogue)
    __half* s_lo;
    int nb;                  // blocks per sweep = np / TB
};

__device__ __forceinline__ void split16(float v, __half& hi, __half& lo) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// rows [r0, r1) of the diagonal block's padded upper triangle -> smem (cp.async)
__device__ __forceinline__ void load_tri_rows(float* jtri, const float* J32, int np, int b0, int r0, int r1,
                                              int t, int nthreads) {
    for (int f = r0 * (TB / 4) + t; f < r1 * (TB / 4); f += nthreads) {
        const int i = f / (TB / 4), k = (f % (TB / 4)) * 4;
        if (k >= tri_k0(i))
            cp_async16(jtri + tri_row_off_rt(i) + k - tri_k0(i), J32 + static_cast<size_t>(b0 + i) * np + b0 + k);
    }
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

// ---- the in-block Gauss-Seidel walk.  Two levels: SB-spin sub-blocks walked with a fully
// unrolled body (fold expressions), inside a runtime loop over the block; before sub-block
// s walks, the Delta of every earlier spin of the block (TMEM) is applied to its fields.
// Fields are fp32 pairs so the updates issue as FFMA2; J rows come from smem as 16-byte
// loads issued before the spin's trial so their latency hides under the tanh.  The compact
// loop keeps the hot code in the instruction cache (a fully unrolled 128-spin triangle is
// ~220 KB of SASS, streamed from L2 by every SM).

struct SubCtx {
    const float* jtri;
    const float* h;       // field slice or nullptr
    float invT;           // 1/T, or 0 at the quench
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

template <int I, bool FULL, bool HAS_H, bool NEXT>
__device__ __forceinline__ void sub_step(float2 (&p)[SB / 2], float2 (&cn)[SB / 2], const float (&old)[SB],
                                         float (&nv)[SB], int k0, SubCtx& c) {
    if (FULL || k0 + I < c.lim) {
        const int i = k0 + I;
        const float* row = c.jtri + tri_row_off_rt(i) - tri_k0(i) + k0;   // row[m] = J[i][k0+m]
        // J[i][k0 + 4g ..] for the groups this spin updates, issued before the trial
        float4 jr[SB / 4];
        if constexpr (I + 1 < SB) {
#pragma unroll
            for (int g = ((I + 1) & ~3) / 4; g < SB / 4; ++g) jr[g] = *reinterpret_cast<const float4*>(row + 4 * g);
        }
        float4 jn[SB / 4];
        if constexpr (NEXT) {
#pragma unroll
            for (int g = 0; g < SB / 4; ++g) jn[g] = *reinterpret_cast<const float4*>(row + SB + 4 * g);
        }
        const float x = (I & 1 ? p[I / 2].y : p[I / 2].x) + (HAS_H ? __ldg(c.h + k0 + I) : 0.0f);
        // tanh_trial (solvers.cpp:145-148): -tanh(phi/t), or -sign(phi) at the quench
        const float sgn = x > 0.0f ? -1.0f : (x < 0.0f ? 1.0f : 0.0f);
        const float th = -tanhf(x * c.invT);
        const float trial = c.quench ? sgn : th;
        const float delta = trial - old[I];
        nv[I] = trial;
        c.dmax = fmaxf(c.dmax, fabsf(delta));
        if constexpr (I + 1 < SB)
            sub_update<I>(p, jr, delta, std::make_integer_sequence<int, SB / 4 - ((I + 1) & ~3) / 4>{});
        if constexpr (NEXT) {
            // this spin's contribution to the next sub-block's fields (right-looking, off the chain)
#pragma unroll
            for (int g = 0; g < SB / 4; ++g) {
                cn[2 * g] = ffma2(make_float2(jn[g].x, jn[g].y), delta, cn[2 * g]);
                cn[2 * g + 1] = ffma2(make_float2(jn[g].z, jn[g].w), delta, cn[2 * g + 1]);
            }
        }
    } else {
        nv[I] = old[I];
    }
}

template <bool FULL, bool HAS_H, bool NEXT, int... I>
__device__ __forceinline__ void sub_walk(float2 (&p)[SB / 2], float2 (&cn)[SB / 2], const float (&old)[SB],
                                         float (&nv)[SB], int k0, SubCtx& c, std::integer_sequence<int, I...>) {
    (sub_step<I, FULL, HAS_H, NEXT>(p, cn, old, nv, k0, c), ...);
}

template <bool HAS_H>
__device__ __forceinline__ void walk_dispatch(float2 (&p)[SB / 2], float2 (&cn)[SB / 2], const float (&old)[SB],
                                              float (&nv)[SB], int k0, bool next, SubCtx& c) {
    constexpr auto seq = std::make_integer_sequence<int, SB>{};
    if (k0 + SB <= c.lim) {
        if (next) sub_walk<true, HAS_H, true>(p, cn, old, nv, k0, c, seq);
        else sub_walk<true, HAS_H, false>(p, cn, old, nv, k0, c, seq);
    } else {
        sub_walk<false, HAS_H, false>(p, cn, old, nv, k0, c, seq);
    }
}

// fields of sub-block k0 += J[j][k0..k0+SB) * Delta_j for the 16 spins j of sub-block `sb`
__device__ __forceinline__ void apply_deltas(float2 (&pf)[SB / 2], const float* jtri, std::uint32_t tdel,
                                             int sb, int k0) {
    float dv[SB];
    tmem_ld16(tdel + sb * SB, dv);
#pragma unroll
    for (int jj = 0; jj < SB; ++jj) {
        const int j = sb * SB + jj;
        const float4* jr = reinterpret_cast<const float4*>(jtri + tri_row_off_rt(j) + k0 - tri_k0(j));
#pragma unroll
        for (int m = 0; m < SB / 4; ++m) {
            const float4 jv = jr[m];
            pf[2 * m] = ffma2(make_float2(jv.x, jv.y), dv[jj], pf[2 * m]);
            pf[2 * m + 1] = ffma2(make_float2(jv.z, jv.w), dv[jj], pf[2 * m + 1]);
        }
    }
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

// the sub-block's new state: fp16 pair planes in HBM (optional) and the tail A operand in TMEM
__device__ __forceinline__ void store_new16(__half* hi, __half* lo, bool to_planes, std::uint32_t tahi,
                                            std::uint32_t talo, const float (&nv)[SB]) {
    std::uint32_t ph[SB / 2], pl[SB / 2];
#pragma unroll
    for (int v = 0; v < SB / 2; ++v) {
        __half h0, l0, h1, l1;
        split16(nv[2 * v], h0, l0);
        split16(nv[2 * v + 1], h1, l1);
        const __half2 hh = __halves2half2(h0, h1), ll = __halves2half2(l0, l1);
        ph[v] = *reinterpret_cast<const std::uint32_t*>(&hh);
        pl[v] = *reinterpret_cast<const std::uint32_t*>(&ll);
    }
    tmem_st8(tahi, ph);
    tmem_st8(talo, pl);
    if (to_planes) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            *reinterpret_cast<uint4*>(hi + v * 8) = make_uint4(ph[4 * v], ph[4 * v + 1], ph[4 * v + 2], ph[4 * v + 3]);
            *reinterpret_cast<uint4*>(lo + v * 8) = make_uint4(pl[4 * v], pl[4 * v + 1], pl[4 * v + 2], pl[4 * v + 3]);
        }
    }
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
    Ctl& ctl = *reinterpret_cast<Ctl*>(base + SMEM_STAGES + SMEM_TRI);

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
            mbar_init(&ctl.chunk_ready[s], NEPI);
        }
        for (int s = 0; s < NSB; ++s) mbar_init(&ctl.asub[s], TM);
        mbar_init(&ctl.mma_done, 1);
        ctl.stop = 0;
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&ctl.tmem_base, TM_COLS);
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
            std::uint32_t g = 0, it = 0;
            for (;;) {
                for (int b = 0; b < nb; ++b, ++g) {
                    for (int j = 0; j < nk; ++j) {
                        const bool tail = j >= nk - CPB;   // block b-1: A comes from TMEM
                        if (tail && g == 0) continue;      // no previous epilogue: no tail
                        if (j == nk - 2 * CPB && g >= 2) {
                            // block b-2's planes are read from HBM: its epilogue must be done
                            if (!mbar_wait_or_stop(&ctl.chunk_ready[g & 1], ((g - 2) >> 1) & 1, &ctl.stop))
                                goto producer_done;
                        }
                        const int s = it % STAGES;
                        const int c = (b * CPB + j) % nk;
                        if (!mbar_wait_or_stop(&ctl.empty[s], ((it / STAGES) & 1) ^ 1, &ctl.stop))
                            goto producer_done;
                        unsigned char* stg = base + s * STAGE_BYTES;
                        const std::uint32_t jbytes = JLO ? 2 * TILE_J : TILE_J;
                        mbar_arrive_expect_tx(&ctl.full[s], tail ? jbytes : 2 * TILE_A + jbytes);
                        if (!tail) {
                            tma_load_2d(stg, &tm_shi, &ctl.full[s], c * KC, row0);
                            tma_load_2d(stg + TILE_A, &tm_slo, &ctl.full[s], c * KC, row0);
                        }
                        tma_load_2d(stg + 2 * TILE_A, &tm_jhi, &ctl.full[s], c * KC, b * TB);
                        if (JLO) tma_load_2d(stg + 2 * TILE_A + TILE_J, &tm_jlo, &ctl.full[s], c * KC, b * TB);
                        ++it;
                    }
                }
            }
        producer_done:
            // drain: every issued TMA load must land before the CTA can exit
            for (std::uint32_t k = (it > STAGES ? it - STAGES : 0); k < it; ++k)
                mbar_wait(&ctl.full[k % STAGES], (k / STAGES) & 1);
        }
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            constexpr std::uint32_t idesc = idesc_f16(TM, TB, 0);
            std::uint32_t g = 0, it = 0;
            for (;;) {
                for (int b = 0; b < nb; ++b, ++g) {
                    const int buf = g & 1;
                    if (!mbar_wait_or_stop(&ctl.tmem_empty[buf], ((g >> 1) & 1) ^ 1, &ctl.stop)) goto mma_done;
                    tc_fence_after();
                    const std::uint32_t d = tmem + TM_ACC + buf * TB;
                    std::uint32_t acc = 0;
                    for (int j = 0; j < nk; ++j) {
                        const bool tail = j >= nk - CPB;
                        if (tail && g == 0) continue;
                        const int s = it % STAGES;
                        if (!mbar_wait_or_stop(&ctl.full[s], (it / STAGES) & 1, &ctl.stop)) goto mma_done;
                        tc_fence_after();
                        const std::uint32_t stg = smem_u32(base + s * STAGE_BYTES);
#pragma unroll
                        for (int kk = 0; kk < KC / 16; ++kk) {
                            const std::uint64_t jhi = desc_k_sw128(stg + 2 * TILE_A + kk * 32);
                            const std::uint64_t jlo = desc_k_sw128(stg + 2 * TILE_A + TILE_J + kk * 32);
                            if (!tail) {
                                const std::uint64_t ahi = desc_k_sw128(stg + kk * 32);
                                const std::uint64_t alo = desc_k_sw128(stg + TILE_A + kk * 32);
                                mma_f16_ss(d, ahi, jhi, idesc, acc);
                                mma_f16_ss(d, alo, jhi, idesc, 1);
                                if (JLO) mma_f16_ss(d, ahi, jlo, idesc, 1);
                            } else {
                                // sub-block sb of block b-1, just walked by the epilogue
                                const int sb = (j - (nk - CPB)) * (KC / 16) + kk;
                                if (!mbar_wait_or_stop(&ctl.asub[sb], (g - 1) & 1, &ctl.stop)) goto mma_done;
                                tc_fence_after();
                                const std::uint32_t ahi = tmem + TM_AHI + sb * (SB / 2);
                                const std::uint32_t alo = tmem + TM_ALO + sb * (SB / 2);
                                mma_f16_ts(d, ahi, jhi, idesc, acc);
                                mma_f16_ts(d, alo, jhi, idesc, 1);
                                if (JLO) mma_f16_ts(d, ahi, jlo, idesc, 1);
                            }
                            acc = 1;
                        }
                        mma_commit(&ctl.empty[s]);
                        ++it;
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
        // current one; a pair-private named barrier hands each finished sub-block over.
        // Side 0 owns the slot state machine and publishes it to side 1 at sweep ends.
        const int q = warp & 3;                            // TMEM lane quarter
        const int side = warp >= EPI0 + 4 ? 1 : 0;
        const int r = q * 32 + lane;                       // slot = TMEM lane
        const int et = threadIdx.x - EPI0 * 32;            // 0..255 for cooperative loads
        const int tside = q * 32 + lane;                   // 0..127 within this side
        // hand-off of sub-block h uses named barrier 2 + 2q + (h & 1): two IDs per pair, so a
        // producer running ahead can never complete the phase its partner has not reached
        const int pair_bar = 2 + 2 * q;
        const std::uint32_t lane_base = tmem + (static_cast<std::uint32_t>(q * 32) << 16);
        const std::uint32_t tdel = lane_base + TM_DEL;
        __half* hi_row = up.s_hi + static_cast<size_t>(row0 + r) * np;
        __half* lo_row = up.s_lo + static_cast<size_t>(row0 + r) * np;

        Slot slot;
        slot.run = -1;
        int mode = kIdle, old_run = -1, new_run = -1;
        float invT = 0.0f;
        bool quench = false;
        if (side == 0) {
            new_run = claim_run(a);
            mode = new_run >= 0 ? kLoading : kIdle;
            ctl.xc[r] = mode;
            ctl.xa[r] = new_run;
        }
        epi_sync();
        if (side == 1) {
            mode = ctl.xc[r];
            new_run = ctl.xa[r];
        }
        std::uint32_t g = 0;
        bool tri_prefetched = false;       // rows [0, 96) of this block's triangle already in flight
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
                const long long t0 = clock64();
                // the diagonal block's upper triangle -> smem (rows the prefetch did not cover)
                epi_sync();
                load_tri_rows(Jtri, a.J32, np, b0, tri_prefetched ? 6 * SB : 0, TB, et, NEPI);
                const int buf = g & 1;
                const long long t1 = clock64();
                mbar_wait(&ctl.tmem_full[buf], (g >> 1) & 1);
                long long t2 = clock64();
                c_wait += t2 - t1;
                cp_async_wait_all();
                epi_sync();
                tri_prefetched = false;
                const long long t2b = clock64();
                c_loads += (t1 - t0) + (t2b - t2);
                t2 = t2b;
                tc_fence_after();
                const std::uint32_t tacc = lane_base + TM_ACC + buf * TB;
                const bool walkers = __any_sync(0xffffffffu, active);
                SubCtx ctx{Jtri, a.h32 ? a.h32 + b0 : nullptr, invT, quench, lim, 0.0f};

                for (int s = side; s < NSB; s += 2) {
                    const int k0 = s * SB;
                    const bool walk = walkers && s < nsub;
                    const bool next = walk && s + 1 < nsub;
                    float old[SB], nv[SB];
                    load_old16(hi_row + b0 + k0, lo_row + b0 + k0, old);
                    float2 pf[SB / 2];
#pragma unroll
                    for (int j = 0; j < SB / 2; ++j) pf[j] = make_float2(0.0f, 0.0f);
                    long long tp = clock64();
                    // ---- fields of sub-block s, part 1: the Delta of sub-blocks < s-1 (final
                    // while the partner is still walking s-1) -- warp-uniform; lanes of
                    // inactive slots compute but their results are discarded
                    if (walk)
                        for (int sb = 0; sb + 1 < s; ++sb) apply_deltas(pf, Jtri, tdel, sb, k0);
                    if (s == NSB - 1 && nsub == NSB) {
                        // every warp is past its reads of triangle rows [0, 96) (side 0 has
                        // finished sub-block 6, side 1 its pass over sub-blocks < 6): prefetch the
                        // next block's rows into them (side 1, all of its threads)
                        asm volatile("bar.sync 10, 256;\n" ::: "memory");
                        load_tri_rows(Jtri, a.J32, np, ((b + 1) % nb) * TB, 0, 6 * SB, tside, TM);
                    }
                    if (walk) {
                        const long long ta = clock64();
                        c_pass0 += ta - tp;
                        if (s > 0) {
                            // part 2: the partner folded sub-block s-1's Delta into our
                            // accumulator columns while it walked; wait for the hand-off
                            asm volatile("bar.sync %0, 64;\n" ::"r"(pair_bar + ((s - 1) & 1)) : "memory");
                            tc_fence_after();
                        }
                        const long long tw = clock64();
                        c_hand += tw - ta;
                        float pv[SB];
                        tmem_ld16(tacc + k0, pv);
#pragma unroll
                        for (int j = 0; j < SB / 2; ++j) {
                            pf[j].x += pv[2 * j];
                            pf[j].y += pv[2 * j + 1];
                        }
                        // ---- Gauss-Seidel walk of sub-block s; also accumulates this
                        // sub-block's contribution to the next one's fields (cn)
                        float2 cn[SB / 2];
#pragma unroll
                        for (int j = 0; j < SB / 2; ++j) cn[j] = make_float2(0.0f, 0.0f);
                        if (ctx.h) walk_dispatch<true>(pf, cn, old, nv, k0, next, ctx);
                        else walk_dispatch<false>(pf, cn, old, nv, k0, next, ctx);
                        c_walk += clock64() - tw;
                        ++n_walks;
                        // Delta history (TMEM, this slot's lane) and the next sub-block's fields
                        std::uint32_t du[SB];
#pragma unroll
                        for (int i = 0; i < SB; ++i) du[i] = __float_as_uint(active ? nv[i] - old[i] : 0.0f);
                        tmem_st16(tdel + k0, du);
                        if (next) {
                            float av[SB];
                            tmem_ld16(tacc + k0 + SB, av);
                            std::uint32_t au[SB];
#pragma unroll
                            for (int j = 0; j < SB / 2; ++j) {
                                au[2 * j] = __float_as_uint(av[2 * j] + cn[j].x);
                                au[2 * j + 1] = __float_as_uint(av[2 * j + 1] + cn[j].y);
                            }
                            tmem_st16(tacc + k0 + SB, au);
                        }
                        tmem_st_wait();
                        tc_fence_before();
                        if (next) asm volatile("bar.arrive %0, 64;\n" ::"r"(pair_bar + (s & 1)) : "memory");
                    }
                    // ---- this slot's new state of the sub-block
                    const bool turnover = !active && (mode == kLoading || mode == kDrain);
                    if (turnover && old_run >= 0) {           // round_spins (model.cpp:245)
                        std::int8_t* out = a.spins + static_cast<size_t>(old_run) * n + b0 + k0;
#pragma unroll
                        for (int i = 0; i < SB; ++i)
                            if (k0 + i < lim) out[i] = old[i] < 0.0f ? -1 : 1;
                    }
                    if (!(active && walk)) {
#pragma unroll
                        for (int i = 0; i < SB; ++i) nv[i] = old[i];
                    }
                    if (mode == kLoading && !active) {
                        const float* src = a.s0 + static_cast<size_t>(new_run) * n + b0 + k0;
#pragma unroll
                        for (int i = 0; i < SB; ++i) nv[i] = k0 + i < lim ? src[i] : 0.0f;
                    }
                    store_new16(hi_row + b0 + k0, lo_row + b0 + k0, active || mode == kLoading,
                                lane_base + TM_AHI + s * (SB / 2), lane_base + TM_ALO + s * (SB / 2), nv);
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(&ctl.asub[s]);                 // tail A ready for GEMM(b+1)
                    if (side == 0 && s == NSB - 2 && nsub == NSB)
                        asm volatile("bar.sync 10, 256;\n" ::: "memory");
                }
                tri_prefetched = nsub == NSB;      // side 1 issued rows [0, 96) of the next block
                dmax = fmaxf(dmax, ctx.dmax);
                tc_fence_before();
                mbar_arrive(&ctl.tmem_empty[buf]);
                const long long t3 = clock64();
                c_corr += t3 - t2;
                if (b == nb - 1) {
                    // ---- end of sweep: annealing state machine (solvers.cpp:178-200), side 0
                    epi_sync();
                    if (side == 1) ctl.xa[r] = __float_as_int(dmax);
                    epi_sync();
                    if (side == 0) {
                        dmax = fmaxf(dmax, __int_as_float(ctl.xa[r]));
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
                        invT = quench ? 0.0f : 1.0f / static_cast<float>(slot.T);
                        ctl.xa[r] = new_run;
                        ctl.xb[r] = old_run;
                        ctl.xc[r] = mode | (quench ? 4 : 0);
                        ctl.xd[r] = __float_as_int(invT);
                    }
                    const bool more = epi_any(side == 0 && mode != kIdle);
                    if (side == 1) {
                        new_run = ctl.xa[r];
                        old_run = ctl.xb[r];
                        mode = ctl.xc[r] & 3;
                        quench = (ctl.xc[r] & 4) != 0;
                        invT = __int_as_float(ctl.xd[r]);
                    }
                    fence_proxy_async_global();
                    mbar_arrive(&ctl.chunk_ready[g & 1]);
                    c_wb += clock64() - t3;
                    if (!more) {
                        cp_async_wait_all();
                        if (et == 0) ctl.stop = 1;
                        goto epilogue_done;
                    }
                } else {
                    fence_proxy_async_global();
                    mbar_arrive(&ctl.chunk_ready[g & 1]);
                    c_wb += clock64() - t3;
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
            pr[7] = c_pass1;
            pr[12] = c_walk;
            pr[13] = n_walks;
            pr[14] = c_pass0;
            pr[15] = c_hand;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, TM_COLS);
}

}  // namespace

int relax_dense_umma_slots_per_cta() { return TM; }
int relax_dense_umma_block() { return TB; }
std::size_t relax_dense_umma_plane_rows(int grid) { return static_cast<std::size_t>(grid) * TM; }

cudaError_t launch_relax_dense_umma(const RelaxArgs& a, const UmmaLaunch& u, int grid, cudaStream_t st) {
    UmmaParams up{u.s_hi, u.s_lo, a.np / TB};
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
