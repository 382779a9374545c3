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
// chunks wait for that epilogue's state write-back (released per 64-spin half block);
// two TMEM accumulators ping-pong.
//
// Epilogue (walker / helper).  The in-block walk is a serial chain per run.  A walker warp
// walks every SB-spin sub-block of its 32 runs; before sub-block t it needs the fields
// corrected by the Deltas of sub-blocks 0..t-1.  The helper warp of the same lane quarter
// applies sub-blocks 0..t-2 (Delta history in TMEM, triangle rows in smem) while the walker
// walks t-1, and writes the fields back to TMEM; the walker then applies only sub-block t-1
// (from its registers) before walking t.  So the chain per sub-block is one 16 x 16
// rectangle plus the 16-spin walk.  Walker <-> helper hand-offs are mbarriers (two per
// direction per quarter, alternating, so neither side can lap the other).
// A finished slot is refilled without stalling the pipeline: for one "loading" sweep the
// epilogue streams the old run's final spins out and the new run's initial state in, block
// by block, in Gauss-Seidel order, so every GEMM always reads a consistent state.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2..5 = walkers, 6..9 = helpers (warp w accesses TMEM lanes 32*(w%4) .. +31).
//
// Global layout: state planes S_hi/S_lo [grid*TM][np] fp16 (row per slot, K-major for
// UMMA), couplings J_hi/J_lo [np][np] fp16 (J symmetric, so row i of J is column i: the
// K-major B operand of block b is the row block J[b*TB .. b*TB+TB)[*]), J32 [np][np] fp32
// for the epilogue's diagonal block.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>

#include "kernels.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

using namespace umma;

constexpr int TM = 128;      // runs per CTA = TMEM lanes = UMMA M
constexpr int TB = 128;      // spins per Gauss-Seidel block = UMMA N
// K per pipeline stage: one 64-byte swizzle atom row of fp16.  Small stages, many of them:
// the operand stream (state + coupling tiles from L2/HBM) is latency bound, so what sets the
// GEMM rate is the bytes in flight -- 5 x 32 KB stages keep ~4 loads outstanding where the
// former 2 x 64 KB ring kept ~1 (measured: the MMA waited on TMA, not on SMEM or the pipe).
#ifndef MARS_UMMA_KC
#define MARS_UMMA_KC 64
#endif
constexpr int KC = MARS_UMMA_KC;   // 32: SWIZZLE_64B rows; 64: SWIZZLE_128B rows (A/B variant)
constexpr int CPB = TB / KC; // chunks per block
// The diagonal block's triangle (33 KB) is double buffered (the helpers stage block b+1's
// during block b).  MARS_JTRI_BUFS=1 single-buffers it (staged once the walkers are past the
// block, inside their wait for the next GEMM) and spends the 33 KB on two more operand
// stages: measured 0.8% slower on cfg2 (same box) -- the MMA's wait for operand data did not
// shrink, so the ring depth is not what limits the GEMM (the shared-memory port is: an N=128
// SS-MMA reads 96 B/clk of operands per SM on top of 64 B/clk of TMA writes).
// All of a stage's MMAs under one elect (1) or one elect per MMA (0)
#ifndef MARS_UMMA_STAGE_ISSUE
#define MARS_UMMA_STAGE_ISSUE (MARS_UMMA_KC == 32)
#endif
// Issue order of the three split products per K step (A/B experiment; 0: hi*hi, lo*hi, hi*lo;
// measured no difference)
#ifndef MARS_UMMA_ORDER_A
#define MARS_UMMA_ORDER_A 0
#endif
#ifndef MARS_JTRI_BUFS
#define MARS_JTRI_BUFS 2
#endif
constexpr int JBUFS = MARS_JTRI_BUFS;
constexpr int STAGES = (JBUFS == 1 ? 8 : 6) * 32 / KC;
constexpr int NT = 320;      // 2 control warps + 4 walker warps + 4 helper warps
constexpr int EPI_W = 2;     // first walker warp
constexpr int EPI_H = 6;     // first helper warp
constexpr int NW = 128;      // walker (= helper) threads
// CTA pair (cluster of 2, cta_group::2): the leader issues M = 2*TM MMAs; each CTA holds its own
// TM state rows and half (TB/2 rows) of every coupling tile, so each SM loads and feeds to the
// tensor core only half of J -- the operand stream per SM per block drops by a quarter.
constexpr int TBH = TB / 2;  // coupling rows per CTA of the pair
constexpr std::uint32_t TILE_A = TM * KC * 2;   // 8 KB
constexpr std::uint32_t TILE_J = TBH * KC * 2;  // 4 KB
constexpr std::uint32_t STAGE_BYTES = 2 * TILE_A + 2 * TILE_J;
// TMEM: two 128-column field accumulators (ping-pong across blocks) + the current block's
// Delta history (one column per spin, lane = run)
constexpr std::uint32_t TMEM_COLS = 512;
constexpr std::uint32_t DEL_COL = 2 * TB;

enum : int { kIdle = 0, kActive = 1, kLoading = 2, kDrain = 3 };

struct __align__(8) Ctl {
    std::uint64_t full[STAGES];
    std::uint64_t empty[STAGES];
    std::uint64_t tmem_full[2];
    std::uint64_t tmem_empty[2];
    std::uint64_t part_ready[2];    // split-K: the other pairs' partial fields of a block in L2
    std::uint64_t jready[2];        // diagonal triangle staged (per block parity)
    std::uint64_t wdone;            // walkers past a block (JBUFS == 1: the triangle may go)
    std::uint64_t fready[4][2];     // helper -> walker: pre-corrected fields (per lane quarter)
    std::uint64_t dready[4][2];     // walker -> helper: a sub-block's Deltas in TMEM
    std::uint64_t mma_done;
    std::uint64_t pair_more[2];     // end-of-sweep consensus with the peer CTA (per sweep parity)
    std::uint32_t peer_more[2];     // written remotely by the peer
    std::uint32_t more_all;
    std::uint32_t tmem_base;
    // Write-back counters, per 64-spin half block: +1 per walker warp of pair 0 (same half)
    // each time it has written that half of a block back (so 4*(g+1) after block g).  A
    // monotonic count, not an mbarrier: with split-K a pair whose K range misses a block need
    // not wait for it, so the walkers may be any number of blocks past such a pair's producer.
    std::uint32_t wb[2];
    std::uint64_t chunk_ready[2];   // SPLIT == 1: the same signal as an mbarrier (NW arrivals per
                                    // half block; the producer reads every block, so its parity
                                    // waits cannot alias) -- the hardware wake-up is faster
    volatile std::uint32_t stop;    // end of the batch (set by pair 0's walkers in every CTA)
    volatile std::uint32_t poison;  // 1 + the sequence number of the stage the leader producer
                                    // arrived on without data when it stopped (0 = running)
};

// dynamic smem: [stages: A_hi A_lo J_hi J_lo] [Jtri x 2: upper triangle of the diagonal block,
// fp32, row i stored from column (i+1) rounded down to a multiple of 4 so every row is
// float4-aligned; double buffered so the helpers stage the next block's during this one] [Ctl]
__host__ __device__ constexpr int tri_k0(int i) { return (i + 1) & ~3; }
__host__ __device__ constexpr int tri_row_off(int i) {
    int off = 0;
    for (int r = 0; r < i; ++r) off += TB - tri_k0(r);
    return off;
}
constexpr std::uint32_t SMEM_STAGES = STAGES * STAGE_BYTES;
constexpr std::uint32_t TRI = tri_row_off(TB);
constexpr std::uint32_t SMEM_TRI = ((TRI * 4 + 127) / 128) * 128;
constexpr std::uint32_t SMEM_TOTAL = SMEM_STAGES + JBUFS * SMEM_TRI + sizeof(Ctl);
static_assert(SMEM_TOTAL <= 232448, "shared memory budget");

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

// K-major operand descriptor of this kernel's stage layout (64- or 128-byte swizzled rows)
__device__ __forceinline__ std::uint64_t desc_k(std::uint32_t smem_addr) {
    if constexpr (KC == 64) {
        return desc_k_sw128(smem_addr);
    } else {
        return desc_k_sw64(smem_addr);
    }
}

struct UmmaParams {
    float* xpart;            // split-K: partial fields of pairs 1.. [split-1][2][tile rows][TB] fp32
    const __half* s_hi;      // state planes (generic pointers for the epilogue)
    __half* s_hi_w;
    __half* s_lo_w;
    int nb;                  // blocks per sweep = np / TB
    int pf;                  // L2 prefetch distance of the state tiles, in chunks (0 = off; measured
                             // slower on cfg2 at 8 and 16 -- extra L2 pressure), MARS_UMMA_PF
    int spol;                // L2 policy of the state-tile loads: 0 evict_normal, 1 evict_last,
                             // 2 evict_first (default: measured on cfg2, same box, 3 runs each:
                             // 12.52K vs 12.17K descents/s, DRAM 11.8 vs 14.0 TB per launch,
                             // L2 hit rate 55.6% vs 50.8%), MARS_UMMA_SPOL
    int jpol;                // the same for the coupling tiles (default 1, evict_last), MARS_UMMA_JPOL
    int nowb;                // TIMING EXPERIMENT ONLY (wrong results): the producers do not wait for
                             // the walkers' write-back except at the sweep boundary, MARS_UMMA_NOWB
    int nohelp;              // TIMING EXPERIMENT ONLY (wrong results): the helpers skip their
                             // rectangles (mma.sync), MARS_UMMA_NOHELP
    int gemmonly;            // TIMING EXPERIMENT ONLY (wrong results; with MARS_UMMA_NOWB=1): walkers
                             // and helpers skip the block's epilogue entirely, MARS_UMMA_GEMMONLY
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

// ---- the in-block Gauss-Seidel walk of one SB-spin sub-block (one thread = one run), fully
// unrolled with fold expressions.  Fields are fp32 pairs so the in-sub-block updates issue as
// FFMA2; the J rows (diagonal block's upper triangle in smem) are 16-byte loads issued before
// the spin's trial so their latency hides under the tanh.  Each spin's change Delta is kept
// in a register (del[I]) -- the walker stores the sub-block's Deltas to TMEM for the helper.
constexpr int SB = 16;

// Who applies sub-block t-1's Deltas to sub-block t.  With the helper on mma.sync (default)
// the helper does every rectangle, the last one after the walker's hand-off, and the walker
// only walks (MARS_WALK_FOLD=0: its fold's broadcast loads were the largest shared-memory
// consumer after the UMMA operands).  With the CUDA-core helper the walker folds t-1 into
// its walk of t-1 (off the serial chain) and the helper starts at t = 2.
#ifndef MARS_HELPER_MMA
#define MARS_HELPER_MMA 0
#endif
#ifndef MARS_WALK_FOLD
#define MARS_WALK_FOLD (MARS_HELPER_MMA ? 0 : 1)
#endif
static_assert(MARS_HELPER_MMA || MARS_WALK_FOLD, "the CUDA-core helper needs the walker's fold");
// Load the fold's coupling rows together with the in-sub-block rows, ahead of each spin's trial:
// +2.4% on cfg2 once the walker binds (same box; neutral while the GEMM bound)
#ifndef MARS_WALK_HOIST
#define MARS_WALK_HOIST 1
#endif
constexpr bool kWalkFold = MARS_WALK_FOLD != 0;
constexpr int HT0 = kWalkFold ? 2 : 1;   // first sub-block the helper prepares

// The same for row i = k0 + I with k0 a multiple of 16 and I < 16 a compile-time constant:
// with Q = k0 / 4, a = I / 4, r = I % 4 the closed form of tri_row_off(i) - tri_k0(i) is
//   (128 k0 - 8 Q^2 - k0) + (128 I - 8 a^2 - 4 a (r - 1) - ((I + 1) & ~3)) - Q (4 (r - 1) + 16 a),
// i.e. a per-sub-block base plus a constant minus Q times a constant: one IMAD per row.
struct TriRows {
    const float* base;    // jtri + 128 k0 - 8 Q^2 - k0
    int Q;
    __device__ __forceinline__ TriRows(const float* jtri, int k0) : base(jtri + 127 * k0 - 8 * (k0 >> 2) * (k0 >> 2)), Q(k0 >> 2) {}
    template <int I>
    __device__ __forceinline__ const float* row(int col) const {   // &J[k0 + I][col]
        constexpr int a = I >> 2, r = I & 3;
        constexpr int kc = 128 * I - 8 * a * a - 4 * a * (r - 1) - ((I + 1) & ~3);
        constexpr int kq = 4 * (r - 1) + 16 * a;
        return base + kc - Q * kq + col;
    }
};
static_assert(TB == 128, "TriRows assumes 128-spin blocks");

struct SubCtx {
    const float* jtri;
    TriRows tr;           // rows of the current sub-block
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
__device__ __forceinline__ void sub_step(float2 (&p)[SB / 2], float2 (&an)[SB / 2], const float (&old)[SB],
                                         float (&nv)[SB], float (&del)[SB], int k0, SubCtx& c) {
    if (FULL || k0 + I < c.lim) {
        // J[k0+I][k0 + 4g ..] for the groups this spin updates, issued before the trial
        float4 jr[SB / 4];
#if MARS_WALK_HOIST
        // the fold's row of this spin (coupling to the NEXT sub-block), loaded with the others
        // ahead of the trial
        float4 jn[SB / 4];
        if constexpr (kWalkFold) {
            const float4* src = reinterpret_cast<const float4*>(c.tr.template row<I>(k0 + SB));
#pragma unroll
            for (int g = 0; g < SB / 4; ++g) jn[g] = src[g];
        }
#endif
        if constexpr (I + 1 < SB) {
            const float* row = c.tr.template row<I>(k0);     // row[m] = J[k0+I][k0+m]
#pragma unroll
            for (int g = ((I + 1) & ~3) / 4; g < SB / 4; ++g) jr[g] = *reinterpret_cast<const float4*>(row + 4 * g);
        }
        const float x = (I & 1 ? p[I / 2].y : p[I / 2].x) + (HAS_H ? __ldg(c.h + k0 + I) : 0.0f);
        // tanh_trial (solvers.cpp:145-148): -tanh(phi/t), or -sign(phi) at the quench; phi / t
        // rounded as div.rn does (quotient from the hoisted refined reciprocal plus div.rn's
        // two correction FMAs: bit-identical to __fdiv_rn for these operands)
        const float sgn = x > 0.0f ? -1.0f : (x < 0.0f ? 1.0f : 0.0f);
        const float q0 = fmaf(c.rT, x, 0.0f);
        const float th = -tanhf(fmaf(fmaf(-c.T, q0, x), c.rT, q0));
        const float trial = c.quench ? sgn : th;
        const float delta = trial - old[I];
        del[I] = delta;
        nv[I] = trial;
        c.dmax = fmaxf(c.dmax, fabsf(delta));
        if constexpr (I + 1 < SB)
            sub_update<I>(p, jr, delta, std::make_integer_sequence<int, SB / 4 - ((I + 1) & ~3) / 4>{});
        if constexpr (kWalkFold) {
            // this spin's coupling to the NEXT sub-block's fields, accumulated off the serial
            // chain (added to the next sub-block's fields before it walks)
#if !MARS_WALK_HOIST
            const float4* jn = reinterpret_cast<const float4*>(c.tr.template row<I>(k0 + SB));
#endif
#pragma unroll
            for (int g = 0; g < SB / 4; ++g) {
                const float4 jv = jn[g];
                an[2 * g] = ffma2(make_float2(jv.x, jv.y), delta, an[2 * g]);
                an[2 * g + 1] = ffma2(make_float2(jv.z, jv.w), delta, an[2 * g + 1]);
            }
        }
    } else {
        nv[I] = old[I];
        del[I] = 0.0f;
    }
}

template <bool FULL, bool HAS_H, int... I>
__device__ __forceinline__ void sub_walk(float2 (&p)[SB / 2], float2 (&an)[SB / 2], const float (&old)[SB],
                                         float (&nv)[SB], float (&del)[SB], int k0, SubCtx& c,
                                         std::integer_sequence<int, I...>) {
    (sub_step<I, FULL, HAS_H>(p, an, old, nv, del, k0, c), ...);
}

template <bool HAS_H>
__device__ __forceinline__ void walk_dispatch(float2 (&p)[SB / 2], float2 (&an)[SB / 2], const float (&old)[SB],
                                              float (&nv)[SB], float (&del)[SB], int k0, SubCtx& c) {
    if (k0 + SB <= c.lim)
        sub_walk<true, HAS_H>(p, an, old, nv, del, k0, c, std::make_integer_sequence<int, SB>{});
    else
        sub_walk<false, HAS_H>(p, an, old, nv, del, k0, c, std::make_integer_sequence<int, SB>{});
}

// fields (fp32 pairs) += J[j0 .. j0+16)[col .. col+16)^T * d[0..16): the 16 x 16 rectangle
// coupling one sub-block's Deltas to a later sub-block's fields (rows from the triangle)
// split-K: the other pairs' partial fields (same prescaled units as the TMEM accumulator) for
// 16 columns of this slot's row; L2 loads (written by other SMs this block)
template <int SPLIT>
__device__ __forceinline__ void add_partials(float (&pv)[16], const float* xpart, std::size_t plane, int buf,
                                             std::size_t row, int col) {
    if constexpr (SPLIT > 1) {
#pragma unroll
        for (int p = 0; p < SPLIT - 1; ++p) {
            const float4* src = reinterpret_cast<const float4*>(xpart + ((p * 2 + buf) * plane + row) * TB + col);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float4 x = __ldcg(src + v);
                pv[4 * v] += x.x;
                pv[4 * v + 1] += x.y;
                pv[4 * v + 2] += x.z;
                pv[4 * v + 3] += x.w;
            }
        }
    }
}

template <int J>
__device__ __forceinline__ void rect_row(float2 (&pf)[SB / 2], const TriRows& tr, int col, float d) {
    const float4* jr = reinterpret_cast<const float4*>(tr.template row<J>(col));
#pragma unroll
    for (int m = 0; m < SB / 4; ++m) {
        const float4 jv = jr[m];
        pf[2 * m] = ffma2(make_float2(jv.x, jv.y), d, pf[2 * m]);
        pf[2 * m + 1] = ffma2(make_float2(jv.z, jv.w), d, pf[2 * m + 1]);
    }
}

template <int... J>
__device__ __forceinline__ void rect_rows(float2 (&pf)[SB / 2], const TriRows& tr, int col, const float (&d)[SB],
                                          std::integer_sequence<int, J...>) {
    (rect_row<J>(pf, tr, col, d[J]), ...);
}

// fields (fp32 pairs) += J[j0 .. j0+16)[col .. col+16)^T * d[0..16): the 16 x 16 rectangle
// coupling one sub-block's Deltas to a later sub-block's fields (rows from the triangle)
__device__ __forceinline__ void apply_rect16(float2 (&pf)[SB / 2], const float* jtri, int j0, int col,
                                             const float (&d)[SB]) {
    rect_rows(pf, TriRows(jtri, j0), col, d, std::make_integer_sequence<int, SB>{});
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

__device__ __forceinline__ void tmem_st16f(std::uint32_t taddr, const float (&v)[16]) {
    std::uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[i]);
    tmem_st16(taddr, r);
}

// ---- helper rectangles on the warp-level tensor core (mma.sync.m16n8k16, fp16 hi/lo split,
// fp32 accumulate).  A helper warp's 32 runs are two 16-run m-tiles (TMEM lanes 32q..+15,
// 32q+16..+31).  tcgen05.ld/st .16x256b hand each thread exactly the mma fragment layout:
// register e of a 16 x 8-column group is (lane g + 8*(e>>1), column 2c + (e&1)), g = lane/4,
// c = lane%4 -- the f32 C/D fragment, and, packed in pairs, the f16 A fragment.  The coupling
// fragments (8 fp32 values per 16 x 16 rectangle, from the diagonal triangle) are loaded per
// thread with distinct addresses, instead of 64 warp-broadcast LDS.128 per rectangle.
__device__ __forceinline__ void tmem_ld_16x256_x2(std::uint32_t taddr, float (&v)[8]) {
    std::uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st_16x256_x2(std::uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}

__device__ __forceinline__ std::uint32_t h2_bits(__half2 h) { return *reinterpret_cast<std::uint32_t*>(&h); }

// x0, x1 (x0 at the lower index) -> packed fp16 hi pair and lo pair (x = hi + lo)
__device__ __forceinline__ void split_pair(float x0, float x1, std::uint32_t& hi, std::uint32_t& lo) {
    const __half2 h = __floats2half2_rn(x0, x1);
    const float2 hf = __half22float2(h);
    hi = h2_bits(h);
    lo = h2_bits(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
}

__device__ __forceinline__ void mma_16816(float& c0, float& c1, float& c2, float& c3, const std::uint32_t (&a)[4],
                                          std::uint32_t b0, std::uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// fields f[m][8] (m-tile m: 16 runs x 16 columns of target sub-block t, prescaled units) +=
// Delta_u (TMEM history, this warp's runs) x J[u rows][t columns] * jup, jup = 2^jexp (the
// couplings in the same prescaled units, inside fp16's range)
__device__ __forceinline__ void rect_mma(float (&f)[2][8], std::uint32_t tdel, const float* jtri, int u, int t,
                                         float jup, int lane) {
    const int g = lane >> 2, c = lane & 3;
    // coupling fragments: B[k][n] = J[16u + k][16t + 8nt + n]; this thread: k = 2c, 2c+1, 2c+8, 2c+9, n = g
    std::uint32_t bh[2][2], bl[2][2];
    {
        float jv[2][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int i = 16 * u + 2 * c + (kk & 1) + 8 * (kk >> 1);
            const float* row = jtri + tri_row_off_rt(i) - tri_k0(i) + 16 * t + g;
            jv[0][kk] = row[0] * jup;
            jv[1][kk] = row[8] * jup;
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            split_pair(jv[nt][0], jv[nt][1], bh[nt][0], bl[nt][0]);
            split_pair(jv[nt][2], jv[nt][3], bh[nt][1], bl[nt][1]);
        }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        float d[8];
        tmem_ld_16x256_x2(tdel + (static_cast<std::uint32_t>(16 * m) << 16) + u * SB, d);
        std::uint32_t ah[4], al[4];
        split_pair(d[0], d[1], ah[0], al[0]);
        split_pair(d[2], d[3], ah[1], al[1]);
        split_pair(d[4], d[5], ah[2], al[2]);
        split_pair(d[6], d[7], ah[3], al[3]);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            float* acc = &f[m][4 * nt];
            mma_16816(acc[0], acc[1], acc[2], acc[3], ah, bh[nt][0], bh[nt][1]);
            mma_16816(acc[0], acc[1], acc[2], acc[3], al, bh[nt][0], bh[nt][1]);
            mma_16816(acc[0], acc[1], acc[2], acc[3], ah, bl[nt][0], bl[nt][1]);
        }
    }
}

struct Old16 {
    uint4 h[2], l[2];
};

__device__ __forceinline__ void fetch_old16(const __half* hi, const __half* lo, Old16& o) {
    o.h[0] = *reinterpret_cast<const uint4*>(hi);
    o.h[1] = *reinterpret_cast<const uint4*>(hi + 8);
    o.l[0] = *reinterpret_cast<const uint4*>(lo);
    o.l[1] = *reinterpret_cast<const uint4*>(lo + 8);
}

__device__ __forceinline__ void unpack_old16(const Old16& o, float (&old)[SB]) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const __half* h8 = reinterpret_cast<const __half*>(&o.h[v]);
        const __half* l8 = reinterpret_cast<const __half*>(&o.l[v]);
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
// arrive on `bar` once every cp.async this thread issued so far has landed (no pending-count
// increment: the barrier's expected count includes this arrival)
__device__ __forceinline__ void cp_async_arrive_noinc(std::uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// the diagonal block's upper triangle (fp32) -> packed smem layout, cooperative over the
// helper warps (128 threads)
__device__ __forceinline__ void issue_jtri(float* dst, const float* J32, int np, int b0, int ht) {
    for (int f = ht; f < TB * TB / 4; f += TM) {
        const int i = f / (TB / 4), k = (f % (TB / 4)) * 4;
        if (k >= tri_k0(i)) cp_async16(dst + tri_row_off_rt(i) + k - tri_k0(i), J32 + static_cast<size_t>(b0 + i) * np + b0 + k);
    }
}

// End-of-sweep consensus of the CTA pair (walkers + helpers of both CTAs): the pair runs its
// blocks in lock step (one MMA stream), so it stops only when neither CTA has a slot left.
// Called by all 256 epilogue threads with their CTA-local vote; `lead` is one walker thread.
__device__ __forceinline__ bool pair_any(Ctl& ctl, bool local, bool lead, std::uint32_t rank, long long sweep) {
    // sweep: 0-based index; consecutive sweeps alternate between two barrier/flag slots
    const std::uint32_t par = static_cast<std::uint32_t>(sweep) & 1u;
    if (lead) {
        const std::uint32_t peer = rank ^ 1u;
        st_cluster_u32(mapa_shared(smem_u32(&ctl.peer_more[par]), peer), local ? 1u : 0u);
        mbar_arrive_cluster(mapa_shared(smem_u32(&ctl.pair_more[par]), peer));
        mbar_wait_cluster(&ctl.pair_more[par], (static_cast<std::uint32_t>(sweep) >> 1) & 1u);
        ctl.more_all = (local || ctl.peer_more[par] != 0) ? 1u : 0u;
    }
    asm volatile("bar.sync 1, 256;\n" ::: "memory");
    return ctl.more_all != 0;
}

// a walker warp has written half `hb` of a block back: count it in this CTA and in the CTAs
// of the other pairs on the same runs (same half).  Each lane's stores are ordered before the
// producer's TMA reads by its proxy fence, the warp barrier and lane 0's release.
template <int SPLIT>
__device__ __forceinline__ void signal_writeback(Ctl& ctl, int hb, int half, int lane) {
    fence_proxy_async_global();
    if constexpr (SPLIT == 1) {
        mbar_arrive(&ctl.chunk_ready[hb]);
        return;
    }
    __syncwarp();
    if (lane == 0) {
        red_add_release_cta(&ctl.wb[hb], 1u);
        for (int p = 1; p < SPLIT; ++p) red_add_release_cluster(mapa_shared(smem_u32(&ctl.wb[hb]), 2 * p + half), 1u);
    }
}

// wait until half `hb` of block target/4 - 1 has been written back (the counter reaches
// `target`, 4 per block; SPLIT == 1: that block's mbarrier phase)
template <int SPLIT>
__device__ __forceinline__ void wait_writeback(Ctl& ctl, int hb, std::uint32_t target) {
    if constexpr (SPLIT == 1) {
        mbar_wait(&ctl.chunk_ready[hb], (target / 4 - 1) & 1);
        return;
    }
    if (ld_acquire_cluster(&ctl.wb[hb]) >= target) return;
    std::uint64_t h0 = 0;
    for (std::uint32_t spin = 1; ld_acquire_cluster(&ctl.wb[hb]) < target; ++spin) {
        if (spin > 64) __nanosleep(32);
        if (hang_check(h0, spin)) mbar_hang(&ctl.tmem_full[0], 0x100u + hb);   // (reported as 0x10h)
    }
}

// SPLIT > 1 (large N): a cluster of 2*SPLIT CTAs = SPLIT pairs on the SAME 256 runs; pair p runs
// the GEMM over the K chunks [p*nk/SPLIT, (p+1)*nk/SPLIT) and pairs 1.. export their partial
// fields through L2 to pair 0, whose walkers and helpers add them (fp32) to their own before
// the walk.  Only pair 0 owns run slots; the other pairs' producers follow its write-backs.
template <bool JLO, int SPLIT>
__global__ void __launch_bounds__(NT, 1)
relax_dense_umma_kernel(RelaxArgs a, UmmaParams up, const __grid_constant__ CUtensorMap tm_shi,
                        const __grid_constant__ CUtensorMap tm_slo,
                        const __grid_constant__ CUtensorMap tm_jhi,
                        const __grid_constant__ CUtensorMap tm_jlo) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw;   // SWIZZLE_128B tiles need 1024-byte alignment (checked)
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0) __trap();
    float* Jtri0 = reinterpret_cast<float*>(base + SMEM_STAGES);
    Ctl& ctl = *reinterpret_cast<Ctl*>(base + SMEM_STAGES + JBUFS * SMEM_TRI);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int np = a.np, n = a.n, nb = up.nb, nk = np / KC;
    const std::uint32_t rank = cluster_ctarank();
    const int pair = static_cast<int>(rank >> 1), half = static_cast<int>(rank & 1);
    const bool leader = half == 0;
    const int tile = blockIdx.x / (2 * SPLIT);
    const int row0 = (2 * tile + half) * TM;             // this CTA's 128 state rows
    const int c_lo = pair * (nk / SPLIT), c_hi = c_lo + nk / SPLIT;   // this pair's K chunks

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&ctl.full[s], 1);
            mbar_init(&ctl.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.tmem_full[s], 1);
            mbar_init(&ctl.tmem_empty[s], 2 * NW);   // leader's: both CTAs' walkers
            mbar_init(&ctl.pair_more[s], 1);
            ctl.wb[s] = 0;
            mbar_init(&ctl.chunk_ready[s], NW);
            mbar_init(&ctl.part_ready[s], NW * (SPLIT - 1) + (SPLIT == 1));
            mbar_init(&ctl.jready[s], NW);
            if (s == 0) mbar_init(&ctl.wdone, NW);
        }
        for (int q = 0; q < 4; ++q)
            for (int s = 0; s < 2; ++s) {
                mbar_init(&ctl.fready[q][s], 32);
                mbar_init(&ctl.dready[q][s], 32);
            }
        mbar_init(&ctl.mma_done, 1);
        ctl.stop = 0;
        ctl.poison = 0;
        fence_mbar_init();
        if (a.prof && blockIdx.x == 0)
            printf("mars: relax_dense_umma Ctl at smem 0x%x (full +0, empty +%d, tmem_full +%d, tmem_empty +%d, "
                   "wb +%d, part_ready +%d, jready +%d, fready +%d, dready +%d, mma_done +%d, pair_more +%d)\n",
                   smem_u32(&ctl), int(offsetof(Ctl, empty)), int(offsetof(Ctl, tmem_full)), int(offsetof(Ctl, tmem_empty)),
                   int(offsetof(Ctl, wb)), int(offsetof(Ctl, part_ready)), int(offsetof(Ctl, jready)),
                   int(offsetof(Ctl, fready)), int(offsetof(Ctl, dready)), int(offsetof(Ctl, mma_done)),
                   int(offsetof(Ctl, pair_more)));
    }
    cluster_sync_all();                      // the peers' barriers exist before any remote arrive
    if (warp == 1) tmem_alloc_pair(&ctl.tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = ctl.tmem_base;

    if (warp == 0) {
        // ================================================================ TMA producer
        // Whole warp converged; one elected lane issues.  Stage / phase / chunk advance
        // incrementally (no division in the loop).
        if (lane == 0) {
            tma_prefetch_desc(&tm_shi);
            tma_prefetch_desc(&tm_slo);
            tma_prefetch_desc(&tm_jhi);
            if (JLO) tma_prefetch_desc(&tm_jlo);
        }
        __syncwarp();
        const std::uint64_t jpol = up.jpol == 1 ? policy_evict_last() : up.jpol == 2 ? policy_evict_first() : policy_evict_normal();
        const std::uint64_t spol = up.spol == 1 ? policy_evict_last() : up.spol == 2 ? policy_evict_first() : policy_evict_normal();
        const std::uint32_t smem0 = smem_u32(base);
        const std::uint32_t full0 = smem_u32(&ctl.full[0]);
        const std::uint32_t tx = 2 * (JLO ? STAGE_BYTES : STAGE_BYTES - TILE_J);   // both CTAs' bytes
        std::uint32_t g = 0, s = 0, ph = 0, seq = 0;   // seq: stages issued so far
        long long w_ready = 0, w_empty = 0;
        for (;;) {
            for (int b = 0; b < nb; ++b, ++g) {
                int c = b * CPB;                               // chunk order: block b first
                for (int j = 0; j < nk; ++j) {
                    const bool mine = c >= c_lo && c < c_hi;   // in this pair's K range
                    // The last chunks of GEMM(b) are block b-1: a pair that reads them waits until
                    // the walkers have written that half block back.  At GEMM(0) every pair waits
                    // for the end of the previous sweep (block nb-1, second half): the walkers
                    // raise `stop` before that write-back, so both producers of a pair stop at
                    // this same point of their stage sequence.
                    const bool sweep_end = b == 0 && j == nk - CPB / 2;
                    if ((j == nk - CPB || j == nk - CPB / 2) && g > 0 && (mine || sweep_end) && (!up.nowb || sweep_end)) {
                        const long long t0 = clock64();
                        wait_writeback<SPLIT>(ctl, j == nk - CPB ? 0 : 1, 4u * g);
                        w_ready += clock64() - t0;
                        if (sweep_end && ctl.stop) {
                            // end of the batch: the next stage carries no data; the leader names
                            // it for its MMA issuer, which consumes every stage before it
                            mbar_wait(&ctl.empty[s], ph ^ 1);
                            if (lane == 0) {
                                if (leader) {
                                    ctl.poison = seq + 1;
                                    mbar_arrive(&ctl.full[s]);
                                }
                                if (a.prof) {
                                    a.prof[blockIdx.x * kProfSlots + 8] = w_ready;
                                    a.prof[blockIdx.x * kProfSlots + 9] = w_empty;
                                }
                            }
                            goto producer_done;
                        }
                    }
                    if (!mine) {                              // another pair's K range
                        if (++c == nk) c = 0;
                        continue;
                    }
                    const long long t1 = clock64();
                    mbar_wait(&ctl.empty[s], ph ^ 1);
                    w_empty += clock64() - t1;
                    const std::uint32_t st = smem0 + s * STAGE_BYTES;
                    const std::uint32_t fb = full0 + s * 8;
                    if (leader) mbar_arrive_expect_tx_elect(&ctl.full[s], tx);
                    tma_load_2d_pair_elect(st, &tm_shi, fb, c * KC, row0, spol);
                    tma_load_2d_pair_elect(st + TILE_A, &tm_slo, fb, c * KC, row0, spol);
                    // the coupling tiles are read by every CTA every sweep: keep them in L2
                    // ahead of the per-CTA state planes; this CTA's half of the block's rows
                    tma_load_2d_pair_elect(st + 2 * TILE_A, &tm_jhi, fb, c * KC, b * TB + half * TBH, jpol);
                    if (JLO) tma_load_2d_pair_elect(st + 2 * TILE_A + TILE_J, &tm_jlo, fb, c * KC, b * TB + half * TBH, jpol);
                    if (up.pf > 0) {
                        // warm L2 with this CTA's state tiles up.pf chunks ahead (same block;
                        // a chunk of block b-1 fetched early is refreshed in L2 by the walker's
                        // write-back, so the later TMA load still reads the new values)
                        int cp = c + up.pf;
                        if (cp >= nk) cp -= nk;
                        if (j + up.pf < nk) {
                            tma_prefetch_2d_elect(&tm_shi, cp * KC, row0);
                            tma_prefetch_2d_elect(&tm_slo, cp * KC, row0);
                        }
                    }
                    if (++c == nk) c = 0;
                    ++seq;
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    producer_done:;
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        // Leader CTA only.  Whole warp converged (descriptors are warp-uniform: uniform
        // registers); one elected lane issues each tcgen05.mma / commit for the pair.
        if (!leader) goto mma_skip;
        {
        constexpr std::uint32_t idesc = idesc_f16(2 * TM, TB, 0);
        const std::uint32_t smem0 = smem_u32(base);
        std::uint32_t g = 0, s = 0, ph = 0, seq = 0;   // seq: stages consumed so far
        long long w_full = 0, w_tmem = 0;
        for (;;) {
            for (int b = 0; b < nb; ++b, ++g) {
                const int buf = g & 1;
                const long long t0 = clock64();
                mbar_wait(&ctl.tmem_empty[buf], ((g >> 1) & 1) ^ 1);
                w_tmem += clock64() - t0;
                tc_fence_after();
                const std::uint32_t d = tmem + buf * TB;
                for (int j = 0, c = b * CPB, cnt = 0; j < nk; ++j, c = c + 1 == nk ? 0 : c + 1) {
                    if (c < c_lo || c >= c_hi) continue;    // another pair's K range
                    const long long t1 = clock64();
                    mbar_wait(&ctl.full[s], ph);
                    w_full += clock64() - t1;
                    // the producers' stop point is the chunk at nk - CPB/2 of GEMM(0), or (a pair
                    // whose K range ends before it) the first chunk of GEMM(1)
                    if ((b == 0 ? j >= nk - CPB / 2 : b == 1 && cnt == 0) && ctl.poison == seq + 1) {
                        if (a.prof && lane == 0) {
                            a.prof[blockIdx.x * kProfSlots + 10] = w_full;
                            a.prof[blockIdx.x * kProfSlots + 11] = w_tmem;
                        }
                        goto mma_done;
                    }
                    tc_fence_after();
                    const std::uint32_t st = smem0 + s * STAGE_BYTES;
#if MARS_UMMA_STAGE_ISSUE
                    static_assert(KC == 32 || !MARS_UMMA_STAGE_ISSUE, "one stage = two K steps of 16");
                    mma_stage_split_pair_elect<JLO>(d, desc_k(st), desc_k(st + TILE_A), desc_k(st + 2 * TILE_A),
                                                    desc_k(st + 2 * TILE_A + TILE_J), idesc, cnt != 0);
#else
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk) {
                        const std::uint64_t ahi = desc_k(st + kk * 32);
                        const std::uint64_t alo = desc_k(st + TILE_A + kk * 32);
                        const std::uint64_t jhi = desc_k(st + 2 * TILE_A + kk * 32);
#if MARS_UMMA_ORDER_A
                        // the two products sharing A_hi back to back
                        mma_f16_ss_pair_elect(d, ahi, jhi, idesc, (cnt | kk) != 0);
                        if (JLO) {
                            const std::uint64_t jlo = desc_k(st + 2 * TILE_A + TILE_J + kk * 32);
                            mma_f16_ss_pair_elect(d, ahi, jlo, idesc, 1);
                        }
                        mma_f16_ss_pair_elect(d, alo, jhi, idesc, 1);
#else
                        mma_f16_ss_pair_elect(d, ahi, jhi, idesc, (cnt | kk) != 0);
                        mma_f16_ss_pair_elect(d, alo, jhi, idesc, 1);
                        if (JLO) {
                            const std::uint64_t jlo = desc_k(st + 2 * TILE_A + TILE_J + kk * 32);
                            mma_f16_ss_pair_elect(d, ahi, jlo, idesc, 1);
                        }
#endif
                    }
#endif
                    mma_commit_pair_mc_elect(&ctl.empty[s], pair);
                    ++cnt;
                    ++seq;
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                mma_commit_pair_mc_elect(&ctl.tmem_full[buf], pair);
            }
        }
    mma_done:
        mma_commit_pair_mc_elect(&ctl.mma_done, pair);
        mbar_wait(&ctl.mma_done, 0);
        }
    mma_skip:
        __syncwarp();
    } else if (SPLIT > 1 && pair > 0) {
        // ================================================================ exporters (split-K)
        // Pairs 1..: the walker warps hand this pair's partial fields of every block to pair 0
        // through L2; the helper warps have nothing to do.
        if (warp < EPI_H) {
            const int q = warp & 3;
            const int r = q * 32 + lane;
            const std::uint32_t lane_t = static_cast<std::uint32_t>(q * 32) << 16;
            const std::size_t plane = static_cast<std::size_t>(gridDim.x / (2 * SPLIT)) * 2 * TM;
            const std::uint32_t tmem_empty_leader = mapa_shared(smem_u32(&ctl.tmem_empty[0]), 2 * pair);
            const std::uint32_t part_ready0 = mapa_shared(smem_u32(&ctl.part_ready[0]), half);
            for (std::uint32_t g = 0;; ++g) {
                const int buf = g & 1;
                std::uint64_t t0 = 0;
                for (std::uint32_t spin = 1; !mbar_try_wait(&ctl.tmem_full[buf], (g >> 1) & 1); ++spin) {
                    if (ctl.stop) goto exporter_done;
                    if (hang_check(t0, spin)) mbar_hang(&ctl.tmem_full[buf], (g >> 1) & 1);
                }
                tc_fence_after();
                // xpart[buf] last held block g-2: pair 0 is done with it once its walkers are
                // past that block (its helpers finish a block before its walkers do)
                if (g >= 2) wait_writeback<SPLIT>(ctl, 1, 4u * (g - 1));
                float* dst = up.xpart + (((pair - 1) * 2 + buf) * plane + row0 + r) * static_cast<std::size_t>(TB);
#pragma unroll 1
                for (int cc = 0; cc < TB / 16; ++cc) {
                    float v[16];
                    tmem_ld16(tmem + lane_t + buf * TB + cc * 16, v);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        __stcg(reinterpret_cast<float4*>(dst + cc * 16) + k,
                               make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
                }
                tc_fence_before();
                mbar_arrive_cluster(part_ready0 + buf * 8);           // pair 0, same half
                mbar_arrive_cluster(tmem_empty_leader + buf * 8);     // this pair's leader MMA
            }
        exporter_done:;
        }
    } else if (warp < EPI_H) {
        // ================================================================ walkers (W)
        // Warp w owns the runs of TMEM lane quarter q = w % 4 (slot r = 32q + lane) and walks
        // every sub-block of every block in ascending spin order.  Before walking sub-block t
        // it takes the fields the helper pre-corrected (GEMM + Deltas of sub-blocks < t-1,
        // written back to TMEM) and applies the previous sub-block's Deltas from its own
        // registers, so the serial chain per sub-block is one 16 x 16 rectangle + the walk.
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const int wt = threadIdx.x - EPI_W * 32;           // 0..127
        const std::uint32_t lane_t = static_cast<std::uint32_t>(q * 32) << 16;
        __half* hi_row = up.s_hi_w + static_cast<size_t>(row0 + r) * np;
        __half* lo_row = up.s_lo_w + static_cast<size_t>(row0 + r) * np;
        Slot slot;
        slot.run = -1;
        int new_run = claim_run(a);
        int mode = new_run >= 0 ? kLoading : kIdle, old_run = -1;
        float rT = 1.0f, Tf = 1.0f;
        bool quench = false;
        std::uint32_t g = 0, fe = 0, de = 0;                // block, F-event and D-event counters
        const std::uint32_t tmem_empty_leader = mapa_shared(smem_u32(&ctl.tmem_empty[0]), 0);
        const std::size_t xplane = static_cast<std::size_t>(gridDim.x / (2 * SPLIT)) * 2 * TM;
        long long c_wait = 0, c_f = 0, c_apply = 0, c_walk = 0, c_turn = 0, c_st = 0, n_sweeps = 0;
        const long long c_start = clock64();

        for (;;) {
            ++n_sweeps;
            const bool active = mode == kActive;
            float dmax = 0.0f;
            for (int b = 0; b < nb; ++b, ++g) {
                const int b0 = b * TB;
                const int lim = min(TB, n - b0);
                const int nsub = (lim + SB - 1) / SB;
                const float* jtri = Jtri0 + (JBUFS == 2 ? (g & 1) * (SMEM_TRI / 4) : 0);
                const int buf = g & 1;
                long long t0 = clock64();
                if (!active && (mode == kLoading || mode == kDrain)) {
                    // ---- slot turnover, block by block: the old run's rounded spins out, the
                    // new run's initial state in (before this block's chunks are re-read)
                    if (old_run >= 0) {
                        std::int8_t* out = a.spins + static_cast<size_t>(old_run) * n + b0;
                        for (int i = 0; i < lim; ++i) {                 // round_spins (model.cpp:245)
                            const float s = __half2float(hi_row[b0 + i]) + __half2float(lo_row[b0 + i]);
                            out[i] = s < 0.0f ? -1 : 1;
                            if (a.state_out) a.state_out[static_cast<size_t>(old_run) * n + b0 + i] = s;
                        }
                    }
                    if (mode == kLoading) {
                        const float* src = a.s0 + static_cast<size_t>(new_run) * n + b0;
                        for (int v = 0; v < TB / 8; ++v) {
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
                long long t1 = clock64();
                c_turn += t1 - t0;
                Old16 pre;
                fetch_old16(hi_row + b0, lo_row + b0, pre);
                mbar_wait(&ctl.jready[buf], (g >> 1) & 1);
                mbar_wait(&ctl.tmem_full[buf], (g >> 1) & 1);
                if (SPLIT > 1) mbar_wait_cluster(&ctl.part_ready[buf], (g >> 1) & 1);
                tc_fence_after();
                t0 = clock64();
                c_wait += t0 - t1;
                const std::uint32_t tacc = tmem + lane_t + buf * TB;
                SubCtx ctx{jtri, TriRows(jtri, 0), a.h32 ? a.h32 + b0 : nullptr, Tf, rT, quench, lim, 0.0f};
                float prev[SB];                                 // this sub-block's Deltas
                float2 an[SB / 2];                              // previous sub-block's coupling
#pragma unroll                                                  // to this one (built during its walk)
                for (int j = 0; j < SB / 2; ++j) an[j] = make_float2(0.0f, 0.0f);
                for (int t = 0; t < (up.gemmonly ? 0 : nsub); ++t) {
                    const int k0 = t * SB;
                    const long long tpre = clock64();
                    float old[SB];
                    unpack_old16(pre, old);
                    if (t + 1 < nsub) fetch_old16(hi_row + b0 + k0 + SB, lo_row + b0 + k0 + SB, pre);
                    t1 = clock64();
                    c_apply += t1 - tpre;                       // the old-state load wait
                    if (t >= HT0) {
                        mbar_wait(&ctl.fready[q][fe & 1], (fe >> 1) & 1);
                        ++fe;
                        tc_fence_after();
                    }
                    float pv[SB];
                    tmem_ld16(tacc + k0, pv);
                    if (t < HT0) add_partials<SPLIT>(pv, up.xpart, xplane, buf, row0 + r, k0);
                    // raw GEMM fields (t < HT0) are on the prescaled couplings; the helper's are not
                    const float sc = t >= HT0 ? 1.0f : a.jscale;
                    float2 pf[SB / 2];
#pragma unroll
                    for (int j = 0; j < SB / 2; ++j) {
                        pf[j] = make_float2(fmaf(pv[2 * j], sc, an[j].x), fmaf(pv[2 * j + 1], sc, an[j].y));
                        an[j] = make_float2(0.0f, 0.0f);
                    }
                    t0 = clock64();
                    c_f += t0 - t1;
                    t1 = t0;
                    float nv[SB];
                    ctx.tr = TriRows(jtri, k0);
                    if (ctx.h) walk_dispatch<true>(pf, an, old, nv, prev, k0, ctx);
                    else walk_dispatch<false>(pf, an, old, nv, prev, k0, ctx);
                    t0 = clock64();
                    c_walk += t0 - t1;
                    if (active) store_new16(hi_row + b0 + k0, lo_row + b0 + k0, nv);
                    if (t == 0 || t + HT0 < nsub) {
                        // the helper needs this sub-block's Deltas (for sub-blocks >= t + HT0)
                        tmem_st16f(tmem + lane_t + DEL_COL + k0, prev);
                        tmem_st_wait();
                        tc_fence_before();
                        mbar_arrive(&ctl.dready[q][de & 1]);
                        ++de;
                    }
                    if (t == min(TB / 2 / SB, nsub) - 1) {
                        // first 64-spin chunk of this block written back: its GEMM chunk may go
                        signal_writeback<SPLIT>(ctl, 0, half, lane);
                    }
                    c_st += clock64() - t0;
                }
                dmax = fmaxf(dmax, ctx.dmax);
                if (JBUFS == 1 || up.gemmonly) mbar_arrive(&ctl.wdone);   // done with this block's triangle
                tc_fence_before();
                mbar_arrive_cluster(tmem_empty_leader + buf * 8);   // the leader's MMA reuses the buffer
                if (b == nb - 1) {
                    // ---- end of sweep: annealing state machine (solvers.cpp:178-200)
                    if (active) {
                        const int code = slot_after_sweep(slot, dmax, a);
                        if (code != kSlotContinue) {
                            slot_finish(slot, code, a);
                            old_run = slot.run;
                            new_run = claim_run(a);
                            mode = new_run >= 0 ? kLoading : kDrain;
                        }
                    } else if (mode == kLoading) {
                        if (old_run >= 0) log_retired(a, old_run);   // its spins went out this sweep
                        slot_start(slot, new_run, a);
                        mode = kActive;
                        old_run = -1;
                    } else if (mode == kDrain) {
                        if (old_run >= 0) log_retired(a, old_run);
                        mode = kIdle;
                        old_run = -1;
                    }
                    quench = mode == kActive && slot_quench(slot);
                    Tf = static_cast<float>(slot.T);
                    rT = quench ? 0.0f : recip_for_div(Tf);
                    const bool more = pair_any(ctl, epi_any(mode != kIdle), wt == 0, rank, n_sweeps - 1);
                    if (!more && wt == 0) {
                        ctl.stop = 1;
                        for (int p = 1; p < SPLIT; ++p) st_cluster_u32(mapa_shared(smem_u32(const_cast<std::uint32_t*>(&ctl.stop)), 2 * p + half), 1u);
                    }
                    signal_writeback<SPLIT>(ctl, 1, half, lane);   // after `stop` (lane 0 of warp 2)
                    if (!more) goto walker_done;
                } else {
                    signal_writeback<SPLIT>(ctl, 1, half, lane);
                }
            }
        }
    walker_done:
        if (a.prof && wt == 0) {
            long long* pr = a.prof + blockIdx.x * kProfSlots;
            pr[0] = n_sweeps;
            pr[1] = clock64() - c_start;
            pr[2] = c_wait;
            pr[3] = c_f;
            pr[4] = c_apply;
            pr[5] = c_walk;
            pr[6] = nb;
            pr[7] = c_turn;
            pr[12] = c_st;
        }
    } else {
        // ================================================================ helpers (H)
        // Warp w (quarter q = w % 4, same runs as walker warp w - 4) prepares the fields of
        // sub-block t >= 2: GEMM fields + the Deltas of sub-blocks 0 .. t-2 (history in TMEM,
        // triangle rows from smem), written back to TMEM for the walker.  It also stages the
        // next block's diagonal triangle into the other smem buffer.
        const int q = warp & 3;
        const int ht = threadIdx.x - EPI_H * 32;           // 0..127
        const std::uint32_t lane_t = static_cast<std::uint32_t>(q * 32) << 16;
        std::uint32_t g = 0, fe = 0, de = 0;
        long long c_dw = 0, c_work = 0, c_tw = 0, h_sweeps = 0;
        const std::size_t xplane = static_cast<std::size_t>(gridDim.x / (2 * SPLIT)) * 2 * TM;
        const std::uint32_t tdel = tmem + lane_t + DEL_COL;   // this quarter's Delta history
        const float jup = 1.0f / a.jscale;                    // 2^jexp (exact)
        issue_jtri(Jtri0, a.J32, np, 0, ht);
        cp_async_arrive_noinc(&ctl.jready[0]);
        for (;;) {
            for (int b = 0; b < nb; ++b, ++g) {
                const int b0 = b * TB;
                const int lim = min(TB, n - b0);
                const int nsub = (lim + SB - 1) / SB;
                const float* jtri = Jtri0 + (JBUFS == 2 ? (g & 1) * (SMEM_TRI / 4) : 0);
                const int buf = g & 1;
                long long t0 = clock64();
                mbar_wait(&ctl.jready[buf], (g >> 1) & 1);
                mbar_wait(&ctl.tmem_full[buf], (g >> 1) & 1);
                if (SPLIT > 1) mbar_wait_cluster(&ctl.part_ready[buf], (g >> 1) & 1);
                tc_fence_after();
                long long t1 = clock64();
                c_tw += t1 - t0;
                const std::uint32_t tacc = tmem + lane_t + buf * TB;
                bool staged = false;
                if (up.gemmonly && JBUFS == 2) {
                    // the walkers are past block g-1 (so they have taken that buffer's previous phase)
                    if (g >= 1) mbar_wait(&ctl.wdone, (g - 1) & 1);
                    const int nb0 = (b + 1 == nb) ? 0 : b0 + TB;
                    issue_jtri(Jtri0 + ((g + 1) & 1) * (SMEM_TRI / 4), a.J32, np, nb0, ht);
                    cp_async_arrive_noinc(&ctl.jready[(g + 1) & 1]);
                }
                for (int t = HT0; !up.gemmonly && t <= nsub + HT0 - 1; ++t) {
                    // target sub-block t (t < nsub); D-event for sub-block t-HT0 (always for
                    // sub-block 0, else only while t < nsub) -- mirrors the walker's arrivals
                    const bool target = t < nsub;
                    if (!target && t - HT0 > 0) break;
#if MARS_HELPER_MMA
                    float f[2][8];
                    if (target) {
#pragma unroll
                        for (int m = 0; m < 2; ++m)
                            tmem_ld_16x256_x2(tmem + (static_cast<std::uint32_t>(q * 32 + 16 * m) << 16) + buf * TB + t * SB, f[m]);
                        if constexpr (SPLIT > 1) {
                            const int gq = lane >> 2, cq = lane & 3;
#pragma unroll
                            for (int pp = 0; pp < SPLIT - 1; ++pp)
#pragma unroll
                                for (int m = 0; m < 2; ++m)
#pragma unroll
                                    for (int pr = 0; pr < 4; ++pr) {
                                        const std::size_t row = row0 + q * 32 + 16 * m + gq + 8 * (pr & 1);
                                        const int col = t * SB + 8 * (pr >> 1) + 2 * cq;
                                        const float2 x = __ldcg(reinterpret_cast<const float2*>(
                                            up.xpart + ((pp * 2 + buf) * xplane + row) * TB + col));
                                        f[m][2 * pr] += x.x;
                                        f[m][2 * pr + 1] += x.y;
                                    }
                        }
                        // Deltas already final: sub-blocks 0 .. t-HT0-1
                        if (!up.nohelp)
                            for (int u = 0; u + HT0 + 1 <= t; ++u) rect_mma(f, tdel, jtri, u, t, jup, lane);
                    }
#else
                    float2 pf[SB / 2];
                    if (target) {
                        float pv[SB];
                        tmem_ld16(tacc + t * SB, pv);
                        add_partials<SPLIT>(pv, up.xpart, xplane, buf, row0 + (q * 32 + lane), t * SB);
#pragma unroll
                        for (int j = 0; j < SB / 2; ++j) pf[j] = make_float2(pv[2 * j] * a.jscale, pv[2 * j + 1] * a.jscale);
                        // Deltas already final: sub-blocks 0 .. t-3
                        for (int u = 0; u + 3 <= t; ++u) {
                            float du[SB];
                            tmem_ld16(tmem + lane_t + DEL_COL + u * SB, du);
                            apply_rect16(pf, jtri, u * SB, t * SB, du);
                        }
                    }
#endif
                    t0 = clock64();
                    c_work += t0 - t1;
                    mbar_wait(&ctl.dready[q][de & 1], (de >> 1) & 1);
                    ++de;
                    tc_fence_after();
                    t1 = clock64();
                    c_dw += t1 - t0;
                    if (JBUFS == 2 && t == HT0 && !staged) {
                        // the walker is past the previous block: stage the next block's triangle
                        const int nb0 = (b + 1 == nb) ? 0 : b0 + TB;
                        issue_jtri(Jtri0 + ((g + 1) & 1) * (SMEM_TRI / 4), a.J32, np, nb0, ht);
                        cp_async_arrive_noinc(&ctl.jready[(g + 1) & 1]);
                        staged = true;
                    }
                    if (!target) break;
#if MARS_HELPER_MMA
                    if (!up.nohelp) rect_mma(f, tdel, jtri, t - HT0, t, jup, lane);
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) f[m][e] *= a.jscale;
                        tmem_st_16x256_x2(tmem + (static_cast<std::uint32_t>(q * 32 + 16 * m) << 16) + buf * TB + t * SB, f[m]);
                    }
#else
                    float du[SB];
                    tmem_ld16(tmem + lane_t + DEL_COL + (t - 2) * SB, du);
                    apply_rect16(pf, jtri, (t - 2) * SB, t * SB, du);
                    float pv[SB];
#pragma unroll
                    for (int j = 0; j < SB / 2; ++j) {
                        pv[2 * j] = pf[j].x;
                        pv[2 * j + 1] = pf[j].y;
                    }
                    tmem_st16f(tacc + t * SB, pv);
#endif
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(&ctl.fready[q][fe & 1]);
                    ++fe;
                    t0 = clock64();
                    c_work += t0 - t1;
                    t1 = t0;
                }
                if (JBUFS == 1) {
                    // the walkers are past this block: stage the next block's triangle over it
                    mbar_wait(&ctl.wdone, g & 1);
                    const int nb0 = (b + 1 == nb) ? 0 : b0 + TB;
                    issue_jtri(Jtri0, a.J32, np, nb0, ht);
                    cp_async_arrive_noinc(&ctl.jready[(g + 1) & 1]);
                }
                if (b == nb - 1) {
                    ++h_sweeps;
                    const bool more = pair_any(ctl, epi_any(false), false, rank, h_sweeps - 1);
                    if (!more) goto helper_done;
                }
            }
        }
    helper_done:
        cp_async_wait_all();
        if (a.prof && ht == 0) {
            long long* pr = a.prof + blockIdx.x * kProfSlots;
            pr[13] = c_dw;
            pr[14] = c_work;
            pr[15] = c_tw;
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();                      // both CTAs done with the pair's TMEM
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, TMEM_COLS);
}

using UmmaKernel = void (*)(RelaxArgs, UmmaParams, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap);

UmmaKernel umma_kernel(int split, bool jlo) {
    return split == 1   ? (jlo ? relax_dense_umma_kernel<true, 1> : relax_dense_umma_kernel<false, 1>)
           : split == 2 ? (jlo ? relax_dense_umma_kernel<true, 2> : relax_dense_umma_kernel<false, 2>)
                        : (jlo ? relax_dense_umma_kernel<true, 4> : relax_dense_umma_kernel<false, 4>);
}

int clamp_split(int split) { return split >= 4 ? 4 : (split >= 2 ? 2 : 1); }

cudaLaunchConfig_t umma_config(int grid, int split, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = SMEM_TOTAL;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;        // split CTA pairs (cta_group::2)
    attr[0].val.clusterDim.x = 2 * split;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

}  // namespace

int relax_dense_umma_slots_per_cta() { return TM; }
int relax_dense_umma_block() { return TB; }
int relax_dense_umma_kc() { return KC; }
int relax_dense_umma_j_rows() { return TBH; }
std::size_t relax_dense_umma_plane_rows(int grid) { return static_cast<std::size_t>(grid) * TM; }

// How many clusters of 2*split CTAs the device keeps resident at once: the persistent grid
// must fit in one wave (a cluster's pairs wait on each other, and on nothing outside it, but
// a cluster left for a second wave would start only after the whole first wave retired).
int relax_dense_umma_max_clusters(int split, bool jlo) {
    split = clamp_split(split);
    UmmaKernel kern = umma_kernel(split, jlo);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL) != cudaSuccess) return -1;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = umma_config(2 * split, split, nullptr, attr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return -1;
    return n;
}

// The host-mapped hang record (umma.cuh) of this translation unit's kernels, allocated once
// per process and pointed to from each device's symbol on first use there; *host receives the
// host view.  Thread-safe: the multi-GPU driver launches from one host thread per device.
cudaError_t relax_dense_umma_hang_log(unsigned long long** host) {
    static std::mutex mu;
    static unsigned long long* h = nullptr;
    static std::uint64_t devs_set = 0;   // bit d: device d's symbol points at h
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (!h) {
        if ((e = cudaHostAlloc(reinterpret_cast<void**>(&h), 8 * sizeof(unsigned long long),
                               cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess) {
            h = nullptr;
            return e;
        }
        for (int i = 0; i < 8; ++i) h[i] = 0;
    }
    if (dev < 64 && !(devs_set >> dev & 1u)) {
        unsigned long long* d = nullptr;
        if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0)) != cudaSuccess) return e;
        if ((e = cudaMemcpyToSymbol(g_hang_log, &d, sizeof(d))) != cudaSuccess) return e;
        if (const char* hs = std::getenv("MARS_HANG_S")) {
            const unsigned long long ns = static_cast<unsigned long long>(std::atof(hs) * 1e9);
            if ((e = cudaMemcpyToSymbol(g_hang_ns, &ns, sizeof(ns))) != cudaSuccess) return e;
        }
        devs_set |= std::uint64_t(1) << dev;
    }
    *host = h;
    return cudaSuccess;
}

cudaError_t launch_relax_dense_umma(const RelaxArgs& a, const UmmaLaunch& u, int grid, cudaStream_t st) {
    unsigned long long* hang = nullptr;
    if (cudaError_t e = relax_dense_umma_hang_log(&hang)) return e;
    const char* pf = std::getenv("MARS_UMMA_PF");
    const char* sp = std::getenv("MARS_UMMA_SPOL");
    const char* jp = std::getenv("MARS_UMMA_JPOL");
    const char* nw = std::getenv("MARS_UMMA_NOWB");
    const char* nh = std::getenv("MARS_UMMA_NOHELP");
    UmmaParams up{u.xpart, u.s_hi, u.s_hi, u.s_lo, a.np / TB, pf ? std::atoi(pf) : 0, sp ? std::atoi(sp) : 2,
                  jp ? std::atoi(jp) : 1, nw ? std::atoi(nw) : 0, nh ? std::atoi(nh) : 0,
                  std::getenv("MARS_UMMA_GEMMONLY") ? std::atoi(std::getenv("MARS_UMMA_GEMMONLY")) : 0};
    const int split = clamp_split(u.split);
    if (a.np % TB != 0 || grid % (2 * split) != 0 || (a.np / KC) % split != 0) return cudaErrorInvalidValue;
    UmmaKernel kern = umma_kernel(split, u.jlo);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = umma_config(grid, split, st, attr);
    return cudaLaunchKernelEx(&cfg, kern, a, up, u.tm_shi, u.tm_slo, u.tm_jhi, u.tm_jlo);
}

}  // namespace marsb200
