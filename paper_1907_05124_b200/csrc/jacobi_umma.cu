// jacobi_umma.cu -- NMFA and SimCIM (the paper's synchronous mean-field baselines) on tcgen05.
//
// Replaces, for tiles of 128 runs per CTA (CTA pairs, cta_group::2, M = 256):
//   nmfa_step / nmfa_run     solvers.cpp:374-408   s <- alpha*tanh_trial((h + J s)/norm + noise, t)
//                                                     + (1 - alpha)*s
//   simcim_step / simcim_run solvers.cpp:412-443   x <- clamp(x + step*(pump*x - J x / 2) + noise, -1, 1)
//   schedule_at              solvers.cpp:118-123   (expanded per iteration on the host)
//
// Both are Jacobi updates: every field of an iteration comes from the previous iteration's
// state, so an iteration is one plain GEMM F = S * J over all runs of a tile -- no Gauss-Seidel
// chain -- with the update fused into the GEMM epilogue.  The state is double buffered
// (read buffer k & 1, write buffer (k + 1) & 1) as fp16 hi/lo planes; the field GEMM is the
// same fp32-accurate 3-product split as the MARS kernel (J_hi*S_hi + J_hi*S_lo + J_lo*S_hi,
// J prescaled by a power of two, fp32 accumulation in TMEM).  The noise is the reference's
// per-run stream (mt19937_64 seeded by sub_seed(base, index), Box-Muller with a spare, drawn in
// spin order: mt_device.cuh), so a run's noise sequence is the reference's.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (leader CTA
// of the pair), warps 2..5 epilogue (one run per thread, TMEM lane = run).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "mt_device.cuh"
#include "slot.cuh"
#include "umma.cuh"

namespace marsb200 {
namespace {

using namespace umma;

constexpr int TM = 128;
constexpr int TB = 128;
constexpr int TBH = TB / 2;
constexpr int KC = 32;
constexpr int CPB = TB / KC;
constexpr int STAGES = 8;
constexpr int NT = 192;
constexpr int EPI0 = 2;
constexpr int NE = 128;
constexpr std::uint32_t TILE_A = TM * KC * 2;
constexpr std::uint32_t TILE_J = TBH * KC * 2;
constexpr std::uint32_t STAGE_BYTES = 2 * TILE_A + 2 * TILE_J;
constexpr std::uint32_t TMEM_COLS = 256;

struct __align__(8) Ctl {
    std::uint64_t full[STAGES];
    std::uint64_t empty[STAGES];
    std::uint64_t tmem_full[2];
    std::uint64_t tmem_empty[2];
    std::uint64_t iter_ready;       // an iteration's state fully written (or a tile initialised)
    std::uint64_t mma_done;
    std::uint64_t pair_more[2];
    std::uint32_t peer_more[2];
    std::uint32_t more_all;
    std::uint32_t tmem_base;
    volatile std::uint32_t stop;
    volatile std::uint32_t poison;
};
constexpr std::uint32_t SMEM_TOTAL = STAGES * STAGE_BYTES + sizeof(Ctl);
static_assert(SMEM_TOTAL <= 232448, "shared memory budget");

__device__ __forceinline__ bool epi_any(bool v) {
    std::uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "barrier.cta.red.or.pred q, 1, 128, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}\n"
        : "=r"(r)
        : "r"(static_cast<std::uint32_t>(v))
        : "memory");
    return r != 0;
}

// the pair agrees on whether either CTA still has a tile (one epilogue thread exchanges)
__device__ __forceinline__ bool pair_any(Ctl& ctl, bool local, bool lead, std::uint32_t rank, long long round) {
    const std::uint32_t par = static_cast<std::uint32_t>(round) & 1u;
    if (lead) {
        const std::uint32_t peer = rank ^ 1u;
        st_cluster_u32(mapa_shared(smem_u32(&ctl.peer_more[par]), peer), local ? 1u : 0u);
        mbar_arrive_cluster(mapa_shared(smem_u32(&ctl.pair_more[par]), peer));
        mbar_wait_cluster(&ctl.pair_more[par], (static_cast<std::uint32_t>(round) >> 1) & 1u);
        ctl.more_all = (local || ctl.peer_more[par] != 0) ? 1u : 0u;
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");
    return ctl.more_all != 0;
}

__device__ __forceinline__ void split16(float v, __half& hi, __half& lo) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
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

template <bool JLO>
__global__ void __launch_bounds__(NT, 1)
jacobi_umma_kernel(JacobiArgs a, const __grid_constant__ CUtensorMap tm_s0hi, const __grid_constant__ CUtensorMap tm_s0lo,
                   const __grid_constant__ CUtensorMap tm_s1hi, const __grid_constant__ CUtensorMap tm_s1lo,
                   const __grid_constant__ CUtensorMap tm_jhi, const __grid_constant__ CUtensorMap tm_jlo) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw;
    Ctl& ctl = *reinterpret_cast<Ctl*>(base + STAGES * STAGE_BYTES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int np = a.np, n = a.n, nb = np / TB, nk = np / KC;
    const int row0 = blockIdx.x * TM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&ctl.full[s], 1);
            mbar_init(&ctl.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ctl.tmem_full[s], 1);
            mbar_init(&ctl.tmem_empty[s], 2 * NE);
            mbar_init(&ctl.pair_more[s], 1);
        }
        mbar_init(&ctl.iter_ready, NE);
        mbar_init(&ctl.mma_done, 1);
        ctl.stop = 0;
        ctl.poison = 0;
        fence_mbar_init();
    }
    const std::uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    cluster_sync_all();
    if (warp == 1) tmem_alloc_pair(&ctl.tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = ctl.tmem_base;

    if (warp == 0) {
        // ================================================================ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_s0hi);
            tma_prefetch_desc(&tm_s1hi);
            tma_prefetch_desc(&tm_jhi);
        }
        __syncwarp();
        const std::uint64_t jpol = policy_evict_last();
        const std::uint64_t spol = policy_evict_normal();
        const std::uint32_t smem0 = smem_u32(base);
        const std::uint32_t full0 = smem_u32(&ctl.full[0]);
        const std::uint32_t tx = 2 * (JLO ? STAGE_BYTES : STAGE_BYTES - TILE_J);
        std::uint32_t s = 0, ph = 0, ir = 0;
        for (;;) {                                         // tiles
            for (int k = 0; k < a.iters; ++k) {
                // the state read this iteration (tile initialisation or the previous
                // iteration's update) is fully written
                mbar_wait(&ctl.iter_ready, ir & 1);
                ++ir;
                if (k == 0 && ctl.stop) {
                    mbar_wait(&ctl.empty[s], ph ^ 1);
                    if (lane == 0 && leader) {
                        ctl.poison = 1;
                        mbar_arrive(&ctl.full[s]);
                    }
                    goto producer_done;
                }
                const CUtensorMap* thi = (k & 1) ? &tm_s1hi : &tm_s0hi;
                const CUtensorMap* tlo = (k & 1) ? &tm_s1lo : &tm_s0lo;
                for (int b = 0; b < nb; ++b) {
                    for (int c = 0; c < nk; ++c) {
                        mbar_wait(&ctl.empty[s], ph ^ 1);
                        const std::uint32_t st = smem0 + s * STAGE_BYTES;
                        const std::uint32_t fb = full0 + s * 8;
                        if (leader) mbar_arrive_expect_tx_elect(&ctl.full[s], tx);
                        tma_load_2d_pair_elect(st, thi, fb, c * KC, row0, spol);
                        tma_load_2d_pair_elect(st + TILE_A, tlo, fb, c * KC, row0, spol);
                        tma_load_2d_pair_elect(st + 2 * TILE_A, &tm_jhi, fb, c * KC, b * TB + rank * TBH, jpol);
                        if (JLO) tma_load_2d_pair_elect(st + 2 * TILE_A + TILE_J, &tm_jlo, fb, c * KC, b * TB + rank * TBH, jpol);
                        if (++s == STAGES) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
            // the tile's last iteration written: the next tile may re-initialise the state
            mbar_wait(&ctl.iter_ready, ir & 1);
            ++ir;
        }
    producer_done:;
    } else if (warp == 1) {
        // ================================================================ MMA issuer (leader)
        if (!leader) goto mma_skip;
        {
            constexpr std::uint32_t idesc = idesc_f16(2 * TM, TB, 0);
            const std::uint32_t smem0 = smem_u32(base);
            std::uint32_t g = 0, s = 0, ph = 0;
            for (;;) {
                for (int k = 0; k < a.iters; ++k) {
                    for (int b = 0; b < nb; ++b, ++g) {
                        const int buf = g & 1;
                        mbar_wait(&ctl.tmem_empty[buf], ((g >> 1) & 1) ^ 1);
                        tc_fence_after();
                        const std::uint32_t d = tmem + buf * TB;
                        for (int c = 0; c < nk; ++c) {
                            mbar_wait(&ctl.full[s], ph);
                            if (k == 0 && b == 0 && c == 0 && ctl.poison) goto mma_done;
                            tc_fence_after();
                            const std::uint32_t st = smem0 + s * STAGE_BYTES;
#pragma unroll
                            for (int kk = 0; kk < KC / 16; ++kk) {
                                const std::uint64_t ahi = desc_k_sw64(st + kk * 32);
                                const std::uint64_t alo = desc_k_sw64(st + TILE_A + kk * 32);
                                const std::uint64_t jhi = desc_k_sw64(st + 2 * TILE_A + kk * 32);
                                mma_f16_ss_pair_elect(d, ahi, jhi, idesc, (c | kk) != 0);
                                mma_f16_ss_pair_elect(d, alo, jhi, idesc, 1);
                                if (JLO) {
                                    const std::uint64_t jlo = desc_k_sw64(st + 2 * TILE_A + TILE_J + kk * 32);
                                    mma_f16_ss_pair_elect(d, ahi, jlo, idesc, 1);
                                }
                            }
                            mma_commit_pair_mc_elect(&ctl.empty[s]);
                            if (++s == STAGES) {
                                s = 0;
                                ph ^= 1;
                            }
                        }
                        mma_commit_pair_mc_elect(&ctl.tmem_full[buf]);
                    }
                }
            }
        mma_done:
            mma_commit_pair_mc_elect(&ctl.mma_done);
            mbar_wait(&ctl.mma_done, 0);
        }
    mma_skip:
        __syncwarp();
    } else {
        // ================================================================ epilogue
        const int q = warp & 3;
        const int r = q * 32 + lane;                       // slot = TMEM lane
        const int et = threadIdx.x - EPI0 * 32;
        const std::uint32_t lane_t = static_cast<std::uint32_t>(q * 32) << 16;
        const std::uint32_t tmem_empty_leader = mapa_shared(smem_u32(&ctl.tmem_empty[0]), 0);
        const size_t row = static_cast<size_t>(row0 + r) * np;
        DevStream rng;
        rng.st = a.mt + (row0 + r);
        rng.stride = a.slots;
        std::uint32_t g = 0;
        long long round = 0;
        for (;; ++round) {
            const int run = claim_run(a.queue_head, a.queue_len, a.order);
            if (!pair_any(ctl, epi_any(run >= 0), et == 0, rank, round)) {
                if (et == 0) ctl.stop = 1;
                fence_proxy_async_global();
                mbar_arrive(&ctl.iter_ready);
                break;
            }
            // tile start: state buffer 0 = 0 (nmfa_run / simcim_run start from zeros)
            __half* w_hi = a.s_hi[0] + row;
            __half* w_lo = a.s_lo[0] + row;
            for (int v = 0; v < np / 8; ++v) {
                *reinterpret_cast<uint4*>(w_hi + 8 * v) = make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(w_lo + 8 * v) = make_uint4(0, 0, 0, 0);
            }
            if (run >= 0) rng.seed(a.seeds[run]);
            const unsigned long long t_start = global_ns();
            fence_proxy_async_global();
            mbar_arrive(&ctl.iter_ready);
            for (int k = 0; k < a.iters; ++k) {
                const double sched = a.sched[k];                // temperature (NMFA) / pump (SimCIM)
                const float tf = static_cast<float>(sched);
                const bool quench = sched < kTempFloor;
                const float rT = quench ? 0.0f : recip_for_div(tf);
                const float pump = tf;
                const __half* r_hi = a.s_hi[k & 1] + row;
                const __half* r_lo = a.s_lo[k & 1] + row;
                __half* o_hi = a.s_hi[(k + 1) & 1] + row;
                __half* o_lo = a.s_lo[(k + 1) & 1] + row;
                const bool last = k + 1 == a.iters;
                for (int b = 0; b < nb; ++b, ++g) {
                    const int buf = g & 1;
                    mbar_wait(&ctl.tmem_full[buf], (g >> 1) & 1);
                    tc_fence_after();
                    for (int cc = 0; cc < TB / 16; ++cc) {
                        const int j0 = b * TB + cc * 16;
                        float f[16];
                        tmem_ld16(tmem + lane_t + buf * TB + cc * 16, f);
                        uint4 hv[2], lv[2];
                        const uint4 oh0 = *reinterpret_cast<const uint4*>(r_hi + j0);
                        const uint4 oh1 = *reinterpret_cast<const uint4*>(r_hi + j0 + 8);
                        const uint4 ol0 = *reinterpret_cast<const uint4*>(r_lo + j0);
                        const uint4 ol1 = *reinterpret_cast<const uint4*>(r_lo + j0 + 8);
                        const __half* ohp[2] = {reinterpret_cast<const __half*>(&oh0), reinterpret_cast<const __half*>(&oh1)};
                        const __half* olp[2] = {reinterpret_cast<const __half*>(&ol0), reinterpret_cast<const __half*>(&ol1)};
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int j = j0 + i;
                            const float s_old = __half2float(ohp[i >> 3][i & 7]) + __half2float(olp[i >> 3][i & 7]);
                            float s_new = 0.0f;
                            if (j < n && run >= 0) {
                                const float field = f[i] * a.jscale;          // J * s (J prescaled by 2^k)
                                if (a.solver == 0) {
                                    // nmfa_step (solvers.cpp:374-390)
                                    const float raw = field + (a.h32 ? a.h32[j] : 0.0f);
                                    const float nrm = a.norm[j];
                                    float phi = nrm > 0.0f ? __fdiv_rn(raw, nrm) : 0.0f;
                                    if (a.noise_sigma > 0.0)
                                        phi = static_cast<float>(static_cast<double>(phi) + a.noise_sigma * rng.gaussian());
                                    const float trial = tanh_trial_r(phi, tf, rT, quench);
                                    s_new = a.alpha_f * trial + a.one_minus_alpha_f * s_old;
                                } else {
                                    // simcim_step (solvers.cpp:412-424)
                                    const float grad = -0.5f * field;
                                    double next = static_cast<double>(s_old + a.step_f * (pump * s_old + grad));
                                    if (a.noise_sigma > 0.0) next += a.noise_sigma * rng.gaussian();
                                    s_new = static_cast<float>(fmin(fmax(next, -1.0), 1.0));
                                }
                            }
                            split16(s_new, reinterpret_cast<__half*>(&hv[i >> 3])[i & 7],
                                    reinterpret_cast<__half*>(&lv[i >> 3])[i & 7]);
                            if (last && run >= 0 && j < n) {
                                const float sv = __half2float(reinterpret_cast<__half*>(&hv[i >> 3])[i & 7]) +
                                                 __half2float(reinterpret_cast<__half*>(&lv[i >> 3])[i & 7]);
                                a.spins[static_cast<size_t>(run) * n + j] = sv < 0.0f ? -1 : 1;   // round_spins
                                if (a.state_out) a.state_out[static_cast<size_t>(run) * n + j] = sv;
                            }
                        }
                        *reinterpret_cast<uint4*>(o_hi + j0) = hv[0];
                        *reinterpret_cast<uint4*>(o_hi + j0 + 8) = hv[1];
                        *reinterpret_cast<uint4*>(o_lo + j0) = lv[0];
                        *reinterpret_cast<uint4*>(o_lo + j0 + 8) = lv[1];
                    }
                    tc_fence_before();
                    mbar_arrive_cluster(tmem_empty_leader + buf * 8);
                }
                fence_proxy_async_global();
                mbar_arrive(&ctl.iter_ready);
            }
            if (run >= 0) {
                const unsigned long long now = global_ns();
                a.status[run] = 0;
                a.iters_out[run] = a.iters;
                a.elapsed[run] = 1e-9 * static_cast<double>(now - t_start);
                if (a.done_ns) a.done_ns[run] = now;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, TMEM_COLS);
}

// TEST-ONLY: one device stream per thread -> its first `count` engine outputs and gaussians
__global__ void rng_probe_kernel(const std::uint64_t* seeds, int streams, int count, std::uint64_t* st,
                                 std::uint64_t* u64, double* gauss) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= streams) return;
    DevStream a{st + t, streams, 0, false, 0.0}, b{st + static_cast<size_t>(kMtN) * streams + t, streams, 0, false, 0.0};
    a.seed(seeds[t]);
    b.seed(seeds[t]);
    for (int k = 0; k < count; ++k) {
        u64[static_cast<size_t>(t) * count + k] = a.next();
        gauss[static_cast<size_t>(t) * count + k] = b.gaussian();
    }
}

}  // namespace

cudaError_t launch_rng_probe(const std::uint64_t* seeds, int streams, int count, std::uint64_t* st, std::uint64_t* u64,
                             double* gauss, cudaStream_t s) {
    rng_probe_kernel<<<(streams + 63) / 64, 64, 0, s>>>(seeds, streams, count, st, u64, gauss);
    return cudaGetLastError();
}

int jacobi_umma_slots_per_cta() { return TM; }
int jacobi_umma_kc() { return KC; }   // its operand maps' box width (independent of the relaxation kernel's)

cudaError_t launch_jacobi_umma(const JacobiArgs& a, const JacobiLaunch& l, int grid, cudaStream_t st) {
    if (a.np % TB != 0 || grid % 2 != 0) return cudaErrorInvalidValue;
    void (*kern)(JacobiArgs, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap) =
        l.jlo ? jacobi_umma_kernel<true> : jacobi_umma_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = SMEM_TOTAL;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, l.tm_s[0][0], l.tm_s[0][1], l.tm_s[1][0], l.tm_s[1][1], l.tm_jhi,
                              l.tm_jlo);
}

}  // namespace marsb200
