// umma.cuh -- thin inline-PTX layer for sm_100a: mbarriers, TMA, tcgen05 (UMMA + TMEM).
//
// Only what the dense relaxation kernel needs, written against the PTX ISA directly:
//   * mbarrier init / arrive / expect_tx / try_wait.parity
//   * cp.async.bulk.tensor.2d (TMA) global -> shared, completing on an mbarrier
//   * tcgen05.alloc / dealloc / relinquish, tcgen05.mma kind::f16 (A, B from shared memory,
//     D in TMEM), tcgen05.commit -> mbarrier, tcgen05.ld 32x32b, tcgen05 fences
//   * UMMA shared-memory descriptors for K-major SWIZZLE_128B tiles (the layout a TMA load
//     with CU_TENSOR_MAP_SWIZZLE_128B produces: 8-row x 128-byte atoms, SBO = 1024 B)
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace marsb200 {
namespace umma {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(std::uint64_t* bar, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Host-mapped record of the first timed-out wait (set per translation unit by its launcher;
// readable by the host after the trap has torn the context down): {1, block, thread, smem
// address, parity, %globaltimer}
static __device__ unsigned long long* g_hang_log = nullptr;
// wait limit (ns); MARS_HANG_S overrides it for the tcgen05 relaxation kernel
static __device__ unsigned long long g_hang_ns = 120000000000ull;

// A pipeline bug must not hang the GPU: a barrier wait longer than 120 s (profiler replays
// are slow) reports the barrier and traps (the launch then fails with an error).

static __device__ __noinline__ void mbar_hang(std::uint64_t* bar, std::uint32_t parity) {
    if (unsigned long long* h = g_hang_log) {
        if (atomicCAS(h, 0ull, 1ull) == 0ull) {
            volatile unsigned long long* v = h;
            std::uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            v[1] = blockIdx.x;
            v[2] = threadIdx.x;
            v[3] = smem_u32(bar);
            v[4] = parity;
            v[5] = t;
            __threadfence_system();
        }
    }
    printf("mars: mbarrier wait timed out (block %d, thread %d, smem 0x%x, parity %u)\n", blockIdx.x, threadIdx.x,
           smem_u32(bar), parity);
    __trap();
}

__device__ __forceinline__ bool hang_check(std::uint64_t& t0, std::uint32_t spin) {
    if ((spin & 1023u) != 0) return false;
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t0 == 0) t0 = t;
    return t - t0 > g_hang_ns;
}

// Wait until the phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    std::uint64_t t0 = 0;
    for (std::uint32_t spin = 1;; ++spin) {
        if (mbar_try_wait(bar, parity)) return;
        if (hang_check(t0, spin)) mbar_hang(bar, parity);
    }
}

// ------------------------------------------------------------------ TMA

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(tmap)) : "memory");
}

// 2D tiled load: box at (c0 = inner/contiguous coordinate, c1 = row) into smem, completing
// `bytes` of transaction count on `bar`.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, std::uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<std::uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// L2 eviction-priority policies for the TMA loads (createpolicy): operands re-read by every
// CTA (the coupling tiles) stay in L2 ahead of per-CTA streams.
__device__ __forceinline__ std::uint64_t policy_evict_last() {
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ std::uint64_t policy_evict_normal() {
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ std::uint64_t policy_evict_first() {
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}

// tma_load_2d with an L2 cache-eviction hint.
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const void* tmap, std::uint64_t* bar,
                                                 int c0, int c1, std::uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<std::uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

// 1D bulk copy global -> shared (TMA engine, no tensor map): `bytes` and both addresses
// multiples of 16; completes `bytes` of transaction count on `bar`.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, std::uint32_t bytes,
                                          std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(reinterpret_cast<std::uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Generic-proxy global writes -> visible to later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05

__device__ __forceinline__ void tmem_alloc(std::uint32_t* dst_smem, std::uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(std::uint32_t taddr, std::uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16/bf16 in, fp32 accumulate), one CTA.
__device__ __forceinline__ void mma_f16_ss(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                           std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread has completed.
__device__ __forceinline__ void mma_commit(std::uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns: thread t of the warp gets TMEM lane
// (base lane + t), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, float (&v)[32]) {
    std::uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// ------------------------------------------------------------------ descriptors

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B canonical layout (8 rows x 128 B
// atoms, SBO = 1024 B between 8-row groups, LBO unused = 1), sm_100 version bit.
// The tile base must be 1024-byte aligned; advancing K by 16 fp16 adds 32 B (>> 4 = 2) to
// the start-address field.
__device__ __forceinline__ std::uint64_t desc_k_sw128(std::uint32_t smem_addr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<std::uint64_t>(1u) << 16;                 // LBO (ignored for SW128 K-major)
    d |= static_cast<std::uint64_t>(1024u >> 4) << 32;         // SBO
    d |= static_cast<std::uint64_t>(1u) << 46;                 // version = 1 (sm_100)
    d |= static_cast<std::uint64_t>(2u) << 61;                 // SWIZZLE_128B
    return d;
}

// K-major SWIZZLE_64B canonical layout (8 rows x 64 B atoms, SBO = 512 B): the layout a TMA
// load with CU_TENSOR_MAP_SWIZZLE_64B and a 32-element fp16 box row produces.  Tile base
// 512-byte aligned; advancing K by 16 fp16 adds 32 B to the start address.
__device__ __forceinline__ std::uint64_t desc_k_sw64(std::uint32_t smem_addr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<std::uint64_t>(1u) << 16;                 // LBO (ignored for swizzled K-major)
    d |= static_cast<std::uint64_t>(512u >> 4) << 32;          // SBO
    d |= static_cast<std::uint64_t>(1u) << 46;                 // version = 1 (sm_100)
    d |= static_cast<std::uint64_t>(4u) << 61;                 // SWIZZLE_64B
    return d;
}

// Instruction descriptor, kind::f16: A/B fp16 (fmt 0) or bf16 (fmt 1), D fp32, both K-major.
__host__ __device__ constexpr std::uint32_t idesc_f16(int M, int N, int ab_format = 0) {
    return (1u << 4)                                   // D format f32
           | (static_cast<std::uint32_t>(ab_format) << 7)   // A format
           | (static_cast<std::uint32_t>(ab_format) << 10)  // B format
           | (static_cast<std::uint32_t>(N >> 3) << 17)     // N >> 3
           | (static_cast<std::uint32_t>(M >> 4) << 24);    // M >> 4
}

}  // namespace umma
}  // namespace marsb200

namespace marsb200 {
namespace umma {

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16.  A (M=128 rows on lanes, K=16 fp16 per
// instruction) occupies 8 consecutive 32-bit TMEM columns, two fp16 per column.
__device__ __forceinline__ void mma_f16_ts(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t bdesc,
                                           std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 lanes x 32 bit x 8 columns store: thread t of the warp writes lane (base + t).
__device__ __forceinline__ void tmem_st8(std::uint32_t taddr, const std::uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_st16(std::uint32_t taddr, const std::uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

}  // namespace umma
}  // namespace marsb200

namespace marsb200 {
namespace umma {

// ---- warp-converged issue: the whole warp executes these, one elected lane issues.  The
// operands are warp-uniform, so they stay in uniform registers and no per-instruction
// "waterfall" loop is generated (a single-lane `if (lane == 0)` issue loop costs ~100+
// instructions per pipeline stage and was measured to bound the GEMM at ~40% of the pipe).

__device__ __forceinline__ void mma_f16_ss_elect(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                                 std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 q, %4, 0;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit_elect(std::uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx_elect(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 st;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_elect(std::uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 st;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_elect(std::uint32_t smem_dst, const void* tmap, std::uint32_t bar,
                                                  int c0, int c1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];\n\t}\n" ::"r"(smem_dst),
        "l"(reinterpret_cast<std::uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_hint_elect(std::uint32_t smem_dst, const void* tmap, std::uint32_t bar,
                                                       int c0, int c1, std::uint64_t policy) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;\n\t}\n" ::"r"(smem_dst),
        "l"(reinterpret_cast<std::uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

}  // namespace umma
}  // namespace marsb200

namespace marsb200 {
namespace umma {

// ---- CTA pair (cluster of 2, cta_group::2): the leader (rank 0) issues M = 256 MMAs whose A
// rows come half from each CTA's shared memory and whose B (N) columns are split between the
// two CTAs' shared memory; each CTA's TMEM holds its own 128 rows of the accumulator.

__device__ __forceinline__ std::uint32_t cluster_ctarank() {
    std::uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// shared::cta address -> the same object's shared::cluster address in CTA `rank`
__device__ __forceinline__ std::uint32_t mapa_shared(std::uint32_t addr, std::uint32_t rank) {
    std::uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(std::uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ void st_cluster_u32(std::uint32_t cluster_addr, std::uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(cluster_addr), "r"(v) : "memory");
}

// monotonic shared-memory counters (cannot alias the way a parity wait on an mbarrier can
// when the signalling side runs two phases ahead)
__device__ __forceinline__ void red_add_release_cta(std::uint32_t* ctr, std::uint32_t v) {
    asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;\n" ::"r"(smem_u32(ctr)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_cluster(std::uint32_t cluster_addr, std::uint32_t v) {
    asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], %1;\n" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_acquire_cluster(const std::uint32_t* ctr) {
    std::uint32_t v;
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(ctr)) : "memory");
    return v;
}

// wait with cluster-scope acquire (data written by the peer CTA before its remote arrive)
__device__ __forceinline__ void mbar_wait_cluster(std::uint64_t* bar, std::uint32_t parity) {
    std::uint32_t ok = 0;
    std::uint64_t t0 = 0;
    for (std::uint32_t spin = 0;; ++spin) {
        if (hang_check(t0, spin)) mbar_hang(bar, parity);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
    }
}

__device__ __forceinline__ void tmem_alloc_pair(std::uint32_t* dst_smem, std::uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc_pair(std::uint32_t taddr, std::uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void mma_f16_ss_pair_elect(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                                      std::uint32_t idesc, std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 q, %4, 0;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// One operand stage of the fp32-accurate split on a CTA pair: for two K steps of 16 (the
// descriptors of the second are the first's + 32 bytes, i.e. +2 in the address field),
// A_hi*J_hi (accumulating unless `accumulate` is 0 on the first), A_lo*J_hi and, with JLO,
// A_hi*J_lo -- all issued by one elected lane under one elect (the per-MMA elect / uniform-
// register broadcast sequence was ~18 instructions per MMA).
template <bool JLO>
__device__ __forceinline__ void mma_stage_split_pair_elect(std::uint32_t d_tmem, std::uint64_t ahi, std::uint64_t alo,
                                                           std::uint64_t jhi, std::uint64_t jlo, std::uint32_t idesc,
                                                           std::uint32_t accumulate) {
    if constexpr (JLO) {
        asm volatile(
            "{\n\t.reg .pred p, q, t;\n\t.reg .b64 a1, l1, h1, g1;\n\t"
            "setp.ne.b32 q, %6, 0;\n\t"
            "setp.eq.b32 t, 0, 0;\n\t"
            "add.s64 a1, %1, 2;\n\t"
            "add.s64 l1, %2, 2;\n\t"
            "add.s64 h1, %3, 2;\n\t"
            "add.s64 g1, %4, 2;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %5, q;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %4, %5, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], a1, h1, %5, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], l1, h1, %5, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], a1, g1, %5, t;\n\t}\n" ::"r"(d_tmem),
            "l"(ahi), "l"(alo), "l"(jhi), "l"(jlo), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p, q, t;\n\t.reg .b64 a1, l1, h1;\n\t"
            "setp.ne.b32 q, %5, 0;\n\t"
            "setp.eq.b32 t, 0, 0;\n\t"
            "add.s64 a1, %1, 2;\n\t"
            "add.s64 l1, %2, 2;\n\t"
            "add.s64 h1, %3, 2;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %4, q;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %4, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], a1, h1, %4, t;\n\t"
            "@p tcgen05.mma.cta_group::2.kind::f16 [%0], l1, h1, %4, t;\n\t}\n" ::"r"(d_tmem),
            "l"(ahi), "l"(alo), "l"(jhi), "r"(idesc), "r"(accumulate)
            : "memory");
        (void)jlo;
    }
}

// commit the pair's MMAs to the barrier at the same offset in both CTAs of pair `pair` of the
// cluster (ranks 2*pair, 2*pair + 1)
__device__ __forceinline__ void mma_commit_pair_mc_elect(std::uint64_t* bar, int pair = 0) {
    const std::uint16_t mask = static_cast<std::uint16_t>(3u << (2 * pair));
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
            smem_u32(bar)), "h"(mask)
        : "memory");
}

// L2 prefetch of a 2D tensor tile (no shared memory, no completion): raises memory-level
// parallelism ahead of the ring (elected lane)
__device__ __forceinline__ void tma_prefetch_2d_elect(const void* tmap, int c0, int c1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n\t}\n" ::"l"(
            reinterpret_cast<std::uint64_t>(tmap)),
        "r"(c0), "r"(c1)
        : "memory");
}

// 2-SM TMA load: into this CTA's shared memory, transaction bytes counted on the LEADER's
// barrier (the peer bit of the barrier address cleared)
__device__ __forceinline__ void tma_load_2d_pair_elect(std::uint32_t smem_dst, const void* tmap, std::uint32_t bar,
                                                       int c0, int c1, std::uint64_t policy) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;\n\t}\n" ::"r"(smem_dst),
        "l"(reinterpret_cast<std::uint64_t>(tmap)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

}  // namespace umma
}  // namespace marsb200
