// mars_host.cpp -- C-ABI implementation (include/mars_b200.h): the coupling store, the
// host-side plan, the staged batch driver and the reference's index-order aggregation.
//
// Host responsibilities mirror the reference's non-kernel code:
//   validate / run_count / run_plan     solvers.cpp:35-52, 202-227
//   IsingProblem construction+metadata  model.cpp:20-131
//   run_batch / run_batch_with          runner.cpp:81-178 (aggregation 126-167)
// The per-run work itself (descents, energies, best-of-R) runs in the sm_100a kernels.
#include <atomic>
#include <mutex>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <thread>
#include <utility>
#include <queue>
#include <vector>

#include "../../include/mars_b200.h"
#include "kernels.cuh"
#include "host_internal.hpp"
#include "rng.hpp"
#include "tma_host.hpp"

using namespace marsb200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// an asynchronous kernel fault surfaces at whichever call comes next: the tcgen05 kernel's
// hang-detector record (if it fired) is appended to the message
#define CUDA_TRY(expr)                                                                                  \
    do {                                                                                                \
        const cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                          \
            return fail(MARS_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_) +               \
                                           (e_ == cudaErrorLaunchFailure ? ::marsb200::hang_note() : "")); \
    } while (0)

constexpr double kSparseDensityThreshold = 0.05;      // model.hpp:31
constexpr std::uint64_t kStartTempTag = 0x74656d7073746172ull;  // solvers.cpp:23

bool is_integral_value(double v) { return std::nearbyint(v) == v && std::isfinite(v); }

int round_up(int x, int m) { return (x + m - 1) / m * m; }

int host_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(hc, 64u)));
}

template <class F>
void parallel_for(std::int64_t count, F&& f) {
    const int nt = static_cast<int>(std::min<std::int64_t>(host_threads(), std::max<std::int64_t>(count / 64, 1)));
    if (nt <= 1) {
        f(0, count);
        return;
    }
    std::vector<std::thread> th;
    const std::int64_t chunk = (count + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const std::int64_t lo = t * chunk, hi = std::min(count, lo + chunk);
        if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto& x : th) x.join();
}

// solvers.cpp:35-41
int check_params(const mars_params_t* p) {
    if (!p) return fail(MARS_ERR_INPUT, "mars: null parameters");
    if (!(p->t_min >= 0.0)) return fail(MARS_ERR_INPUT, "mars: t_min must be >= 0");
    if (!(p->t_max > p->t_min)) return fail(MARS_ERR_INPUT, "mars: t_max must exceed t_min");
    if (!(p->t_step > 0.0)) return fail(MARS_ERR_INPUT, "mars: t_step must be positive");
    if (!(p->c_step > 0.0)) return fail(MARS_ERR_INPUT, "mars: c_step must be positive");
    if (!(p->d_min > 0.0)) return fail(MARS_ERR_INPUT, "mars: d_min must be positive");
    if (p->start_mode != MARS_GRID_SWEEP && p->start_mode != MARS_UNIFORM_RANDOM)
        return fail(MARS_ERR_INPUT, "mars: unknown start mode");
    if (p->sweep_cap < 0) return fail(MARS_ERR_INPUT, "mars: sweep_cap must be >= 0");
    return MARS_OK;
}

// solvers.cpp:215-227 (GridSweep slot k at t_min + k*t_step; UniformRandom via the tagged stream)
void plan_of(const mars_params_t* prm, std::uint64_t base, std::int64_t idx, bool* skipped,
             double* t, std::uint64_t* seed) {
    *seed = sub_seed(base, static_cast<std::uint64_t>(idx));
    if (prm->start_mode == MARS_GRID_SWEEP) {
        *t = prm->t_min + static_cast<double>(idx) * prm->t_step;
        *skipped = !(*t > 0.0);
    } else {
        Stream r(splitmix64(*seed ^ kStartTempTag));
        *t = prm->t_min + r.open01() * (prm->t_max - prm->t_min);
        *skipped = false;
    }
}

}  // namespace

// ============================================================================ problem store

struct mars_problem {
    // staged batches borrow this problem's stream and buffer pool: one reference for the handle
    // and one per live batch; whichever of mars_problem_destroy / mars_batch_destroy drops the
    // last reference frees the problem (a single atomic count: no double delete)
    std::atomic<int> refs{1};
    std::mutex pool_mu;             // the buffer pool is shared by concurrent batches
    int n = 0;
    bool dense = true;              // storage choice of the reference (model.cpp:91)
    bool integral = true;
    bool has_field = false;
    double coupling_sum = 0.0;
    std::int64_t nnz = 0;
    int device = 0;
    int kernel = MARS_KERNEL_DENSE_SIMT;
    int np = 0;                     // padded size for the dense kernels
    int num_sms = 148;
    std::vector<double> J;          // dense row-major (dense storage)
    std::vector<int> off, idx;      // CSR (adjacency storage)
    std::vector<double> wt;
    std::vector<double> h;
    cudaStream_t stream = nullptr;
    // device copies
    float* dJ32 = nullptr;          // [np][np] fp32, zero padded (dense kernels)
    double* dJ64 = nullptr;         // [n][n]   fp64 (exact energy, dense storage)
    int* dOff = nullptr;            // CSR of the reference storage (exact energy)
    int* dIdx = nullptr;
    double* dW64 = nullptr;
    // level-scheduled sparse relaxation layout (relax_csr.cu), built from the sorted nonzeros
    int nlev = 0, nchunks = 0, max_level_chunks = 0, cw = 32;
    bool unit = false;              // every |J_ij| == 1
    // torus stencil layout (relax_stencil.cu), when the adjacency is an L^dims +-1 torus
    bool stencil = false;
    int st_dims = 0, st_L = 0, st_nlev = 0, st_maxw = 0;
    int* dStLvl = nullptr;
    unsigned* dStCoords = nullptr;
    unsigned buf_bytes = 0, wbuf_off = 0;
    std::size_t chunk_bytes = 0;    // all chunk blocks (+ weights), bytes
    int* dLvlChunk = nullptr;
    int4* dCtab = nullptr;
    int* dBlk = nullptr;
    double* dWblk = nullptr;
    float* dH32 = nullptr;
    double* dH64 = nullptr;
    __half* dJhi = nullptr;         // [np][np] fp16 split of J * 2^jexp (tcgen05 kernels)
    __half* dJlo = nullptr;
    bool jlo = true;                // J_lo nonzero somewhere (non-integer couplings)
    int jexp = 0;                   // power-of-two prescale of the fp16 planes
    int np16 = 0;                   // padded size of the fp16 planes (multiple of 128)
    CUtensorMap tm_jhi{}, tm_jlo{};          // relaxation kernel's boxes (relax_dense_umma_kc() wide)
    CUtensorMap tm_jhi_j{}, tm_jlo_j{};      // the Jacobi kernel's (jacobi_umma_kc() wide)
    float* dNorm = nullptr;         // NMFA normalisers (lazily, fp32 [np16])
    // Buffer pool for the batches run on this problem: repeated run_batch calls reuse their
    // pinned host and device allocations (a 65536 x 2000 fp64 plan is 1 GB pinned) instead of
    // allocating and freeing them every call.
    struct PoolBuf {
        void* ptr;
        std::size_t bytes;
        bool pinned;
    };
    std::vector<PoolBuf> pool;

    void* take(std::size_t bytes, bool pinned) {
        std::lock_guard<std::mutex> lk(pool_mu);
        bytes = std::max<std::size_t>(bytes, 16);
        for (std::size_t k = 0; k < pool.size(); ++k)
            if (pool[k].pinned == pinned && pool[k].bytes >= bytes && pool[k].bytes <= 2 * bytes + 4096) {
                void* ptr = pool[k].ptr;
                pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(k));
                return ptr;
            }
        // no pooled block fits: release the idle blocks of this kind first, so a problem that
        // runs batches of changing sizes keeps one batch's worth of memory, not every size seen
        for (std::size_t k = pool.size(); k-- > 0;)
            if (pool[k].pinned == pinned) {
                void* q = pool[k].ptr;
                if (pinned) cudaFreeHost(q);
                else cudaFree(q);
                for (std::size_t z = 0; z < sizes.size(); ++z)
                    if (sizes[z].first == q) {
                        sizes.erase(sizes.begin() + static_cast<std::ptrdiff_t>(z));
                        break;
                    }
                pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(k));
            }
        void* ptr = nullptr;
        if ((pinned ? cudaMallocHost(&ptr, bytes) : cudaMalloc(&ptr, bytes)) != cudaSuccess) return nullptr;
        sizes.emplace_back(ptr, bytes);
        return ptr;
    }
    void give(void* ptr, bool pinned) {
        if (!ptr) return;
        std::lock_guard<std::mutex> lk(pool_mu);
        for (const auto& sz : sizes)
            if (sz.first == ptr) {
                pool.push_back({ptr, sz.second, pinned});
                return;
            }
    }
    std::vector<std::pair<void*, std::size_t>> sizes;   // every block this pool allocated

    ~mars_problem() {
        cudaSetDevice(device);
        for (const auto& b : pool) {
            if (b.pinned) cudaFreeHost(b.ptr);
            else cudaFree(b.ptr);
        }
        cudaFree(dJhi);
        cudaFree(dJlo);
        cudaFree(dNorm);
        cudaSetDevice(device);
        cudaFree(dJ32);
        cudaFree(dJ64);
        cudaFree(dOff);
        cudaFree(dIdx);
        cudaFree(dW64);
        cudaFree(dStLvl);
        cudaFree(dStCoords);
        cudaFree(dLvlChunk);
        cudaFree(dCtab);
        cudaFree(dBlk);
        cudaFree(dWblk);
        cudaFree(dH32);
        cudaFree(dH64);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

// model.cpp:20-45 -- metadata in storage order
void finalize_metadata(mars_problem* p) {
    p->coupling_sum = 0.0;
    p->nnz = 0;
    p->integral = true;
    if (p->dense) {
        for (std::size_t k = 0; k < p->J.size(); ++k) {
            const double w = p->J[k];
            p->coupling_sum += w;
            if (w != 0.0) ++p->nnz;
            if (p->integral && !is_integral_value(w)) p->integral = false;
        }
    } else {
        for (double w : p->wt) {
            p->coupling_sum += w;
            ++p->nnz;
            if (p->integral && !is_integral_value(w)) p->integral = false;
        }
    }
    p->has_field = false;
    for (double v : p->h) {
        if (v != 0.0) p->has_field = true;
        if (p->integral && !is_integral_value(v)) p->integral = false;
    }
}

template <class T>
int upload(T** dst, const T* src, std::size_t count) {
    CUDA_TRY(cudaMalloc(dst, std::max<std::size_t>(count, 1) * sizeof(T)));
    if (count) CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return MARS_OK;
}

// Instances whose nonzero density is below this run on the fp64 CSR kernel even when the
// reference stores them dense (e.g. the G1-shape 6% graph): its summation over the sorted
// nonzeros is bit-identical to the dense row_dot (zeros add nothing), and it is cheaper.
constexpr double kCsrDensity = 0.10;

int resolve_kernel(mars_problem* p, int requested) {
    if (requested == MARS_KERNEL_AUTO) {
        const double density = static_cast<double>(p->nnz) / (static_cast<double>(p->n) * p->n);
        return (!p->dense || density < kCsrDensity) ? MARS_KERNEL_CSR : MARS_KERNEL_DENSE_UMMA;
    }
    if (requested == MARS_KERNEL_DENSE_SIMT || requested == MARS_KERNEL_CSR ||
        requested == MARS_KERNEL_DENSE_UMMA)
        return requested;
    return -1;
}

// Torus recognition for the stencil kernel: n = L^dims (dims 2 or 3, 3 <= L <= 256), every
// coupling +-1, and every adjacency row exactly the 2*dims lattice neighbours of the site
// (site i = c0 + L*c1 + L^2*c2, bonds to c_d +- 1 mod L) in ascending order.  Builds the
// level lists (coordinate sums) and one sign byte per site (bit k: k-th row entry is -1).
int try_stencil(mars_problem* p, const std::vector<int>& off, const std::vector<int>& idx,
                const std::vector<double>& w) {
    const int n = p->n;
    for (int dims = 2; dims <= 3; ++dims) {
        const int L = static_cast<int>(std::lround(std::pow(static_cast<double>(n), 1.0 / dims)));
        std::int64_t nn = 1;
        for (int d = 0; d < dims; ++d) nn *= L;
        if (nn != n || L < 3 || L > 256) continue;
        std::vector<unsigned char> signs(n, 0);
        bool ok = true;
        for (int i = 0; i < n && ok; ++i) {
            if (off[i + 1] - off[i] != 2 * dims) { ok = false; break; }
            int nb[6], stride = 1;
            for (int d = 0; d < dims; ++d) {
                const int c = (i / stride) % L;
                nb[2 * d] = c ? i - stride : i + (L - 1) * stride;
                nb[2 * d + 1] = c < L - 1 ? i + stride : i - (L - 1) * stride;
                stride *= L;
            }
            std::sort(nb, nb + 2 * dims);
            for (int k = 0; k < 2 * dims; ++k) {
                const int e = off[i] + k;
                if (idx[e] != nb[k] || (w[e] != 1.0 && w[e] != -1.0)) { ok = false; break; }
                if (w[e] < 0.0) signs[i] |= static_cast<unsigned char>(1u << k);
            }
        }
        if (!ok) continue;
        const int nlev = dims * (L - 1) + 1;
        std::vector<std::vector<unsigned>> lv(nlev);
        for (int i = 0; i < n; ++i) {
            int c[3] = {0, 0, 0}, stride = 1, sum = 0;
            for (int d = 0; d < dims; ++d) {
                c[d] = (i / stride) % L;
                sum += c[d];
                stride *= L;
            }
            lv[sum].push_back(static_cast<unsigned>(c[0]) | static_cast<unsigned>(c[1]) << 8 |
                              static_cast<unsigned>(c[2]) << 16 | static_cast<unsigned>(signs[i]) << 24);
        }
        std::vector<int> lvl_off{0};
        std::vector<unsigned> coords;
        int maxw = 0;
        for (const auto& l : lv) {
            coords.insert(coords.end(), l.begin(), l.end());
            lvl_off.push_back(static_cast<int>(coords.size()));
            maxw = std::max(maxw, static_cast<int>(l.size()));
        }
        if (int rc = upload(&p->dStLvl, lvl_off.data(), lvl_off.size())) return rc;
        if (int rc = upload(&p->dStCoords, coords.data(), coords.size())) return rc;
        p->stencil = true;
        p->st_dims = dims;
        p->st_L = L;
        p->st_nlev = nlev;
        p->st_maxw = maxw;
        return MARS_OK;
    }
    return MARS_OK;
}

// Gauss-Seidel levels of the ascending sweep (relax_csr.cu): level(i) = 1 + max level of
// the lower neighbours.  Each level is cut into 32-spin chunks; chunk c's neighbour lists are
// stored interleaved, entry k of lane l at chunk_base[c] + 32k + l, padded to the chunk's
// longest list with the +0.0 slot n (weight 0.0).
int build_levels(mars_problem* p, const std::vector<int>& off, const std::vector<int>& idx,
                 const std::vector<double>& w) {
    const int n = p->n;
    p->np = n + 1;
    std::vector<int> level(n, 0);
    int nlev = 1;
    p->unit = true;
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int k = off[i]; k < off[i + 1]; ++k) {
            if (idx[k] < i) l = std::max(l, level[idx[k]] + 1);
            if (w[k] != 1.0 && w[k] != -1.0) p->unit = false;
        }
        level[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<std::vector<int>> by_level(nlev);
    for (int i = 0; i < n; ++i) by_level[level[i]].push_back(i);
    // within a level the order is free (no couplings): group similar degrees so a chunk's
    // lanes pad less to its longest list
    for (auto& m : by_level)
        std::stable_sort(m.begin(), m.end(), [&](int x, int y) { return off[x + 1] - off[x] > off[y + 1] - off[y]; });
    // chunk width.  Warp-per-run kernel (state small enough for >= 4 runs per SM): 16 for
    // narrow levels (two runs per warp), 64 for wide ones (two spins per lane), else 32.
    // Level-parallel kernel: 16 when 32-wide chunks would leave most lanes idle, else 32.
    std::size_t chunks32 = 0, chunks16 = 0;
    for (const auto& m : by_level) {
        chunks32 += (m.size() + 31) / 32;
        chunks16 += (m.size() + 15) / 16;
    }
    const char* kern = std::getenv("MARS_SPARSE_KERNEL");
    const bool spmm_layout = !(kern && std::string(kern) == "levels") &&
                             (static_cast<std::size_t>(n) + 1) * sizeof(double) * 4 <= 180 * 1024;
    const double per_level = static_cast<double>(n) / nlev;
    int cw = static_cast<double>(n) / (32.0 * chunks32) < 0.5 && chunks16 < 2 * chunks32 ? 16 : 32;
    if (spmm_layout) cw = per_level < 20 ? 16 : 32;   // 64 (two spins per lane) measured slower
    if (const char* v = std::getenv("MARS_SPARSE_CW")) {
        const int want = std::atoi(v);
        cw = want == 16 ? 16 : (want == 64 && spmm_layout ? 64 : 32);
    }
    p->cw = cw;
    // chunk blocks [md,0,0,0][spin x cw][idx: md x cw] (+ weights [md x cw] when non-unit)
    std::vector<int> lvl_chunk{0}, blk;
    std::vector<int4> ctab;
    std::vector<double> wblk;
    int max_chunks = 0, max_md = 0;
    std::size_t max_blen = 0;
    std::vector<int> lanes(cw);
    for (const auto& members : by_level) {
        const int chunks = static_cast<int>((members.size() + cw - 1) / cw);
        max_chunks = std::max(max_chunks, chunks);
        for (int c = 0; c < chunks; ++c) {
            int md = 0;
            for (int l = 0; l < cw; ++l) {
                const std::size_t m = static_cast<std::size_t>(c) * cw + l;
                lanes[l] = m < members.size() ? members[m] : -1;
                if (lanes[l] >= 0) md = std::max(md, off[lanes[l] + 1] - off[lanes[l]]);
            }
            md = (md + 3) / 4 * 4;   // the warp-per-run kernel gathers in groups of 4
            const std::size_t boff = blk.size(), woff = wblk.size();
            blk.insert(blk.end(), {md, 0, 0, 0});
            blk.insert(blk.end(), lanes.begin(), lanes.end());
            for (int k = 0; k < md; ++k)
                for (int l = 0; l < cw; ++l) {
                    const int sp = lanes[l];
                    const bool real = sp >= 0 && k < off[sp + 1] - off[sp];
                    const int e = real ? off[sp] + k : -1;
                    int code = real ? idx[e] : n;
                    if (p->unit && real && w[e] < 0.0) code |= static_cast<int>(0x80000000u);
                    blk.push_back(code);
                    if (!p->unit) wblk.push_back(real ? w[e] : 0.0);
                }
            const std::size_t blen = blk.size() - boff;
            if (blk.size() > 0x7fffffffu || wblk.size() > 0x7fffffffu)
                return fail(MARS_ERR_INPUT, "sparse layout exceeds 2^31 entries");
            ctab.push_back(make_int4(static_cast<int>(boff), static_cast<int>(blen), static_cast<int>(woff), md));
            max_blen = std::max(max_blen, blen);
            max_md = std::max(max_md, md);
        }
        lvl_chunk.push_back(static_cast<int>(ctab.size()));
    }
    p->nlev = nlev;
    p->nchunks = static_cast<int>(ctab.size());
    p->max_level_chunks = max_chunks;
    p->chunk_bytes = blk.size() * 4 + wblk.size() * 8;
    p->wbuf_off = static_cast<unsigned>((max_blen * 4 + 15) / 16 * 16);
    p->buf_bytes = p->wbuf_off + (p->unit ? 0u : static_cast<unsigned>(max_md) * cw * 8u);
    if (int rc = upload(&p->dLvlChunk, lvl_chunk.data(), lvl_chunk.size())) return rc;
    if (int rc = upload(&p->dCtab, ctab.data(), ctab.size())) return rc;
    if (int rc = upload(&p->dBlk, blk.data(), blk.size())) return rc;
    if (!p->unit)
        if (int rc = upload(&p->dWblk, wblk.data(), wblk.size())) return rc;
    return MARS_OK;
}

// fp16 split operand planes of the tcgen05 kernels: J * 2^jexp = J_hi + J_lo, [np16][np16],
// zero padded, plus their TMA maps.  The power-of-two prescale keeps every coupling inside
// fp16's range (|J_hi| < 2^14) and J_lo out of fp16 subnormals for the bulk of the couplings;
// it is exact, and the kernels scale the fp32 GEMM fields back by 2^-jexp.  Integer couplings
// up to 2048 are exact in J_hi unscaled (no J_lo product, integer fields stay exact).
int build_umma_planes(mars_problem* p) {
    if (p->dJhi) return MARS_OK;
    const int n = p->n;
    p->np16 = round_up(n, relax_dense_umma_block());
    const int np = p->np16;
    std::vector<double> w(static_cast<std::size_t>(np) * np, 0.0);
    double jmax = 0.0;
    if (p->dense) {
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) w[static_cast<std::size_t>(i) * np + j] = p->J[static_cast<std::size_t>(i) * n + j];
    } else {
        for (int i = 0; i < n; ++i)
            for (int k = p->off[i]; k < p->off[i + 1]; ++k) w[static_cast<std::size_t>(i) * np + p->idx[k]] += p->wt[k];
    }
    for (double v : w) jmax = std::max(jmax, std::fabs(v));
    p->jexp = 0;
    if (!(p->integral && jmax <= 2048.0) && jmax > 0.0)
        p->jexp = std::max(-120, std::min(120, 13 - static_cast<int>(std::floor(std::log2(jmax)))));
    const double sc = std::ldexp(1.0, p->jexp);
    std::vector<__half> jh(w.size()), jl(w.size());
    p->jlo = false;
    for (std::size_t k = 0; k < w.size(); ++k) {
        const double v = w[k] * sc;
        jh[k] = __double2half(v);
        jl[k] = __double2half(v - static_cast<double>(__half2float(jh[k])));
        if (__half2float(jl[k]) != 0.0f) p->jlo = true;
    }
    if (int rc = upload(&p->dJhi, jh.data(), jh.size())) return rc;
    if (int rc = upload(&p->dJlo, jl.data(), jl.size())) return rc;
    if (!make_tmap_f16(&p->tm_jhi, p->dJhi, np, np, relax_dense_umma_kc(), relax_dense_umma_j_rows()) ||
        !make_tmap_f16(&p->tm_jlo, p->dJlo, np, np, relax_dense_umma_kc(), relax_dense_umma_j_rows()) ||
        !make_tmap_f16(&p->tm_jhi_j, p->dJhi, np, np, jacobi_umma_kc(), relax_dense_umma_j_rows()) ||
        !make_tmap_f16(&p->tm_jlo_j, p->dJlo, np, np, jacobi_umma_kc(), relax_dense_umma_j_rows()))
        return fail(MARS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the coupling planes");
    return MARS_OK;
}

// Device copies in the layouts the kernels use.
int build_device_store(mars_problem* p) {
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (p->device < 0 || p->device >= ndev)
        return fail(MARS_ERR_CUDA, "device " + std::to_string(p->device) + " not present (" +
                                       std::to_string(ndev) + " visible)");
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    const int n = p->n;
    // exact-order energy operands (reference storage)
    if (p->dense) {
        if (int rc = upload(&p->dJ64, p->J.data(), p->J.size())) return rc;
    } else {
        if (int rc = upload(&p->dOff, p->off.data(), p->off.size())) return rc;
        if (int rc = upload(&p->dIdx, p->idx.data(), p->idx.size())) return rc;
        if (int rc = upload(&p->dW64, p->wt.data(), p->wt.size())) return rc;
    }
    if (p->has_field) {
        std::vector<float> h32(p->h.begin(), p->h.end());
        if (int rc = upload(&p->dH64, p->h.data(), p->h.size())) return rc;
        if (int rc = upload(&p->dH32, h32.data(), h32.size())) return rc;
    }
    // relaxation operands
    if (p->kernel == MARS_KERNEL_DENSE_SIMT || p->kernel == MARS_KERNEL_DENSE_UMMA) {
        p->np = round_up(n, p->kernel == MARS_KERNEL_DENSE_UMMA ? relax_dense_umma_block()
                                                                 : relax_dense_simt_block());
        std::vector<float> j32(static_cast<std::size_t>(p->np) * p->np, 0.0f);
        if (p->dense) {
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    j32[static_cast<std::size_t>(i) * p->np + j] =
                        static_cast<float>(p->J[static_cast<std::size_t>(i) * n + j]);
        } else {
            for (int i = 0; i < n; ++i)
                for (int k = p->off[i]; k < p->off[i + 1]; ++k)
                    j32[static_cast<std::size_t>(i) * p->np + p->idx[k]] += static_cast<float>(p->wt[k]);
        }
        if (int rc = upload(&p->dJ32, j32.data(), j32.size())) return rc;
        if (p->kernel == MARS_KERNEL_DENSE_UMMA)
            if (int rc = build_umma_planes(p)) return rc;
    } else {
        // relaxation CSR: the reference's sorted adjacency, or the nonzeros of a dense store in
        // ascending columns (row_dot order minus zero terms, which add nothing: acc is never -0)
        std::vector<int> off, idx;
        std::vector<double> w64;
        if (p->dense) {
            off.assign(n + 1, 0);
            for (int i = 0; i < n; ++i) {
                for (int j = 0; j < n; ++j) {
                    const double w = p->J[static_cast<std::size_t>(i) * n + j];
                    if (w != 0.0) {
                        idx.push_back(j);
                        w64.push_back(w);
                    }
                }
                off[i + 1] = static_cast<int>(idx.size());
            }
        }
        if (int rc = build_levels(p, p->dense ? off : p->off, p->dense ? idx : p->idx, p->dense ? w64 : p->wt))
            return rc;
        if (int rc = try_stencil(p, p->dense ? off : p->off, p->dense ? idx : p->idx, p->dense ? w64 : p->wt))
            return rc;
    }
    return MARS_OK;
}

int finish_problem(mars_problem* p, int device, int kernel, mars_problem_t** out) {
    p->device = device;
    finalize_metadata(p);
    p->kernel = resolve_kernel(p, kernel);
    if (p->kernel < 0) {
        delete p;
        return fail(MARS_ERR_INPUT, "unknown kernel selection " + std::to_string(kernel));
    }
    if (int rc = build_device_store(p)) {
        delete p;
        return rc;
    }
    *out = p;
    return MARS_OK;
}

}  // namespace

// ============================================================================ batch

struct mars_batch {
    mars_problem* p = nullptr;
    mars_params_t prm{};
    std::int64_t runs = 0;          // effective batch size (run_count)
    std::uint64_t base_seed = 0;
    std::int64_t first = 0, count = 0;
    int queue_len = 0;
    int grid = 0, slots = 0;
    bool uploaded = false, executed = false;
    // host plan
    std::vector<std::uint8_t> skipped;
    std::vector<double> temp;
    void* h_s0 = nullptr;           // pinned [count][n], fp32 or fp64 per kernel
    std::size_t s0_elem = 4;
    int* h_order = nullptr;         // pinned [count]
    double* h_temp = nullptr;       // pinned [count]
    std::uint8_t* h_status = nullptr;  // pinned [count]
    // device
    void* d_s0 = nullptr;
    double* d_temp = nullptr;
    int* d_order = nullptr;
    void* d_work = nullptr;
    std::size_t work_bytes = 0;
    int* d_queue = nullptr;
    std::uint8_t* d_status = nullptr;
    long long* d_iters = nullptr;
    double* d_elapsed = nullptr;
    unsigned long long* d_done = nullptr;  // [count] retirement %globaltimer (time-to-best)
    double* d_failT = nullptr;             // [count] level temperature of a Diverged run
    float* d_xpart = nullptr;              // split-K partial-field exchange (dense tcgen05)
    std::int8_t* d_spins = nullptr;
    double* d_energy = nullptr;
    double* d_cut = nullptr;
    double* d_part_e = nullptr;
    long long* d_part_i = nullptr;
    long long* d_best = nullptr;
    int best_grid = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    UmmaLaunch umma{};
    SparseLaunch sparse{};
    SpmmLaunch spmm{};
    bool use_spmm = false;
    StencilLaunch stencil{};
    bool use_stencil = false;
    bool use_small = false;   // relax_small.cu instead of the tensor-core kernel
    int small_warps = 0;      // its warps (= run slots) per CTA

    ~mars_batch() {
        if (!p) return;
        cudaSetDevice(p->device);
        cudaStreamSynchronize(p->stream);
        for (void* h : {static_cast<void*>(h_s0), static_cast<void*>(h_order), static_cast<void*>(h_temp),
                        static_cast<void*>(h_status)})
            p->give(h, true);
        for (void* d : {d_s0, static_cast<void*>(d_temp), static_cast<void*>(d_order), d_work,
                        static_cast<void*>(d_queue), static_cast<void*>(d_status), static_cast<void*>(d_iters),
                        static_cast<void*>(d_elapsed), static_cast<void*>(d_done), static_cast<void*>(d_failT), static_cast<void*>(d_xpart), static_cast<void*>(d_spins), static_cast<void*>(d_energy),
                        static_cast<void*>(d_cut), static_cast<void*>(d_part_e), static_cast<void*>(d_part_i),
                        static_cast<void*>(d_best)})
            p->give(d, false);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

SparseLevels sparse_levels(const mars_problem* p) {
    return SparseLevels{p->nlev, p->dLvlChunk, p->dCtab, p->dBlk, p->dWblk, p->nchunks, p->buf_bytes, p->wbuf_off, p->unit};
}

// Launch shape of the level-scheduled sparse kernel.  A CTA relaxes (32/cw)*r runs in
// lockstep; warps per CTA from the level widths (at most the widest level's chunk count);
// state in shared memory when it fits beside the warps' chunk buffers (else global rows,
// kept L2-resident by bounding the grid).  MARS_SPARSE_STATE=smem|global, MARS_SPARSE_R,
// MARS_SPARSE_WARPS and MARS_SPARSE_GRID override (tuning).
// Warp-per-run SpMM kernel when its shared memory holds at least 4 consumer warps of runs:
// RUNS = warps * (32/cw) state rows + a `ring`-slot chunk ring, one CTA per SM.
// MARS_SPARSE_KERNEL=spmm|levels, MARS_SPMM_WARPS, MARS_SPMM_RING_KB override.
bool spmm_config(mars_batch* b) {
    mars_problem* p = b->p;
    SpmmLaunch& l = b->spmm;
    const char* k = std::getenv("MARS_SPARSE_KERNEL");
    if (k && std::string(k) == "levels") return false;
    constexpr std::size_t kSmem = 220 * 1024;
    l.cw = p->cw;
    if (l.cw > 32 && k && std::string(k) == "levels") return false;
    // runs per warp: two 16-lane groups for 16-wide chunks, else one run per warp
    l.h = env_int("MARS_SPMM_H", l.cw == 16 ? 2 : 1);
    if (!relax_spmm_shape_ok(l.cw, l.h)) l.h = l.cw == 16 ? 2 : 1;
    // runs per lane group: 2 (interleaved, one 16-byte gather serves both) needs one spin per lane
    l.r = env_int("MARS_SPMM_R", 1) == 2 && l.cw * l.h == 32 ? 2 : 1;
    // byte ring: the largest block plus ~3 average blocks in flight (MARS_SPMM_RING_KB)
    const std::size_t avg = p->nchunks ? p->chunk_bytes / p->nchunks : p->buf_bytes;
    std::size_t ring_bytes = std::max<std::size_t>(p->buf_bytes + 3 * avg, 2 * p->buf_bytes);
    if (const int kb = env_int("MARS_SPMM_RING_KB", 0)) ring_bytes = static_cast<std::size_t>(kb) * 1024;
    ring_bytes = std::max<std::size_t>((ring_bytes + 15) / 16 * 16, p->buf_bytes);
    l.ring_bytes = static_cast<int>(ring_bytes);
    const std::size_t warp_bytes = relax_spmm_smem(p->np, l.h * l.r, 1, 0);
    if (ring_bytes + 4 * warp_bytes > kSmem && !(k && std::string(k) == "spmm")) return false;
    // CTAs per SM (each with its own ring): smaller CTAs couple fewer warps to one ring
    const int per_sm = std::max(1, env_int("MARS_SPMM_CTAS_PER_SM", 1));
    const std::size_t budget = (kSmem + 1024) / per_sm - 1024;
    int warps = static_cast<int>((budget - std::min(budget, ring_bytes)) / warp_bytes);
    warps = std::max(1, std::min({relax_spmm_max_warps(), warps, env_int("MARS_SPMM_WARPS", 64)}));
    const int runs_per_cta = warps * l.h * l.r;
    l.warps = warps;
    l.grid = std::max(1, std::min(per_sm * p->num_sms, (b->queue_len + runs_per_cta - 1) / runs_per_cta));
    l.grid = env_int("MARS_SPARSE_GRID", l.grid);
    return relax_spmm_smem(p->np, l.h * l.r, l.warps, l.ring_bytes) <= 227 * 1024;
}

int sparse_config(mars_batch* b) {
    mars_problem* p = b->p;
    SparseLaunch& l = b->sparse;
    l.cw = p->cw;
    if (l.cw > 32) return fail(MARS_ERR_INPUT, "64-wide chunk layout needs the warp-per-run kernel");
    const int groups = 32 / l.cw;
    const std::size_t col_bytes = static_cast<std::size_t>(p->np) * sizeof(double);
    constexpr std::size_t kSmem = 220 * 1024;
    l.r = env_int("MARS_SPARSE_R", 1);
    if (!relax_sparse_shape_ok(l.cw, l.r)) return fail(MARS_ERR_INPUT, "MARS_SPARSE_R must be 1, 2 or 4");
    const int runs = groups * l.r;
    const std::size_t state_bytes = col_bytes * runs;
    const double avg = static_cast<double>(p->nchunks) / std::max(p->nlev, 1);
    int warps = std::max(1, std::min(16, static_cast<int>(std::ceil(avg))));
    const auto bufs = [&](int w) { return static_cast<std::size_t>(w) * 2 * p->buf_bytes; };
    l.smem_state = state_bytes + bufs(warps) <= kSmem;
    if (l.smem_state) {
        // few CTAs per SM: widen toward the widest level so the SM has work in flight
        const int per_sm = std::max<int>(1, static_cast<int>(kSmem / (state_bytes + bufs(warps) + 1024)));
        while (per_sm * warps < 16 && 2 * warps <= std::min(16, p->max_level_chunks) &&
               state_bytes + bufs(2 * warps) <= kSmem)
            warps *= 2;
    }
    // every warp must own a chunk of the widest level (the per-warp chunk streams cycle)
    l.warps = std::max(1, std::min({16, p->max_level_chunks, env_int("MARS_SPARSE_WARPS", warps)}));
    if (const char* v = std::getenv("MARS_SPARSE_STATE")) l.smem_state = std::string(v) != "global";
    if (l.smem_state && state_bytes + bufs(l.warps) > kSmem) l.smem_state = false;
    const int occ = relax_sparse_occupancy(l, sparse_levels(p), p->n);
    if (occ <= 0) return fail(MARS_ERR_CUDA, "sparse kernel does not fit on the device (n = " + std::to_string(p->n) + ")");
    int grid = occ * p->num_sms;
    if (!l.smem_state) {
        // keep the live state rows within ~80 MB of L2
        const int l2_ctas = static_cast<int>((80ull << 20) / state_bytes);
        grid = std::min(grid, std::max(p->num_sms, l2_ctas / p->num_sms * p->num_sms));
    }
    l.grid = std::max(1, env_int("MARS_SPARSE_GRID", grid));
    return MARS_OK;
}

// A run's expected work for the large-N schedule: its level count (the descent relaxes once
// per temperature level from its start temperature down to t_min).
double run_work(double t0, const mars_params_t& prm) {
    return std::floor(std::max(0.0, t0 - prm.t_min) / prm.t_step) + 1.0;
}

// Greedy longest-first makespan of `work` (queue order) over `slots` identical slots.
double greedy_makespan(const double* work, std::int64_t count, int slots) {
    std::priority_queue<double, std::vector<double>, std::greater<double>> q;
    for (int i = 0; i < slots; ++i) q.push(0.0);
    double end = 0.0;
    for (std::int64_t k = 0; k < count; ++k) {
        const double t = q.top() + work[k];
        q.pop();
        q.push(t);
        end = std::max(end, t);
    }
    return end;
}

// Split-K choice for np >= 8192 (K1 "Split-K"): among split 1 / 2 / 4 (or only
// `forced`), the split and tile count (pairs) minimising greedy_makespan / per-run sweep rate,
// a tile count limited by the pairs the batch asks for, the resident clusters of that split
// and the SMs.  Rates from the measured cfg5 cycles per block (276K / 151K / 106K).  A near
// tie (< 2%) keeps the smaller split.  Returns the split; *tiles_out the tile count.
int choose_split(const double* work, std::int64_t count, int pairs, const int resident[3], int num_sms, int nkc,
                 int forced, int slots_per_cta, int* tiles_out) {
    static const double kSpeed[5] = {0.0, 1.0, 1.83, 0.0, 2.6};
    int split = 1, tiles = std::max(1, std::min(pairs, num_sms / 2));
    double best = -1.0;
    for (int sp : {1, 2, 4}) {
        if ((forced > 1 && sp != forced) || nkc % sp != 0) continue;
        const int tl = std::min({pairs, resident[sp == 1 ? 0 : sp == 2 ? 1 : 2], num_sms / (2 * sp)});
        if (tl < 1) continue;
        const double est = greedy_makespan(work, count, tl * 2 * slots_per_cta) / kSpeed[sp];
        if (best < 0.0 || est < best * 0.98) {
            best = est;
            split = sp;
            tiles = tl;
        }
    }
    *tiles_out = tiles;
    return split;
}

int batch_alloc(mars_batch* b) {
    mars_problem* p = b->p;
    const std::size_t cnt = static_cast<std::size_t>(std::max<std::int64_t>(b->count, 1));
    const std::size_t n = static_cast<std::size_t>(p->n);
    CUDA_TRY(cudaSetDevice(p->device));
    b->s0_elem = p->kernel == MARS_KERNEL_CSR ? sizeof(double) : sizeof(float);
    if (!(b->h_s0 = static_cast<decltype(b->h_s0)>(p->take(cnt * n * b->s0_elem, true))))
        return fail(MARS_ERR_CUDA, "pinned host allocation failed");
    if (!(b->h_order = static_cast<decltype(b->h_order)>(p->take(cnt * sizeof(int), true))))
        return fail(MARS_ERR_CUDA, "pinned host allocation failed");
    if (!(b->h_temp = static_cast<decltype(b->h_temp)>(p->take(cnt * sizeof(double), true))))
        return fail(MARS_ERR_CUDA, "pinned host allocation failed");
    if (!(b->h_status = static_cast<decltype(b->h_status)>(p->take(cnt, true))))
        return fail(MARS_ERR_CUDA, "pinned host allocation failed");
    if (!(b->d_s0 = static_cast<decltype(b->d_s0)>(p->take(cnt * n * b->s0_elem, false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_temp = static_cast<decltype(b->d_temp)>(p->take(cnt * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_order = static_cast<decltype(b->d_order)>(p->take(cnt * sizeof(int), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_queue = static_cast<decltype(b->d_queue)>(p->take(sizeof(int), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_status = static_cast<decltype(b->d_status)>(p->take(cnt, false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_iters = static_cast<decltype(b->d_iters)>(p->take(cnt * sizeof(long long), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_elapsed = static_cast<decltype(b->d_elapsed)>(p->take(cnt * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_failT = static_cast<decltype(b->d_failT)>(p->take(cnt * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_done = static_cast<decltype(b->d_done)>(p->take(cnt * sizeof(unsigned long long), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_spins = static_cast<decltype(b->d_spins)>(p->take(cnt * n, false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_energy = static_cast<decltype(b->d_energy)>(p->take(cnt * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_cut = static_cast<decltype(b->d_cut)>(p->take(cnt * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    b->best_grid = static_cast<int>(std::min<std::int64_t>((b->count + 255) / 256, 2 * p->num_sms));
    b->best_grid = std::max(b->best_grid, 1);
    if (!(b->d_part_e = static_cast<decltype(b->d_part_e)>(p->take(b->best_grid * sizeof(double), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_part_i = static_cast<decltype(b->d_part_i)>(p->take(b->best_grid * sizeof(long long), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (!(b->d_best = static_cast<decltype(b->d_best)>(p->take(sizeof(long long), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    for (auto& e : b->ev) CUDA_TRY(cudaEventCreate(&e));
    // plan (host, cheap) decides the queue length and hence the grid
    b->skipped.assign(cnt, 0);
    b->temp.assign(cnt, 0.0);
    std::vector<std::uint64_t> seeds(cnt);
    parallel_for(b->count, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t k = lo; k < hi; ++k) {
            bool sk;
            plan_of(&b->prm, b->base_seed, b->first + k, &sk, &b->temp[k], &seeds[k]);
            b->skipped[k] = sk;
        }
    });
    std::vector<int> order;
    for (std::int64_t k = 0; k < b->count; ++k)
        if (!b->skipped[k]) order.push_back(static_cast<int>(k));
    // longest-expected descents first: the level count grows with the start temperature
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return b->temp[x] > b->temp[y]; });
    b->queue_len = static_cast<int>(order.size());
    std::copy(order.begin(), order.end(), b->h_order);
    for (std::int64_t k = 0; k < b->count; ++k) {
        b->h_temp[k] = b->temp[k];
        b->h_status[k] = b->skipped[k] ? MARS_RUN_SKIPPED : 255;
    }
    int tm = 1;
    std::size_t per_cta = 0;
    int max_grid = p->num_sms;
    if (p->kernel == MARS_KERNEL_DENSE_SIMT) {
        tm = relax_dense_simt_slots_per_cta();
        per_cta = relax_dense_simt_work_bytes(p->np);
    } else if (p->kernel == MARS_KERNEL_DENSE_UMMA) {
        // Small integer instances run on the on-chip warp-per-run kernel unless the batch
        // fills the tensor-core kernel: a warp per run walks a sweep with less latency than
        // the 128-run tcgen05 tile.  Measured (SK N=256 +-1, descents/s, small vs tcgen05):
        // 1024 runs 16.0K vs 12.5K, 2368: 34.4K vs 29.1K, 4736: 69K vs 58K, 9472: 104K vs
        // 93K, 18944: 139K vs 183K -- so up to 4 x 16 warps x SMs runs.
        // MARS_DENSE_SMALL=1 forces it (when eligible), =0 forbids it.
        const bool small_ok = !p->jlo && p->jexp == 0 && p->n <= relax_small_max_n();
        const int small_env = env_int("MARS_DENSE_SMALL", -1);
        const std::int64_t small_max_runs = static_cast<std::int64_t>(4) * relax_small_slots_per_cta() * p->num_sms;
        b->use_small = small_ok && (small_env == 1 || (small_env < 0 && b->queue_len <= small_max_runs));
        if (b->use_small) {
            // one CTA per SM, as many warps (runs) per CTA as spread the batch over every SM:
            // the descents are latency-bound chains, so fewer warps per SM finish each sooner
            const int spread = static_cast<int>((b->queue_len + p->num_sms - 1) / p->num_sms);
            b->small_warps = std::max(1, std::min(relax_small_slots_per_cta(),
                                                  env_int("MARS_SMALL_WARPS", spread)));
            tm = b->small_warps;
            per_cta = 0;
        } else {
            tm = relax_dense_umma_slots_per_cta();
            per_cta = static_cast<std::size_t>(2) * tm * p->np * sizeof(__half);   // S_hi + S_lo rows
            // Persistent CTAs (in pairs): when the fp16 J planes fit in L2, only as many CTAs as
            // keep their state planes (re-read by every spin block's GEMM) in 90% of L2 beside
            // J.  cfg2 (N = 2000, round 2 kernel, power-capped): 11.5K descents/s at 148 CTAs,
            // 12.6K at 110 (one box); 11.81K at 92, 12.0K at 98, 11.85K at 104 (another box,
            // same call).  This rule: 98.  MARS_UMMA_GRID overrides.
            int l2 = 0;
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device);
            const std::size_t jbytes = static_cast<std::size_t>(2) * p->np * p->np * sizeof(__half);
            int fit = p->num_sms;
            const std::size_t l2use = static_cast<std::size_t>(l2) * 90 / 100;   // headroom: J32 diag, s0, spins
            if (l2 > 0 && jbytes < l2use)
                fit = static_cast<int>((l2use - jbytes) / per_cta);
            fit = std::max(p->num_sms / 2, std::min(p->num_sms, fit));
            max_grid = std::max(1, std::min(p->num_sms, env_int("MARS_UMMA_GRID", fit)));
        }
    } else {
        const char* kk = std::getenv("MARS_SPARSE_KERNEL");
        b->use_stencil = p->stencil && !(kk && std::string(kk) != "stencil");
        if (b->use_stencil) {
            // One run per CTA.  The run's level chain (gathers + fp64 tanh per level) is latency
            // bound, so throughput comes from runs in flight: up to 8 CTAs of <= 256 threads per SM
            // (measured: EA-2D 1.5K -> 2.7K descents/s from 1 to 8 CTAs/SM with the state rows in
            // global memory, beyond L2 capacity; EA-3D best at 4 x 256).  State in shared memory
            // only when that still leaves >= 2 CTAs per SM.
            StencilLaunch& l = b->stencil;
            l.threads = std::min(256, std::max(32, (p->st_maxw + 31) / 32 * 32));
            l.threads = std::max(32, std::min(1024, env_int("MARS_STENCIL_THREADS", l.threads)) / 32 * 32);
            const std::size_t smem = relax_stencil_smem(p->n, p->st_nlev, true);
            l.smem_state = 2 * (smem + 1024) <= 228 * 1024;
            if (const char* v = std::getenv("MARS_SPARSE_STATE")) l.smem_state = smem <= 220 * 1024 && std::string(v) != "global";
            const int fit = std::min(2048 / l.threads, 64 * 1024 / (l.threads * 64));
            const int per_sm = std::max(1, env_int("MARS_STENCIL_CTAS_PER_SM",
                                                   l.smem_state ? std::min<int>(fit, (228 * 1024) / (smem + 1024))
                                                                : std::min(8, fit)));
            tm = 1;
            max_grid = env_int("MARS_SPARSE_GRID", per_sm * p->num_sms);
            per_cta = l.smem_state ? 0 : static_cast<std::size_t>(p->np) * sizeof(double);
        } else if ((b->use_spmm = spmm_config(b))) {
            tm = b->spmm.warps * b->spmm.h * b->spmm.r;
            max_grid = b->spmm.grid;
            per_cta = 0;
        } else {
            if (int rc = sparse_config(b)) return rc;
            tm = (32 / b->sparse.cw) * b->sparse.r;
            max_grid = b->sparse.grid;
            per_cta = b->sparse.smem_state ? 0 : static_cast<std::size_t>(p->np) * tm * sizeof(double);
        }
    }
    b->grid = std::max(1, std::min(max_grid, (b->queue_len + tm - 1) / tm));
    int split = 1;
    if (p->kernel == MARS_KERNEL_DENSE_UMMA && !b->use_small) {
        b->grid = std::max(2, b->grid + (b->grid & 1));   // CTA pairs (cta_group::2)
        // Split-K for large N (np >= 8192): the field GEMM of a block (K = N) dwarfs its walk,
        // so a 256-run tile's K range is split over 2 or 4 CTA pairs of one cluster, which
        // makes each of its runs sweep faster (cfg5, cycles per block: 276K / 151K / 106K at
        // split 1 / 2 / 4).  A batch lasts as long as its slowest slot, and runs are queued
        // longest first (descending start temperature), so fewer but faster slots can win:
        // pick the split and tile count minimising a greedy longest-first makespan estimate
        // (work of a run ~ its level count).  cfg5 (8192 runs), measured: split 2 on 32 tiles
        // (8192 slots) 11.2 descents/s; split 4 on 15 tiles (3840 slots) 17.9.  Every
        // candidate keeps the whole grid one wave of resident clusters.
        // MARS_UMMA_SPLIT=1/2/4 forces the split (tiles: as many as fit).
        const int se = env_int("MARS_UMMA_SPLIT", -1);
        const int nkc = p->np / relax_dense_umma_kc();
        const int pairs = b->grid / 2;                        // tiles the batch asks for
        if (se > 1 || (se < 0 && p->np >= 8192)) {
            std::vector<double> work;                          // queue order (longest first)
            work.reserve(static_cast<std::size_t>(b->queue_len));
            for (int k = 0; k < b->queue_len; ++k)
                work.push_back(run_work(b->temp[static_cast<std::size_t>(b->h_order[k])], b->prm));
            const int resident[3] = {relax_dense_umma_max_clusters(1, p->jlo), relax_dense_umma_max_clusters(2, p->jlo),
                                     relax_dense_umma_max_clusters(4, p->jlo)};
            int tiles = 0;
            split = choose_split(work.data(), static_cast<std::int64_t>(work.size()), pairs, resident, p->num_sms,
                                 nkc, se > 1 ? se : 0, relax_dense_umma_slots_per_cta(), &tiles);
            b->grid = 2 * tiles;
        }
        if (std::getenv("MARS_UMMA_DEBUG"))
            std::fprintf(stderr, "[mars umma] pairs %d split %d resident clusters %d/%d/%d (split 1/2/4)\n", b->grid / 2,
                         split, relax_dense_umma_max_clusters(1, p->jlo), relax_dense_umma_max_clusters(2, p->jlo),
                         relax_dense_umma_max_clusters(4, p->jlo));
        b->umma.split = split;
        b->grid *= split;
    }
    b->sparse.grid = b->grid;
    b->spmm.grid = b->grid;
    b->stencil.grid = b->grid;
    b->slots = b->grid / split * tm;
    b->work_bytes = per_cta * (b->grid / split);
    if (!(b->d_work = static_cast<decltype(b->d_work)>(p->take(std::max<std::size_t>(b->work_bytes, 16), false))))
        return fail(MARS_ERR_CUDA, "device allocation failed");
    if (p->kernel == MARS_KERNEL_DENSE_UMMA && !b->use_small) {
        const std::size_t rows = relax_dense_umma_plane_rows(b->grid / split);
        b->umma.xpart = nullptr;
        if (split > 1) {
            const std::size_t bytes = static_cast<std::size_t>(split - 1) * 2 * rows * relax_dense_umma_block() * sizeof(float);
            if (!(b->d_xpart = static_cast<float*>(p->take(bytes, false))))
                return fail(MARS_ERR_CUDA, "device allocation failed");
            b->umma.xpart = b->d_xpart;
        }
        b->umma.s_hi = static_cast<__half*>(b->d_work);
        b->umma.s_lo = b->umma.s_hi + rows * p->np;
        b->umma.tm_jhi = p->tm_jhi;
        b->umma.tm_jlo = p->tm_jlo;
        b->umma.jlo = p->jlo;
        if (!make_tmap_f16(&b->umma.tm_shi, b->umma.s_hi, rows, p->np, relax_dense_umma_kc(), tm) ||
            !make_tmap_f16(&b->umma.tm_slo, b->umma.s_lo, rows, p->np, relax_dense_umma_kc(), tm))
            return fail(MARS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the state planes");
    }
    return MARS_OK;
}

}  // namespace

namespace marsb200 {

int host_fail(int code, const std::string& msg) { return fail(code, msg); }

// the tcgen05 kernel's hang detector record (umma.cuh), as text for an error message
std::string hang_note() {
    unsigned long long* h = nullptr;
    if (relax_dense_umma_hang_log(&h) != cudaSuccess || !h) return "";
    const volatile unsigned long long* v = h;
    if (v[0] == 0) return "";
    char buf[160];
    std::snprintf(buf, sizeof buf, "; mbarrier wait timed out in block %llu thread %llu (smem 0x%llx, parity %llu)",
                  v[1], v[2], v[3], v[4]);
    return buf;
}

int batch_device_view(mars_batch_t* b, BatchDevView* v) {
    if (!b || !v) return fail(MARS_ERR_INPUT, "null argument");
    if (!b->executed) return fail(MARS_ERR_RUNTIME, "batch viewed before execute");
    *v = BatchDevView{b->p->device, b->p->stream, b->p->n, b->first, b->count, b->d_status, b->d_energy,
                      b->d_cut, b->d_iters, b->d_elapsed, b->d_spins, b->d_best};
    return MARS_OK;
}

int plan_start_temps(const mars_params_t* prm, std::uint64_t base_seed, std::int64_t total, double* out) {
    parallel_for(total, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t k = lo; k < hi; ++k) {
            bool sk;
            std::uint64_t seed;
            plan_of(prm, base_seed, k, &sk, &out[k], &seed);
        }
    });
    return MARS_OK;
}

}  // namespace marsb200

// ============================================================================ C-ABI

extern "C" {

const char* mars_last_error(void) { return g_err.c_str(); }

int mars_debug_choose_split(const double* start_temps, int64_t count, const mars_params_t* prm, int32_t pairs,
                            const int32_t resident[3], int32_t num_sms, int32_t np, int32_t forced, int32_t* split,
                            int32_t* tiles) {
    if (!start_temps || !prm || !resident || !split || !tiles || count < 0 || pairs < 1 || num_sms < 2 || np < 128)
        return fail(MARS_ERR_INPUT, "mars_debug_choose_split: bad arguments");
    std::vector<double> work(static_cast<std::size_t>(count));
    for (int64_t k = 0; k < count; ++k) work[static_cast<std::size_t>(k)] = run_work(start_temps[k], *prm);
    std::stable_sort(work.begin(), work.end(), std::greater<double>());   // the queue's longest-first order
    const int res[3] = {resident[0], resident[1], resident[2]};
    int t = 0;
    *split = choose_split(work.data(), count, pairs, res, num_sms, np / relax_dense_umma_kc(), forced,
                          relax_dense_umma_slots_per_cta(), &t);
    *tiles = t;
    return MARS_OK;
}

int mars_device_count(int* out) {
    CUDA_TRY(cudaGetDeviceCount(out));
    return MARS_OK;
}

uint64_t mars_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t mars_sub_seed(uint64_t b, uint64_t i) { return sub_seed(b, i); }

int mars_validate_params(const mars_params_t* prm) { return check_params(prm); }

// solvers.cpp:202-213 (+ mars_grid_count 43-48)
int mars_run_count(const mars_params_t* prm, int64_t requested, int64_t* out) {
    if (int rc = check_params(prm)) return rc;
    if (prm->start_mode == MARS_GRID_SWEEP) {
        const double slots = std::floor((prm->t_max - prm->t_min) / prm->t_step);
        if (!(slots >= 0.0) || slots > 1e9)
            return fail(MARS_ERR_INPUT, "mars: grid of " + std::to_string(slots) +
                                            " temperatures is not usable");
        const std::int64_t count = static_cast<std::int64_t>(slots) + 1;
        if (count == 1 && !(prm->t_min > 0.0))
            return fail(MARS_ERR_INPUT,
                        "mars: the temperature grid contains no positive starting temperature");
        *out = count;
        return MARS_OK;
    }
    if (requested < 1) return fail(MARS_ERR_INPUT, "mars: UniformRandom mode needs runs >= 1");
    *out = requested;
    return MARS_OK;
}

int mars_run_plan(const mars_params_t* prm, uint64_t base_seed, int64_t index, int32_t* skipped,
                  double* start_temp, uint64_t* seed) {
    if (int rc = check_params(prm)) return rc;
    bool sk;
    plan_of(prm, base_seed, index, &sk, start_temp, seed);
    *skipped = sk;
    return MARS_OK;
}

int mars_initial_state(uint64_t seed, int32_t n, double* s) {
    Stream r(seed);
    for (int i = 0; i < n; ++i) s[i] = r.open_sym();
    return MARS_OK;
}

}  // extern "C"

namespace {

// Host side of IsingProblem::dense (model.cpp:47-72): validation and the stored copy.
int host_dense(int32_t n, const double* J, const double* h, mars_problem** out) {
    if (n <= 0) return fail(MARS_ERR_INPUT, "problem size must be positive");
    if (!J || !out) return fail(MARS_ERR_INPUT, "null argument");
    for (int i = 0; i < n; ++i) {                                          // model.cpp:55-64
        if (J[static_cast<std::size_t>(i) * n + i] != 0.0)
            return fail(MARS_ERR_INPUT, "coupling diagonal must be zero (row " + std::to_string(i) + ")");
        for (int j = i + 1; j < n; ++j)
            if (J[static_cast<std::size_t>(i) * n + j] != J[static_cast<std::size_t>(j) * n + i])
                return fail(MARS_ERR_INPUT, "coupling matrix must be symmetric (entries " +
                                                std::to_string(i) + "," + std::to_string(j) + ")");
    }
    auto* p = new mars_problem;
    p->n = n;
    p->dense = true;
    p->J.assign(J, J + static_cast<std::size_t>(n) * n);
    p->h.assign(n, 0.0);
    if (h) std::copy(h, h + n, p->h.begin());
    *out = p;
    return MARS_OK;
}

// Host side of IsingProblem::from_edges (model.cpp:74-131): validation, the 5% storage rule,
// dense accumulation or the canonical (sorted) adjacency.
int host_edges(int32_t n, int64_t m, const int32_t* u, const int32_t* v, const double* w, const double* h,
               mars_problem** out) {
    if (n <= 0) return fail(MARS_ERR_INPUT, "problem size must be positive");
    if (!out || (m > 0 && (!u || !v || !w))) return fail(MARS_ERR_INPUT, "null argument");
    for (std::int64_t k = 0; k < m; ++k) {                                  // model.cpp:80-84
        if (u[k] < 0 || u[k] >= n || v[k] < 0 || v[k] >= n)
            return fail(MARS_ERR_INPUT, "edge endpoint out of range");
        if (u[k] == v[k]) return fail(MARS_ERR_INPUT, "self-coupling is not allowed");
    }
    auto* p = new mars_problem;
    p->n = n;
    p->h.assign(n, 0.0);
    if (h) std::copy(h, h + n, p->h.begin());
    const double max_pairs = 0.5 * static_cast<double>(n) * (n - 1);
    const double density = max_pairs > 0 ? static_cast<double>(m) / max_pairs : 1.0;
    if (density >= kSparseDensityThreshold) {                               // model.cpp:91-98
        p->dense = true;
        p->J.assign(static_cast<std::size_t>(n) * n, 0.0);
        for (std::int64_t k = 0; k < m; ++k) {
            p->J[static_cast<std::size_t>(u[k]) * n + v[k]] += w[k];
            p->J[static_cast<std::size_t>(v[k]) * n + u[k]] += w[k];
        }
    } else {                                                                // model.cpp:99-128
        p->dense = false;
        std::vector<int> deg(n, 0);
        for (std::int64_t k = 0; k < m; ++k) {
            ++deg[u[k]];
            ++deg[v[k]];
        }
        p->off.assign(n + 1, 0);
        for (int i = 0; i < n; ++i) p->off[i + 1] = p->off[i] + deg[i];
        p->idx.resize(2 * m);
        p->wt.resize(2 * m);
        std::vector<int> cur(p->off.begin(), p->off.end() - 1);
        for (std::int64_t k = 0; k < m; ++k) {
            p->idx[cur[u[k]]] = v[k];
            p->wt[cur[u[k]]++] = w[k];
            p->idx[cur[v[k]]] = u[k];
            p->wt[cur[v[k]]++] = w[k];
        }
        std::vector<std::pair<int, double>> row;
        for (int i = 0; i < n; ++i) {                                       // canonical order
            row.clear();
            for (int k = p->off[i]; k < p->off[i + 1]; ++k) row.emplace_back(p->idx[k], p->wt[k]);
            std::sort(row.begin(), row.end());
            for (int k = p->off[i]; k < p->off[i + 1]; ++k) {
                p->idx[k] = row[k - p->off[i]].first;
                p->wt[k] = row[k - p->off[i]].second;
            }
        }
    }
    *out = p;
    return MARS_OK;
}

// problem_hash (io.cpp:260-290): FNV-1a over n, the stored upper-triangle couplings in
// visit_upper order (model.cpp:184-196) and the nonzero field entries, little-endian bytes.
std::uint64_t hash_of(const mars_problem* p) {
    std::uint64_t hv = 0xcbf29ce484222325ull;
    auto mix64 = [&hv](std::uint64_t x) {
        for (int b = 0; b < 8; ++b) {
            hv ^= (x >> (8 * b)) & 0xffu;
            hv *= 0x100000001b3ull;
        }
    };
    auto mix_double = [&](double d) {
        std::uint64_t bits;
        std::memcpy(&bits, &d, sizeof bits);
        mix64(bits);
    };
    const int n = p->n;
    mix64(static_cast<std::uint64_t>(n));
    for (int i = 0; i < n; ++i) {
        if (p->dense) {
            for (int k = i + 1; k < n; ++k) {
                const double w = p->J[static_cast<std::size_t>(i) * n + k];
                if (w != 0.0) {
                    mix64(static_cast<std::uint64_t>(i));
                    mix64(static_cast<std::uint64_t>(k));
                    mix_double(w);
                }
            }
        } else {
            for (int e = p->off[i]; e < p->off[i + 1]; ++e)
                if (p->idx[e] > i) {
                    mix64(static_cast<std::uint64_t>(i));
                    mix64(static_cast<std::uint64_t>(p->idx[e]));
                    mix_double(p->wt[e]);
                }
        }
    }
    for (int i = 0; i < n; ++i)
        if (p->h[i] != 0.0) {
            mix64(static_cast<std::uint64_t>(i));
            mix_double(p->h[i]);
        }
    return hv;
}

}  // namespace

extern "C" {

int mars_problem_dense(int32_t n, const double* J, const double* h, int32_t device,
                       int32_t kernel, mars_problem_t** out) {
    mars_problem* p = nullptr;
    if (int rc = host_dense(n, J, h, &p)) return rc;
    return finish_problem(p, device, kernel, out);
}

int mars_problem_from_edges(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                            const double* w, const double* h, int32_t device, int32_t kernel,
                            mars_problem_t** out) {
    mars_problem* p = nullptr;
    if (int rc = host_edges(n, m, u, v, w, h, &p)) return rc;
    return finish_problem(p, device, kernel, out);
}

// A copy of the problem on another device (same host data, same kernel family): the replicas
// mars_run_batch_multi shards a batch over.
int mars_problem_replicate(const mars_problem_t* src, int32_t device, mars_problem_t** out) {
    if (!src || !out) return fail(MARS_ERR_INPUT, "null argument");
    auto* p = new mars_problem;
    p->n = src->n;
    p->dense = src->dense;
    p->J = src->J;
    p->off = src->off;
    p->idx = src->idx;
    p->wt = src->wt;
    p->h = src->h;
    return finish_problem(p, device, src->kernel, out);
}

int mars_problem_hash(const mars_problem_t* p, uint64_t* out) {
    if (!p || !out) return fail(MARS_ERR_INPUT, "null argument");
    *out = hash_of(p);
    return MARS_OK;
}

int mars_instance_hash(int32_t n, const double* J, int64_t m, const int32_t* u, const int32_t* v,
                       const double* w, const double* h, uint64_t* out) {
    if (!out) return fail(MARS_ERR_INPUT, "null argument");
    mars_problem* p = nullptr;
    if (int rc = J ? host_dense(n, J, h, &p) : host_edges(n, m, u, v, w, h, &p)) return rc;
    *out = hash_of(p);
    delete p;
    return MARS_OK;
}

int mars_problem_rows(const mars_problem_t* p, double* out) {
    if (!p || !out) return fail(MARS_ERR_INPUT, "null argument");
    const int n = p->n;
    if (p->dense) {
        std::copy(p->J.begin(), p->J.end(), out);
    } else {                                                                // row_values, model.cpp:173-182
        std::fill(out, out + static_cast<std::size_t>(n) * n, 0.0);
        for (int i = 0; i < n; ++i)
            for (int e = p->off[i]; e < p->off[i + 1]; ++e) out[static_cast<std::size_t>(i) * n + p->idx[e]] = p->wt[e];
    }
    return MARS_OK;
}

void mars_problem_destroy(mars_problem_t* p) {
    if (!p) return;
    if (--p->refs == 0) delete p;
}

int mars_problem_info(const mars_problem_t* p, mars_problem_info_t* out) {
    if (!p || !out) return fail(MARS_ERR_INPUT, "null argument");
    out->n = p->n;
    out->uses_adjacency = !p->dense;
    out->integral = p->integral;
    out->has_field = p->has_field;
    out->coupling_sum = p->coupling_sum;
    out->nonzeros = p->nnz;
    out->device = p->device;
    out->kernel = p->kernel;
    out->levels = p->kernel == MARS_KERNEL_CSR ? (p->stencil ? p->st_nlev : p->nlev) : 0;
    out->reserved = 0;
    return MARS_OK;
}

int mars_energy(const mars_problem_t* p, const int8_t* spins, double* energy, double* cut) {
    if (!p || !spins) return fail(MARS_ERR_INPUT, "null argument");
    for (int i = 0; i < p->n; ++i)
        if (spins[i] != 1 && spins[i] != -1) return fail(MARS_ERR_INPUT, "spins must be +1/-1");
    CUDA_TRY(cudaSetDevice(p->device));
    std::int8_t* ds = nullptr;
    std::uint8_t* dst = nullptr;
    double* dout = nullptr;
    CUDA_TRY(cudaMalloc(&ds, p->n));
    CUDA_TRY(cudaMalloc(&dst, 1));
    CUDA_TRY(cudaMalloc(&dout, 2 * sizeof(double)));
    CUDA_TRY(cudaMemcpyAsync(ds, spins, p->n, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemsetAsync(dst, 0, 1, p->stream));
    EnergyArgs ea{p->n, p->dJ64, p->dOff, p->dIdx, p->dW64, p->dH64, p->coupling_sum, 1, ds,
                  dst, dout, dout + 1};
    CUDA_TRY(launch_energy(ea, p->stream));
    double out[2];
    CUDA_TRY(cudaMemcpyAsync(out, dout, sizeof out, cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    cudaFree(ds);
    cudaFree(dst);
    cudaFree(dout);
    if (energy) *energy = out[0];
    if (cut) *cut = out[1];
    return MARS_OK;
}

int mars_batch_create(mars_problem_t* p, const mars_params_t* prm, int64_t runs,
                      uint64_t base_seed, int64_t first, int64_t count, mars_batch_t** out) {
    if (!p || !out) return fail(MARS_ERR_INPUT, "null argument");
    std::int64_t total = 0;
    if (int rc = mars_run_count(prm, runs, &total)) return rc;
    if (first < 0 || count < 0 || first + count > total)
        return fail(MARS_ERR_INPUT, "shard [" + std::to_string(first) + ", " +
                                        std::to_string(first + count) + ") outside the batch of " +
                                        std::to_string(total) + " runs");
    auto* b = new mars_batch;
    b->p = p;
    ++p->refs;
    b->prm = *prm;
    if (b->prm.sweep_cap == 0) b->prm.sweep_cap = kSweepCap;
    b->runs = total;
    b->base_seed = base_seed;
    b->first = first;
    b->count = count;
    if (int rc = batch_alloc(b)) {
        mars_batch_destroy(b);
        return rc;
    }
    *out = b;
    return MARS_OK;
}

// Initial states: s_i = Rng(seed).uniform_open_sym(), i ascending (solvers.cpp:184-187),
// generated on host threads straight into pinned memory, then one H2D copy per array.
int mars_batch_upload(mars_batch_t* b) {
    if (!b) return fail(MARS_ERR_INPUT, "null argument");
    mars_problem* p = b->p;
    const int n = p->n;
    parallel_for(b->count, [&](std::int64_t lo, std::int64_t hi) {
        for (std::int64_t k = lo; k < hi; ++k) {
            if (b->skipped[k]) continue;
            Stream r(sub_seed(b->base_seed, static_cast<std::uint64_t>(b->first + k)));
            if (b->s0_elem == sizeof(double)) {
                double* row = static_cast<double*>(b->h_s0) + static_cast<std::size_t>(k) * n;
                for (int i = 0; i < n; ++i) row[i] = r.open_sym();
            } else {
                float* row = static_cast<float*>(b->h_s0) + static_cast<std::size_t>(k) * n;
                for (int i = 0; i < n; ++i) row[i] = static_cast<float>(r.open_sym());
            }
        }
    });
    CUDA_TRY(cudaSetDevice(p->device));
    const std::size_t cnt = static_cast<std::size_t>(b->count);
    CUDA_TRY(cudaMemcpyAsync(b->d_s0, b->h_s0, cnt * n * b->s0_elem, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_temp, b->h_temp, cnt * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_order, b->h_order, std::max(b->queue_len, 1) * sizeof(int),
                             cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_status, b->h_status, cnt, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    b->uploaded = true;
    b->executed = false;
    return MARS_OK;
}

}  // extern "C"

namespace {

// The device work of one batch (relax -> energy -> reduce).  fixed_sweeps / d_state_out are
// the test-only fixed-temperature mode of mars_debug_sweeps (RelaxArgs::fixed_sweeps).
// Progress during the batch (mars_run_batch_progress): the relaxation kernels append each run
// whose rounded spins are written to a host-mapped log (completion order); the calling thread
// polls it while the kernel runs, evaluates those runs' exact energies on a side stream and
// calls progress(index, best so far) once per run, like the reference's mutex-serialised
// worker callback (runner.cpp:107-113).  Skipped grid slots are reported first.
struct ProgressCtx {
    void (*cb)(int64_t, double, void*);
    void* user;
};

int report_progress(mars_batch_t* b, const ProgressCtx& pc, int* h_log, int* d_list_buf, double* d_e, std::uint8_t* d_st,
                    int* h_list, double* h_e, std::uint8_t* h_st) {
    mars_problem* p = b->p;
    double best = std::numeric_limits<double>::infinity();
    for (std::int64_t k = 0; k < b->count; ++k)
        if (b->skipped[k]) pc.cb(b->first + k, best, pc.user);
    cudaStream_t side = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    struct S {
        cudaStream_t s;
        ~S() { cudaStreamDestroy(s); }
    } sg{side};
    cudaEvent_t done = nullptr;
    CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    struct E {
        cudaEvent_t e;
        ~E() { cudaEventDestroy(e); }
    } eg{done};
    const int total = b->queue_len;
    int seen = 0, reported = 0, job = 0;
    bool inflight = false;
    const volatile int* log = h_log;
    while (reported < total) {
        if (!inflight && seen < total) {
            int k = 0;
            while (seen < total && log[seen] >= 0 && k < total) h_list[k++] = log[seen++];
            if (k > 0) {
                job = k;
                CUDA_TRY(cudaMemcpyAsync(d_list_buf, h_list, k * sizeof(int), cudaMemcpyHostToDevice, side));
                EnergyArgs ea{p->n, p->dJ64, p->dOff, p->dIdx, p->dW64, p->dH64, p->coupling_sum, k, b->d_spins,
                              b->d_status, nullptr, nullptr};
                CUDA_TRY(launch_energy_list(ea, d_list_buf, d_e, d_st, side));
                CUDA_TRY(cudaMemcpyAsync(h_e, d_e, k * sizeof(double), cudaMemcpyDeviceToHost, side));
                CUDA_TRY(cudaMemcpyAsync(h_st, d_st, k, cudaMemcpyDeviceToHost, side));
                CUDA_TRY(cudaEventRecord(done, side));
                inflight = true;
            }
        }
        if (inflight) {
            const cudaError_t q = cudaEventQuery(done);
            if (q == cudaSuccess) {
                for (int k = 0; k < job; ++k) {
                    if (h_st[k] == MARS_RUN_OK && h_e[k] < best) best = h_e[k];
                    pc.cb(b->first + h_list[k], best, pc.user);
                }
                reported += job;
                inflight = false;
                continue;
            }
            if (q != cudaErrorNotReady) return fail(MARS_ERR_CUDA, std::string("progress: ") + cudaGetErrorString(q));
        }
        const cudaError_t k = cudaStreamQuery(p->stream);          // a relaxation fault ends the wait
        if (k != cudaSuccess && k != cudaErrorNotReady) return fail(MARS_ERR_CUDA, cudaGetErrorString(k));
        if (k == cudaSuccess && !inflight && seen == total && reported < total)
            return fail(MARS_ERR_RUNTIME, "progress: the relaxation kernel ended with runs unreported");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    return MARS_OK;
}

int execute_impl(mars_batch_t* b, mars_timing_t* timing, int fixed_sweeps, float* d_state_out,
                 const ProgressCtx* prog = nullptr) {
    if (!b) return fail(MARS_ERR_INPUT, "null argument");
    if (!b->uploaded) return fail(MARS_ERR_RUNTIME, "batch executed before upload");
    mars_problem* p = b->p;
    cudaStream_t st = p->stream;
    CUDA_TRY(cudaSetDevice(p->device));
    if (b->executed)  // re-execution: restore the pending statuses
        CUDA_TRY(cudaMemcpyAsync(b->d_status, b->h_status, b->count, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(b->d_queue, 0, sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(b->d_work, 0, b->work_bytes, st));
    RelaxArgs ra{};
    ra.n = p->n;
    ra.np = p->np;
    ra.J32 = p->dJ32;
    ra.h32 = p->dH32;
    ra.h64 = p->dH64;
    ra.queue_len = b->queue_len;
    ra.order = b->d_order;
    ra.s0 = static_cast<const float*>(b->d_s0);
    ra.s0_64 = b->d_s0;
    ra.start_temp = b->d_temp;
    ra.c_step = b->prm.c_step;
    ra.d_min = b->prm.d_min;
    ra.sweep_cap = b->prm.sweep_cap;
    ra.work = b->d_work;
    ra.queue_head = b->d_queue;
    ra.status = b->d_status;
    ra.iters = b->d_iters;
    ra.elapsed = b->d_elapsed;
    ra.done_ns = b->d_done;
    ra.spins = b->d_spins;
    ra.fixed_sweeps = fixed_sweeps;
    ra.jscale = static_cast<float>(std::ldexp(1.0, -p->jexp));
    ra.fail_temp = b->d_failT;
    // progress buffers: host-mapped completion log + device counter + side-stream scratch
    int* h_log = nullptr;
    int* d_head = nullptr;
    int* d_list = nullptr;
    double* d_pe = nullptr;
    std::uint8_t* d_pst = nullptr;
    std::vector<int> h_list;
    std::vector<double> h_pe;
    std::vector<std::uint8_t> h_pst;
    struct ProgFree {
        int** hl;
        std::vector<void*> d;
        ~ProgFree() {
            if (*hl) cudaFreeHost(*hl);
            for (void* x : d) cudaFree(x);
        }
    } pfree{&h_log, {}};
    if (prog && b->queue_len > 0) {
        const std::size_t q = static_cast<std::size_t>(b->queue_len);
        CUDA_TRY(cudaHostAlloc(&h_log, q * sizeof(int), cudaHostAllocMapped));
        std::fill(h_log, h_log + q, -1);
        int* d_log = nullptr;
        CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_log), h_log, 0));
        CUDA_TRY(cudaMalloc(&d_head, sizeof(int)));
        pfree.d.push_back(d_head);
        CUDA_TRY(cudaMalloc(&d_list, q * sizeof(int)));
        pfree.d.push_back(d_list);
        CUDA_TRY(cudaMalloc(&d_pe, q * sizeof(double)));
        pfree.d.push_back(d_pe);
        CUDA_TRY(cudaMalloc(&d_pst, q));
        pfree.d.push_back(d_pst);
        CUDA_TRY(cudaMemsetAsync(d_head, 0, sizeof(int), st));
        h_list.resize(q);
        h_pe.resize(q);
        h_pst.resize(q);
        ra.retire_log = d_log;
        ra.retire_head = d_head;
    }
    ra.state_out = d_state_out;
    if (p->kernel == MARS_KERNEL_DENSE_UMMA && !b->use_small && std::getenv("MARS_L2_PERSIST")) {
        // experiment: a persisting-L2 carve-out (evict_last lines) and an access-policy window
        // over the state planes (MARS_L2_PERSIST=1: carve-out only, =2: + window)
        int maxp = 0, maxw = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, p->device);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, p->device);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<std::size_t>(maxp));
        if (std::atoi(std::getenv("MARS_L2_PERSIST")) >= 2) {
            cudaStreamAttrValue v{};
            v.accessPolicyWindow.base_ptr = b->d_work;
            v.accessPolicyWindow.num_bytes = std::min<std::size_t>(b->work_bytes, static_cast<std::size_t>(maxw));
            v.accessPolicyWindow.hitRatio =
                std::min(1.0f, static_cast<float>(maxp) / static_cast<float>(v.accessPolicyWindow.num_bytes));
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
        }
        if (std::getenv("MARS_UMMA_DEBUG"))
            std::fprintf(stderr, "[mars umma] persisting L2 max %d B, window max %d B, state planes %zu B\n", maxp, maxw,
                         b->work_bytes);
    }
    std::int64_t launches = 0;
    const bool prof = std::getenv("MARS_PROFILE") != nullptr;
    long long* dprof = nullptr;
    if (prof) {
        CUDA_TRY(cudaMalloc(&dprof, sizeof(long long) * kProfSlots * b->grid));
        CUDA_TRY(cudaMemsetAsync(dprof, 0, sizeof(long long) * kProfSlots * b->grid, st));
    }
    ra.prof = dprof;
    CUDA_TRY(cudaEventRecord(b->ev[0], st));
    if (b->queue_len > 0) {
        if (p->kernel == MARS_KERNEL_DENSE_SIMT)
            CUDA_TRY(launch_relax_dense_simt(ra, b->grid, st));
        else if (p->kernel == MARS_KERNEL_DENSE_UMMA && b->use_small)
            CUDA_TRY(launch_relax_small(ra, p->dJhi, b->grid, b->small_warps, st));
        else if (p->kernel == MARS_KERNEL_DENSE_UMMA)
            CUDA_TRY(launch_relax_dense_umma(ra, b->umma, b->grid, st));
        else
            CUDA_TRY(b->use_stencil
                         ? launch_relax_stencil(ra, StencilArgs{p->st_dims, p->st_L, p->st_nlev, p->dStLvl, p->dStCoords},
                                                b->stencil, st)
                         : b->use_spmm ? launch_relax_spmm(ra, sparse_levels(p), b->spmm, st)
                                       : launch_relax_sparse(ra, sparse_levels(p), b->sparse, st));
        ++launches;
        if (std::getenv("MARS_SYNC_CHECK")) {          // attribute an asynchronous fault to the relaxation
            const cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess)
                return fail(MARS_ERR_CUDA, std::string("relaxation kernel: ") + cudaGetErrorString(e) + ::marsb200::hang_note());
        }
    }
    if (prog) {
        if (b->queue_len > 0) {
            if (int rc = report_progress(b, *prog, h_log, d_list, d_pe, d_pst, h_list.data(), h_pe.data(), h_pst.data()))
                return rc;
        } else {
            for (std::int64_t k = 0; k < b->count; ++k)
                prog->cb(b->first + k, std::numeric_limits<double>::infinity(), prog->user);
        }
    }
    CUDA_TRY(cudaEventRecord(b->ev[1], st));
    EnergyArgs ea{p->n, p->dJ64, p->dOff, p->dIdx, p->dW64, p->dH64, p->coupling_sum,
                  b->count, b->d_spins, b->d_status, b->d_energy, b->d_cut};
    if (b->count > 0) {
        CUDA_TRY(launch_energy(ea, st));
        ++launches;
    }
    CUDA_TRY(cudaEventRecord(b->ev[2], st));
    BestArgs ba{b->count, b->d_status, b->d_energy, b->d_part_e, b->d_part_i, b->d_best};
    CUDA_TRY(launch_best(ba, b->best_grid, st));
    launches += 2;
    CUDA_TRY(cudaEventRecord(b->ev[3], st));
    CUDA_TRY(cudaStreamSynchronize(st));
    b->executed = true;
    if (prof) {
        std::vector<long long> h(static_cast<std::size_t>(kProfSlots) * b->grid);
        CUDA_TRY(cudaMemcpy(h.data(), dprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        cudaFree(dprof);
        double acc[kProfSlots] = {0};
        for (int c = 0; c < b->grid; ++c)
            for (int k = 0; k < kProfSlots; ++k) acc[k] += static_cast<double>(h[c * kProfSlots + k]);
        if (p->kernel == MARS_KERNEL_CSR && b->use_spmm && acc[0] > 0) {
            const double per = acc[0] * p->nchunks;   // warp-chunks
            std::fprintf(stderr, "[mars prof] spmm: %.0f warp-sweeps; per warp-chunk: wait %.0f, sum %.0f, trial %.0f cycles\n",
                         acc[0], acc[1] / per, acc[2] / per, acc[3] / per);
        }
        const double blocks = acc[0] * (h[6] ? h[6] : 1);
        if (p->kernel == MARS_KERNEL_DENSE_UMMA && !b->use_small)
            std::fprintf(stderr,
                         "[mars prof] grid %d: sweeps/cta %.1f, cycles/cta %.3g | per block, walker: turnover %.0f, "
                         "wait jready+tmem_full %.0f, wait fields+ld %.0f, old-state load %.0f, walk %.0f, store/arrive %.0f | "
                         "helper: wait tmem_full %.0f, work %.0f, wait deltas %.0f | producer wait ready %.0f empty %.0f | "
                         "mma wait full %.0f tmem_empty %.0f\n",
                         b->grid, acc[0] / b->grid, acc[1] / b->grid, acc[7] / blocks, acc[2] / blocks, acc[3] / blocks,
                         acc[4] / blocks, acc[5] / blocks, acc[12] / blocks, acc[15] / blocks, acc[14] / blocks,
                         acc[13] / blocks, acc[8] / blocks, acc[9] / blocks, acc[10] / blocks, acc[11] / blocks);
    }
    if (timing) {
        float ms[3];
        CUDA_TRY(cudaEventElapsedTime(&ms[0], b->ev[0], b->ev[1]));
        CUDA_TRY(cudaEventElapsedTime(&ms[1], b->ev[1], b->ev[2]));
        CUDA_TRY(cudaEventElapsedTime(&ms[2], b->ev[2], b->ev[3]));
        timing->relax_ms = ms[0];
        timing->energy_ms = ms[1];
        timing->reduce_ms = ms[2];
        timing->total_ms = static_cast<double>(ms[0]) + ms[1] + ms[2];
        timing->launches = launches;
        timing->grid = b->grid;
        timing->slots = b->slots;
        timing->kernel = b->use_small ? 4 : p->kernel;
        timing->split = (p->kernel == MARS_KERNEL_DENSE_UMMA && !b->use_small) ? std::max(1, b->umma.split) : 1;
        std::vector<long long> it(static_cast<std::size_t>(b->count));
        std::vector<std::uint8_t> stt(static_cast<std::size_t>(b->count));
        if (b->count) {
            CUDA_TRY(cudaMemcpy(it.data(), b->d_iters, b->count * sizeof(long long), cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(stt.data(), b->d_status, b->count, cudaMemcpyDeviceToHost));
        }
        long long tot = 0;
        for (std::int64_t k = 0; k < b->count; ++k)
            if (stt[k] != MARS_RUN_SKIPPED) tot += it[k];
        timing->total_sweeps = tot;
    }
    return MARS_OK;
}

}  // namespace

extern "C" {

int mars_batch_execute(mars_batch_t* b, mars_timing_t* timing) { return execute_impl(b, timing, 0, nullptr); }

// TEST-ONLY (include/mars_b200.h): `sweeps` Gauss-Seidel sweeps at fixed temperatures through
// the problem's dense relaxation kernel, from caller-given fp32 states.
int mars_debug_sweeps(mars_problem_t* p, int64_t count, const float* s_in, const double* temps,
                      int32_t sweeps, float* s_out, int32_t* kernel_used) {
    if (!p || !s_in || !temps || !s_out) return fail(MARS_ERR_INPUT, "null argument");
    if (count < 1 || sweeps < 1) return fail(MARS_ERR_INPUT, "count and sweeps must be positive");
    if (p->kernel != MARS_KERNEL_DENSE_UMMA && p->kernel != MARS_KERNEL_DENSE_SIMT)
        return fail(MARS_ERR_INPUT, "mars_debug_sweeps needs a dense (fp32-state) kernel");
    for (std::int64_t k = 0; k < count; ++k)
        if (!(temps[k] >= 0.0)) return fail(MARS_ERR_INPUT, "temperatures must be >= 0");
    const mars_params_t prm{0.0, 1.0, 1.0, 1.0, 1e-4, MARS_UNIFORM_RANDOM, 0, 0};
    mars_batch_t* b = nullptr;
    if (int rc = mars_batch_create(p, &prm, count, 0, 0, count, &b)) return rc;
    struct Guard {
        mars_batch_t* b;
        float* d = nullptr;
        ~Guard() {
            if (d) cudaFree(d);
            mars_batch_destroy(b);
        }
    } g{b};
    const std::size_t n = static_cast<std::size_t>(p->n), cnt = static_cast<std::size_t>(count);
    std::memcpy(b->h_s0, s_in, cnt * n * sizeof(float));
    for (std::int64_t k = 0; k < count; ++k) {
        b->h_temp[k] = temps[k];
        b->h_order[k] = static_cast<int>(k);
        b->h_status[k] = 255;
    }
    b->queue_len = static_cast<int>(count);
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaMalloc(&g.d, cnt * n * sizeof(float)));
    CUDA_TRY(cudaMemcpyAsync(b->d_s0, b->h_s0, cnt * n * sizeof(float), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_temp, b->h_temp, cnt * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_order, b->h_order, cnt * sizeof(int), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(b->d_status, b->h_status, cnt, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    b->uploaded = true;
    mars_timing_t t{};
    if (int rc = execute_impl(b, &t, sweeps, g.d)) return rc;
    CUDA_TRY(cudaMemcpy(s_out, g.d, cnt * n * sizeof(float), cudaMemcpyDeviceToHost));
    if (kernel_used) *kernel_used = t.kernel;
    return MARS_OK;
}

int mars_batch_fetch(mars_batch_t* b, mars_records_t* rec, int64_t* best_index,
                     int8_t* best_spins) {
    if (!b) return fail(MARS_ERR_INPUT, "null argument");
    if (!b->executed) return fail(MARS_ERR_RUNTIME, "batch fetched before execute");
    mars_problem* p = b->p;
    cudaStream_t st = p->stream;
    const std::size_t cnt = static_cast<std::size_t>(b->count);
    CUDA_TRY(cudaSetDevice(p->device));
    std::vector<std::uint8_t> status(cnt);
    std::vector<long long> iters(cnt);
    if (cnt) {
        CUDA_TRY(cudaMemcpyAsync(status.data(), b->d_status, cnt, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(iters.data(), b->d_iters, cnt * sizeof(long long), cudaMemcpyDeviceToHost, st));
    }
    if (rec) {
        if (rec->energy && cnt) CUDA_TRY(cudaMemcpyAsync(rec->energy, b->d_energy, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (rec->cut && cnt) CUDA_TRY(cudaMemcpyAsync(rec->cut, b->d_cut, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (rec->elapsed_seconds && cnt) CUDA_TRY(cudaMemcpyAsync(rec->elapsed_seconds, b->d_elapsed, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (rec->spins && cnt) CUDA_TRY(cudaMemcpyAsync(rec->spins, b->d_spins, cnt * p->n, cudaMemcpyDeviceToHost, st));
        if (rec->fail_temp && cnt) CUDA_TRY(cudaMemcpyAsync(rec->fail_temp, b->d_failT, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    long long best = -1;
    CUDA_TRY(cudaMemcpyAsync(&best, b->d_best, sizeof best, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (best >= 0 && best_spins)
        CUDA_TRY(cudaMemcpy(best_spins, b->d_spins + static_cast<std::size_t>(best) * p->n, p->n, cudaMemcpyDeviceToHost));
    for (std::size_t k = 0; k < cnt; ++k)
        if (status[k] > MARS_RUN_DIVERGED)
            return fail(MARS_ERR_RUNTIME, "run " + std::to_string(b->first + k) + " was never executed");
    if (rec) {
        if (rec->status) std::copy(status.begin(), status.end(), rec->status);
        if (rec->descent_iters)
            for (std::size_t k = 0; k < cnt; ++k) rec->descent_iters[k] = status[k] == MARS_RUN_SKIPPED ? 0 : iters[k];
        if (rec->start_temp) std::copy(b->temp.begin(), b->temp.begin() + cnt, rec->start_temp);
        // skipped slots carry zero records (runner.cpp:35-39)
        for (std::size_t k = 0; k < cnt; ++k) {
            if (status[k] != MARS_RUN_SKIPPED) continue;
            if (rec->energy) rec->energy[k] = 0.0;
            if (rec->cut) rec->cut[k] = 0.0;
            if (rec->elapsed_seconds) rec->elapsed_seconds[k] = 0.0;
            if (rec->spins) std::memset(rec->spins + k * p->n, 0, p->n);
        }
    }
    if (best_index) *best_index = best < 0 ? -1 : b->first + best;
    return MARS_OK;
}

int mars_batch_fetch_finish(mars_batch_t* b, double* finish_seconds) {
    if (!b || !finish_seconds) return fail(MARS_ERR_INPUT, "null argument");
    if (!b->executed) return fail(MARS_ERR_RUNTIME, "batch fetched before execute");
    mars_problem* p = b->p;
    cudaStream_t st = p->stream;
    const std::size_t cnt = static_cast<std::size_t>(b->count);
    if (!cnt) return MARS_OK;
    CUDA_TRY(cudaSetDevice(p->device));
    std::vector<std::uint8_t> status(cnt);
    std::vector<double> elapsed(cnt);
    std::vector<unsigned long long> done(cnt);
    CUDA_TRY(cudaMemcpyAsync(status.data(), b->d_status, cnt, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(elapsed.data(), b->d_elapsed, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(done.data(), b->d_done, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    // origin = the earliest descent start of the launch (retirement - its own elapsed)
    long double origin = 0.0L;
    bool any = false;
    for (std::size_t k = 0; k < cnt; ++k) {
        if (status[k] > MARS_RUN_DIVERGED || status[k] == MARS_RUN_SKIPPED) continue;
        const long double t0 = static_cast<long double>(done[k]) - 1e9L * elapsed[k];
        if (!any || t0 < origin) origin = t0;
        any = true;
    }
    for (std::size_t k = 0; k < cnt; ++k) {
        const bool ran = status[k] <= MARS_RUN_DIVERGED && status[k] != MARS_RUN_SKIPPED;
        finish_seconds[k] = ran ? static_cast<double>((static_cast<long double>(done[k]) - origin) * 1e-9L) : 0.0;
    }
    return MARS_OK;
}

void mars_batch_destroy(mars_batch_t* b) {
    if (!b) return;
    mars_problem* p = b->p;
    delete b;
    if (p && --p->refs == 0) delete p;
}

// runner.cpp:126-167 -- index-order aggregation; the all-failed batch is an error (153-155)
int mars_aggregate(int64_t count, const uint8_t* status, const double* energy, const double* cut,
                   const double* elapsed, double tol, double total_seconds, mars_stats_t* s) {
    if (!s || (count > 0 && (!status || !energy || !cut)))
        return fail(MARS_ERR_INPUT, "null argument");
    *s = mars_stats_t{};
    double cut_sum = 0.0, energy_sum = 0.0, run_seconds = 0.0;
    std::int64_t best = -1;
    for (std::int64_t i = 0; i < count; ++i) {
        if (status[i] == MARS_RUN_SKIPPED) {
            ++s->skipped_runs;
            continue;
        }
        if (status[i] == MARS_RUN_DIVERGED) {
            ++s->failed_runs;
            continue;
        }
        ++s->completed_runs;
        energy_sum += energy[i];
        cut_sum += cut[i];
        if (elapsed) run_seconds += elapsed[i];
        if (best < 0 || energy[i] < s->best_energy) {
            s->best_energy = energy[i];
            best = i;
        }
        if (s->best_cut < cut[i] || s->completed_runs == 1) s->best_cut = cut[i];
    }
    s->best_index = best;
    s->total_seconds = total_seconds;
    if (s->completed_runs == 0)
        return fail(MARS_ERR_ALL_FAILED, "batch failed: no run completed (" +
                                             std::to_string(s->failed_runs) + " diverged, " +
                                             std::to_string(s->skipped_runs) + " skipped)");
    s->mean_energy = energy_sum / static_cast<double>(s->completed_runs);
    s->mean_cut = cut_sum / static_cast<double>(s->completed_runs);
    for (std::int64_t i = 0; i < count; ++i)
        if (status[i] == MARS_RUN_OK && std::abs(energy[i] - s->best_energy) <= tol) ++s->hit_count;
    s->success_probability = static_cast<double>(s->hit_count) / static_cast<double>(s->completed_runs);
    s->mean_seconds_per_run = run_seconds / static_cast<double>(s->completed_runs);
    return MARS_OK;
}

int mars_run_shard(mars_problem_t* p, const mars_params_t* prm, int64_t runs, uint64_t base_seed,
                   int64_t first, int64_t count, mars_records_t* rec) {
    mars_batch_t* b = nullptr;
    if (int rc = mars_batch_create(p, prm, runs, base_seed, first, count, &b)) return rc;
    int rc = mars_batch_upload(b);
    if (!rc) rc = mars_batch_execute(b, nullptr);
    if (!rc) rc = mars_batch_fetch(b, rec, nullptr, nullptr);
    mars_batch_destroy(b);
    return rc;
}

int mars_run_batch(mars_problem_t* p, const mars_params_t* prm, int64_t runs, uint64_t base_seed,
                   mars_records_t* records, mars_stats_t* stats, int8_t* best_spins) {
    return mars_run_batch_progress(p, prm, runs, base_seed, records, stats, best_spins, nullptr, nullptr);
}

int mars_run_batch_progress(mars_problem_t* p, const mars_params_t* prm, int64_t runs, uint64_t base_seed,
                            mars_records_t* records, mars_stats_t* stats, int8_t* best_spins,
                            void (*progress)(int64_t, double, void*), void* user) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!p || !stats) return fail(MARS_ERR_INPUT, "null argument");
    std::int64_t total = 0;
    if (int rc = mars_run_count(prm, runs, &total)) return rc;   // InputError before any run
    mars_batch_t* b = nullptr;
    if (int rc = mars_batch_create(p, prm, runs, base_seed, 0, total, &b)) return rc;
    std::vector<std::uint8_t> status(total);
    std::vector<double> energy(total), cut(total), elapsed(total);
    mars_records_t own{status.data(), energy.data(), cut.data(), nullptr, nullptr, elapsed.data(),
                       records ? records->spins : nullptr, records ? records->fail_temp : nullptr};
    if (records) {
        own.start_temp = records->start_temp;
        own.descent_iters = records->descent_iters;
    }
    std::int64_t best = -1;
    const ProgressCtx pc{progress, user};
    int rc = mars_batch_upload(b);
    if (!rc) rc = execute_impl(b, nullptr, 0, nullptr, progress ? &pc : nullptr);
    if (!rc) rc = mars_batch_fetch(b, &own, &best, best_spins);
    mars_batch_destroy(b);
    if (rc) return rc;
    if (records) {
        if (records->status) std::copy(status.begin(), status.end(), records->status);
        if (records->energy) std::copy(energy.begin(), energy.end(), records->energy);
        if (records->cut) std::copy(cut.begin(), cut.end(), records->cut);
        if (records->elapsed_seconds) std::copy(elapsed.begin(), elapsed.end(), records->elapsed_seconds);
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rc = mars_aggregate(total, status.data(), energy.data(), cut.data(), elapsed.data(),
                        p->integral ? 0.0 : 1e-9, secs, stats);
    if (rc) return rc;
    if (stats->best_index != best)
        return fail(MARS_ERR_RUNTIME, "device best-of-R index " + std::to_string(best) +
                                          " disagrees with the host aggregation " +
                                          std::to_string(stats->best_index));
    return MARS_OK;
}

}  // extern "C"

namespace {

// schedule_at (solvers.cpp:118-123): the stored sequence stretched / compressed by index
double schedule_at(const double* sched, std::int64_t len, std::int64_t k, std::int64_t iters) {
    if (len == iters) return sched[k];
    const std::int64_t idx = std::min(len - 1, k * len / iters);
    return sched[idx];
}

// Device-owning scratch of one synchronous-solver batch.
struct JacobiScratch {
    std::vector<void*> bufs;
    ~JacobiScratch() {
        for (void* b : bufs) cudaFree(b);
    }
    template <class T>
    int alloc(T** p, std::size_t count) {
        void* q = nullptr;
        CUDA_TRY(cudaMalloc(&q, std::max<std::size_t>(count, 1) * sizeof(T)));
        bufs.push_back(q);
        *p = static_cast<T*>(q);
        return MARS_OK;
    }
};

// run_batch for NmfaParams / SimCimParams (runner.cpp:31-60, 81-178): every run index through
// the tcgen05 Jacobi kernel, exact energies, best-of-R, then the reference's aggregation.
int run_jacobi(mars_problem* p, int solver, std::int64_t iters, const double* sched, std::int64_t sched_len,
               double alpha, double noise_sigma, double step_size, std::int64_t runs, std::uint64_t base_seed,
               mars_records_t* records, mars_stats_t* stats, std::int8_t* best_spins) {
    const auto t0 = std::chrono::steady_clock::now();
    if (runs < 1) return fail(MARS_ERR_INPUT, "batch needs runs >= 1");            // effective_runs
    if (runs > (1 << 30)) return fail(MARS_ERR_INPUT, "batch too large");
    CUDA_TRY(cudaSetDevice(p->device));
    if (int rc = build_umma_planes(p)) return rc;
    const int n = p->n, np = p->np16;
    cudaStream_t st = p->stream;
    if (solver == 0 && !p->dNorm) {
        // nmfa_normalizers (solvers.cpp:364-372): sqrt(h_i^2 + row_sumsq(i)), row_sumsq in the
        // storage order of model.cpp:165-175
        std::vector<float> nrm(np, 0.0f);
        for (int i = 0; i < n; ++i) {
            double acc = 0.0;
            if (p->dense) {
                const double* row = p->J.data() + static_cast<std::size_t>(i) * n;
                for (int j = 0; j < n; ++j) acc += row[j] * row[j];
            } else {
                for (int k = p->off[i]; k < p->off[i + 1]; ++k) acc += p->wt[k] * p->wt[k];
            }
            nrm[i] = static_cast<float>(std::sqrt(p->h[i] * p->h[i] + acc));
        }
        if (int rc = upload(&p->dNorm, nrm.data(), nrm.size())) return rc;
    }
    const int count = static_cast<int>(runs);
    const int tm = jacobi_umma_slots_per_cta();
    int grid = std::min((count + tm - 1) / tm, p->num_sms & ~1);
    grid = std::max(2, grid + (grid & 1));
    const int slots = grid * tm;
    JacobiScratch sc;
    JacobiArgs a{};
    a.n = n;
    a.np = np;
    a.solver = solver;
    a.iters = static_cast<int>(iters);
    a.noise_sigma = noise_sigma;
    a.alpha_f = static_cast<float>(alpha);
    a.one_minus_alpha_f = static_cast<float>(1.0 - alpha);
    a.step_f = static_cast<float>(step_size);
    a.jscale = static_cast<float>(std::ldexp(1.0, -p->jexp));
    a.norm = p->dNorm;
    a.h32 = p->dH32;
    a.queue_len = count;
    a.slots = slots;
    std::vector<double> sv(static_cast<std::size_t>(iters));
    for (std::int64_t k = 0; k < iters; ++k) sv[k] = schedule_at(sched, sched_len, k, iters);
    std::vector<std::uint64_t> seeds(count);
    std::vector<int> order(count);
    for (int k = 0; k < count; ++k) {
        seeds[k] = sub_seed(base_seed, static_cast<std::uint64_t>(k));           // runner.cpp:55
        order[k] = k;
    }
    double *d_sched, *d_elapsed, *d_energy, *d_cut, *d_part_e;
    std::uint64_t *d_seeds, *d_mt;
    int *d_order, *d_queue;
    std::uint8_t* d_status;
    long long *d_iters, *d_part_i, *d_best;
    unsigned long long* d_done;
    std::int8_t* d_spins;
    __half* planes[4];
    const int best_grid = std::max(1, std::min((count + 255) / 256, 2 * p->num_sms));
    for (auto& pl : planes)
        if (int rc = sc.alloc(&pl, static_cast<std::size_t>(slots) * np)) return rc;
    if (int rc = sc.alloc(&d_sched, sv.size())) return rc;
    if (int rc = sc.alloc(&d_seeds, seeds.size())) return rc;
    if (int rc = sc.alloc(&d_order, order.size())) return rc;
    if (int rc = sc.alloc(&d_queue, 1)) return rc;
    if (int rc = sc.alloc(&d_mt, static_cast<std::size_t>(kMtWords) * slots)) return rc;
    if (int rc = sc.alloc(&d_status, count)) return rc;
    if (int rc = sc.alloc(&d_iters, count)) return rc;
    if (int rc = sc.alloc(&d_elapsed, count)) return rc;
    if (int rc = sc.alloc(&d_done, count)) return rc;
    if (int rc = sc.alloc(&d_spins, static_cast<std::size_t>(count) * n)) return rc;
    if (int rc = sc.alloc(&d_energy, count)) return rc;
    if (int rc = sc.alloc(&d_cut, count)) return rc;
    if (int rc = sc.alloc(&d_part_e, best_grid)) return rc;
    if (int rc = sc.alloc(&d_part_i, best_grid)) return rc;
    if (int rc = sc.alloc(&d_best, 1)) return rc;
    CUDA_TRY(cudaMemcpyAsync(d_sched, sv.data(), sv.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d_seeds, seeds.data(), seeds.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d_order, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(d_queue, 0, sizeof(int), st));
    CUDA_TRY(cudaMemsetAsync(d_status, 255, count, st));
    a.sched = d_sched;
    a.seeds = d_seeds;
    a.order = d_order;
    a.queue_head = d_queue;
    a.mt = d_mt;
    a.s_hi[0] = planes[0];
    a.s_lo[0] = planes[1];
    a.s_hi[1] = planes[2];
    a.s_lo[1] = planes[3];
    a.status = d_status;
    a.iters_out = d_iters;
    a.elapsed = d_elapsed;
    a.done_ns = d_done;
    a.spins = d_spins;
    a.state_out = nullptr;
    JacobiLaunch l{};
    for (int bsel = 0; bsel < 2; ++bsel)
        for (int pl = 0; pl < 2; ++pl)
            if (!make_tmap_f16(&l.tm_s[bsel][pl], planes[2 * bsel + pl], slots, np, jacobi_umma_kc(), tm))
                return fail(MARS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the state planes");
    l.tm_jhi = p->tm_jhi_j;
    l.tm_jlo = p->tm_jlo_j;
    l.jlo = p->jlo;
    CUDA_TRY(launch_jacobi_umma(a, l, grid, st));
    EnergyArgs ea{n, p->dJ64, p->dOff, p->dIdx, p->dW64, p->dH64, p->coupling_sum,
                  count, d_spins, d_status, d_energy, d_cut};
    CUDA_TRY(launch_energy(ea, st));
    BestArgs ba{count, d_status, d_energy, d_part_e, d_part_i, d_best};
    CUDA_TRY(launch_best(ba, best_grid, st));
    std::vector<std::uint8_t> status(count);
    std::vector<double> energy(count), cut(count), elapsed(count);
    long long best = -1;
    CUDA_TRY(cudaMemcpyAsync(status.data(), d_status, count, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(energy.data(), d_energy, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(cut.data(), d_cut, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(elapsed.data(), d_elapsed, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&best, d_best, sizeof(long long), cudaMemcpyDeviceToHost, st));
    if (records && records->spins)
        CUDA_TRY(cudaMemcpyAsync(records->spins, d_spins, static_cast<std::size_t>(count) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int k = 0; k < count; ++k)
        if (status[k] != MARS_RUN_OK) return fail(MARS_ERR_RUNTIME, "run " + std::to_string(k) + " did not complete");
    if (best_spins && best >= 0)
        CUDA_TRY(cudaMemcpy(best_spins, d_spins + static_cast<std::size_t>(best) * n, n, cudaMemcpyDeviceToHost));
    if (records) {
        if (records->status) std::copy(status.begin(), status.end(), records->status);
        if (records->energy) std::copy(energy.begin(), energy.end(), records->energy);
        if (records->cut) std::copy(cut.begin(), cut.end(), records->cut);
        if (records->elapsed_seconds) std::copy(elapsed.begin(), elapsed.end(), records->elapsed_seconds);
        if (records->start_temp) std::fill(records->start_temp, records->start_temp + count, sched[0]);
        if (records->descent_iters) std::fill(records->descent_iters, records->descent_iters + count, iters);
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (int rc = mars_aggregate(count, status.data(), energy.data(), cut.data(), elapsed.data(),
                                p->integral ? 0.0 : 1e-9, secs, stats))
        return rc;
    if (stats->best_index != best)
        return fail(MARS_ERR_RUNTIME, "device best-of-R index disagrees with the host aggregation");
    return MARS_OK;
}

}  // namespace

extern "C" {

// TEST-ONLY (include/mars_b200.h): the device copy of the reference's stream
int mars_debug_rng(const uint64_t* seeds, int32_t streams, int32_t count, uint64_t* u64, double* gauss) {
    if (!seeds || !u64 || !gauss || streams < 1 || count < 1) return fail(MARS_ERR_INPUT, "bad argument");
    JacobiScratch sc;
    std::uint64_t *d_seeds, *d_st, *d_u;
    double* d_g;
    if (int rc = sc.alloc(&d_seeds, streams)) return rc;
    if (int rc = sc.alloc(&d_st, static_cast<std::size_t>(2) * kMtWords * streams)) return rc;
    if (int rc = sc.alloc(&d_u, static_cast<std::size_t>(streams) * count)) return rc;
    if (int rc = sc.alloc(&d_g, static_cast<std::size_t>(streams) * count)) return rc;
    CUDA_TRY(cudaMemcpy(d_seeds, seeds, streams * sizeof(std::uint64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(launch_rng_probe(d_seeds, streams, count, d_st, d_u, d_g, nullptr));
    CUDA_TRY(cudaMemcpy(u64, d_u, static_cast<std::size_t>(streams) * count * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(gauss, d_g, static_cast<std::size_t>(streams) * count * sizeof(double), cudaMemcpyDeviceToHost));
    return MARS_OK;
}

// run_batch with NmfaParams (validate: solvers.cpp:89-96; run: solvers.cpp:392-408)
int mars_run_batch_nmfa(mars_problem_t* p, const mars_nmfa_params_t* prm, int64_t runs, uint64_t base_seed,
                        mars_records_t* records, mars_stats_t* stats, int8_t* best_spins) {
    if (!p || !prm || !stats) return fail(MARS_ERR_INPUT, "null argument");
    if (!(prm->alpha > 0.0 && prm->alpha <= 1.0)) return fail(MARS_ERR_INPUT, "nmfa: alpha must lie in (0,1]");
    if (!(prm->noise_sigma >= 0.0)) return fail(MARS_ERR_INPUT, "nmfa: noise_sigma must be >= 0");
    if (prm->iters < 1) return fail(MARS_ERR_INPUT, "nmfa: iters must be >= 1");
    if (prm->schedule_len < 1 || !prm->schedule)
        return fail(MARS_ERR_INPUT, "nmfa: temperature schedule must not be empty");
    for (std::int64_t k = 0; k < prm->schedule_len; ++k)
        if (!(prm->schedule[k] >= 0.0)) return fail(MARS_ERR_INPUT, "nmfa: schedule temperatures must be >= 0");
    if (prm->iters > (1 << 30)) return fail(MARS_ERR_INPUT, "nmfa: iters too large");
    return run_jacobi(p, 0, prm->iters, prm->schedule, prm->schedule_len, prm->alpha, prm->noise_sigma, 0.0, runs,
                      base_seed, records, stats, best_spins);
}

// run_batch with SimCimParams (validate: solvers.cpp:98-103; run: solvers.cpp:426-443)
int mars_run_batch_simcim(mars_problem_t* p, const mars_simcim_params_t* prm, int64_t runs, uint64_t base_seed,
                          mars_records_t* records, mars_stats_t* stats, int8_t* best_spins) {
    if (!p || !prm || !stats) return fail(MARS_ERR_INPUT, "null argument");
    if (!(prm->step_size > 0.0)) return fail(MARS_ERR_INPUT, "simcim: step_size must be positive");
    if (!(prm->noise_sigma >= 0.0)) return fail(MARS_ERR_INPUT, "simcim: noise_sigma must be >= 0");
    if (prm->iters < 1) return fail(MARS_ERR_INPUT, "simcim: iters must be >= 1");
    if (prm->pump_schedule_len < 1 || !prm->pump_schedule)
        return fail(MARS_ERR_INPUT, "simcim: pump schedule must not be empty");
    if (prm->iters > (1 << 30)) return fail(MARS_ERR_INPUT, "simcim: iters too large");
    return run_jacobi(p, 1, prm->iters, prm->pump_schedule, prm->pump_schedule_len, 0.0, prm->noise_sigma,
                      prm->step_size, runs, base_seed, records, stats, best_spins);
}

// brute_force_ground_state (model.cpp:296-324): exhaustive Gray-code scan on the device
// (brute_force.cu), ties toward the lexicographically smallest spins; the energy reported is
// recomputed in the reference's exact order.
int mars_brute_force(const mars_problem_t* p, int32_t max_n, double* energy_out, int8_t* spins) {
    if (!p || !spins) return fail(MARS_ERR_INPUT, "null argument");
    const int n = p->n;
    if (n > max_n)
        return fail(MARS_ERR_INPUT, "brute force refused: n = " + std::to_string(n) + " exceeds guard " +
                                        std::to_string(max_n));
    if (n > brute_force_max_n())
        return fail(MARS_ERR_INPUT, "brute force supports n <= " + std::to_string(brute_force_max_n()));
    CUDA_TRY(cudaSetDevice(p->device));
    std::vector<double> J(static_cast<std::size_t>(n) * n, 0.0);
    CUDA_TRY(mars_problem_rows(p, J.data()) == MARS_OK ? cudaSuccess : cudaErrorInvalidValue);
    const int blocks = std::max(1, std::min(p->num_sms * 4, static_cast<int>(((1ull << n) + 255) / 256)));
    double* dJ = nullptr;
    double* dh = nullptr;
    double* de = nullptr;
    unsigned* dk = nullptr;
    CUDA_TRY(cudaMalloc(&dJ, J.size() * sizeof(double)));
    CUDA_TRY(cudaMalloc(&dh, n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&de, blocks * sizeof(double)));
    CUDA_TRY(cudaMalloc(&dk, blocks * sizeof(unsigned)));
    CUDA_TRY(cudaMemcpyAsync(dJ, J.data(), J.size() * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(dh, p->h.data(), n * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(launch_brute_force(dJ, dh, n, de, dk, blocks, p->stream));
    std::vector<double> e(blocks);
    std::vector<unsigned> k(blocks);
    CUDA_TRY(cudaMemcpyAsync(e.data(), de, blocks * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaMemcpyAsync(k.data(), dk, blocks * sizeof(unsigned), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    cudaFree(dJ);
    cudaFree(dh);
    cudaFree(de);
    cudaFree(dk);
    int best = 0;
    for (int b = 1; b < blocks; ++b)
        if (e[b] < e[best] || (e[b] == e[best] && k[b] < k[best])) best = b;
    for (int i = 0; i < n; ++i)   // key = bit-reversed mask: bit (n-1-i) of the key is spin i
        spins[i] = ((k[best] >> (n - 1 - i)) & 1u) ? 1 : -1;
    return energy_out ? mars_energy(p, spins, energy_out, nullptr) : MARS_OK;
}

// ------------------------------------------------------------ instance generators

void mars_gen_sk_gaussian(int32_t n, uint64_t seed, double* J) {           // io.cpp:151-163
    Stream r(seed);
    std::memset(J, 0, sizeof(double) * static_cast<std::size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = r.gaussian();
            J[static_cast<std::size_t>(i) * n + k] = w;
            J[static_cast<std::size_t>(k) * n + i] = w;
        }
}

void mars_gen_sk_pm1(int32_t n, uint64_t seed, double* J) {
    Stream r(seed);
    std::memset(J, 0, sizeof(double) * static_cast<std::size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = r.coin();
            J[static_cast<std::size_t>(i) * n + k] = w;
            J[static_cast<std::size_t>(k) * n + i] = w;
        }
}

int64_t mars_gen_er(int32_t n, double prob, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    Stream r(seed);
    std::int64_t m = 0;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            if (r.open01() < prob) {
                if (u) {
                    u[m] = a;
                    v[m] = b;
                    w[m] = 1.0;
                }
                ++m;
            }
    return m;
}

int64_t mars_gen_ea(int32_t L, int32_t dims, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    Stream r(seed);
    std::int64_t nsite = 1;
    for (int d = 0; d < dims; ++d) nsite *= L;
    std::int64_t m = 0;
    for (std::int64_t i = 0; i < nsite; ++i) {
        std::int64_t stride = 1;
        for (int d = 0; d < dims; ++d) {
            const std::int64_t c = (i / stride) % L;
            const std::int64_t j = i + (c == L - 1 ? -static_cast<std::int64_t>(L - 1) * stride : stride);
            const double wt = r.coin();
            if (u) {
                u[m] = static_cast<int32_t>(i);
                v[m] = static_cast<int32_t>(j);
                w[m] = wt;
            }
            ++m;
            stride *= L;
        }
    }
    return m;
}

}  // extern "C"
