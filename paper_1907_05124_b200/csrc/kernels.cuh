// kernels.cuh -- device-side interface shared by the host driver and the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace marsb200 {

// Run-slot state machine constants (solvers.cpp:19, solvers.hpp:116).
constexpr double kTempFloor = 1e-12;
constexpr std::int64_t kSweepCap = 1000000;

// Everything the persistent relaxation kernels need.  One launch relaxes `queue_len`
// descents: slots pull queue positions from an atomic counter, so the longest-expected
// runs (highest start temperature, placed first by the host) start first.
struct RelaxArgs {
    int n;             // spins
    int np;            // padded spins (multiple of the kernel's block size)
    // dense couplings, fp32 row-major [np][np], zero padded
    const float* J32;
    const float* h32;          // [n] external field, or nullptr (fp32 kernels)
    const double* h64;         // [n] external field, or nullptr (fp64 kernels)
    // the runs of this launch
    int queue_len;             // descents to run
    const int* order;          // [queue_len] local run index, processing order
    const float* s0;           // [count][n] initial states, fp32 (dense fp32 kernels)
    const void* s0_64;         // [count][n] initial states, fp64 as drawn (fp64 kernels)
    const double* start_temp;  // [count]
    double c_step, d_min;
    long long sweep_cap;
    // scratch
    void* work;                // per-CTA slot state, kernel-specific layout
    int* queue_head;           // atomic counter, zero before launch
    // per-run outputs (local run index)
    std::uint8_t* status;
    long long* iters;
    double* elapsed;
    unsigned long long* done_ns;  // [count] %globaltimer when the run retired, or nullptr
    double* fail_temp;         // [count] level temperature of a Diverged run, or nullptr
    std::int8_t* spins;        // [count][n] rounded final state (round_spins, model.cpp:245)
    // optional per-CTA phase counters (clock64 cycles), kProfSlots per CTA, or nullptr
    long long* prof;
    // TEST-ONLY fixed-temperature mode (mars_debug_sweeps, dense kernels): when > 0 every run
    // does exactly this many Gauss-Seidel sweeps at T = start_temp[run] (no annealing
    // schedule, no convergence test) and its final continuous state goes to state_out
    // ([count][n] fp32) -- the device counterpart of mars_relax_sweep (solvers.cpp:150-161)
    int fixed_sweeps;
    float* state_out;
    // tcgen05 kernel: the field GEMM runs on J * 2^k (fp16 range); fields scale back by 2^-k
    float jscale;
    // progress during the batch (mars_run_batch_progress): when a run's rounded spins are in
    // memory its index is appended here (host-mapped, completion order), or nullptr
    int* retire_log;
    int* retire_head;          // device counter of retire_log entries
};
constexpr int kProfSlots = 16;

// Exact-order energy evaluation (model.cpp:203-229) over `count` rounded spin vectors.
struct EnergyArgs {
    int n;
    const double* J64;         // dense [n][n] fp64 (reference order), or nullptr
    const int* off;
    const int* idx;
    const double* w64;         // CSR weights fp64
    const double* h64;         // [n] or nullptr
    double coupling_sum;
    long long count;
    const std::int8_t* spins;  // [count][n]
    const std::uint8_t* status;
    double* energy;
    double* cut;
};

struct BestArgs {
    long long count;
    const std::uint8_t* status;
    const double* energy;
    double* part_energy;       // [grid]
    long long* part_index;     // [grid]
    long long* best_index;     // [1]
};

// Launchers (return cudaGetLastError()).
cudaError_t launch_relax_dense_simt(const RelaxArgs& a, int grid, cudaStream_t st);
int relax_dense_simt_slots_per_cta();
int relax_dense_simt_block();
std::size_t relax_dense_simt_work_bytes(int np);

// tcgen05 dense kernel (CTA pairs: grid must be even): TMA maps over the fp16 state planes
// ([grid*128][np], per batch) and the fp16 coupling planes ([np][np], per problem).
struct UmmaLaunch {
    CUtensorMap tm_shi, tm_slo, tm_jhi, tm_jlo;
    __half* s_hi;
    __half* s_lo;
    bool jlo;   // Gaussian couplings need the J_lo product; integer ones are exact in J_hi
    int split;  // 1, or 2: two CTA pairs per 256-run tile split the K range (large N)
    float* xpart;  // split 2: partial-field exchange [2][tile rows][128] fp32
};
cudaError_t launch_relax_dense_umma(const RelaxArgs& a, const UmmaLaunch& u, int grid, cudaStream_t st);
int relax_dense_umma_slots_per_cta();
int relax_dense_umma_block();
int relax_dense_umma_kc();      // K per pipeline stage (the TMA box width of both operand maps)
int relax_dense_umma_j_rows();  // coupling-tile rows per CTA of the pair (TMA box height of J maps)
std::size_t relax_dense_umma_plane_rows(int grid);
int relax_dense_umma_max_clusters(int split, bool jlo);   // resident clusters of 2*split CTAs
cudaError_t relax_dense_umma_hang_log(unsigned long long** host);   // host view of the hang record

// Synchronous mean-field baselines on tcgen05 (jacobi_umma.cu): NMFA (solver 0) and SimCIM
// (solver 1), solvers.cpp:374-443.  CTA pairs (grid even); 128 runs per CTA per tile round.
struct JacobiArgs {
    int n, np;
    int solver;                // 0 = NMFA, 1 = SimCIM
    int iters;
    const double* sched;       // [iters] schedule_at(...) per iteration: temperature / pump
    double noise_sigma;
    float alpha_f, one_minus_alpha_f, step_f;
    float jscale;              // 2^-k: the GEMM runs on J * 2^k (fp16 range)
    const float* norm;         // [np] NMFA normalisers sqrt(h_i^2 + sum_j J_ij^2) (fp32)
    const float* h32;          // [np] field or nullptr
    int queue_len;
    int* queue_head;
    const int* order;          // [queue_len] run index
    const std::uint64_t* seeds;   // [count] per-run rng seed (sub_seed(base, index))
    std::uint64_t* mt;         // [312][slots] mt19937_64 states (word-major)
    int slots;
    __half* s_hi[2];           // state double buffer, fp16 hi/lo planes [slots][np]
    __half* s_lo[2];
    std::uint8_t* status;
    long long* iters_out;
    double* elapsed;
    unsigned long long* done_ns;
    std::int8_t* spins;        // [count][n]
    float* state_out;          // TEST-ONLY final states [count][n] fp32, or nullptr
};
struct JacobiLaunch {
    CUtensorMap tm_s[2][2];    // [buffer][hi, lo]
    CUtensorMap tm_jhi, tm_jlo;
    bool jlo;
};
cudaError_t launch_jacobi_umma(const JacobiArgs& a, const JacobiLaunch& l, int grid, cudaStream_t st);
constexpr int kMtWords = 312;   // mt19937_64 state words per run slot (mt_device.cuh)
cudaError_t launch_rng_probe(const std::uint64_t* seeds, int streams, int count, std::uint64_t* st,
                             std::uint64_t* u64, double* gauss, cudaStream_t s);
int jacobi_umma_slots_per_cta();
int jacobi_umma_kc();            // K per stage of the Jacobi kernel (the TMA box width of its maps)

// Level-scheduled sparse kernel (relax_csr.cu).  Spins grouped by Gauss-Seidel level,
// levels cut into cw-spin chunks, each chunk's neighbour lists interleaved [k][cw].
struct SparseLevels {
    int nlev;
    const int* lvl_chunk;      // [nlev + 1] first chunk of each level
    const int4* ctab;          // [nchunks] {block offset (ints), block length (ints),
                               //            weight offset (doubles), md}
    const int* blk;            // chunk blocks: [md,0,0,0][spin x cw (-1 pad)][idx: md x cw]
                               //  idx n = the +0.0 padding row; unit couplings carry the
                               //  weight's sign in bit 31
    const double* wblk;        // non-unit couplings: weight blocks [md x cw], padding 0.0
    int nchunks;               // chunks per sweep
    unsigned buf_bytes;        // one chunk buffer in shared memory (16-byte multiple)
    unsigned wbuf_off;         // weight block offset inside a chunk buffer
    bool unit;                 // every |J_ij| == 1
};
struct SparseLaunch {
    int grid;
    int warps;                 // warps per CTA (<= 16)
    int cw;                    // chunk width (spins per chunk): 32 or 16, as the layout was built
    int r;                     // runs per lane: 1, 2 or 4; a CTA holds (32/cw)*r run slots
    bool smem_state;           // state in shared memory ([n+1] doubles) or a global row
};
cudaError_t launch_relax_sparse(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l,
                                cudaStream_t st);
int relax_sparse_occupancy(const SparseLaunch& l, const SparseLevels& g, int n);
bool relax_sparse_shape_ok(int cw, int r);

// Warp-per-run sparse kernel (relax_spmm.cu): one CTA per SM, `warps` consumer warps each
// holding 32/cw runs in shared memory, plus a producer warp streaming the chunk blocks
// through a `ring_bytes` TMA byte ring (>= the largest block, 16-byte multiple).
struct SpmmLaunch {
    int grid;
    int warps;
    int ring_bytes;
    int cw;                    // chunk (layout) width: 16, 32 or 64
    int h;                     // lane groups per warp (1 or 2); spins per lane = cw * h / 32 (1 or 2)
    int r;                     // runs per lane group (1, or 2 with one spin per lane), interleaved
};
cudaError_t launch_relax_spmm(const RelaxArgs& a, const SparseLevels& g, const SpmmLaunch& l, cudaStream_t st);
std::size_t relax_spmm_smem(int np, int runs_per_warp, int warps, int ring_bytes);
int relax_spmm_max_warps();
bool relax_spmm_shape_ok(int layout_width, int runs_per_warp);

// Torus stencil kernel (relax_stencil.cu): L^dims lattice with unit couplings.
struct StencilArgs {
    int dims;                  // 2 or 3
    int L;                     // side (3..256)
    int nlev;                  // dims*(L-1)+1 Gauss-Seidel levels (coordinate sums)
    const int* lvl_off;        // [nlev + 1] first site of each level in `coords`
    const unsigned* coords;    // [n] sites by level: c0 | c1 << 8 | c2 << 16 | signs << 24,
                               //  sign bit k = the k-th smallest neighbour's coupling is -1
};
struct StencilLaunch {
    int grid;
    int threads;               // per CTA (one run per CTA)
    bool smem_state;           // state in shared memory, else a global row per CTA
};
cudaError_t launch_relax_stencil(const RelaxArgs& a, const StencilArgs& g, const StencilLaunch& l, cudaStream_t st);
std::size_t relax_stencil_smem(int n, int nlev, bool smem_state);

// Small dense instances with integer couplings (relax_small.cu): one warp per run, J (fp16)
// and fields on chip; for batches too small to fill the tensor-core kernel.
cudaError_t launch_relax_small(const RelaxArgs& a, const __half* J, int grid, int warps, cudaStream_t st);
int relax_small_max_n();
int relax_small_slots_per_cta();

// Exhaustive ground-state scan (brute_force.cu), n <= brute_force_max_n().
int brute_force_max_n();
cudaError_t launch_brute_force(const double* J, const double* h, int n, double* part_e, unsigned* part_key,
                               int blocks, cudaStream_t st);

cudaError_t launch_energy(const EnergyArgs& a, cudaStream_t st);
// energies of the runs list[0..a.count) (thread per run), compact outputs out_e / out_st [a.count]
cudaError_t launch_energy_list(const EnergyArgs& a, const int* list, double* out_e, std::uint8_t* out_st,
                               cudaStream_t st);
cudaError_t launch_best(const BestArgs& a, int grid, cudaStream_t st);

}  // namespace marsb200
