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
    std::int8_t* spins;        // [count][n] rounded final state (round_spins, model.cpp:245)
    // optional per-CTA phase counters (clock64 cycles), kProfSlots per CTA, or nullptr
    long long* prof;
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

// tcgen05 dense kernel: TMA maps over the fp16 state planes ([grid*128][np], per batch)
// and the fp16 coupling planes ([np][np], per problem).
struct UmmaLaunch {
    CUtensorMap tm_shi, tm_slo, tm_jhi, tm_jlo;
    __half* s_hi;
    __half* s_lo;
    bool jlo;   // Gaussian couplings need the J_lo product; integer ones are exact in J_hi
};
cudaError_t launch_relax_dense_umma(const RelaxArgs& a, const UmmaLaunch& u, int grid, cudaStream_t st);
int relax_dense_umma_slots_per_cta();
int relax_dense_umma_block();
std::size_t relax_dense_umma_plane_rows(int grid);

// Level-scheduled sparse kernel (relax_csr.cu).  Spins grouped by Gauss-Seidel level,
// levels cut into 32-spin chunks, each chunk's neighbour lists interleaved [k][32].
struct SparseLevels {
    int nlev;
    const int* lvl_chunk;      // [nlev + 1] first chunk of each level
    const int* chunk_base;     // [nchunks] offset of the chunk's [md][32] neighbour block
    const int* chunk_md;       // [nchunks] longest neighbour list in the chunk
    const int* spin;           // [nchunks * 32] spin of each lane, -1 for padding
    const int* nidx;           // interleaved neighbour indices (n = the +0.0 padding slot);
                               //  unit couplings carry the weight's sign in bit 31
    const double* nw;          // interleaved weights (non-unit couplings), padding 0.0
    bool unit;                 // every |J_ij| == 1
};
struct SparseLaunch {
    int grid;
    int warps;                 // warps per CTA (one run slot per CTA)
    bool smem_state;           // state in shared memory ([n+1] doubles) or a global row
};
cudaError_t launch_relax_sparse(const RelaxArgs& a, const SparseLevels& g, const SparseLaunch& l,
                                cudaStream_t st);
int relax_sparse_occupancy(const SparseLaunch& l, bool unit, int n);

cudaError_t launch_energy(const EnergyArgs& a, cudaStream_t st);
cudaError_t launch_best(const BestArgs& a, int grid, cudaStream_t st);

}  // namespace marsb200
