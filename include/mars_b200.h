/*
 * mars_b200.h -- C-ABI of the B200-native MARS batched-descent engine.
 *
 * This is the drop-in seam for the reference's batch API.  The reference (a C++20 header
 * library under /root/reference/proj) has no FFI of its own; the natural replacement point
 * is `mars::run_batch(const IsingProblem&, const BatchSpec&) -> BatchStats`
 * (include/mars/runner.hpp:55-56).  Each entry point below names the reference interface
 * it replaces.  Plain pointers and sizes only; all host arrays are caller-owned.
 *
 * Every compute call runs hand-written sm_100a kernels on the problem's device.  There is
 * no CPU fallback: with no usable CUDA device, problem creation fails with MARS_ERR_CUDA.
 */
#ifndef MARS_B200_H
#define MARS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (C++ wrappers rethrow the reference's exception classes) ---------- */
enum {
    MARS_OK = 0,
    MARS_ERR_INPUT = 1,      /* mars::InputError (errors.hpp:16)                            */
    MARS_ERR_RUNTIME = 2,    /* mars::Error (errors.hpp:11)                                  */
    MARS_ERR_CUDA = 3,       /* CUDA runtime failure or no device                            */
    MARS_ERR_NCCL = 4,       /* NCCL missing or a collective of the multi-GPU exchange failed */
    MARS_ERR_ALL_FAILED = 5  /* "batch failed: no run completed" (runner.cpp:153-155)        */
};

/* RunStatus (solvers.hpp:95) */
enum { MARS_RUN_OK = 0, MARS_RUN_SKIPPED = 1, MARS_RUN_DIVERGED = 2 };

/* StartMode (solvers.hpp:18) */
enum { MARS_GRID_SWEEP = 0, MARS_UNIFORM_RANDOM = 1 };

/* Kernel family selection for a problem handle. AUTO picks by storage (dense vs CSR). */
enum { MARS_KERNEL_AUTO = 0, MARS_KERNEL_DENSE_SIMT = 1, MARS_KERNEL_CSR = 2,
       MARS_KERNEL_DENSE_UMMA = 3 };

/* MarsParams (solvers.hpp:20-27).  sweep_cap = 0 means kMarsSweepCap = 10^6
 * (solvers.hpp:116); a positive value overrides it (fault injection in tests). */
typedef struct {
    double t_min, t_max, t_step, c_step, d_min;
    int32_t start_mode;
    int32_t reserved;
    int64_t sweep_cap;
} mars_params_t;

/* IsingProblem metadata (model.hpp:52-70). */
typedef struct {
    int32_t n;
    int32_t uses_adjacency;  /* CSR storage (edge density < 5%, model.cpp:91)            */
    int32_t integral;
    int32_t has_field;
    double coupling_sum;     /* ordered sum in storage order (model.cpp:20-45)           */
    int64_t nonzeros;
    int32_t device;
    int32_t kernel;          /* MARS_KERNEL_* actually used by mars_run_* on this handle  */
    int32_t levels;          /* Gauss-Seidel levels of one sweep (sparse layouts; 0 dense) */
    int32_t reserved;
} mars_problem_info_t;

/* RunResult fields (solvers.hpp:97-106), one entry per run index, caller-allocated.
 * Any pointer may be NULL.  spins is [count * n] int8 (+1/-1), row per run. */
typedef struct {
    uint8_t* status;
    double* energy;
    double* cut;
    double* start_temp;
    int64_t* descent_iters;
    double* elapsed_seconds;
    int8_t* spins;
    double* fail_temp;       /* Diverged runs: the level temperature T of DivergedError's
                                "relaxation exceeded the sweep cap at T = " (solvers.cpp:169) */
} mars_records_t;

/* BatchStats scalars (runner.hpp:29-44); best_index is the run index of best_result. */
typedef struct {
    double best_energy, mean_energy, best_cut, mean_cut;
    int64_t hit_count;
    double success_probability, total_seconds, mean_seconds_per_run;
    int64_t best_index, completed_runs, skipped_runs, failed_runs;
} mars_stats_t;

/* Device-side timing of the last executed batch (CUDA events on the handle's stream). */
typedef struct {
    double relax_ms;         /* the persistent relaxation kernel (dominant kernel)          */
    double energy_ms;        /* round + exact energy/cut kernel                              */
    double reduce_ms;        /* best-of-R reduction                                          */
    double total_ms;         /* first to last event of mars_batch_execute                   */
    int64_t launches;        /* kernels launched by mars_batch_execute                      */
    int64_t total_sweeps;    /* sum of descent_iters over the batch                          */
    int32_t grid;            /* CTAs of the relaxation kernel                                */
    int32_t slots;           /* concurrent descents (run slots) on the device                */
    int32_t kernel;          /* relaxation kernel this batch ran: MARS_KERNEL_* or 4 = small  */
    int32_t split;           /* tcgen05 kernel: CTA pairs per 256-run tile (K split), else 1  */
} mars_timing_t;

typedef struct mars_problem mars_problem_t;
typedef struct mars_batch mars_batch_t;

/* Thread-local message of the last failing call on this thread. */
const char* mars_last_error(void);

/* Library / device facts. */
int mars_device_count(int* out);

/* ---- problem store (IsingProblem, model.hpp:23-101) -------------------------------- */

/* IsingProblem::dense (model.hpp:41, model.cpp:47-72): J is n*n row-major fp64, symmetric
 * with zero diagonal; h may be NULL.  Copies the couplings to `device` in the layouts the
 * kernels use.  kernel = MARS_KERNEL_*. */
int mars_problem_dense(int32_t n, const double* J, const double* h, int32_t device,
                       int32_t kernel, mars_problem_t** out);

/* IsingProblem::from_edges (model.hpp:46, model.cpp:74-131): same 5% dense/CSR rule. */
int mars_problem_from_edges(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                            const double* w, const double* h, int32_t device, int32_t kernel,
                            mars_problem_t** out);

/* Staged batches (mars_batch_*) keep their problem alive: the handle and every live batch
 * hold one reference; the last of mars_problem_destroy / mars_batch_destroy frees it. */
void mars_problem_destroy(mars_problem_t* p);
int mars_problem_info(const mars_problem_t* p, mars_problem_info_t* out);

/* problem_hash (io.hpp, io.cpp:260-290): FNV-1a over n, the stored upper-triangle couplings in
 * visit_upper order and the nonzero field entries.  mars_instance_hash hashes an instance
 * given as dense J (J != NULL) or an edge list, with the same validation and storage rule as
 * the constructors, without touching a device. */
int mars_problem_hash(const mars_problem_t* p, uint64_t* out);
int mars_instance_hash(int32_t n, const double* J, int64_t m, const int32_t* u, const int32_t* v,
                       const double* w, const double* h, uint64_t* out);

/* brute_force_ground_state (model.hpp:139, model.cpp:296-324): exhaustive 2^n Gray-code scan
 * on the device, n <= max_n (and <= 26); ties toward the lexicographically smallest spins
 * (-1 before +1).  Exact for integer couplings. */
int mars_brute_force(const mars_problem_t* p, int32_t max_n, double* energy, int8_t* spins);

/* All n rows of IsingProblem::row_values (model.cpp:173-182) into out[n*n] (write_matrix). */
int mars_problem_rows(const mars_problem_t* p, double* out);

/* energy / cut_value of one spin vector, on the device, exact reference order
 * (model.cpp:203-229). */
int mars_energy(const mars_problem_t* p, const int8_t* spins, double* energy, double* cut);

/* ---- parameters and plan (solvers.hpp:18-35,133-139; solvers.cpp:35-52,202-227) -------- */

int mars_validate_params(const mars_params_t* prm);                 /* validate(MarsParams) */
int mars_run_count(const mars_params_t* prm, int64_t requested, int64_t* out);
int mars_run_plan(const mars_params_t* prm, uint64_t base_seed, int64_t index,
                  int32_t* skipped, double* start_temp, uint64_t* seed);
/* The descent's initial state s_i = Rng(seed).uniform_open_sym() (solvers.cpp:184-187). */
int mars_initial_state(uint64_t seed, int32_t n, double* s);
uint64_t mars_splitmix64(uint64_t x);                               /* rng.hpp:13  */
uint64_t mars_sub_seed(uint64_t base_seed, uint64_t run_index);     /* rng.hpp:20  */

/* ---- the batch (run_batch, runner.hpp:55-56 / runner.cpp:170-178) ------------------------
 *
 * One call = validate, plan on host threads, H2D of initial states and start
 * temperatures, persistent relaxation kernel, exact energy/cut kernel, best-of-R
 * reduction, D2H of the per-run records, and the reference's index-order aggregation
 * (runner.cpp:126-167).  `runs` has the reference meaning (ignored by GridSweep).
 * `records` and `best_spins` (n bytes) may be NULL. */
int mars_run_batch(mars_problem_t* p, const mars_params_t* prm, int64_t runs,
                   uint64_t base_seed, mars_records_t* records, mars_stats_t* stats,
                   int8_t* best_spins);

/* run_batch with a ProgressFn (runner.hpp:52-56): progress(run index, best energy so far,
 * user) is called from the calling thread once per run while the batch runs -- in completion
 * order, best_so_far non-increasing, skipped grid slots first -- as the reference's worker
 * pool does (runner.cpp:107-113).  The kernels log each run into host-mapped memory when its
 * rounded spins are written; the finished runs' exact energies are evaluated on a side stream
 * (concurrently with the relaxation kernel when it leaves SMs free, else right after it). */
int mars_run_batch_progress(mars_problem_t* p, const mars_params_t* prm, int64_t runs,
                            uint64_t base_seed, mars_records_t* records, mars_stats_t* stats,
                            int8_t* best_spins, void (*progress)(int64_t index, double best_so_far, void* user),
                            void* user);

/* A contiguous shard [first, first+count) of the batch's run indices (for multi-GPU:
 * each rank runs its shard, the records are gathered, then mars_aggregate). */
int mars_run_shard(mars_problem_t* p, const mars_params_t* prm, int64_t runs,
                   uint64_t base_seed, int64_t first, int64_t count, mars_records_t* records);

/* ---- multi-GPU inside one call (SURVEY.md 8(b) device set, 8(e)) ------------------------
 *
 * mars_problem_replicate: the same problem (host copy, kernel family) stored on `device`.
 * mars_run_batch_multi: run_batch over `count` replicas on distinct devices -- the run
 * indices split into contiguous shards, one host thread + stream per device running its
 * shard, then one exchange over NCCL (loaded at run time; ncclCommInitAll over the devices):
 * AllReduce(min) of the shard best energies, AllReduce(min) of the first index attaining the
 * batch best, Broadcast of that run's spins from its owner, AllGather of every shard's
 * records; the index-order aggregation then runs once.  Results are identical to mars_run_batch
 * on one device (every run depends only on its index).  MARS_ERR_NCCL when NCCL is missing
 * or a collective fails.  count == 1 is mars_run_batch. */
int mars_problem_replicate(const mars_problem_t* p, int32_t device, mars_problem_t** out);
int mars_run_batch_multi(mars_problem_t* const* replicas, int32_t count, const mars_params_t* prm,
                         int64_t runs, uint64_t base_seed, mars_records_t* records, mars_stats_t* stats,
                         int8_t* best_spins);
/* TEST-ONLY: the shard / exchange logic of mars_run_batch_multi on host memory (the four
 * collectives between `ranks` host threads) over caller-given full-batch records (status,
 * energy, cut, descent_iters, elapsed, spins [total*n]); fills records/stats/best_spins like
 * the multi-device call.  Lets a machine without GPUs test the multi-GPU path. */
int mars_debug_exchange(int32_t ranks, int64_t total, int32_t n, const uint8_t* status, const double* energy,
                        const double* cut, const int64_t* iters, const double* elapsed, const int8_t* spins,
                        double energy_tolerance, mars_records_t* records, mars_stats_t* stats,
                        int8_t* best_spins);

/* TEST-ONLY: the tcgen05 kernel's large-N split-K choice (K1 "Split-K") on host
 * data: runs with the given start temperatures, `pairs` CTA pairs asked for, the resident
 * clusters of 2 / 4 / 8 CTAs, the SM count, the padded size np; forced = 2 or 4 forces the
 * split (0: choose).  Returns the split (1, 2, 4) and the tile (CTA-pair) count. */
int mars_debug_choose_split(const double* start_temps, int64_t count, const mars_params_t* prm, int32_t pairs,
                            const int32_t resident[3], int32_t num_sms, int32_t np, int32_t forced,
                            int32_t* split, int32_t* tiles);

/* The reference's aggregation (runner.cpp:126-167) over `count` records in index order.
 * energy_tolerance: 0 for integral problems, 1e-9 otherwise (model.hpp:82). */
int mars_aggregate(int64_t count, const uint8_t* status, const double* energy,
                   const double* cut, const double* elapsed_seconds, double energy_tolerance,
                   double total_seconds, mars_stats_t* stats);

/* ---- staged batch (for device-resident timing; mars_run_* are built from these) -------- */

int mars_batch_create(mars_problem_t* p, const mars_params_t* prm, int64_t runs,
                      uint64_t base_seed, int64_t first, int64_t count, mars_batch_t** out);
/* Host plan + H2D of the initial states (pinned staging). */
int mars_batch_upload(mars_batch_t* b);
/* Device work only (relax -> energy -> reduce), blocks until done; fills timing. */
int mars_batch_execute(mars_batch_t* b, mars_timing_t* timing);
/* D2H of the records (and optional per-run spins), best index and best spins. */
int mars_batch_fetch(mars_batch_t* b, mars_records_t* records, int64_t* best_index,
                     int8_t* best_spins);
/* Time-to-best support: per run, seconds from the launch's first descent
 * start to that run's retirement on the device (%globaltimer); 0 for skipped runs.  No
 * reference counterpart (the reference records only per-run elapsed_seconds). */
int mars_batch_fetch_finish(mars_batch_t* b, double* finish_seconds);
void mars_batch_destroy(mars_batch_t* b);

/* ---- the synchronous mean-field baselines (solvers.hpp:62-82, 154-158) ------------------
 *
 * run_batch with NmfaParams / SimCimParams (runner.cpp:31-60: run index k uses the stream
 * Rng(sub_seed(base_seed, k))): every run on the tcgen05 Jacobi kernel (one GEMM per
 * iteration, update + the run's Box-Muller noise fused into the epilogue), exact energies,
 * best-of-R and the reference's aggregation.  Same validation and messages as
 * validate(NmfaParams) / validate(SimCimParams).  The schedule is stretched over `iters` like
 * schedule_at (solvers.cpp:118-123); records.start_temp = schedule[0], descent_iters = iters. */
typedef struct {
    double noise_sigma;          /* NmfaParams::noise_sigma (0.15)                          */
    double alpha;                /* NmfaParams::alpha (0.15), in (0, 1]                     */
    int64_t iters;
    const double* schedule;      /* temperatures, >= 0 (nmfa_defaults: 2.0 -> 0.02, 64)    */
    int64_t schedule_len;
} mars_nmfa_params_t;
typedef struct {
    double step_size;            /* SimCimParams::step_size (0.1)                           */
    double noise_sigma;          /* SimCimParams::noise_sigma (0.03)                        */
    int64_t iters;
    const double* pump_schedule; /* simcim_defaults: -2.0 -> 1.0, 64 points                 */
    int64_t pump_schedule_len;
} mars_simcim_params_t;
int mars_run_batch_nmfa(mars_problem_t* p, const mars_nmfa_params_t* prm, int64_t runs, uint64_t base_seed,
                        mars_records_t* records, mars_stats_t* stats, int8_t* best_spins);
int mars_run_batch_simcim(mars_problem_t* p, const mars_simcim_params_t* prm, int64_t runs,
                          uint64_t base_seed, mars_records_t* records, mars_stats_t* stats,
                          int8_t* best_spins);

/* ---- TEST-ONLY hook: single sweeps through the device kernels -------------------------
 *
 * mars_relax_sweep (solvers.cpp:150-161) from caller-given states: for each of `count`
 * states s_in[k*n ..] (fp32), `sweeps` in-order Gauss-Seidel sweeps at the fixed temperature
 * temps[k] (T < 1e-12 is the quench) through the problem's dense relaxation kernel -- the
 * same kernel, launch shape and precision scheme mars_run_batch uses for this handle and
 * batch size (MARS_DENSE_SMALL applies) -- final states to s_out (fp32).  kernel_used
 * (may be NULL) receives the kernel that ran (mars_timing_t.kernel).  Dense handles only.
 * Exists so the tests can pin one sweep of the device path against the reference. */
int mars_debug_sweeps(mars_problem_t* p, int64_t count, const float* s_in, const double* temps,
                      int32_t sweeps, float* s_out, int32_t* kernel_used);

/* TEST-ONLY: the device copy of Rng(seed) (mt_device.cuh) for `streams` seeds: the first
 * `count` engine outputs and, from a second copy of the stream, the first `count` gaussian()
 * draws (rng.hpp:27-75), row per stream. */
int mars_debug_rng(const uint64_t* seeds, int32_t streams, int32_t count, uint64_t* u64, double* gauss);

/* ---- instance generators built from the reference Rng --------------- */
void mars_gen_sk_gaussian(int32_t n, uint64_t seed, double* J);     /* io.cpp:151-163 */
void mars_gen_sk_pm1(int32_t n, uint64_t seed, double* J);
int64_t mars_gen_er(int32_t n, double prob, uint64_t seed, int32_t* u, int32_t* v, double* w);
int64_t mars_gen_ea(int32_t L, int32_t dims, uint64_t seed, int32_t* u, int32_t* v, double* w);

#ifdef __cplusplus
}
#endif
#endif
