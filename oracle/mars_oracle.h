/*
 * mars_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Two interchangeable CPU implementations of the MARS hot path sit behind this one
 * C interface, distinguished only by the symbol prefix:
 *
 *   ref_*  oracle/ref_driver.cpp  -- a thin extern "C" shim over the REFERENCE's own
 *          C++ sources (/root/reference/proj/src/{model,solvers,runner}.cpp), compiled by
 *          oracle/Makefile into oracle/_ref/libmars_ref.so.  This is "the reference
 *          itself run here".
 *   orc_*  oracle/mars_oracle.c   -- a plain-C restatement of the same algorithm, each
 *          function citing the reference file:line it follows; compiled into
 *          oracle/libmars_oracle.so.  Pinned bit-for-bit against ref_* and against the
 *          committed golden fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library.  The product (paper_1907_05124_b200/) never links them.
 */
#ifndef MARS_ORACLE_H
#define MARS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* MarsParams (reference include/mars/solvers.hpp:20-27). start_mode: 0 GridSweep, 1 UniformRandom. */
typedef struct {
    double t_min, t_max, t_step, c_step, d_min;
    int32_t start_mode;
    int32_t pad_;
} orc_params_t;

/* RunResult fields as caller-owned arrays (reference solvers.hpp:95-106). Any may be NULL. */
typedef struct {
    uint8_t* status;        /* 0 Ok, 1 Skipped, 2 Diverged */
    double* energy;
    double* cut;
    double* start_temp;
    int64_t* descent_iters;
    double* elapsed_seconds;
    int8_t* spins;          /* [count * n] */
} orc_records_t;

/* BatchStats scalars (reference runner.hpp:29-44) plus the index of best_result. */
typedef struct {
    double best_energy, mean_energy, best_cut, mean_cut;
    int64_t hit_count;
    double success_probability, total_seconds, mean_seconds_per_run;
    int64_t best_index, completed_runs, skipped_runs, failed_runs;
} orc_stats_t;

#define ORC_DECLARE(P)                                                                        \
    uint64_t P##splitmix64(uint64_t x);                                                       \
    uint64_t P##sub_seed(uint64_t base, uint64_t index);                                      \
    /* kind: 0 next_u64, 1 uniform_open01, 2 uniform_open_sym, 3 gaussian, 4 coin_spin,       \
       5 below(arg) */                                                                        \
    void P##rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t count, uint64_t* out_u64, \
                      double* out_f64);                                                       \
    void* P##problem_dense(int n, const double* J, const double* h, char* err, int errlen);   \
    void* P##problem_edges(int n, int64_t m, const int32_t* u, const int32_t* v,              \
                           const double* w, const double* h, char* err, int errlen);          \
    void P##problem_free(void* p);                                                            \
    void P##problem_info(const void* p, int* n, int* adjacency, int* integral,                \
                         double* coupling_sum, int64_t* nnz);                                 \
    double P##energy(const void* p, const int8_t* spins);                                     \
    double P##cut_value(const void* p, const int8_t* spins);                                  \
    double P##coupling_term(const void* p, const int8_t* spins);                              \
    double P##tanh_trial(double phi, double t);                                               \
    double P##relax_sweep(const void* p, double* s, double t);                                \
    int P##relax_to_fixed_point(const void* p, double* s, double t, double d_min,             \
                                int64_t* budget, int64_t* sweeps);                            \
    int P##validate(const orc_params_t* prm, char* err, int errlen);                          \
    int P##run_count(const orc_params_t* prm, int64_t requested, int64_t* out, char* err,     \
                     int errlen);                                                             \
    void P##run_plan(const orc_params_t* prm, uint64_t base_seed, int64_t index,              \
                     int* skipped, double* start_temp, uint64_t* seed);                       \
    void P##initial_state(uint64_t seed, int n, double* s);                                   \
    int P##descent(const void* p, double start_temp, const orc_params_t* prm, uint64_t seed,  \
                   uint8_t* status, double* energy, double* cut, int64_t* iters,              \
                   int8_t* spins, char* err, int errlen);                                     \
    /* run_batch over runs [0, runs) with `workers` threads; records for every index */       \
    int P##run_batch(const void* p, const orc_params_t* prm, int64_t runs, uint64_t base_seed, \
                     int workers, orc_records_t* rec, orc_stats_t* stats, char* err,           \
                     int errlen);                                                             \
    /* instance generators built only from the reference Rng */             \
    void P##gen_sk_gaussian(int n, uint64_t seed, double* J);                                 \
    void P##gen_sk_pm1(int n, uint64_t seed, double* J);                                      \
    int64_t P##gen_er(int n, double prob, uint64_t seed, int32_t* u, int32_t* v, double* w);  \
    int64_t P##gen_ea(int L, int dims, uint64_t seed, int32_t* u, int32_t* v, double* w);

ORC_DECLARE(ref_)
ORC_DECLARE(orc_)

/* port-only test knob: override kMarsSweepCap (0 restores 10^6) */
void orc_set_sweep_cap(int64_t cap);
/* TEST-ONLY (ref_driver.cpp, reference only): run_batch with NmfaParams / SimCimParams. */
int ref_run_batch_nmfa(const void* p, double noise_sigma, double alpha, int64_t iters, const double* sched,
                       int64_t sched_len, int64_t runs, uint64_t base_seed, int workers, orc_records_t* rec,
                       orc_stats_t* st, char* err, int errlen);
int ref_run_batch_simcim(const void* p, double step_size, double noise_sigma, int64_t iters, const double* sched,
                         int64_t sched_len, int64_t runs, uint64_t base_seed, int workers, orc_records_t* rec,
                         orc_stats_t* st, char* err, int errlen);
/* TEST-ONLY measurement tool (mars_oracle.c): the reference descent replayed in fp32
 * (mode 0) or fp32 with J rounded to one fp16 plane (mode 1); dense problems only. */
double orc_relax_sweep_f32(const void* p, float* s, double t);
int orc_replay_batch_f32(const void* p, const orc_params_t* prm, int64_t runs, uint64_t base_seed,
                         int workers, int mode, uint8_t* status, int64_t* iters, int8_t* spins);

#ifdef __cplusplus
}
#endif
#endif
