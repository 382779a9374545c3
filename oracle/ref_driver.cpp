// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// An extern "C" shim over the reference's own C++ library so the parity tests, the golden
// generator and bench.py's CPU baseline can call the reference itself.  Compiled together
// with /root/reference/proj/src/{model,solvers,runner}.cpp by oracle/Makefile into
// oracle/_ref/libmars_ref.so.  Nothing here re-implements the algorithm: every entry
// point forwards to the reference function named in its comment.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mars/errors.hpp"
#include "mars/model.hpp"
#include "mars/rng.hpp"
#include "mars/runner.hpp"
#include "mars/solvers.hpp"

#include "mars_oracle.h"

namespace {

void put_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) {
        std::strncpy(err, msg, static_cast<std::size_t>(errlen) - 1);
        err[errlen - 1] = '\0';
    }
}

mars::MarsParams to_params(const orc_params_t* p) {
    mars::MarsParams m;
    m.t_min = p->t_min;
    m.t_max = p->t_max;
    m.t_step = p->t_step;
    m.c_step = p->c_step;
    m.d_min = p->d_min;
    m.start_mode = p->start_mode ? mars::StartMode::UniformRandom : mars::StartMode::GridSweep;
    return m;
}

const mars::IsingProblem& P(const void* p) { return *static_cast<const mars::IsingProblem*>(p); }

mars::SpinConfig spins_of(const void* p, const int8_t* s) {
    return mars::SpinConfig(s, s + P(p).size());
}

}  // namespace

extern "C" {

uint64_t ref_splitmix64(uint64_t x) { return mars::splitmix64(x); }               // rng.hpp:13
uint64_t ref_sub_seed(uint64_t b, uint64_t i) { return mars::sub_seed(b, i); }    // rng.hpp:20

void ref_rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t count, uint64_t* ou,
                   double* of) {                                                   // rng.hpp:27-83
    mars::Rng r(seed);
    for (int64_t k = 0; k < count; ++k) {
        switch (kind) {
            case 0: ou[k] = r.next_u64(); break;
            case 1: of[k] = r.uniform_open01(); break;
            case 2: of[k] = r.uniform_open_sym(); break;
            case 3: of[k] = r.gaussian(); break;
            case 4: of[k] = r.coin_spin(); break;
            default: ou[k] = r.below(arg); break;
        }
    }
}

void* ref_problem_dense(int n, const double* J, const double* h, char* err, int errlen) {
    try {                                                                          // model.cpp:47
        std::vector<double> j(J, J + static_cast<std::size_t>(n > 0 ? n : 0) * (n > 0 ? n : 0));
        std::vector<double> f;
        if (h) f.assign(h, h + n);
        return new mars::IsingProblem(mars::IsingProblem::dense(n, std::move(j), std::move(f)));
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return nullptr;
    }
}

void* ref_problem_edges(int n, int64_t m, const int32_t* u, const int32_t* v, const double* w,
                        const double* h, char* err, int errlen) {
    try {                                                                          // model.cpp:74
        std::vector<mars::IsingProblem::Edge> edges(static_cast<std::size_t>(m));
        for (int64_t k = 0; k < m; ++k) edges[static_cast<std::size_t>(k)] = {u[k], v[k], w[k]};
        std::vector<double> f;
        if (h) f.assign(h, h + n);
        return new mars::IsingProblem(mars::IsingProblem::from_edges(n, edges, std::move(f)));
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return nullptr;
    }
}

void ref_problem_free(void* p) { delete static_cast<mars::IsingProblem*>(p); }

void ref_problem_info(const void* p, int* n, int* adjacency, int* integral, double* csum,
                      int64_t* nnz) {
    *n = P(p).size();
    *adjacency = P(p).uses_adjacency();
    *integral = P(p).integral();
    *csum = P(p).coupling_sum();
    *nnz = P(p).nonzeros();
}

double ref_energy(const void* p, const int8_t* s) { return mars::energy(P(p), spins_of(p, s)); }
double ref_cut_value(const void* p, const int8_t* s) {
    return mars::cut_value(P(p), spins_of(p, s));
}
double ref_coupling_term(const void* p, const int8_t* s) {
    return mars::coupling_term(P(p), spins_of(p, s));
}
double ref_tanh_trial(double phi, double t) { return mars::tanh_trial(phi, t); }

double ref_relax_sweep(const void* p, double* s, double t) {                     // solvers.cpp:150
    mars::ContinuousState st(s, s + P(p).size());
    const double d = mars::mars_relax_sweep(P(p), st, t);
    std::memcpy(s, st.data(), st.size() * sizeof(double));
    return d;
}

int ref_relax_to_fixed_point(const void* p, double* s, double t, double d_min, int64_t* budget,
                             int64_t* sweeps) {                                    // solvers.cpp:163
    mars::ContinuousState st(s, s + P(p).size());
    int rc = 0;
    try {
        std::int64_t b = *budget;
        *sweeps = mars::relax_to_fixed_point(P(p), st, t, d_min, b);
        *budget = b;
    } catch (const mars::DivergedError& e) {
        st = e.partial_state;
        *sweeps = e.sweeps;
        *budget = 0;
        rc = 1;
    }
    std::memcpy(s, st.data(), st.size() * sizeof(double));
    return rc;
}

int ref_validate(const orc_params_t* prm, char* err, int errlen) {
    try {
        mars::validate(to_params(prm));                                            // solvers.cpp:35
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_run_count(const orc_params_t* prm, int64_t requested, int64_t* out, char* err,
                  int errlen) {
    try {
        *out = mars::mars_run_count(to_params(prm), requested);                   // solvers.cpp:202
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

void ref_run_plan(const orc_params_t* prm, uint64_t base, int64_t idx, int* skipped, double* t,
                  uint64_t* seed) {
    const mars::MarsRunPlan plan = mars::mars_run_plan(to_params(prm), base, idx); // solvers.cpp:215
    *skipped = plan.skipped;
    *t = plan.start_temp;
    *seed = plan.seed;
}

void ref_initial_state(uint64_t seed, int n, double* s) {                          // solvers.cpp:184-187
    mars::Rng rng(seed);
    for (int i = 0; i < n; ++i) s[i] = rng.uniform_open_sym();
}

int ref_descent(const void* p, double start_temp, const orc_params_t* prm, uint64_t seed,
                uint8_t* status, double* energy, double* cut, int64_t* iters, int8_t* spins,
                char* err, int errlen) {
    try {
        const mars::RunResult r = mars::mars_descent(P(p), start_temp, to_params(prm), seed);
        *status = static_cast<uint8_t>(r.status);
        *energy = r.energy;
        *cut = r.cut;
        *iters = r.descent_iters;
        if (spins) std::memcpy(spins, r.spins.data(), r.spins.size());
        return 0;
    } catch (const mars::DivergedError& e) {
        *status = 2;
        *iters = e.sweeps;
        const auto sp = mars::round_spins(e.partial_state);
        *energy = mars::energy(P(p), sp);
        *cut = mars::cut_value(P(p), sp);
        if (spins) std::memcpy(spins, sp.data(), sp.size());
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

namespace {
// BatchStats -> the C records / stats (index order; best_result = first strict minimum)
void fill_batch(const mars::IsingProblem& prob, const mars::BatchStats& s, orc_records_t* rec, orc_stats_t* st) {
    const int n = prob.size();
    int64_t best_index = -1;
    for (std::size_t k = 0; k < s.runs.size(); ++k) {
        const mars::RunResult& r = s.runs[k];
        if (rec) {
            if (rec->status) rec->status[k] = static_cast<uint8_t>(r.status);
            if (rec->energy) rec->energy[k] = r.energy;
            if (rec->cut) rec->cut[k] = r.cut;
            if (rec->start_temp) rec->start_temp[k] = r.start_temp;
            if (rec->descent_iters) rec->descent_iters[k] = r.descent_iters;
            if (rec->elapsed_seconds) rec->elapsed_seconds[k] = r.elapsed_seconds;
            if (rec->spins && r.spins.size() == static_cast<std::size_t>(n))
                std::memcpy(rec->spins + k * static_cast<std::size_t>(n), r.spins.data(),
                            static_cast<std::size_t>(n));
        }
        // best_result is the first strict minimum (runner.cpp:147-150)
        if (best_index < 0 && r.status == mars::RunStatus::Ok && r.energy == s.best_energy)
            best_index = static_cast<int64_t>(k);
    }
    st->best_energy = s.best_energy;
    st->mean_energy = s.mean_energy;
    st->best_cut = s.best_cut;
    st->mean_cut = s.mean_cut;
    st->hit_count = s.hit_count;
    st->success_probability = s.success_probability;
    st->total_seconds = s.total_seconds;
    st->mean_seconds_per_run = s.mean_seconds_per_run;
    st->best_index = best_index;
    st->completed_runs = s.completed_runs;
    st->skipped_runs = s.skipped_runs;
    st->failed_runs = s.failed_runs;
}
}  // namespace

int ref_run_batch(const void* p, const orc_params_t* prm, int64_t runs, uint64_t base_seed,
                  int workers, orc_records_t* rec, orc_stats_t* st, char* err, int errlen) {
    try {
        mars::BatchSpec spec;                                                      // runner.hpp:19
        spec.params = to_params(prm);
        spec.runs = runs;
        spec.base_seed = base_seed;
        spec.workers = workers;
        const mars::BatchStats s = mars::run_batch(P(p), spec);                    // runner.cpp:170
        fill_batch(P(p), s, rec, st);
        return 0;
    } catch (const mars::InputError& e) {
        put_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 5;
    }
}

// --- instance generators: the reference's own Rng driven by the SURVEY.md 8(d) recipes ---

void ref_gen_sk_gaussian(int n, uint64_t seed, double* J) {                        // io.cpp:151-163
    mars::Rng rng(seed);
    std::memset(J, 0, sizeof(double) * static_cast<std::size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = rng.gaussian();
            J[static_cast<std::size_t>(i) * n + k] = w;
            J[static_cast<std::size_t>(k) * n + i] = w;
        }
}

void ref_gen_sk_pm1(int n, uint64_t seed, double* J) {
    mars::Rng rng(seed);
    std::memset(J, 0, sizeof(double) * static_cast<std::size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = rng.coin_spin();
            J[static_cast<std::size_t>(i) * n + k] = w;
            J[static_cast<std::size_t>(k) * n + i] = w;
        }
}

int64_t ref_gen_er(int n, double prob, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    mars::Rng rng(seed);
    int64_t m = 0;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            if (rng.uniform_open01() < prob) {
                if (u) {
                    u[m] = a;
                    v[m] = b;
                    w[m] = 1.0;
                }
                ++m;
            }
    return m;
}

int64_t ref_gen_ea(int L, int dims, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    mars::Rng rng(seed);
    int64_t nsite = 1;
    for (int d = 0; d < dims; ++d) nsite *= L;
    int64_t m = 0;
    for (int64_t i = 0; i < nsite; ++i) {
        int64_t stride = 1;
        for (int d = 0; d < dims; ++d) {
            const int64_t coord = (i / stride) % L;
            const int64_t j = i + (coord == L - 1 ? -(L - 1) * stride : stride);
            const double wt = rng.coin_spin();
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

extern "C" {

// TEST-ONLY: the reference's run_batch with NmfaParams / SimCimParams (runner.cpp:31-60,
// solvers.cpp:374-443) -- the checker for the device's synchronous baselines.
int ref_run_batch_nmfa(const void* p, double noise_sigma, double alpha, int64_t iters, const double* sched,
                       int64_t sched_len, int64_t runs, uint64_t base_seed, int workers, orc_records_t* rec,
                       orc_stats_t* st, char* err, int errlen) {
    try {
        mars::NmfaParams np;
        np.noise_sigma = noise_sigma;
        np.alpha = alpha;
        np.iters = iters;
        np.schedule.assign(sched, sched + sched_len);
        mars::BatchSpec spec;
        spec.params = np;
        spec.runs = runs;
        spec.base_seed = base_seed;
        spec.workers = workers;
        fill_batch(P(p), mars::run_batch(P(p), spec), rec, st);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_run_batch_simcim(const void* p, double step_size, double noise_sigma, int64_t iters, const double* sched,
                         int64_t sched_len, int64_t runs, uint64_t base_seed, int workers, orc_records_t* rec,
                         orc_stats_t* st, char* err, int errlen) {
    try {
        mars::SimCimParams sp;
        sp.step_size = step_size;
        sp.noise_sigma = noise_sigma;
        sp.iters = iters;
        sp.pump_schedule.assign(sched, sched + sched_len);
        mars::BatchSpec spec;
        spec.params = sp;
        spec.runs = runs;
        spec.base_seed = base_seed;
        spec.workers = workers;
        fill_batch(P(p), mars::run_batch(P(p), spec), rec, st);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

}  // extern "C"
