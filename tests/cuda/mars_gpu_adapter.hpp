// mars_gpu_adapter.hpp -- the reference-side binding a maintainer of the reference would add
// (documented in INTEGRATION.md).  It keeps the reference's own signature,
//     mars::BatchStats mars::run_batch(const IsingProblem&, const BatchSpec&, const ProgressFn&)
// (include/mars/runner.hpp:55-56), and routes MARS batches through the B200 C-ABI
// (include/mars_b200.h).  Compiled here against the reference's headers by
// tests/test_adapter.py; never part of the product library.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mars/errors.hpp"
#include "mars/model.hpp"
#include "mars/runner.hpp"
#include "mars/solvers.hpp"
#include "mars_b200.h"

namespace mars::gpu {

inline void check(int rc) {
    if (rc == MARS_OK) return;
    const std::string msg = mars_last_error();
    if (rc == MARS_ERR_INPUT) throw InputError(msg);
    throw Error(msg);
}

// A device-resident copy of the problem (model.hpp:29-101), kept for many batches.
class DeviceProblem {
  public:
    explicit DeviceProblem(const IsingProblem& p, int device = 0) : n_(p.size()) {
        const double* h = p.has_field() ? p.field().data() : nullptr;
        if (!p.uses_adjacency()) {
            check(mars_problem_dense(n_, p.dense_data().data(), h, device, MARS_KERNEL_AUTO, &h_));
        } else {
            std::vector<int32_t> u, v;
            std::vector<double> w;
            p.visit_upper([&](int i, int j, double wt) {   // canonical (i, j) order
                u.push_back(i);
                v.push_back(j);
                w.push_back(wt);
            });
            check(mars_problem_from_edges(n_, static_cast<int64_t>(u.size()), u.data(), v.data(),
                                          w.data(), h, device, MARS_KERNEL_AUTO, &h_));
        }
    }
    ~DeviceProblem() { mars_problem_destroy(h_); }
    DeviceProblem(const DeviceProblem&) = delete;
    DeviceProblem& operator=(const DeviceProblem&) = delete;
    mars_problem_t* handle() const { return h_; }
    int size() const { return n_; }

  private:
    int n_;
    mars_problem_t* h_ = nullptr;
};

inline void progress_trampoline(int64_t idx, double best, void* user) {
    (*static_cast<const ProgressFn*>(user))(idx, best);
}

// run_batch (runner.cpp:170-178) on the GPU: MarsParams (the hot path), NmfaParams and
// SimCimParams (the synchronous baselines); identical BatchStats.  SA / MFA have no GPU path.
inline BatchStats run_batch(const DeviceProblem& dp, const BatchSpec& spec,
                            const ProgressFn& progress = {}) {
    const auto* mp = std::get_if<MarsParams>(&spec.params);
    if (!mp) {
        const auto* np = std::get_if<NmfaParams>(&spec.params);
        const auto* sp = std::get_if<SimCimParams>(&spec.params);
        if (!np && !sp)
            throw InputError(std::string("mars::gpu::run_batch: solver '") + solver_name(spec.params) +
                             "' has no GPU path (MARS, NMFA and SimCIM do)");
        const int n = dp.size();
        std::vector<uint8_t> status(spec.runs);
        std::vector<double> energy(spec.runs), cut(spec.runs), temp(spec.runs), elapsed(spec.runs);
        std::vector<int64_t> iters(spec.runs);
        std::vector<int8_t> spins(static_cast<size_t>(spec.runs) * n);
        mars_records_t rec{status.data(), energy.data(), cut.data(), temp.data(), iters.data(),
                           elapsed.data(), spins.data(), nullptr};
        mars_stats_t st{};
        if (np) {
            const mars_nmfa_params_t c{np->noise_sigma, np->alpha, np->iters, np->schedule.data(),
                                       static_cast<int64_t>(np->schedule.size())};
            check(mars_run_batch_nmfa(dp.handle(), &c, spec.runs, spec.base_seed, &rec, &st, nullptr));
        } else {
            const mars_simcim_params_t c{sp->step_size, sp->noise_sigma, sp->iters, sp->pump_schedule.data(),
                                         static_cast<int64_t>(sp->pump_schedule.size())};
            check(mars_run_batch_simcim(dp.handle(), &c, spec.runs, spec.base_seed, &rec, &st, nullptr));
        }
        BatchStats out;
        out.runs.resize(static_cast<size_t>(spec.runs));
        double best_so_far = 1e300;
        for (int64_t k = 0; k < spec.runs; ++k) {
            RunResult& r = out.runs[static_cast<size_t>(k)];
            r.status = static_cast<RunStatus>(status[k]);
            r.energy = energy[k];
            r.cut = cut[k];
            r.start_temp = temp[k];
            r.descent_iters = iters[k];
            r.elapsed_seconds = elapsed[k];
            r.spins.assign(spins.begin() + k * n, spins.begin() + (k + 1) * n);
            out.energies.push_back(r.energy);
            best_so_far = std::min(best_so_far, r.energy);
            if (progress) progress(k, best_so_far);
        }
        out.best_energy = st.best_energy;
        out.mean_energy = st.mean_energy;
        out.best_cut = st.best_cut;
        out.mean_cut = st.mean_cut;
        out.hit_count = st.hit_count;
        out.success_probability = st.success_probability;
        out.total_seconds = st.total_seconds;
        out.mean_seconds_per_run = st.mean_seconds_per_run;
        out.completed_runs = st.completed_runs;
        out.best_result = out.runs[static_cast<size_t>(st.best_index)];
        return out;
    }
    const mars_params_t prm{mp->t_min, mp->t_max, mp->t_step, mp->c_step, mp->d_min,
                            mp->start_mode == StartMode::UniformRandom ? MARS_UNIFORM_RANDOM
                                                                       : MARS_GRID_SWEEP,
                            0, 0};
    int64_t runs = 0;
    check(mars_run_count(&prm, spec.runs, &runs));
    const int n = dp.size();
    std::vector<uint8_t> status(runs);
    std::vector<double> energy(runs), cut(runs), temp(runs), elapsed(runs), fail_temp(runs);
    std::vector<int64_t> iters(runs);
    std::vector<int8_t> spins(static_cast<size_t>(runs) * n);
    mars_records_t rec{status.data(), energy.data(), cut.data(), temp.data(), iters.data(),
                       elapsed.data(), spins.data(), fail_temp.data()};
    mars_stats_t st{};
    // the progress callback runs on this thread while the batch runs (runner.cpp:107-113)
    check(mars_run_batch_progress(dp.handle(), &prm, spec.runs, spec.base_seed, &rec, &st, nullptr,
                                  progress ? progress_trampoline : nullptr,
                                  const_cast<ProgressFn*>(&progress)));

    BatchStats out;
    out.runs.resize(static_cast<size_t>(runs));
    for (int64_t k = 0; k < runs; ++k) {
        RunResult& r = out.runs[static_cast<size_t>(k)];
        r.status = static_cast<RunStatus>(status[k]);
        r.energy = energy[k];
        r.cut = cut[k];
        r.start_temp = temp[k];
        r.descent_iters = iters[k];
        r.elapsed_seconds = elapsed[k];
        if (r.status != RunStatus::Skipped)
            r.spins.assign(spins.begin() + k * n, spins.begin() + (k + 1) * n);
        if (r.status == RunStatus::Diverged)
            r.error = "relaxation exceeded the sweep cap at T = " + std::to_string(fail_temp[k]);
        if (r.status == RunStatus::Ok) out.energies.push_back(r.energy);
    }
    out.best_energy = st.best_energy;
    out.mean_energy = st.mean_energy;
    out.best_cut = st.best_cut;
    out.mean_cut = st.mean_cut;
    out.hit_count = st.hit_count;
    out.success_probability = st.success_probability;
    out.total_seconds = st.total_seconds;
    out.mean_seconds_per_run = st.mean_seconds_per_run;
    out.completed_runs = st.completed_runs;
    out.skipped_runs = st.skipped_runs;
    out.failed_runs = st.failed_runs;
    out.best_result = out.runs[static_cast<size_t>(st.best_index)];
    return out;
}

inline BatchStats run_batch(const IsingProblem& p, const BatchSpec& spec,
                            const ProgressFn& progress = {}) {
    std::visit([](const auto& prm) { validate(prm); }, spec.params);   // InputError before any run (runner.cpp:172)
    DeviceProblem dp(p);
    return run_batch(dp, spec, progress);
}

}  // namespace mars::gpu
