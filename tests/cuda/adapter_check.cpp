// adapter_check.cpp -- TEST ONLY: the reference's own code path next to the drop-in GPU
// adapter, on the same IsingProblem objects built by the reference library.  Prints one line
// per case: reference vs GPU best energy, identical-spin fraction, hit counts.
#include <cmath>
#include <cstdio>
#include <limits>

#include "mars/io.hpp"
#include "mars/rng.hpp"
#include "mars/runner.hpp"
#include "mars_gpu_adapter.hpp"

// generate_sk's loop (io.cpp:151-163) with the reference's own Rng, without linking io.cpp
static mars::IsingProblem sk(int n, uint64_t seed) {
    mars::Rng rng(seed);
    std::vector<double> j(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = rng.gaussian();
            j[static_cast<size_t>(i) * n + k] = w;
            j[static_cast<size_t>(k) * n + i] = w;
        }
    return mars::IsingProblem::dense(n, std::move(j));
}

int main() {
    using namespace mars;
    int failures = 0;
    auto compare = [&](const char* name, const IsingProblem& p, const MarsParams& mp, int64_t runs,
                       uint64_t seed, double min_same) {
        BatchSpec spec;
        spec.params = mp;
        spec.runs = runs;
        spec.base_seed = seed;
        spec.workers = 0;
        const BatchStats ref = run_batch(p, spec);          // the reference (CPU)
        const BatchStats gpu = gpu::run_batch(p, spec);     // the drop-in (B200)
        int same = 0, total = 0;
        for (size_t k = 0; k < ref.runs.size(); ++k) {
            if (ref.runs[k].status != RunStatus::Ok) continue;
            ++total;
            if (ref.runs[k].spins == gpu.runs[k].spins) {
                ++same;
                if (ref.runs[k].energy != gpu.runs[k].energy) ++failures;   // bit-exact energies
            }
        }
        const double frac = total ? static_cast<double>(same) / total : 1.0;
        // the reference's own result document (io.cpp:480-538) over the
        // GPU batch; identical to the reference's document whenever every run matches
        const std::string dref = result_document_to_string(make_result_document(name, p, mp, ref, DocDetail::Full, false));
        const std::string dgpu = result_document_to_string(make_result_document(name, p, mp, gpu, DocDetail::Full, false));
        int iters_same = 0;
        for (size_t k = 0; k < ref.runs.size(); ++k) iters_same += ref.runs[k].descent_iters == gpu.runs[k].descent_iters;
        const bool all_same = same == total && iters_same == static_cast<int>(ref.runs.size());
        if (all_same && dref != dgpu) ++failures;
        std::printf("    result document: %s (%zu bytes; iters identical %d/%zu)\n",
                    dref == dgpu ? "byte-identical" : "differs", dref.size(), iters_same, ref.runs.size());
        const bool ok = frac >= min_same && gpu.runs.size() == ref.runs.size() &&
                        gpu.skipped_runs == ref.skipped_runs &&
                        std::abs(gpu.best_energy - ref.best_energy) <= 1e-6 * std::abs(ref.best_energy) + 1e-9;
        if (!ok) ++failures;
        std::printf("%-28s ref best %.6f  gpu best %.6f  same spins %d/%d  hits %lld/%lld  %s\n", name,
                    ref.best_energy, gpu.best_energy, same, total, static_cast<long long>(ref.hit_count),
                    static_cast<long long>(gpu.hit_count), ok ? "OK" : "FAIL");
    };
    MarsParams grid;
    grid.t_min = 0;
    grid.t_max = 10;
    grid.t_step = 0.1;
    // acceptance.cpp:59-82 shape: SK(14) grid sweeps
    for (uint64_t i = 1; i <= 3; ++i) compare("sk14 grid (acceptance c1)", sk(14, 900000 + i), grid, 1, i, 0.95);
    MarsParams uni;
    uni.t_min = 0;
    uni.t_max = 16;
    uni.start_mode = StartMode::UniformRandom;
    compare("sk60 uniform", sk(60, 99), uni, 256, 41, 0.9);
    // sparse storage path (CSR kernel)
    std::vector<IsingProblem::Edge> edges;
    Rng r(31);
    for (int a = 0; a < 300; ++a)
        for (int b = a + 1; b < 300; ++b)
            if (r.uniform_open01() < 0.02) edges.push_back({a, b, r.uniform_open01() < 0.5 ? -1.0 : 1.0});
    compare("er300 (CSR)", IsingProblem::from_edges(300, edges), uni, 256, 5, 0.98);
    // ProgressFn (runner.hpp:52; test_runner.cpp:148-162): once per run incl. the skipped slot,
    // non-increasing best, on the calling thread while the GPU batch runs
    {
        MarsParams g2;
        g2.t_min = 0;
        g2.t_max = 10;
        g2.t_step = 1;
        BatchSpec spec;
        spec.params = g2;
        spec.base_seed = 2;
        int calls = 0;
        bool monotone = true;
        double last = std::numeric_limits<double>::infinity();   // test_runner.cpp:151
        const BatchStats gpu = gpu::run_batch(sk(10, 75), spec, [&](std::int64_t, double best) {
            ++calls;
            if (best > last + 1e-12) monotone = false;
            last = best;
        });
        const bool ok = calls == 11 && monotone && gpu.completed_runs == 10 && last == gpu.best_energy;
        if (!ok) ++failures;
        std::printf("%-28s calls %d monotone %d best %.6f  %s\n", "progress (test_runner 148)", calls, monotone,
                    gpu.best_energy, ok ? "OK" : "FAIL");
    }
    // the synchronous baselines through the same seam: identical records to the reference's
    for (int which = 0; which < 2; ++which) {
        BatchSpec spec;
        if (which == 0) spec.params = nmfa_defaults(300);
        else spec.params = simcim_defaults(300);
        spec.runs = 64;
        spec.base_seed = 4;
        const IsingProblem p = sk(128, 17);
        const BatchStats ref = run_batch(p, spec);
        const BatchStats gpu = gpu::run_batch(p, spec);
        int same = 0;
        for (size_t k = 0; k < ref.runs.size(); ++k)
            same += ref.runs[k].spins == gpu.runs[k].spins && ref.runs[k].energy == gpu.runs[k].energy;
        const bool ok = same >= 61 && gpu.best_energy <= ref.best_energy + 1e-9;
        if (!ok) ++failures;
        std::printf("%-28s ref best %.6f  gpu best %.6f  same runs %d/64  %s\n", which ? "simcim sk128" : "nmfa sk128",
                    ref.best_energy, gpu.best_energy, same, ok ? "OK" : "FAIL");
    }
    // SA has no GPU path: InputError (not bad_variant_access)
    {
        BatchSpec spec;
        spec.params = SaParams{};
        spec.runs = 1;
        bool threw = false;
        try {
            gpu::run_batch(sk(10, 1), spec);
        } catch (const InputError&) {
            threw = true;
        }
        if (!threw) ++failures;
        std::printf("%-28s %s\n", "sa -> InputError", threw ? "OK" : "FAIL");
    }
    std::printf("%s\n", failures ? "ADAPTER FAIL" : "ADAPTER OK");
    return failures ? 1 : 0;
}
