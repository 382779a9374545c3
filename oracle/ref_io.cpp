// ref_io.cpp -- TEST ONLY.  An extern "C" shim over the reference's own instance I/O and
// result documents (/root/reference/proj/src/io.cpp, include/mars/io.hpp), compiled with the
// reference's sources by oracle/Makefile into oracle/_ref/libmars_ref_io.so.  The tests use it
// to check the Python mirror (paper_1907_05124_b200/io.py) byte for byte: parse errors and
// their messages, the dense-matrix / G-set writers, problem_hash, and the JSON result
// document of a reference batch.
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "mars/errors.hpp"
#include "mars/io.hpp"
#include "mars/runner.hpp"
#include "mars/solvers.hpp"
#include "mars_oracle.h"

namespace {

// error classes -> codes: 1 ParseError, 2 StructuralError, 3 InputError, 4 other mars::Error
int code_of(const std::exception& e) {
    if (dynamic_cast<const mars::ParseError*>(&e)) return 1;
    if (dynamic_cast<const mars::StructuralError*>(&e)) return 2;
    if (dynamic_cast<const mars::InputError*>(&e)) return 3;
    return 4;
}

int put(const std::string& s, char* out, std::int64_t cap) {
    if (static_cast<std::int64_t>(s.size()) + 1 > cap) return -static_cast<int>(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

mars::IsingProblem make_problem(int n, const double* J, std::int64_t m, const int32_t* u, const int32_t* v,
                                const double* w, const double* h) {
    std::vector<double> field = h ? std::vector<double>(h, h + n) : std::vector<double>{};
    if (J) return mars::IsingProblem::dense(n, std::vector<double>(J, J + static_cast<std::size_t>(n) * n), field);
    std::vector<mars::IsingProblem::Edge> edges;
    for (std::int64_t k = 0; k < m; ++k) edges.push_back({u[k], v[k], w[k]});
    return mars::IsingProblem::from_edges(n, edges, field);
}

}  // namespace

extern "C" {

// parse_gset (io.cpp:77-130) on `text`.  Returns 0 and fills n / m / arrays (capacity `cap`
// edges), or the error code with the exception message in `msg`.
int ref_io_parse_gset(const char* text, int* n, int64_t* m, int32_t* u, int32_t* v, int64_t* w,
                      int64_t cap, char* msg, int64_t msgcap) {
    try {
        std::istringstream in(text);
        const mars::GsetGraph g = mars::parse_gset(in);
        *n = g.n_vertices;
        *m = static_cast<int64_t>(g.edges.size());
        for (std::size_t k = 0; k < g.edges.size() && static_cast<int64_t>(k) < cap; ++k) {
            u[k] = g.edges[k].u;
            v[k] = g.edges[k].v;
            w[k] = g.edges[k].w;
        }
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), msg, msgcap);
        return code_of(e);
    }
}

// read_matrix (io.cpp:187-228): n and the n*n couplings (capacity `cap` doubles).
int ref_io_read_matrix(const char* text, int* n, double* J, int64_t cap, char* msg, int64_t msgcap) {
    try {
        std::istringstream in(text);
        const mars::IsingProblem p = mars::read_matrix(in);
        *n = p.size();
        for (int i = 0; i < p.size(); ++i) {
            const std::vector<double> row = p.row_values(i);
            for (int k = 0; k < p.size(); ++k)
                if (static_cast<int64_t>(i) * p.size() + k < cap) J[static_cast<std::size_t>(i) * p.size() + k] = row[k];
        }
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), msg, msgcap);
        return code_of(e);
    }
}

// detect_format (io.cpp:230-244): 0 G-set, 1 dense matrix, < 0 error (message in msg).
int ref_io_detect_format(const char* text, char* msg, int64_t msgcap) {
    try {
        std::istringstream in(text);
        return mars::detect_format(in) == mars::InstanceFormat::GsetGraph ? 0 : 1;
    } catch (const std::exception& e) {
        put(e.what(), msg, msgcap);
        return -code_of(e);
    }
}

// problem_hash (io.cpp:260-290) of a dense (J != null) or edge-list instance.
uint64_t ref_io_problem_hash(int n, const double* J, int64_t m, const int32_t* u, const int32_t* v,
                             const double* w, const double* h) {
    return mars::problem_hash(make_problem(n, J, m, u, v, w, h));
}

// write_matrix (io.cpp:165-178) / write_gset (io.cpp:138-141) into `out`.
int ref_io_write_matrix(int n, const double* J, int64_t m, const int32_t* u, const int32_t* v, const double* w,
                        char* out, int64_t cap) {
    std::ostringstream os;
    mars::write_matrix(make_problem(n, J, m, u, v, w, nullptr), os);
    return put(os.str(), out, cap);
}

int ref_io_write_gset(int n, int64_t m, const int32_t* u, const int32_t* v, const int64_t* w, char* out,
                      int64_t cap) {
    mars::GsetGraph g;
    g.n_vertices = n;
    for (int64_t k = 0; k < m; ++k) g.edges.push_back({u[k], v[k], w[k]});
    std::ostringstream os;
    mars::write_gset(g, os);
    return put(os.str(), out, cap);
}

// The reference's run_batch on the instance, then make_result_document (io.cpp:480-502) and
// result_document_to_string (io.cpp:504-538) with volatile fields suppressed.
// detail: 0 Summary, 1 Energies, 2 Full.
int ref_io_result_document(int n, const double* J, int64_t m, const int32_t* u, const int32_t* v,
                           const double* w, const double* h, const orc_params_t* prm, int64_t runs,
                           uint64_t base_seed, int detail, const char* problem_id, char* out, int64_t cap) {
    try {
        const mars::IsingProblem p = make_problem(n, J, m, u, v, w, h);
        mars::MarsParams mp;
        mp.t_min = prm->t_min;
        mp.t_max = prm->t_max;
        mp.t_step = prm->t_step;
        mp.c_step = prm->c_step;
        mp.d_min = prm->d_min;
        mp.start_mode = prm->start_mode ? mars::StartMode::UniformRandom : mars::StartMode::GridSweep;
        mars::BatchSpec spec;
        spec.params = mp;
        spec.runs = runs;
        spec.base_seed = base_seed;
        spec.workers = 0;
        const mars::BatchStats stats = mars::run_batch(p, spec);
        const auto doc = mars::make_result_document(problem_id, p, mp, stats,
                                                    static_cast<mars::DocDetail>(detail), false);
        return put(mars::result_document_to_string(doc), out, cap);
    } catch (const std::exception& e) {
        put(e.what(), out, cap);
        return code_of(e);
    }
}

// brute_force_ground_state (model.cpp:296-324) with its default guard and policy.
int ref_io_brute_force(int n, const double* J, int64_t m, const int32_t* u, const int32_t* v, const double* w,
                       const double* h, int max_n, double* energy, int8_t* spins, char* msg, int64_t msgcap) {
    try {
        const mars::GroundState g = mars::brute_force_ground_state(make_problem(n, J, m, u, v, w, h), max_n);
        *energy = g.energy;
        for (int i = 0; i < n; ++i) spins[i] = g.spins[static_cast<std::size_t>(i)];
        return 0;
    } catch (const std::exception& e) {
        put(e.what(), msg, msgcap);
        return code_of(e);
    }
}

}  // extern "C"
