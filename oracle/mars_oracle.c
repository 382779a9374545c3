/*
 * mars_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the reference MARS
 * hot path, used as the parity checker for the B200 product.  It is never linked into,
 * loaded by, or called from the product path (paper_1907_05124_b200/).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  The arithmetic is fp64 in exactly the reference's order, with
 * the same libm calls, so results are bit-identical to the compiled reference
 * (oracle/_ref/libmars_ref.so); tests/test_oracle.py pins that, and pins both against
 * the committed golden fixtures under tests/golden/.
 *
 * Pinned: yes -- against the compiled reference on identical inputs (bitwise) and the
 * reference's only frozen constant splitmix64(0) == 0xE220A8397B1DCDAF
 * (tests/test_io.cpp:157).
 */
#include "mars_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* ------------------------------------------------------------------ RNG (rng.hpp) */

/* include/mars/rng.hpp:13-18 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* include/mars/rng.hpp:20-22 */
uint64_t orc_sub_seed(uint64_t base, uint64_t index) {
    return orc_splitmix64(base + index * 0x9E3779B97F4A7C15ull);
}

/* std::mt19937_64 (ISO C++ [rand.eng.mers], the engine behind rng.hpp:82). */
enum { MT_N = 312, MT_M = 156 };
typedef struct {
    uint64_t mt[MT_N];
    int idx;
    double spare;
    int have_spare;
} orc_rng;

static void mt_seed(orc_rng* r, uint64_t s) {
    r->mt[0] = s;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
    r->spare = 0.0;
    r->have_spare = 0;
}

static uint64_t mt_next(orc_rng* r) {
    if (r->idx >= MT_N) {
        const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
        }
        r->idx = 0;
    }
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

/* rng.hpp:29 -- Rng(seed) seeds the engine with splitmix64(seed) */
static void rng_init(orc_rng* r, uint64_t seed) { mt_seed(r, orc_splitmix64(seed)); }

/* rng.hpp:34-36 */
static double rng_open01(orc_rng* r) { return ((double)(mt_next(r) >> 11) + 0.5) * 0x1.0p-53; }
/* rng.hpp:39 */
static double rng_open_sym(orc_rng* r) { return 2.0 * rng_open01(r) - 1.0; }

/* rng.hpp:45-60 (Lemire rejection) */
static uint64_t rng_below(orc_rng* r, uint64_t n) {
    uint64_t x = mt_next(r);
    __uint128_t m = (__uint128_t)x * n;
    uint64_t lo = (uint64_t)m;
    if (lo < n) {
        const uint64_t t = (0 - n) % n;
        while (lo < t) {
            x = mt_next(r);
            m = (__uint128_t)x * n;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* rng.hpp:63-75 (basic Box-Muller with a cached spare) */
static double rng_gaussian(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = rng_open01(r);
    const double u2 = rng_open01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(a);
    r->have_spare = 1;
    return rad * cos(a);
}

/* rng.hpp:77 */
static int8_t rng_coin(orc_rng* r) { return (mt_next(r) >> 63) ? (int8_t)1 : (int8_t)-1; }

void orc_rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t count, uint64_t* ou,
                   double* of) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t k = 0; k < count; ++k) {
        switch (kind) {
            case 0: ou[k] = mt_next(&r); break;
            case 1: of[k] = rng_open01(&r); break;
            case 2: of[k] = rng_open_sym(&r); break;
            case 3: of[k] = rng_gaussian(&r); break;
            case 4: of[k] = rng_coin(&r); break;
            default: ou[k] = rng_below(&r, arg); break;
        }
    }
}

/* ------------------------------------------------------------ problem (model.cpp) */

typedef struct {
    int n;
    int dense;          /* storage choice, model.cpp:91 */
    int integral;
    int has_field;
    double coupling_sum;
    int64_t nnz;
    double* J;          /* n*n row-major when dense */
    int* off;           /* n+1 when adjacency */
    int* idx;
    double* wt;
    double* h;          /* always n */
} orc_problem;

static void put_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) {
        strncpy(err, msg, (size_t)errlen - 1);
        err[errlen - 1] = '\0';
    }
}

/* model.cpp:16 */
static int is_integral_value(double v) { return nearbyint(v) == v && isfinite(v); }

/* model.cpp:20-45 -- coupling_sum in storage order, nnz, integral flag */
static void finalize_metadata(orc_problem* p) {
    p->coupling_sum = 0.0;
    p->nnz = 0;
    p->integral = 1;
    if (p->dense) {
        for (int i = 0; i < p->n; ++i)
            for (int j = 0; j < p->n; ++j) {
                const double w = p->J[(size_t)i * p->n + j];
                p->coupling_sum += w;
                if (w != 0.0) ++p->nnz;
                if (p->integral && !is_integral_value(w)) p->integral = 0;
            }
    } else {
        const int64_t m = p->off[p->n];
        for (int64_t k = 0; k < m; ++k) {
            p->coupling_sum += p->wt[k];
            ++p->nnz;
            if (p->integral && !is_integral_value(p->wt[k])) p->integral = 0;
        }
    }
    p->has_field = 0;
    for (int i = 0; i < p->n; ++i) {
        if (p->h[i] != 0.0) p->has_field = 1;
        if (p->integral && !is_integral_value(p->h[i])) p->integral = 0;
    }
}

/* model.cpp:47-72 -- IsingProblem::dense with symmetric / zero-diagonal validation */
void* orc_problem_dense(int n, const double* J, const double* h, char* err, int errlen) {
    char msg[160];
    if (n <= 0) {
        put_err(err, errlen, "problem size must be positive");
        return NULL;
    }
    for (int i = 0; i < n; ++i) {
        if (J[(size_t)i * n + i] != 0.0) {
            snprintf(msg, sizeof msg, "coupling diagonal must be zero (row %d)", i);
            put_err(err, errlen, msg);
            return NULL;
        }
        for (int j = i + 1; j < n; ++j)
            if (J[(size_t)i * n + j] != J[(size_t)j * n + i]) {
                snprintf(msg, sizeof msg, "coupling matrix must be symmetric (entries %d,%d)", i, j);
                put_err(err, errlen, msg);
                return NULL;
            }
    }
    orc_problem* p = (orc_problem*)calloc(1, sizeof *p);
    p->n = n;
    p->dense = 1;
    p->J = (double*)malloc(sizeof(double) * (size_t)n * n);
    memcpy(p->J, J, sizeof(double) * (size_t)n * n);
    p->h = (double*)calloc((size_t)n, sizeof(double));
    if (h) memcpy(p->h, h, sizeof(double) * (size_t)n);
    finalize_metadata(p);
    return p;
}

typedef struct {
    int j;
    double w;
} nbr;

/* std::sort of pair<int,double>: by index, then weight (model.cpp:116-127) */
static int nbr_cmp(const void* a, const void* b) {
    const nbr* x = (const nbr*)a;
    const nbr* y = (const nbr*)b;
    if (x->j != y->j) return x->j < y->j ? -1 : 1;
    if (x->w != y->w) return x->w < y->w ? -1 : 1;
    return 0;
}

/* model.cpp:74-131 -- IsingProblem::from_edges with the 5% density storage rule */
void* orc_problem_edges(int n, int64_t m, const int32_t* u, const int32_t* v, const double* w,
                        const double* h, char* err, int errlen) {
    if (n <= 0) {
        put_err(err, errlen, "problem size must be positive");
        return NULL;
    }
    for (int64_t k = 0; k < m; ++k) {
        if (u[k] < 0 || u[k] >= n || v[k] < 0 || v[k] >= n) {
            put_err(err, errlen, "edge endpoint out of range");
            return NULL;
        }
        if (u[k] == v[k]) {
            put_err(err, errlen, "self-coupling is not allowed");
            return NULL;
        }
    }
    const double max_pairs = 0.5 * (double)n * (n - 1);
    const double density = max_pairs > 0 ? (double)m / max_pairs : 1.0;
    orc_problem* p = (orc_problem*)calloc(1, sizeof *p);
    p->n = n;
    p->h = (double*)calloc((size_t)n, sizeof(double));
    if (h) memcpy(p->h, h, sizeof(double) * (size_t)n);
    if (density >= 0.05) {                                   /* kSparseDensityThreshold, model.hpp:31 */
        p->dense = 1;
        p->J = (double*)calloc((size_t)n * n, sizeof(double));
        for (int64_t k = 0; k < m; ++k) {
            p->J[(size_t)u[k] * n + v[k]] += w[k];
            p->J[(size_t)v[k] * n + u[k]] += w[k];
        }
    } else {
        p->dense = 0;
        p->off = (int*)calloc((size_t)n + 1, sizeof(int));
        for (int64_t k = 0; k < m; ++k) {
            ++p->off[u[k] + 1];
            ++p->off[v[k] + 1];
        }
        for (int i = 0; i < n; ++i) p->off[i + 1] += p->off[i];
        p->idx = (int*)malloc(sizeof(int) * (size_t)(2 * m + 1));
        p->wt = (double*)malloc(sizeof(double) * (size_t)(2 * m + 1));
        int* cur = (int*)malloc(sizeof(int) * (size_t)n);
        memcpy(cur, p->off, sizeof(int) * (size_t)n);
        for (int64_t k = 0; k < m; ++k) {
            p->idx[cur[u[k]]] = v[k];
            p->wt[cur[u[k]]++] = w[k];
            p->idx[cur[v[k]]] = u[k];
            p->wt[cur[v[k]]++] = w[k];
        }
        free(cur);
        for (int i = 0; i < n; ++i) {
            const int lo = p->off[i], hi = p->off[i + 1];
            nbr* row = (nbr*)malloc(sizeof(nbr) * (size_t)(hi - lo + 1));
            for (int k = lo; k < hi; ++k) row[k - lo] = (nbr){p->idx[k], p->wt[k]};
            qsort(row, (size_t)(hi - lo), sizeof(nbr), nbr_cmp);
            for (int k = lo; k < hi; ++k) {
                p->idx[k] = row[k - lo].j;
                p->wt[k] = row[k - lo].w;
            }
            free(row);
        }
    }
    finalize_metadata(p);
    return p;
}

void orc_problem_free(void* vp) {
    orc_problem* p = (orc_problem*)vp;
    if (!p) return;
    free(p->J);
    free(p->off);
    free(p->idx);
    free(p->wt);
    free(p->h);
    free(p);
}

void orc_problem_info(const void* vp, int* n, int* adjacency, int* integral, double* csum,
                      int64_t* nnz) {
    const orc_problem* p = (const orc_problem*)vp;
    *n = p->n;
    *adjacency = !p->dense;
    *integral = p->integral;
    *csum = p->coupling_sum;
    *nnz = p->nnz;
}

/* model.cpp:141-151 -- ordered row dot product */
static double row_dot(const orc_problem* p, int i, const double* s) {
    double acc = 0.0;
    if (p->dense) {
        const double* row = p->J + (size_t)i * p->n;
        for (int j = 0; j < p->n; ++j) acc += row[j] * s[j];
    } else {
        for (int k = p->off[i]; k < p->off[i + 1]; ++k) acc += p->wt[k] * s[p->idx[k]];
    }
    return acc;
}

/* model.cpp:153-163 */
static double row_dot_spins(const orc_problem* p, int i, const int8_t* s) {
    double acc = 0.0;
    if (p->dense) {
        const double* row = p->J + (size_t)i * p->n;
        for (int j = 0; j < p->n; ++j) acc += row[j] * s[j];
    } else {
        for (int k = p->off[i]; k < p->off[i + 1]; ++k) acc += p->wt[k] * s[p->idx[k]];
    }
    return acc;
}

/* model.cpp:203-218 (serial policy) */
double orc_coupling_term(const void* vp, const int8_t* s) {
    const orc_problem* p = (const orc_problem*)vp;
    double total = 0.0;
    for (int i = 0; i < p->n; ++i) total += s[i] * row_dot_spins(p, i, s);
    return total;
}

/* model.cpp:220-225 */
double orc_energy(const void* vp, const int8_t* s) {
    const orc_problem* p = (const orc_problem*)vp;
    double total = orc_coupling_term(vp, s);
    for (int i = 0; i < p->n; ++i) total += p->h[i] * s[i];
    return total;
}

/* model.cpp:227-229 */
double orc_cut_value(const void* vp, const int8_t* s) {
    const orc_problem* p = (const orc_problem*)vp;
    return 0.25 * (p->coupling_sum - orc_coupling_term(vp, s));
}

/* model.cpp:245-249 */
static void round_spins(const double* s, int n, int8_t* out) {
    for (int i = 0; i < n; ++i) out[i] = s[i] < 0.0 ? (int8_t)-1 : (int8_t)1;
}

/* ------------------------------------------------------------- MARS (solvers.cpp) */

#define K_TEMP_FLOOR 1e-12                    /* solvers.cpp:19 */
#define K_START_TEMP_TAG 0x74656d7073746172ull /* solvers.cpp:23 */
#define K_SWEEP_CAP 1000000                   /* solvers.hpp:116 */

/* Test-only knob of the port (not in the reference): overrides kMarsSweepCap so the
 * DivergedError record path (runner.cpp:43-53) can be exercised at batch level. */
static int64_t g_sweep_cap = K_SWEEP_CAP;
void orc_set_sweep_cap(int64_t cap) { g_sweep_cap = cap > 0 ? cap : K_SWEEP_CAP; }

/* solvers.cpp:145-148 */
double orc_tanh_trial(double phi, double t) {
    if (t < K_TEMP_FLOOR) return phi > 0.0 ? -1.0 : (phi < 0.0 ? 1.0 : 0.0);
    return -tanh(phi / t);
}

/* solvers.cpp:150-161 -- Gauss-Seidel in ascending index order, in place */
double orc_relax_sweep(const void* vp, double* s, double t) {
    const orc_problem* p = (const orc_problem*)vp;
    double d = 0.0;
    for (int i = 0; i < p->n; ++i) {
        const double phi = row_dot(p, i, s) + p->h[i];
        const double trial = orc_tanh_trial(phi, t);
        const double dd = fabs(trial - s[i]);
        d = d > dd ? d : dd;      /* std::max(d, |.|) keeps d on ties / NaN-free inputs */
        s[i] = trial;
    }
    return d;
}

/* solvers.cpp:163-176 -- returns 1 (DivergedError) when the budget runs out */
int orc_relax_to_fixed_point(const void* vp, double* s, double t, double d_min, int64_t* budget,
                             int64_t* sweeps) {
    int64_t n_sweeps = 0;
    double d;
    do {
        if (*budget <= 0) {
            *sweeps = n_sweeps;
            return 1;
        }
        --*budget;
        d = orc_relax_sweep(vp, s, t);
        ++n_sweeps;
    } while (d > d_min);
    *sweeps = n_sweeps;
    return 0;
}

/* solvers.cpp:35-41 */
int orc_validate(const orc_params_t* p, char* err, int errlen) {
    if (!(p->t_min >= 0.0)) { put_err(err, errlen, "mars: t_min must be >= 0"); return 1; }
    if (!(p->t_max > p->t_min)) { put_err(err, errlen, "mars: t_max must exceed t_min"); return 1; }
    if (!(p->t_step > 0.0)) { put_err(err, errlen, "mars: t_step must be positive"); return 1; }
    if (!(p->c_step > 0.0)) { put_err(err, errlen, "mars: c_step must be positive"); return 1; }
    if (!(p->d_min > 0.0)) { put_err(err, errlen, "mars: d_min must be positive"); return 1; }
    return 0;
}

/* solvers.cpp:43-48 */
static int grid_count(const orc_params_t* p, int64_t* out, char* err, int errlen) {
    const double slots = floor((p->t_max - p->t_min) / p->t_step);
    if (!(slots >= 0.0) || slots > 1e9) {
        put_err(err, errlen, "mars: grid of temperatures is not usable");
        return 1;
    }
    *out = (int64_t)slots + 1;
    return 0;
}

/* solvers.cpp:202-213 */
int orc_run_count(const orc_params_t* p, int64_t requested, int64_t* out, char* err, int errlen) {
    if (orc_validate(p, err, errlen)) return 1;
    if (p->start_mode == 0) {
        int64_t count;
        if (grid_count(p, &count, err, errlen)) return 1;
        if (count == 1 && !(p->t_min > 0.0)) {
            put_err(err, errlen,
                    "mars: the temperature grid contains no positive starting temperature");
            return 1;
        }
        *out = count;
        return 0;
    }
    if (requested < 1) {
        put_err(err, errlen, "mars: UniformRandom mode needs runs >= 1");
        return 1;
    }
    *out = requested;
    return 0;
}

/* solvers.cpp:215-227 (+ mars_grid_temp 50-52) */
void orc_run_plan(const orc_params_t* p, uint64_t base, int64_t index, int* skipped, double* t,
                  uint64_t* seed) {
    *seed = orc_sub_seed(base, (uint64_t)index);
    if (p->start_mode == 0) {
        *t = p->t_min + (double)index * p->t_step;
        *skipped = !(*t > 0.0);
    } else {
        orc_rng r;
        rng_init(&r, orc_splitmix64(*seed ^ K_START_TEMP_TAG));
        *t = p->t_min + rng_open01(&r) * (p->t_max - p->t_min);
        *skipped = 0;
    }
}

/* solvers.cpp:184-187 */
void orc_initial_state(uint64_t seed, int n, double* s) {
    orc_rng r;
    rng_init(&r, seed);
    for (int i = 0; i < n; ++i) s[i] = rng_open_sym(&r);
}

/* solvers.cpp:178-200 (+ finish_result 25-29); returns 0 Ok, 2 Diverged (runner.cpp:43-53
 * record semantics: descent_iters = sweeps of the failing level), 1 input error */
int orc_descent(const void* vp, double start_temp, const orc_params_t* prm, uint64_t seed,
                uint8_t* status, double* energy, double* cut, int64_t* iters, int8_t* spins,
                char* err, int errlen) {
    const orc_problem* p = (const orc_problem*)vp;
    if (orc_validate(prm, err, errlen)) return 1;
    if (!(start_temp > 0.0)) {
        put_err(err, errlen, "mars: start_temp must be positive");
        return 1;
    }
    double* s = (double*)malloc(sizeof(double) * (size_t)p->n);
    int8_t* sp = (int8_t*)malloc((size_t)p->n);
    orc_initial_state(seed, p->n, s);
    int64_t budget = g_sweep_cap, total = 0, sweeps = 0;
    double t_t = start_temp;
    int rc = 0;
    while (t_t > 0.0) {
        t_t -= prm->c_step;
        if (orc_relax_to_fixed_point(vp, s, t_t, prm->d_min, &budget, &sweeps)) {
            rc = 2;
            break;
        }
        total += sweeps;
    }
    round_spins(s, p->n, sp);
    *status = (uint8_t)rc;
    *iters = rc ? sweeps : total;
    *energy = orc_energy(vp, sp);
    *cut = orc_cut_value(vp, sp);
    if (spins) memcpy(spins, sp, (size_t)p->n);
    if (rc) put_err(err, errlen, "relaxation exceeded the sweep cap");
    free(s);
    free(sp);
    return rc;
}

/* ------------------------------------------------------------ batch (runner.cpp) */

typedef struct {
    const orc_problem* p;
    const orc_params_t* prm;
    uint64_t base;
    int64_t runs;
    orc_records_t* rec;
    int8_t* spins;      /* [runs * n] scratch when the caller does not want spins */
    int64_t next;
    pthread_mutex_t mu;
} batch_ctx;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* runner.cpp:31-60 execute_run for MarsParams */
static void execute_run(batch_ctx* c, int64_t k) {
    int skipped;
    double t;
    uint64_t seed;
    orc_run_plan(c->prm, c->base, k, &skipped, &t, &seed);
    c->rec->start_temp[k] = t;
    if (skipped) {
        c->rec->status[k] = 1;
        c->rec->energy[k] = 0.0;
        c->rec->cut[k] = 0.0;
        c->rec->descent_iters[k] = 0;
        c->rec->elapsed_seconds[k] = 0.0;
        return;
    }
    const double t0 = now_s();
    uint8_t st;
    orc_descent(c->p, t, c->prm, seed, &st, &c->rec->energy[k], &c->rec->cut[k],
                &c->rec->descent_iters[k], c->spins + (size_t)k * c->p->n, NULL, 0);
    c->rec->status[k] = st;
    c->rec->elapsed_seconds[k] = now_s() - t0;
}

/* runner.cpp:95-115 -- workers pull indices from a shared counter */
static void* worker(void* arg) {
    batch_ctx* c = (batch_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        const int64_t k = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (k >= c->runs) return NULL;
        execute_run(c, k);
    }
}

int orc_run_batch(const void* vp, const orc_params_t* prm, int64_t runs_req, uint64_t base,
                  int workers, orc_records_t* user, orc_stats_t* st, char* err, int errlen) {
    const orc_problem* p = (const orc_problem*)vp;
    int64_t runs;
    if (orc_run_count(prm, runs_req, &runs, err, errlen)) return 1;   /* runner.cpp:172-173 */
    const double t0 = now_s();
    orc_records_t rec;
    rec.status = (uint8_t*)malloc((size_t)runs);
    rec.energy = (double*)malloc(sizeof(double) * (size_t)runs);
    rec.cut = (double*)malloc(sizeof(double) * (size_t)runs);
    rec.start_temp = (double*)malloc(sizeof(double) * (size_t)runs);
    rec.descent_iters = (int64_t*)malloc(sizeof(int64_t) * (size_t)runs);
    rec.elapsed_seconds = (double*)malloc(sizeof(double) * (size_t)runs);
    batch_ctx c = {p, prm, base, runs, &rec, NULL, 0, PTHREAD_MUTEX_INITIALIZER};
    c.spins = (int8_t*)malloc((size_t)runs * (size_t)p->n);
    /* runner.cpp:20-25 resolve_workers */
    int w = workers;
    if (w <= 0) w = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (w <= 0) w = 1;
    if (w > runs) w = (int)runs;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)w);
    for (int i = 0; i < w; ++i) pthread_create(&th[i], NULL, worker, &c);
    for (int i = 0; i < w; ++i) pthread_join(th[i], NULL);
    free(th);

    /* runner.cpp:126-167 -- aggregation in run-index order */
    memset(st, 0, sizeof *st);
    double cut_sum = 0.0, energy_sum = 0.0, run_seconds = 0.0;
    int64_t best = -1;
    for (int64_t i = 0; i < runs; ++i) {
        if (rec.status[i] == 1) { ++st->skipped_runs; continue; }
        if (rec.status[i] == 2) { ++st->failed_runs; continue; }
        ++st->completed_runs;
        energy_sum += rec.energy[i];
        cut_sum += rec.cut[i];
        run_seconds += rec.elapsed_seconds[i];
        if (best < 0 || rec.energy[i] < st->best_energy) {
            st->best_energy = rec.energy[i];
            best = i;
        }
        if (st->best_cut < rec.cut[i] || st->completed_runs == 1) st->best_cut = rec.cut[i];
    }
    int rc = 0;
    if (st->completed_runs == 0) {
        put_err(err, errlen, "batch failed: no run completed");
        rc = 5;
    } else {
        st->best_index = best;
        st->mean_energy = energy_sum / (double)st->completed_runs;
        st->mean_cut = cut_sum / (double)st->completed_runs;
        const double tol = p->integral ? 0.0 : 1e-9;                   /* model.hpp:82 */
        for (int64_t i = 0; i < runs; ++i)
            if (rec.status[i] == 0 && fabs(rec.energy[i] - st->best_energy) <= tol) ++st->hit_count;
        st->success_probability = (double)st->hit_count / (double)st->completed_runs;
        st->mean_seconds_per_run = run_seconds / (double)st->completed_runs;
        st->total_seconds = now_s() - t0;
    }
    if (user) {
        for (int64_t i = 0; i < runs; ++i) {
            if (user->status) user->status[i] = rec.status[i];
            if (user->energy) user->energy[i] = rec.energy[i];
            if (user->cut) user->cut[i] = rec.cut[i];
            if (user->start_temp) user->start_temp[i] = rec.start_temp[i];
            if (user->descent_iters) user->descent_iters[i] = rec.descent_iters[i];
            if (user->elapsed_seconds) user->elapsed_seconds[i] = rec.elapsed_seconds[i];
        }
        if (user->spins)
            for (int64_t i = 0; i < runs; ++i)
                if (rec.status[i] != 1)
                    memcpy(user->spins + (size_t)i * p->n, c.spins + (size_t)i * p->n, (size_t)p->n);
    }
    free(rec.status); free(rec.energy); free(rec.cut); free(rec.start_temp);
    free(rec.descent_iters); free(rec.elapsed_seconds); free(c.spins);
    return rc;
}

/* ------------------------------------------- instance generators */

/* io.cpp:151-163 generate_sk */
void orc_gen_sk_gaussian(int n, uint64_t seed, double* J) {
    orc_rng r;
    rng_init(&r, seed);
    memset(J, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = rng_gaussian(&r);
            J[(size_t)i * n + k] = w;
            J[(size_t)k * n + i] = w;
        }
}

/* cfg1: J_ab = J_ba = coin_spin() over a<b in row-major order */
void orc_gen_sk_pm1(int n, uint64_t seed, double* J) {
    orc_rng r;
    rng_init(&r, seed);
    memset(J, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int k = i + 1; k < n; ++k) {
            const double w = rng_coin(&r);
            J[(size_t)i * n + k] = w;
            J[(size_t)k * n + i] = w;
        }
}

/* cfg3: edge (a,b,+1) when uniform_open01() < prob, a<b row-major */
int64_t orc_gen_er(int n, double prob, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    orc_rng r;
    rng_init(&r, seed);
    int64_t m = 0;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            if (rng_open01(&r) < prob) {
                if (u) { u[m] = a; v[m] = b; w[m] = 1.0; }
                ++m;
            }
    return m;
}

/* cfg4: site i (x fastest), per dim d a +1-neighbour bond (periodic), w = coin_spin() */
int64_t orc_gen_ea(int L, int dims, uint64_t seed, int32_t* u, int32_t* v, double* w) {
    orc_rng r;
    rng_init(&r, seed);
    int64_t nsite = 1;
    for (int d = 0; d < dims; ++d) nsite *= L;
    int64_t m = 0;
    for (int64_t i = 0; i < nsite; ++i) {
        int64_t stride = 1;
        for (int d = 0; d < dims; ++d) {
            const int64_t coord = (i / stride) % L;
            const int64_t j = i + (coord == L - 1 ? -(int64_t)(L - 1) * stride : stride);
            const double wt = rng_coin(&r);
            if (u) { u[m] = (int32_t)i; v[m] = (int32_t)j; w[m] = wt; }
            ++m;
            stride *= L;
        }
    }
    return m;
}

/* ------------------------------------------------ fp32 replay (TEST-ONLY measurement tool)
 *
 * The reference's mars_descent (solvers.cpp:178-200 with relax_to_fixed_point 163-176,
 * mars_relax_sweep 150-161 and tanh_trial 145-148) replayed with fp32 arithmetic for the
 * state, the fields and tanh -- the precision class of the B200 dense kernels -- while the
 * control flow (temperature steps and the level loop in fp64, d vs d_min, the sweep cap) is
 * kept exactly.  It answers "how often does an fp32 computation of the same descent end on
 * the same spins as the fp64 reference", the floor the dense-kernel parity gate is set
 * from (tests/test_gpu_parity.py).  mode 0: J and h in fp32; mode 1: J rounded to a single
 * fp16 plane (a 2-product split), for the precision study in DESIGN.md.  Dense problems only. */
static float f16_round(float x) {
    /* round-to-nearest-even to an IEEE binary16 value (normal and subnormal range) */
    if (x == 0.0f || !isfinite(x)) return x;
    int e;
    frexpf(x, &e);                                      /* |x| in [2^(e-1), 2^e) */
    int q = e - 11;                                     /* ulp exponent, 11 significant bits */
    if (q < -24) q = -24;                               /* fp16 subnormal spacing */
    return ldexpf(nearbyintf(ldexpf(x, -q)), q);
}

static int replay_descent_f32(const orc_problem* p, const float* Jf, const float* hf, double start_temp,
                              const orc_params_t* prm, uint64_t seed, int8_t* spins, int64_t* iters) {
    const int n = p->n;
    float* s = (float*)malloc(sizeof(float) * (size_t)n);
    double* s64 = (double*)malloc(sizeof(double) * (size_t)n);
    orc_initial_state(seed, n, s64);
    for (int i = 0; i < n; ++i) s[i] = (float)s64[i];
    int64_t budget = g_sweep_cap, total = 0, sweeps = 0;
    double t_t = start_temp;
    int rc = 0;
    while (t_t > 0.0) {
        t_t -= prm->c_step;
        const float tf = (float)t_t;
        const int quench = t_t < K_TEMP_FLOOR;
        double d;
        sweeps = 0;
        do {
            if (budget <= 0) { rc = 2; break; }
            --budget;
            float dm = 0.0f;
            for (int i = 0; i < n; ++i) {
                const float* row = Jf + (size_t)i * n;
                float phi = 0.0f;
                for (int j = 0; j < n; ++j) phi = fmaf(row[j], s[j], phi);
                phi += hf[i];
                const float trial = quench ? (phi > 0.0f ? -1.0f : (phi < 0.0f ? 1.0f : 0.0f)) : -tanhf(phi / tf);
                const float dd = fabsf(trial - s[i]);
                dm = dm > dd ? dm : dd;
                s[i] = trial;
            }
            d = dm;
            ++sweeps;
        } while (d > prm->d_min);
        if (rc) break;
        total += sweeps;
    }
    for (int i = 0; i < n; ++i) spins[i] = s[i] < 0.0f ? -1 : 1;
    *iters = rc ? sweeps : total;
    free(s);
    free(s64);
    return rc;
}

typedef struct {
    const orc_problem* p;
    const orc_params_t* prm;
    const float *Jf, *hf;
    uint64_t base;
    int64_t runs, next;
    uint8_t* status;
    int64_t* iters;
    int8_t* spins;
    pthread_mutex_t mu;
} replay_ctx;

static void* replay_worker(void* arg) {
    replay_ctx* c = (replay_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        const int64_t k = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (k >= c->runs) return NULL;
        int skipped;
        double t;
        uint64_t seed;
        orc_run_plan(c->prm, c->base, k, &skipped, &t, &seed);
        if (skipped) { c->status[k] = 1; c->iters[k] = 0; continue; }
        c->status[k] = (uint8_t)replay_descent_f32(c->p, c->Jf, c->hf, t, c->prm, seed,
                                                   c->spins + (size_t)k * c->p->n, &c->iters[k]);
    }
}

int orc_replay_batch_f32(const void* vp, const orc_params_t* prm, int64_t runs, uint64_t base, int workers,
                         int mode, uint8_t* status, int64_t* iters, int8_t* spins) {
    const orc_problem* p = (const orc_problem*)vp;
    if (!p->dense) return 1;
    const int n = p->n;
    float* Jf = (float*)malloc(sizeof(float) * (size_t)n * n);
    float* hf = (float*)malloc(sizeof(float) * (size_t)n);
    for (size_t k = 0; k < (size_t)n * n; ++k) Jf[k] = mode == 1 ? f16_round((float)p->J[k]) : (float)p->J[k];
    for (int i = 0; i < n; ++i) hf[i] = (float)p->h[i];
    replay_ctx c = {p, prm, Jf, hf, base, runs, 0, status, iters, spins, PTHREAD_MUTEX_INITIALIZER};
    int w = workers > 0 ? workers : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (w < 1) w = 1;
    if (w > runs) w = (int)runs;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)w);
    for (int i = 0; i < w; ++i) pthread_create(&th[i], NULL, replay_worker, &c);
    for (int i = 0; i < w; ++i) pthread_join(th[i], NULL);
    free(th);
    free(Jf);
    free(hf);
    return 0;
}

/* TEST-ONLY: mars_relax_sweep (solvers.cpp:150-161) in fp32 -- fp32 state, row dot accumulated
 * in fp32 in ascending j, tanhf -- the single-sweep fp32 floor the device trajectory gates of
 * tests/test_gpu_trajectory.py are set from (dense problems only; returns d). */
double orc_relax_sweep_f32(const void* vp, float* s, double t) {
    const orc_problem* p = (const orc_problem*)vp;
    const int n = p->n;
    const float tf = (float)t;
    float d = 0.0f;
    for (int i = 0; i < n; ++i) {
        const double* row = p->J + (size_t)i * n;
        float phi = 0.0f;
        for (int j = 0; j < n; ++j) phi = fmaf((float)row[j], s[j], phi);
        phi += (float)p->h[i];
        const float trial = t < K_TEMP_FLOOR ? (phi > 0.0f ? -1.0f : (phi < 0.0f ? 1.0f : 0.0f)) : -tanhf(phi / tf);
        const float dd = fabsf(trial - s[i]);
        d = d > dd ? d : dd;
        s[i] = trial;
    }
    return d;
}
