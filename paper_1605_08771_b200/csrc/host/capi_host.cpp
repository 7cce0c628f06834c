// Host-level C ABI entry points (include/feastlab_b200.h, bottom section):
// the drop-in C++ drivers and contour helpers exported for foreign callers.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "feastlab/drivers.hpp"
#include "feastlab/matrix_market.hpp"
#include "feastlab_b200.h"

namespace feastlab {
namespace detail {
extern thread_local bool keep_first_filtered;
}
}  // namespace feastlab

using namespace feastlab;

namespace {

int fail(fl_err* e, int code, const char* msg) {
    if (e) {
        e->status = code;
        std::snprintf(e->msg, sizeof(e->msg), "%s", msg);
    }
    return code;
}

template <class F>
int guarded(fl_err* err, F&& body) {
    try {
        body();
        return FL_OK;
    } catch (const NotSymmetricError& x) {
        if (err) err->index = x.line;
        return fail(err, FL_NOT_SYMMETRIC, x.what());
    } catch (const MatrixMarketError& x) {
        if (err) err->index = x.line;
        return fail(err, FL_MATRIX_MARKET, x.what());
    } catch (const CholeskyError& x) {
        if (err) {
            err->pivot = x.pivot;
            err->index = x.index;
        }
        return fail(err, FL_CHOLESKY, x.what());
    } catch (const std::invalid_argument& x) {
        return fail(err, FL_INVALID_ARGUMENT, x.what());
    } catch (const std::bad_alloc&) {
        return fail(err, FL_OOM, "host allocation failed");
    } catch (const std::exception& x) {
        return fail(err, FL_RUNTIME_ERROR, x.what());
    }
}

struct ScopedContext {
    explicit ScopedContext(fl_ctx* c) { set_current_context(c); }
    ~ScopedContext() { set_current_context(nullptr); }
};

}  // namespace

extern "C" {

int fl_solve(fl_ctx* ctx, int variant, const double* A, int n, int lda, double lo, double hi,
             const fl_solver_config* c, double* values, double* vectors, double* norms, int* m,
             int* converged, int* iterations, long long* rhs_solved, long long* factorizations,
             int* recovery_events, fl_trace_record* trace, int* ntrace, double* first_filtered,
             fl_err* err) {
    return guarded(err, [&] {
        if (n < 1 || lda < n) throw std::invalid_argument("fl_solve: bad matrix shape");
        ScopedContext sc(ctx);
        const auto t0 = std::chrono::steady_clock::now();
        const SymmetricMatrix S(A, n, lda);
        if (std::getenv("FEASTLAB_TIME"))
            std::fprintf(stderr, "fl_solve: SymmetricMatrix %.3f s\n",
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        SolverConfig cfg;
        cfg.m0 = c->m0;
        cfg.n_c = c->n_c;
        cfg.s = c->s;
        cfg.tol = c->tol;
        cfg.max_iter = c->max_iter;
        cfg.seed = c->seed;
        cfg.orthogonalizer = c->orthogonalizer == 1 ? Orthogonalizer::qr : Orthogonalizer::svd;
        cfg.drop_tol = c->drop_tol;
        cfg.cache_factorizations = c->cache_factorizations != 0;
        cfg.generalized_reduced = c->generalized_reduced != 0;
        const SearchInterval I(lo, hi);
        detail::keep_first_filtered = first_filtered != nullptr;
        struct Reset {
            ~Reset() { detail::keep_first_filtered = false; }
        } reset;
        const auto t1 = std::chrono::steady_clock::now();
        Solution s = variant == 0   ? feast_solve(S, I, cfg)
                     : variant == 1 ? xfeast_solve(S, I, cfg)
                                    : rfeast_solve(S, I, cfg);
        if (std::getenv("FEASTLAB_TIME"))
            std::fprintf(stderr, "fl_solve: driver %.3f s\n",
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count());
        const int k = s.eigenvalues.size();
        *m = k;
        std::memcpy(values, s.eigenvalues.data(), sizeof(double) * k);
        std::memcpy(norms, s.residual_norms.data(), sizeof(double) * k);
        std::memcpy(vectors, s.eigenvectors.data(), sizeof(double) * (size_t)n * k);
        *converged = s.converged ? 1 : 0;
        *iterations = s.iterations;
        *rhs_solved = s.accounting.rhs_solved;
        *factorizations = s.accounting.factorizations;
        *recovery_events = s.recovery_events;
        *ntrace = static_cast<int>(s.trace.records.size());
        for (size_t t = 0; t < s.trace.records.size(); ++t) {
            const TraceRecord& r = s.trace.records[t];
            trace[t] = {r.iter, r.subspace_dim, r.rhs_cumulative, r.max_residual, r.m_found};
        }
        if (first_filtered && s.first_filtered.cols() > 0)
            std::memcpy(first_filtered, s.first_filtered.data(),
                        sizeof(double) * s.first_filtered.size());
    });
}

int fl_gauss_legendre(int n, double* nodes, double* weights, fl_err* err) {
    return guarded(err, [&] {
        GaussLegendreRule g = gauss_legendre(n);
        std::memcpy(nodes, g.nodes.data(), sizeof(double) * n);
        std::memcpy(weights, g.weights.data(), sizeof(double) * n);
    });
}

int fl_build_contour_rule(double lo, double hi, int n_c, double* zr, double* zi, double* wr,
                          double* wi, fl_err* err) {
    return guarded(err, [&] {
        ContourRule r = build_contour_rule(SearchInterval(lo, hi), n_c);
        for (int k = 0; k < n_c; ++k) {
            zr[k] = r.nodes[k].real();
            zi[k] = r.nodes[k].imag();
            wr[k] = r.weights[k].real();
            wi[k] = r.weights[k].imag();
        }
    });
}

double fl_filter_value(int n_c, const double* zr, const double* zi, const double* wr,
                       const double* wi, double lambda) {
    ContourRule r{SearchInterval(-1, 1), {}, {}};
    for (int k = 0; k < n_c; ++k) {
        r.nodes.emplace_back(zr[k], zi[k]);
        r.weights.emplace_back(wr[k], wi[k]);
    }
    return filter_value(r, lambda);
}

int fl_symmetric_matrix(const double* M, int n, int ldm, double sym_tol, double* out, fl_err* err) {
    return guarded(err, [&] {
        if (n < 1 || ldm < n)
            throw std::invalid_argument("SymmetricMatrix: matrix must be square, n >= 1");
        SymmetricMatrix S(M, n, ldm, sym_tol);
        std::memcpy(out, S.mat().data(), sizeof(double) * (size_t)n * n);
    });
}

int fl_mm_read(const char* path, int* n, double* A, int lda, fl_err* err) {
    return guarded(err, [&] {
        if (!path) throw std::invalid_argument("read_matrix_market: null path");
        const int m = read_matrix_market_into(path, A, lda);
        if (n) *n = m;
    });
}

int fl_mm_write(const char* path, const double* A, int n, int lda, int format, fl_err* err) {
    return guarded(err, [&] {
        if (!path || n < 1 || lda < n) throw std::invalid_argument("write_matrix_market: bad arguments");
        write_matrix_market(A, n, lda, path,
                            format ? MatrixMarketFormat::array : MatrixMarketFormat::coordinate);
    });
}

int fl_make_initial_guess(fl_ctx* ctx, int n, int m0, uint64_t seed, double* X, fl_err* err) {
    return guarded(err, [&] {
        ScopedContext sc(ctx);
        MatrixXd G = make_initial_guess(n, m0, seed);
        std::memcpy(X, G.data(), sizeof(double) * G.size());
    });
}

int fl_select_pairs(const double* vals, const double* norms, const unsigned char* inside, int p,
                    int m0, double lo, double hi, int* chosen, int* nchosen, fl_err* err) {
    return guarded(err, [&] {
        std::vector<double> v(vals, vals + p), r(norms, norms + p);
        std::vector<bool> f(inside, inside + p);
        const std::vector<int> idx = select_indices(v, r, f, SelectionPolicy{m0, SearchInterval(lo, hi)});
        for (size_t j = 0; j < idx.size(); ++j) chosen[j] = idx[j];
        *nchosen = static_cast<int>(idx.size());
    });
}

void fl_gaussian_fill(double* out, long long count, uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (long long i = 0; i < count; ++i) out[i] = normal(gen);
}

void fl_uniform_fill(double* out, long long count, double lo, double hi, uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> u(lo, hi);
    for (long long i = 0; i < count; ++i) out[i] = u(gen);
}

}  // extern "C"

int fl_solve_many(const int* devices, int ndev, int per_device, const double* A, int n, int lda,
                  int njobs, const int* variant, const double* lo, const double* hi,
                  const fl_solver_config* cfgs, double* values, int ldv, int* m, int* converged,
                  int* iterations, double* max_residual, int* status, char* errors, fl_err* err) {
    return guarded(err, [&] {
        if (n < 1 || lda < n || njobs < 0 || ndev < 0 || (njobs > 0 && ldv < 1))
            throw std::invalid_argument("fl_solve_many: bad arguments");
        const SymmetricMatrix S(A, n, lda);
        std::vector<SolveJob> jobs;
        for (int j = 0; j < njobs; ++j) {
            const fl_solver_config* c = cfgs + j;
            SolverConfig cfg;
            cfg.m0 = c->m0;
            cfg.n_c = c->n_c;
            cfg.s = c->s;
            cfg.tol = c->tol;
            cfg.max_iter = c->max_iter;
            cfg.seed = c->seed;
            cfg.orthogonalizer = c->orthogonalizer == 1 ? Orthogonalizer::qr : Orthogonalizer::svd;
            cfg.drop_tol = c->drop_tol;
            cfg.cache_factorizations = c->cache_factorizations != 0;
            cfg.generalized_reduced = c->generalized_reduced != 0;
            jobs.emplace_back(variant[j] == 1   ? SolveVariant::xfeast
                              : variant[j] == 2 ? SolveVariant::rfeast
                                                : SolveVariant::feast,
                              SearchInterval(lo[j], hi[j]), cfg);
        }
        std::vector<int> devs(devices, devices + ndev);
        const std::vector<JobResult> res = solve_concurrently(S, jobs, devs, per_device);
        for (int j = 0; j < njobs; ++j) {
            const Solution& sol = res[j].solution;
            const int k = std::min<int>(static_cast<int>(sol.eigenvalues.size()), ldv);
            m[j] = k;
            std::memcpy(values + (size_t)j * ldv, sol.eigenvalues.data(), sizeof(double) * k);
            converged[j] = sol.converged ? 1 : 0;
            iterations[j] = sol.iterations;
            max_residual[j] = sol.trace.records.empty() ? 0.0 : sol.trace.records.back().max_residual;
            status[j] = res[j].failed ? FL_RUNTIME_ERROR : FL_OK;
            if (errors) {
                char* e = errors + (size_t)j * 256;
                std::snprintf(e, 256, "%s", res[j].error.c_str());
            }
        }
    });
}

extern "C" int fl_node_shard(int n_c, int rank, int nranks, int* k_begin, int* k_end) {
    if (nranks < 1 || rank < 0 || rank >= nranks || n_c < 0) return FL_INVALID_ARGUMENT;
    *k_begin = static_cast<int>(static_cast<long long>(n_c) * rank / nranks);
    *k_end = static_cast<int>(static_cast<long long>(n_c) * (rank + 1) / nranks);
    return FL_OK;
}
