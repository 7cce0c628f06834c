// TEST INFRASTRUCTURE ONLY — C entry points over the REFERENCE's own sources.
//
// `make -C oracle ref` compiles /root/reference/proj/src/{contour,matmodel,
// filterop,ritz,drivers}.cpp unmodified (from where they lie; nothing is
// copied) against oracle/eigen_shim (a minimal Eigen-API stand-in on OpenBLAS;
// Eigen itself is absent from this image) together with this file into
// oracle/_ref/libfeastlab_ref.so. The symbols are the `orc_*` entry points of
// feast_oracle.cpp (same names, same signatures), so oracle/__init__.py can
// drive either library and tests/test_ref_pin.py can compare the restatement
// with the reference's own control flow call by call.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "feastlab/contour.hpp"
#include "feastlab/drivers.hpp"
#include "feastlab/filterop.hpp"
#include "feastlab/matmodel.hpp"
#include "feastlab/ritz.hpp"

using namespace feastlab;
using Eigen::MatrixXcd;
using Eigen::MatrixXd;
using Eigen::VectorXd;

namespace {

MatrixXd wrap(const double* p, int r, int c) {
    MatrixXd M(r, c);
    if (static_cast<size_t>(r) * c > 0) std::memcpy(M.data(), p, sizeof(double) * (size_t)r * c);
    return M;
}
ContourRule wrap_rule(int nc, const double* zr, const double* zi, const double* wr,
                      const double* wi) {
    // the interval of a wrapped rule is not read on the filter path
    ContourRule r{SearchInterval(-1.0, 1.0), {}, {}};
    for (int k = 0; k < nc; ++k) {
        r.nodes.emplace_back(zr[k], zi[k]);
        r.weights.emplace_back(wr[k], wi[k]);
    }
    return r;
}
RitzSet wrap_ritz(const double* vals, const double* V, const double* norms,
                  const unsigned char* inside, int n, int p) {
    RitzSet r;
    r.values.resize(p);
    r.residual_norms.resize(p);
    r.inside_flags.resize(p);
    for (int k = 0; k < p; ++k) {
        r.values[k] = vals[k];
        r.residual_norms[k] = norms ? norms[k] : 0.0;
        r.inside_flags[k] = inside ? inside[k] != 0 : false;
    }
    if (V) r.vectors = wrap(V, n, p);
    else r.vectors.resize(0, p);
    return r;
}

}  // namespace

extern "C" {

struct orc_err {
    int status;
    int index;
    double pivot;
    double z_re, z_im;
    char msg[512];
};

static int fail(orc_err* e, int code, const char* m) {
    if (e) {
        e->status = code;
        std::snprintf(e->msg, sizeof(e->msg), "%s", m);
    }
    return code;
}

// The reference reports a singular node as a plain std::runtime_error
// (filterop.cpp:19-22), so code 4 never comes from this library.
#define REF_TRY try {
#define REF_CATCH(e)                                                        \
    }                                                                       \
    catch (const CholeskyError& x) {                                        \
        if (e) { e->pivot = x.pivot; e->index = x.index; }                  \
        return fail(e, 3, x.what());                                        \
    }                                                                       \
    catch (const std::invalid_argument& x) { return fail(e, 1, x.what()); } \
    catch (const std::exception& x) { return fail(e, 2, x.what()); }        \
    return 0;

void orc_set_threads(int t) { scipy_openblas_set_num_threads(t); }
int orc_get_threads(void) { return scipy_openblas_get_num_threads(); }

int orc_gauss_legendre(int n, double* nodes, double* weights, orc_err* e) {
    REF_TRY
    GaussLegendreRule g = gauss_legendre(n);
    std::memcpy(nodes, g.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, g.weights.data(), sizeof(double) * n);
    REF_CATCH(e)
}

int orc_build_contour_rule(double lo, double hi, int nc, double* zr, double* zi, double* wr,
                           double* wi, orc_err* e) {
    REF_TRY
    ContourRule r = build_contour_rule(SearchInterval(lo, hi), nc);
    for (int k = 0; k < nc; ++k) {
        zr[k] = r.nodes[k].real(); zi[k] = r.nodes[k].imag();
        wr[k] = r.weights[k].real(); wi[k] = r.weights[k].imag();
    }
    REF_CATCH(e)
}

double orc_filter_value(int nc, const double* zr, const double* zi, const double* wr,
                        const double* wi, double lambda) {
    return filter_value(wrap_rule(nc, zr, zi, wr, wi), lambda);
}

int orc_predicted_rate(int nc, const double* zr, const double* zi, const double* wr,
                       const double* wi, const double* spectrum, int ns, int m0, double* out,
                       orc_err* e) {
    REF_TRY
    *out = predicted_rate(wrap_rule(nc, zr, zi, wr, wi),
                          std::vector<double>(spectrum, spectrum + ns), m0);
    REF_CATCH(e)
}

int orc_symmetric_matrix(const double* M, int n, double sym_tol, double* out, orc_err* e) {
    REF_TRY
    SymmetricMatrix S(wrap(M, n, n), sym_tol);
    std::memcpy(out, S.mat().data(), sizeof(double) * (size_t)n * n);
    REF_CATCH(e)
}

// generate_spectrum (proj/src/matmodel.cpp:60-110): values ascending + Q.
int orc_generate_spectrum(int n, double in_lo, double in_hi, int in_count, double out_lo,
                          double out_hi, int out_count, int clustered, int num_clusters,
                          double cluster_width, unsigned long long seed, double* values,
                          double* Q, orc_err* e) {
    REF_TRY
    SpectrumLayout L{n, SearchInterval(in_lo, in_hi), in_count, SearchInterval(out_lo, out_hi),
                     out_count, clustered ? Placement::clustered : Placement::uniform,
                     num_clusters, cluster_width, seed};
    EigenDecomposition d = generate_spectrum(L);
    std::memcpy(values, d.values.data(), sizeof(double) * n);
    std::memcpy(Q, d.vectors.data(), sizeof(double) * (size_t)n * n);
    REF_CATCH(e)
}

int orc_assemble_matrix(int n, const double* values, const double* Q, double* A, orc_err* e) {
    REF_TRY
    EigenDecomposition d;
    d.values = Eigen::Map<VectorXd>(values, n);
    d.vectors = wrap(Q, n, n);
    SymmetricMatrix S = assemble_matrix(d);
    std::memcpy(A, S.mat().data(), sizeof(double) * (size_t)n * n);
    REF_CATCH(e)
}

// NodeFactorization(A, z).solve(B) with complex B (interleaved).
int orc_node_solve(const double* A, int n, double zr, double zi, const double* B, int p, double* W,
                   orc_err* e) {
    REF_TRY
    SymmetricMatrix S(wrap(A, n, n));
    NodeFactorization f(S, {zr, zi}, -1);
    MatrixXcd Bm(n, p);
    std::memcpy(static_cast<void*>(Bm.data()), B, sizeof(double) * 2 * (size_t)n * p);
    MatrixXcd Wm = f.solve(Bm);
    std::memcpy(W, Wm.data(), sizeof(double) * 2 * (size_t)n * p);
    REF_CATCH(e)
}

int orc_apply_filter(const double* A, int n, int nc, const double* zr, const double* zi,
                     const double* wr, const double* wi, const double* X, int xr, int p,
                     int cache, int napply, double* Y, long long* rhs, long long* facts,
                     orc_err* e) {
    REF_TRY
    SymmetricMatrix S(wrap(A, n, n));
    ContourRule rule = wrap_rule(nc, zr, zi, wr, wi);
    FilterApplier ap(S, rule, cache != 0);
    SolveAccounting acc{*rhs, *facts};
    MatrixXd Xm = wrap(X, xr, p);
    MatrixXd Ym;
    for (int i = 0; i < napply; ++i) Ym = ap.apply(Xm, acc);
    std::memcpy(Y, Ym.data(), sizeof(double) * (size_t)xr * p);
    *rhs = acc.rhs_solved;
    *facts = acc.factorizations;
    REF_CATCH(e)
}

int orc_orthonormalize(const double* X, int n, int p, double drop_tol, int method, double* U,
                       int* rank, orc_err* e) {
    REF_TRY
    auto [Um, r] = orthonormalize(wrap(X, n, p), drop_tol,
                                  method == 1 ? Orthogonalizer::qr : Orthogonalizer::svd);
    std::memcpy(U, Um.data(), sizeof(double) * (size_t)n * r);
    *rank = r;
    REF_CATCH(e)
}

int orc_rayleigh_ritz(const double* A, int n, const double* X, int xr, int p, double lo, double hi,
                      double* vals, double* V, double* norms, unsigned char* inside, orc_err* e) {
    REF_TRY
    SymmetricMatrix S(wrap(A, n, n));
    RitzSet r = rayleigh_ritz(S, wrap(X, xr, p), SearchInterval(lo, hi));
    std::memcpy(vals, r.values.data(), sizeof(double) * p);
    std::memcpy(V, r.vectors.data(), sizeof(double) * (size_t)n * p);
    std::memcpy(norms, r.residual_norms.data(), sizeof(double) * p);
    for (int k = 0; k < p; ++k) inside[k] = r.inside_flags[k];
    REF_CATCH(e)
}

int orc_residual_block(const double* A, int n, const double* vals, const double* V, int p,
                       double* R, orc_err* e) {
    REF_TRY
    SymmetricMatrix S(wrap(A, n, n));
    MatrixXd Rm = compute_residual_block(S, wrap_ritz(vals, V, nullptr, nullptr, n, p));
    std::memcpy(R, Rm.data(), sizeof(double) * (size_t)n * p);
    REF_CATCH(e)
}

// select_pairs: the chosen indices. The reference returns the gathered pairs,
// not the indices, so the values array carries each pair's index in through
// a one-row "vectors" block and the selection is read back from it.
int orc_select_pairs(const double* vals, const double* norms, const unsigned char* inside, int p,
                     int m0, double lo, double hi, int* chosen, int* nchosen, orc_err* e) {
    REF_TRY
    std::vector<double> tag(p);
    for (int k = 0; k < p; ++k) tag[k] = k;
    RitzSet r = wrap_ritz(vals, tag.data(), norms, inside, 1, p);
    RitzSet s = select_pairs(r, SelectionPolicy{m0, SearchInterval(lo, hi)});
    for (int j = 0; j < s.size(); ++j) chosen[j] = static_cast<int>(s.vectors(0, j));
    *nchosen = s.size();
    REF_CATCH(e)
}

int orc_make_initial_guess(int n, int m0, unsigned long long seed, double* X, orc_err* e) {
    REF_TRY
    MatrixXd M = make_initial_guess(n, m0, seed);
    std::memcpy(X, M.data(), sizeof(double) * (size_t)n * m0);
    REF_CATCH(e)
}

struct orc_config {
    int m0, n_c, s;
    double tol;
    int max_iter;
    unsigned long long seed;
    int orthogonalizer;
    double drop_tol;
    int cache_factorizations, generalized_reduced;
};

struct orc_trace {
    int iter, subspace_dim;
    long long rhs_cumulative;
    double max_residual;
    int m_found;
};

// variant: 0 feast, 1 xfeast, 2 rfeast. first_filtered is not part of the
// reference's Solution and is left untouched.
int orc_solve(int variant, const double* A, int n, double lo, double hi, const orc_config* c,
              double* values, double* vectors, double* norms, int* m, int* converged,
              int* iterations, long long* rhs, long long* facts, int* recovery, orc_trace* trace,
              int* ntrace, double* first_filtered, orc_err* e) {
    (void)first_filtered;
    REF_TRY
    SolverConfig cfg;
    cfg.m0 = c->m0; cfg.n_c = c->n_c; cfg.s = c->s; cfg.tol = c->tol; cfg.max_iter = c->max_iter;
    cfg.seed = c->seed;
    cfg.orthogonalizer = c->orthogonalizer == 1 ? Orthogonalizer::qr : Orthogonalizer::svd;
    cfg.drop_tol = c->drop_tol;
    cfg.cache_factorizations = c->cache_factorizations != 0;
    cfg.generalized_reduced = c->generalized_reduced != 0;
    SymmetricMatrix S(wrap(A, n, n));
    SearchInterval I(lo, hi);
    Solution s = variant == 0 ? feast_solve(S, I, cfg)
                 : variant == 1 ? xfeast_solve(S, I, cfg)
                                : rfeast_solve(S, I, cfg);
    const int mm = static_cast<int>(s.eigenvalues.size());
    *m = mm;
    std::memcpy(values, s.eigenvalues.data(), sizeof(double) * mm);
    std::memcpy(norms, s.residual_norms.data(), sizeof(double) * mm);
    std::memcpy(vectors, s.eigenvectors.data(), sizeof(double) * (size_t)n * mm);
    *converged = s.converged;
    *iterations = s.iterations;
    *rhs = s.accounting.rhs_solved;
    *facts = s.accounting.factorizations;
    *recovery = s.recovery_events;
    *ntrace = static_cast<int>(s.trace.records.size());
    for (size_t t = 0; t < s.trace.records.size(); ++t) {
        const TraceRecord& q = s.trace.records[t];
        trace[t] = {q.iter, q.subspace_dim, q.rhs_cumulative, q.max_residual, q.m_found};
    }
    REF_CATCH(e)
}

}  // extern "C"
