// FEAST / XFEAST / RFEAST drivers (proj/src/drivers.cpp:13-252), host C++
// orchestration over device-resident blocks: only Ritz values, residual norms
// and flags (<= s*m0 scalars per iteration) cross PCIe; the subspace blocks,
// the filter and the Rayleigh-Ritz algebra stay in HBM.
#include "feastlab/drivers.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <numeric>
#include <ostream>
#include <random>
#include <stdexcept>

#include "feastlab/device.hpp"

namespace feastlab {

namespace detail {
// set by the C ABI entry point when the caller wants Y_1 back (parity hook)
thread_local bool keep_first_filtered = false;
}  // namespace detail

void write_trace_csv(std::ostream& os, const ConvergenceTrace& trace) {
    os << "iter,subspace_dim,rhs_cumulative,max_residual,m_found\n";
    for (const TraceRecord& t : trace.records) {
        char line[160];
        std::snprintf(line, sizeof(line), "%d,%d,%lld,%.17g,%d\n", t.iter, t.subspace_dim,
                      t.rhs_cumulative, t.max_residual, t.m_found);
        os << line;
    }
}

namespace {

// FEASTLAB_TIME=1: per-phase wall time of the feast_solve loop on stderr
// (the context is synchronised at each phase boundary)
struct PhaseTimer {
    bool on = std::getenv("FEASTLAB_TIME") != nullptr;
    fl_ctx* ctx;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double filter = 0, orth = 0, rr = 0, host = 0, setup = 0, upload = 0, guess = 0;
    explicit PhaseTimer(fl_ctx* c) : ctx(c) {}
    void lap(double& acc) {
        if (!on) return;
        fl_err e{};
        fl_ctx_sync(ctx, &e);
        const auto t = std::chrono::steady_clock::now();
        acc += std::chrono::duration<double>(t - t0).count();
        t0 = t;
    }
    ~PhaseTimer() {
        if (on)
            std::fprintf(stderr, "feast_solve phases [s]: matrix upload %.3f initial guess %.3f "
                                 "setup %.3f filter %.3f orthonormalize %.3f rayleigh_ritz %.3f "
                                 "host %.3f\n", upload, guess, setup, filter, orth, rr, host);
    }
};

// Ritz pairs with the vectors left on the device
struct DevRitz {
    std::vector<double> values, norms;
    std::vector<bool> inside;
    DeviceBlock vectors;
    explicit DevRitz(fl_ctx* ctx, int n) : vectors(ctx, n, 1) {}
    int size() const { return static_cast<int>(values.size()); }
};

void rr_device(fl_ctx* ctx, const DeviceMatrix& A, const DeviceBlock& X,
               const SearchInterval& I, DevRitz& out) {
    const int p = X.cols();
    out.values.assign(p, 0.0);
    out.norms.assign(p, 0.0);
    std::vector<unsigned char> flags(p);
    fl_err err{};
    check(fl_rayleigh_ritz(ctx, A.get(), X.get(), I.lo, I.hi, out.values.data(),
                           out.vectors.get(), out.norms.data(), flags.data(), &err),
          err);
    out.inside.assign(flags.begin(), flags.end());
}

int orth_device(fl_ctx* ctx, const DeviceBlock& X, const SolverConfig& cfg, DeviceBlock& U) {
    int rank = 0;
    fl_err err{};
    check(fl_orthonormalize(ctx, X.get(), cfg.drop_tol,
                            cfg.orthogonalizer == Orthogonalizer::qr ? 1 : 0, U.get(), &rank, &err),
          err);
    return rank;
}

void gather(const DeviceBlock& src, const std::vector<int>& idx, DeviceBlock& dst) {
    fl_err err{};
    check(fl_block_gather(dst.get(), src.get(), idx.data(), static_cast<int>(idx.size()), &err),
          err);
}

// select_pairs (ritz.cpp:124-166): host ordering, device column gather
void select_device(fl_ctx* ctx, const DevRitz& rr, const SelectionPolicy& pol, DevRitz& out) {
    const std::vector<int> idx = select_indices(rr.values, rr.norms, rr.inside, pol);
    const int k = static_cast<int>(idx.size());
    out.values.resize(k);
    out.norms.resize(k);
    out.inside.resize(k);
    for (int j = 0; j < k; ++j) {
        out.values[j] = rr.values[idx[j]];
        out.norms[j] = rr.norms[idx[j]];
        out.inside[j] = rr.inside[idx[j]];
    }
    gather(rr.vectors, idx, out.vectors);
    (void)ctx;
}

void validate_config(const SymmetricMatrix& A, const SolverConfig& c) {  // drivers.cpp:42-48
    if (c.m0 < 1 || c.m0 > A.dim()) throw std::invalid_argument("SolverConfig: require 1 <= m0 <= n");
    if (c.s < 1) throw std::invalid_argument("SolverConfig: require s >= 1");
    if (!(c.tol > 0.0)) throw std::invalid_argument("SolverConfig: require tol > 0");
    if (c.max_iter < 1) throw std::invalid_argument("SolverConfig: require max_iter >= 1");
}

// inside pairs by ascending residual, ties by index (drivers.cpp:51-61)
std::vector<int> inside_by_residual(const DevRitz& rr) {
    std::vector<int> idx;
    for (int k = 0; k < rr.size(); ++k)
        if (rr.inside[k]) idx.push_back(k);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) {
        return rr.norms[a] != rr.norms[b] ? rr.norms[a] < rr.norms[b] : a < b;
    });
    return idx;
}

double max_residual(const DevRitz& rr, const std::vector<int>& idx) {
    double r = 0.0;
    for (int k : idx) r = std::max(r, rr.norms[k]);
    return r;
}

// pairs into the solution, ascending eigenvalue (drivers.cpp:70-82)
void fill_solution(fl_ctx* ctx, Solution& sol, const DevRitz& rr, std::vector<int> idx) {
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return rr.values[a] < rr.values[b]; });
    const int m = static_cast<int>(idx.size());
    sol.eigenvalues.resize(m);
    sol.residual_norms.resize(m);
    for (int j = 0; j < m; ++j) {
        sol.eigenvalues[j] = rr.values[idx[j]];
        sol.residual_norms[j] = rr.norms[idx[j]];
    }
    DeviceBlock V(ctx, rr.vectors.rows(), std::max(m, 1));
    gather(rr.vectors, idx, V);
    sol.eigenvectors = V.download();
}

void record(Solution& sol, int iter, int dim, double r, int m_found) {
    sol.trace.records.push_back({iter, dim, sol.accounting.rhs_solved, r, m_found});
    sol.iterations = iter;
}

DeviceBlock initial_block(fl_ctx* ctx, const SymmetricMatrix& A, const SolverConfig& cfg) {
    DeviceBlock X(ctx, A.dim(), cfg.m0);
    X.set(make_initial_guess(A.dim(), cfg.m0, cfg.seed));
    return X;
}

}  // namespace

// drivers.cpp:23-38: mt19937_64(seed ^ golden), N(0,1), column-major; the
// rank check is the reference's (ColPivHouseholderQR, threshold 1e-10:
// drivers.cpp:33-36) on the device (fl_block_rank -> column-pivoted QR).
MatrixXd make_initial_guess(int n, int m0, std::uint64_t seed) {
    if (m0 < 1 || m0 > n) throw std::invalid_argument("make_initial_guess: require 1 <= m0 <= n");
    std::mt19937_64 gen(seed ^ 0x9e3779b97f4a7c15ULL);
    std::normal_distribution<double> normal(0.0, 1.0);
    MatrixXd X(n, m0);
    double* x = X.data();
    for (size_t e = 0; e < X.size(); ++e) x[e] = normal(gen);
    fl_ctx* ctx = current_context();
    DeviceBlock dX(ctx, n, m0);
    dX.set(X);
    int rank = 0;
    fl_err err{};
    check(fl_block_rank(ctx, dX.get(), 1e-10, &rank, &err), err);
    if (rank < m0) throw std::runtime_error("make_initial_guess: guess block is rank deficient");
    return X;
}

Solution feast_solve(const SymmetricMatrix& A, const SearchInterval& interval,
                     const SolverConfig& config) {
    validate_config(A, config);
    fl_ctx* ctx = current_context();
    PhaseTimer timer(ctx);
    const ContourRule rule = build_contour_rule(interval, config.n_c);
    FilterApplier filt(A, rule, config.cache_factorizations);
    timer.lap(timer.upload);
    const int n = A.dim();
    Solution sol;
    DeviceBlock X = initial_block(ctx, A, config);
    timer.lap(timer.guess);
    DeviceBlock Y(ctx, n, config.m0), U(ctx, n, config.m0);
    DevRitz rr(ctx, n);
    int last_m_found = 0;
    timer.lap(timer.setup);
    for (int iter = 1; iter <= config.max_iter; ++iter) {
        timer.lap(timer.host);
        filt.apply(X, Y, sol.accounting);
        timer.lap(timer.filter);
        if (iter == 1 && detail::keep_first_filtered) sol.first_filtered = Y.download();
        int dim;
        if (config.generalized_reduced) {
            rr_device(ctx, filt.device_matrix(), Y, interval, rr);
            dim = Y.cols();
            timer.lap(timer.rr);
        } else {
            const int rank = orth_device(ctx, Y, config, U);
            timer.lap(timer.orth);
            if (rank < last_m_found)
                throw std::runtime_error(
                    "feast_solve: filtered subspace rank collapsed below the inside "
                    "eigenpair count; m0 may be too small");
            rr_device(ctx, filt.device_matrix(), U, interval, rr);
            timer.lap(timer.rr);
            dim = rank;
        }
        const std::vector<int> inside = inside_by_residual(rr);
        const double r = max_residual(rr, inside);
        record(sol, iter, dim, r, static_cast<int>(inside.size()));
        last_m_found = static_cast<int>(inside.size());
        if (r <= config.tol) {
            sol.converged = true;
            fill_solution(ctx, sol, rr, inside);
            return sol;
        }
        // X <- the Ritz vectors by a device copy into X's own storage (not a
        // buffer swap): the filter's launch key (X, Y, p) then repeats from
        // iteration to iteration and the application is replayed from its
        // CUDA graph instead of re-captured (cfg4: ~0.4 s per iteration)
        fl_err err{};
        check(fl_block_copy(X.get(), rr.vectors.get(), &err), err);
    }
    fill_solution(ctx, sol, rr, inside_by_residual(rr));
    return sol;
}

Solution xfeast_solve(const SymmetricMatrix& A, const SearchInterval& interval,
                      const SolverConfig& config) {
    validate_config(A, config);
    if (static_cast<long>(config.s) * config.m0 > A.dim())
        std::fprintf(stderr, "xfeast_solve: warning: s*m0 = %ld exceeds matrix dimension %d\n",
                     static_cast<long>(config.s) * config.m0, A.dim());
    const ContourRule rule = build_contour_rule(interval, config.n_c);
    FilterApplier filt(A, rule, config.cache_factorizations);
    fl_ctx* ctx = current_context();
    const int n = A.dim();
    const SelectionPolicy policy{config.m0, interval};
    Solution sol;
    std::deque<DeviceBlock> window;
    window.push_back(initial_block(ctx, A, config));
    // the filter writes one fixed block and the window takes a copy, so the
    // application's launch key repeats and its CUDA graph is replayed
    DeviceBlock filtered(ctx, n, config.m0);
    auto push_filtered = [&](const DeviceBlock& src) {
        filt.apply(src, filtered, sol.accounting);
        if (sol.first_filtered.cols() == 0 && detail::keep_first_filtered)
            sol.first_filtered = filtered.download();
        DeviceBlock next(ctx, n, config.m0);
        fl_err err{};
        check(fl_block_copy(next.get(), filtered.get(), &err), err);
        window.push_back(std::move(next));
    };
    // pre-expansion: [X0, rho X0, ..., rho^{s-2} X0] (drivers.cpp:155-158)
    for (int k = 2; k < config.s; ++k) push_filtered(window.back());
    DeviceBlock estimate(ctx, n, config.m0);
    {
        fl_err err{};
        check(fl_block_copy(estimate.get(), window.back().get(), &err), err);
    }
    DeviceBlock stacked(ctx, n, config.s * config.m0), U(ctx, n, config.s * config.m0);
    DevRitz rr(ctx, n), sel(ctx, n);
    for (int iter = 1; iter <= config.max_iter; ++iter) {
        push_filtered(estimate);
        while (static_cast<int>(window.size()) > config.s) window.pop_front();
        // hconcat(window) (drivers.cpp:84-94)
        {
            fl_err err{};
            check(fl_block_copy(stacked.get(), window.front().get(), &err), err);
            for (size_t w = 1; w < window.size(); ++w)
                check(fl_block_append(stacked.get(), window[w].get(), &err), err);
        }
        const int rank = orth_device(ctx, stacked, config, U);
        rr_device(ctx, filt.device_matrix(), U, interval, rr);
        select_device(ctx, rr, policy, sel);
        const std::vector<int> inside = inside_by_residual(sel);
        const double r = max_residual(sel, inside);
        record(sol, iter, rank, r, static_cast<int>(inside.size()));
        if (r <= config.tol) {
            sol.converged = true;
            fill_solution(ctx, sol, sel, inside);
            return sol;
        }
        fl_err err{};  // copy, not swap: estimate keeps its storage (graph replay)
        check(fl_block_copy(estimate.get(), sel.vectors.get(), &err), err);
    }
    fill_solution(ctx, sol, sel, inside_by_residual(sel));
    return sol;
}

Solution rfeast_solve(const SymmetricMatrix& A, const SearchInterval& interval,
                      const SolverConfig& config) {
    validate_config(A, config);
    if (static_cast<long>(config.s + 1) * config.m0 > A.dim())
        std::fprintf(stderr, "rfeast_solve: warning: (s+1)*m0 = %ld exceeds matrix dimension %d\n",
                     static_cast<long>(config.s + 1) * config.m0, A.dim());
    const ContourRule rule = build_contour_rule(interval, config.n_c);
    FilterApplier filt(A, rule, config.cache_factorizations);
    fl_ctx* ctx = current_context();
    const int n = A.dim();
    const SelectionPolicy policy{config.m0, interval};
    Solution sol;
    DeviceBlock X = initial_block(ctx, A, config);
    DeviceBlock Xp(ctx, n, config.s * config.m0), U(ctx, n, config.s * config.m0);
    DeviceBlock R(ctx, n, config.m0);
    DevRitz rr(ctx, n), sel(ctx, n);
    int m_expected = 0;
    auto trimmed_inside = [&]() {
        std::vector<int> inside = inside_by_residual(sel);
        if (static_cast<int>(inside.size()) > m_expected) inside.resize(m_expected);
        return inside;
    };
    for (int iter = 1; iter <= config.max_iter; ++iter) {
        filt.apply(X, Xp, sol.accounting);
        if (iter == 1 && detail::keep_first_filtered) sol.first_filtered = Xp.download();
        int dim = Xp.cols();
        for (int j = 1; j <= config.s; ++j) {
            try {
                rr_device(ctx, filt.device_matrix(), Xp, interval, rr);
            } catch (const CholeskyError&) {
                // one-shot recovery by orthonormalising the expanded subspace
                // (drivers.cpp:212-219)
                ++sol.recovery_events;
                orth_device(ctx, Xp, config, U);
                std::swap(Xp, U);
                rr_device(ctx, filt.device_matrix(), Xp, interval, rr);
            }
            if (j == 1) m_expected = static_cast<int>(std::count(rr.inside.begin(), rr.inside.end(), true));
            select_device(ctx, rr, policy, sel);
            if (j < config.s) {
                fl_err err{};
                check(fl_residual_block(ctx, filt.device_matrix().get(), sel.vectors.get(),
                                        sel.values.data(), R.get(), &err),
                      err);
                check(fl_block_append(Xp.get(), R.get(), &err), err);
                dim = Xp.cols();
            }
        }
        const std::vector<int> inside = trimmed_inside();
        const double r = max_residual(sel, inside);
        record(sol, iter, dim, r, m_expected);
        if (r <= config.tol) {
            sol.converged = true;
            fill_solution(ctx, sol, sel, inside);
            return sol;
        }
        fl_err err{};  // copy, not swap: X keeps its storage (graph replay)
        check(fl_block_copy(X.get(), sel.vectors.get(), &err), err);
    }
    fill_solution(ctx, sol, sel, trimmed_inside());
    return sol;
}

}  // namespace feastlab
