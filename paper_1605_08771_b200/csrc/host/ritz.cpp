// Drop-in Rayleigh-Ritz API (proj/src/ritz.cpp:11-170): GEMMs, Cholesky,
// eigensolve, normalisation and residuals on the device; pair selection is a
// host sort of <= s*m0 scalars.
#include "feastlab/ritz.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "feastlab/device.hpp"

namespace feastlab {

CholeskyError::CholeskyError(double pivot_, int index_)
    : std::runtime_error("rayleigh_ritz: B' not numerically SPD, pivot " + std::to_string(pivot_) +
                         " at index " + std::to_string(index_)),
      pivot(pivot_),
      index(index_) {}

std::pair<MatrixXd, int> orthonormalize(const MatrixXd& X, double drop_tol, Orthogonalizer method) {
    if (X.cols() < 1 || X.rows() < 1) throw std::invalid_argument("orthonormalize: empty block");
    fl_ctx* ctx = current_context();
    DeviceBlock dX(ctx, X.rows(), X.cols()), dU(ctx, X.rows(), X.cols());
    dX.set(X);
    int rank = 0;
    fl_err err{};
    check(fl_orthonormalize(ctx, dX.get(), drop_tol, method == Orthogonalizer::qr ? 1 : 0, dU.get(),
                            &rank, &err),
          err);
    return {dU.download(), rank};
}

RitzSet rayleigh_ritz(const SymmetricMatrix& A, const MatrixXd& X, const SearchInterval& interval) {
    if (X.rows() != A.dim())
        throw std::invalid_argument("rayleigh_ritz: block/matrix dimension mismatch");
    const int p = X.cols();
    if (p < 1) throw std::invalid_argument("rayleigh_ritz: empty block");
    fl_ctx* ctx = current_context();
    const DeviceMatrix& dA = A.device(ctx);
    DeviceBlock dX(ctx, X.rows(), p), dV(ctx, X.rows(), p);
    dX.set(X);
    RitzSet out;
    out.values.resize(p);
    out.residual_norms.resize(p);
    std::vector<unsigned char> inside(p);
    fl_err err{};
    check(fl_rayleigh_ritz(ctx, dA.get(), dX.get(), interval.lo, interval.hi, out.values.data(),
                           dV.get(), out.residual_norms.data(), inside.data(), &err),
          err);
    out.vectors = dV.download();
    out.inside_flags.assign(inside.begin(), inside.end());
    return out;
}

MatrixXd compute_residual_block(const SymmetricMatrix& A, const RitzSet& ritz) {
    fl_ctx* ctx = current_context();
    const DeviceMatrix& dA = A.device(ctx);
    DeviceBlock dV(ctx, ritz.vectors.rows(), std::max(1, ritz.vectors.cols()));
    DeviceBlock dR(ctx, ritz.vectors.rows(), std::max(1, ritz.vectors.cols()));
    dV.set(ritz.vectors);
    fl_err err{};
    check(fl_residual_block(ctx, dA.get(), dV.get(), ritz.values.data(), dR.get(), &err), err);
    return dR.download();
}

std::vector<int> select_indices(const std::vector<double>& values,
                                const std::vector<double>& residual_norms,
                                const std::vector<bool>& inside_flags,
                                const SelectionPolicy& policy) {
    const int p = static_cast<int>(values.size());
    if (p == 0) throw std::invalid_argument("select_pairs: empty RitzSet");
    const double c = policy.interval.center();
    // (residual asc, |lambda - c| asc, index asc): ritz.cpp:128-134
    auto order = [&](int a, int b) {
        if (residual_norms[a] != residual_norms[b]) return residual_norms[a] < residual_norms[b];
        const double da = std::abs(values[a] - c), db = std::abs(values[b] - c);
        if (da != db) return da < db;
        return a < b;
    };
    std::vector<int> in, out;
    for (int k = 0; k < p; ++k) (inside_flags[k] ? in : out).push_back(k);
    std::sort(in.begin(), in.end(), order);
    std::sort(out.begin(), out.end(), order);
    std::vector<int> chosen;
    const size_t m0 = static_cast<size_t>(std::max(policy.target_count, 0));
    for (const auto* group : {&in, &out})
        for (int k : *group) {
            if (chosen.size() >= m0) break;
            chosen.push_back(k);
        }
    return chosen;
}

RitzSet select_pairs(const RitzSet& ritz, const SelectionPolicy& policy) {
    std::vector<double> vals(ritz.values.data(), ritz.values.data() + ritz.size());
    std::vector<double> res(ritz.residual_norms.data(), ritz.residual_norms.data() + ritz.size());
    const std::vector<int> idx = select_indices(vals, res, ritz.inside_flags, policy);
    RitzSet out;
    const int k = static_cast<int>(idx.size());
    out.values.resize(k);
    out.residual_norms.resize(k);
    out.vectors.resize(ritz.vectors.rows(), k);
    out.inside_flags.resize(k);
    for (int j = 0; j < k; ++j) {
        out.values[j] = ritz.values[idx[j]];
        out.residual_norms[j] = ritz.residual_norms[idx[j]];
        out.inside_flags[j] = ritz.inside_flags[idx[j]];
        std::copy(ritz.vectors.col(idx[j]), ritz.vectors.col(idx[j]) + ritz.vectors.rows(),
                  out.vectors.col(j));
    }
    return out;
}

int count_inside(const RitzSet& ritz) {
    return static_cast<int>(std::count(ritz.inside_flags.begin(), ritz.inside_flags.end(), true));
}

}  // namespace feastlab
