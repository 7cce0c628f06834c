// Drop-in for proj/include/feastlab/matmodel.hpp: SymmetricMatrix, the
// hot-path input container. (The synthetic-spectrum generator of the
// reference is fixture code outside the filter path: SURVEY.md §8(f)(1).)
#pragma once

#include <memory>

#include "feastlab/contour.hpp"
#include "feastlab/matrix.hpp"
#include "feastlab_b200.h"

namespace feastlab {

class DeviceMatrix;

/// Dense real-symmetric operator, symmetrised exactly as (M + M^T)/2 at
/// construction (matmodel.cpp:10-19); immutable afterwards.
class SymmetricMatrix {
public:
    explicit SymmetricMatrix(MatrixXd entries, double sym_tol = 1e-12);
    /// Same, reading a column-major n x n matrix (leading dimension lda) in
    /// place: no intermediate copy of the caller's buffer.
    SymmetricMatrix(const double* entries, int n, long lda, double sym_tol = 1e-12);
    int dim() const { return mat_.rows(); }
    const MatrixXd& mat() const { return mat_; }
    double operator()(int i, int j) const { return mat_(i, j); }
    /// The matrix resident in HBM on `ctx`: uploaded on first use and shared
    /// by every later NodeFactorization / FilterApplier / rayleigh_ritz /
    /// compute_residual_block call on that context (the matrix is immutable,
    /// so one upload per context suffices).
    const DeviceMatrix& device(fl_ctx* ctx) const;

private:
    void init(const double* entries, int n, long lda, double sym_tol);
    MatrixXd mat_;
    struct DeviceCache;
    std::shared_ptr<DeviceCache> dev_;
};

}  // namespace feastlab
