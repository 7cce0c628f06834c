// SymmetricMatrix (proj/src/matmodel.cpp:10-19): square check, relative
// asymmetry check, exact symmetrisation (M + M^T)/2.
#include "feastlab/matmodel.hpp"

#include "feastlab/device.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

namespace feastlab {

SymmetricMatrix::SymmetricMatrix(MatrixXd entries, double sym_tol) {
    const int n = entries.rows();
    if (n < 1 || n != entries.cols())
        throw std::invalid_argument("SymmetricMatrix: matrix must be square, n >= 1");
    init(entries.data(), n, n, sym_tol);
}

SymmetricMatrix::SymmetricMatrix(const double* entries, int n, long lda, double sym_tol) {
    if (n < 1 || lda < n) throw std::invalid_argument("SymmetricMatrix: matrix must be square, n >= 1");
    init(entries, n, lda, sym_tol);
}

void SymmetricMatrix::init(const double* e, int n, long lde, double sym_tol) {
    // 64 x 64 tile pairs (I, J <= I): both tiles are read while cache
    // resident instead of striding through the transpose, and one parallel
    // pass both checks and writes (the destination is not pre-zeroed, so its
    // pages are first touched here, by all threads); the same max and
    // (a + b) / 2 arithmetic as the reference
    constexpr int T = 64;
    const int nt = (n + T - 1) / T;
    double scale = 1.0, asym = 0.0;
    MatrixXd out(n, n, uninitialized);
    double* m = out.data();
#pragma omp parallel for schedule(dynamic, 1) reduction(max : scale, asym)
    for (int J = 0; J < nt; ++J)
        for (int I = J; I < nt; ++I)
            for (int j = J * T; j < std::min(n, J * T + T); ++j)
                for (int i = I * T; i < std::min(n, I * T + T); ++i) {
                    const double a = e[(size_t)j * lde + i], b = e[(size_t)i * lde + j];
                    scale = std::max(scale, std::max(std::abs(a), std::abs(b)));
                    asym = std::max(asym, std::abs(a - b));
                    const double v = 0.5 * (a + b);
                    m[(size_t)j * n + i] = v;
                    m[(size_t)i * n + j] = v;
                }
    if (asym > sym_tol * scale)
        throw std::invalid_argument("SymmetricMatrix: input not symmetric (max |A - A^T| = " +
                                    std::to_string(asym) + ")");
    mat_ = std::move(out);
    dev_ = std::make_shared<DeviceCache>();
}

// One device copy per context, uploaded on first use (contexts are
// per-thread / per-GPU, so concurrent solves each get their own).
struct SymmetricMatrix::DeviceCache {
    std::mutex mu;
    std::map<fl_ctx*, std::unique_ptr<DeviceMatrix>> copies;
};

const DeviceMatrix& SymmetricMatrix::device(fl_ctx* ctx) const {
    // dev_ is created at construction time (see init) so the const accessor
    // never races on the pointer itself
    std::lock_guard<std::mutex> lk(dev_->mu);
    auto& slot = dev_->copies[ctx];
    if (!slot) slot = std::make_unique<DeviceMatrix>(ctx, mat_);
    return *slot;
}

}  // namespace feastlab
