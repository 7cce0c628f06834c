// SymmetricMatrix (proj/src/matmodel.cpp:10-19): square check, relative
// asymmetry check, exact symmetrisation (M + M^T)/2.
#include "feastlab/matmodel.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

namespace feastlab {

SymmetricMatrix::SymmetricMatrix(MatrixXd entries, double sym_tol) {
    const int n = entries.rows();
    if (n < 1 || n != entries.cols())
        throw std::invalid_argument("SymmetricMatrix: matrix must be square, n >= 1");
    double scale = 1.0, asym = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            scale = std::max(scale, std::abs(entries(i, j)));
            asym = std::max(asym, std::abs(entries(i, j) - entries(j, i)));
        }
    if (asym > sym_tol * scale)
        throw std::invalid_argument("SymmetricMatrix: input not symmetric (max |A - A^T| = " +
                                    std::to_string(asym) + ")");
    mat_ = MatrixXd(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) mat_(i, j) = 0.5 * (entries(i, j) + entries(j, i));
}

}  // namespace feastlab
