// Drop-in filter operator (proj/src/filterop.cpp:9-84) over the C ABI: the
// shift, LU, solves and ascending-k accumulation all run on the B200.
#include "feastlab/filterop.hpp"

#include <stdexcept>
#include <string>
#include <vector>

namespace feastlab {

namespace {

void check_block(int n, const MatrixXd& X) {  // filterop.cpp:40-46
    if (X.rows() != n)
        throw std::invalid_argument("apply_filter: block dimension " + std::to_string(X.rows()) +
                                    " != matrix dimension " + std::to_string(n));
    if (X.cols() < 1) throw std::invalid_argument("apply_filter: block must have p >= 1");
}

void split_rule(const ContourRule& rule, std::vector<double>& zr, std::vector<double>& zi,
                std::vector<double>& wr, std::vector<double>& wi) {
    for (int k = 0; k < rule.num_points(); ++k) {
        zr.push_back(rule.nodes[k].real());
        zi.push_back(rule.nodes[k].imag());
        wr.push_back(rule.weights[k].real());
        wi.push_back(rule.weights[k].imag());
    }
}

}  // namespace

NodeFactorization::NodeFactorization(const SymmetricMatrix& A, std::complex<double> z,
                                     int node_index)
    : z_(z), node_index_(node_index) {
    // factor once up front into an owned device factor; a singular shift
    // throws here with the reference's message (filterop.cpp:13-23)
    fl_ctx* ctx = current_context();
    fl_node* nd = nullptr;
    fl_err err{};
    const int st = fl_node_create(ctx, A.device(ctx).get(), z.real(), z.imag(), node_index, &nd, &err);
    if (st == FL_SINGULAR_NODE)
        throw std::runtime_error("factorize_node: singular factorization at node " +
                                 std::to_string(node_index_) + " (z = " + std::to_string(z_.real()) +
                                 "+" + std::to_string(z_.imag()) + "i)");
    check(st, err);
    node_.reset(nd, [](fl_node* p) { fl_node_destroy(p); });
}

MatrixXcd NodeFactorization::solve(const MatrixXcd& X) const {
    MatrixXcd W(X.rows(), X.cols());
    fl_err err{};
    check(fl_node_factor_solve(node_.get(), reinterpret_cast<const double*>(X.data()), X.cols(),
                               reinterpret_cast<double*>(W.data()), &err),
          err);
    return W;
}

MatrixXcd NodeFactorization::solve(const MatrixXd& X) const {
    MatrixXcd B(X.rows(), X.cols());
    for (int j = 0; j < X.cols(); ++j)
        for (int i = 0; i < X.rows(); ++i) B(i, j) = std::complex<double>(X(i, j), 0.0);
    return solve(B);
}

NodeFactorization factorize_node(const SymmetricMatrix& A, std::complex<double> z) {
    return NodeFactorization(A, z);
}

MatrixXd apply_filter(const SymmetricMatrix& A, const ContourRule& rule, const MatrixXd& X,
                      SolveAccounting& accounting) {
    FilterApplier applier(A, rule);
    return applier.apply(X, accounting);
}

FilterApplier::FilterApplier(const SymmetricMatrix& A, const ContourRule& rule,
                             bool cache_factorizations)
    : A_(A), rule_(rule), cache_(cache_factorizations) {
    fl_ctx* ctx = current_context();
    dA_ = &A.device(ctx);
    std::vector<double> zr, zi, wr, wi;
    split_rule(rule, zr, zi, wr, wi);
    fl_err err{};
    check(fl_filter_create(ctx, dA_->get(), rule.num_points(), zr.data(), zi.data(), wr.data(),
                           wi.data(), cache_ ? 1 : 0, &filt_, &err),
          err);
}

FilterApplier::~FilterApplier() { fl_filter_destroy(filt_); }

MatrixXd FilterApplier::apply(const MatrixXd& X, SolveAccounting& accounting) {
    check_block(A_.dim(), X);
    MatrixXd Y(X.rows(), X.cols());
    fl_err err{};
    check(fl_filter_apply_raw(filt_, X.data(), X.rows(), X.cols(), Y.data(), Y.rows(), FL_HOST,
                              &accounting.rhs_solved, &accounting.factorizations, &err),
          err);
    return Y;
}

void FilterApplier::apply(const DeviceBlock& X, DeviceBlock& Y, SolveAccounting& accounting) {
    fl_err err{};
    check(fl_filter_apply(filt_, X.get(), Y.get(), &accounting.rhs_solved,
                          &accounting.factorizations, &err),
          err);
}

}  // namespace feastlab
