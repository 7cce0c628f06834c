// RAII wrappers and status -> exception mapping for the drop-in C++ layer.
#include "feastlab/device.hpp"

#include <cstdlib>
#include <memory>
#include <stdexcept>

#include "feastlab/ritz.hpp"

namespace feastlab {

void throw_status(int status, const fl_err& err) {
    switch (status) {
        case FL_OK:
            return;
        case FL_INVALID_ARGUMENT:
            throw std::invalid_argument(err.msg);
        case FL_CHOLESKY:
            throw CholeskyError(err.pivot, err.index);
        default:
            throw std::runtime_error(err.msg);
    }
}

namespace {
struct CtxOwner {
    fl_ctx* ctx = nullptr;
    ~CtxOwner() {
        if (ctx) fl_ctx_destroy(ctx);
    }
};
thread_local CtxOwner tl_default;
thread_local fl_ctx* tl_current = nullptr;
}  // namespace

fl_ctx* current_context() {
    if (tl_current) return tl_current;
    if (!tl_default.ctx) {
        int dev = 0;
        if (const char* e = std::getenv("FEASTLAB_DEVICE")) dev = std::atoi(e);
        fl_err err{};
        check(fl_ctx_create(dev, &tl_default.ctx, &err), err);
    }
    return tl_default.ctx;
}

void set_current_context(fl_ctx* ctx) { tl_current = ctx; }

DeviceMatrix::DeviceMatrix(fl_ctx* ctx, const MatrixXd& A) : n_(A.rows()) {
    fl_err err{};
    check(fl_matrix_create(ctx, A.data(), A.rows(), A.rows(), FL_HOST, &m_, &err), err);
}

DeviceMatrix::~DeviceMatrix() { fl_matrix_destroy(m_); }

DeviceBlock::DeviceBlock(fl_ctx* ctx, int n, int cap_cols) : ctx_(ctx) {
    fl_err err{};
    check(fl_block_create(ctx, n, cap_cols, &b_, &err), err);
}

DeviceBlock::~DeviceBlock() { fl_block_destroy(b_); }

DeviceBlock& DeviceBlock::operator=(DeviceBlock&& o) noexcept {
    if (this != &o) {
        fl_block_destroy(b_);
        b_ = o.b_;
        ctx_ = o.ctx_;
        o.b_ = nullptr;
    }
    return *this;
}

int DeviceBlock::rows() const { return fl_block_rows(b_); }
int DeviceBlock::cols() const { return fl_block_cols(b_); }

void DeviceBlock::set(const MatrixXd& X) {
    fl_err err{};
    check(fl_block_set(b_, X.data(), X.rows() > 0 ? X.rows() : 1, X.cols(), FL_HOST, &err), err);
}

MatrixXd DeviceBlock::download() const {
    MatrixXd X(rows(), cols());
    fl_err err{};
    check(fl_block_get(b_, X.data(), X.rows(), FL_HOST, &err), err);
    return X;
}

}  // namespace feastlab
