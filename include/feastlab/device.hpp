// RAII wrappers over the C ABI (include/feastlab_b200.h) used by the drop-in
// C++ layer. fl_status codes are rethrown as the reference exception types.
#pragma once

#include <string>

#include "feastlab/matrix.hpp"
#include "feastlab_b200.h"

namespace feastlab {

/// Throws the exception the reference would (std::invalid_argument,
/// std::runtime_error, CholeskyError) for a non-OK status.
void throw_status(int status, const fl_err& err);
inline void check(int status, const fl_err& err) {
    if (status != FL_OK) throw_status(status, err);
}

/// The context used by the calling thread: set explicitly (multi-GPU ranks,
/// concurrent solves) or created lazily on device $FEASTLAB_DEVICE (default 0).
fl_ctx* current_context();
/// Install `ctx` (not owned) for the calling thread; nullptr restores the default.
void set_current_context(fl_ctx* ctx);

class DeviceMatrix {
public:
    DeviceMatrix(fl_ctx* ctx, const MatrixXd& A);
    ~DeviceMatrix();
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    fl_matrix* get() const { return m_; }
    int dim() const { return n_; }

private:
    fl_matrix* m_ = nullptr;
    int n_ = 0;
};

class DeviceBlock {
public:
    DeviceBlock(fl_ctx* ctx, int n, int cap_cols = 1);
    ~DeviceBlock();
    DeviceBlock(const DeviceBlock&) = delete;
    DeviceBlock& operator=(const DeviceBlock&) = delete;
    DeviceBlock(DeviceBlock&& o) noexcept : b_(o.b_), ctx_(o.ctx_) { o.b_ = nullptr; }
    DeviceBlock& operator=(DeviceBlock&& o) noexcept;
    fl_block* get() const { return b_; }
    fl_ctx* ctx() const { return ctx_; }
    int rows() const;
    int cols() const;
    void set(const MatrixXd& X);
    MatrixXd download() const;

private:
    fl_block* b_ = nullptr;
    fl_ctx* ctx_ = nullptr;
};

}  // namespace feastlab
