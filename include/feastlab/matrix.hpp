// Eigen-free dense containers for the drop-in feastlab API.
//
// The reference API is typed on Eigen::MatrixXd / MatrixXcd / VectorXd
// (proj/include/feastlab/*.hpp). Eigen is not part of this build, so these
// minimal column-major (ld = rows, Eigen's default storage) stand-ins keep the
// member names callers use: rows(), cols(), size(), data(), operator()(i, j),
// operator[](i), col(j), and Zero / Identity factories.
#pragma once

#include <algorithm>
#include <complex>
#include <cstddef>
#include <memory>
#include <new>
#include <utility>
#include <stdexcept>
#include <vector>

namespace feastlab {

// Allocator whose value-less construct() default-initialises: a Matrix made
// with `uninitialized` skips the serial zero fill (2 GB at n = 16384), so the
// caller's parallel loop is the first touch of every page.
template <class T>
struct DefaultInitAllocator : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAllocator<U>;
    };
    DefaultInitAllocator() = default;
    template <class U>
    DefaultInitAllocator(const DefaultInitAllocator<U>&) {}
    template <class U>
    void construct(U* p) {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};

struct Uninitialized {};
constexpr Uninitialized uninitialized{};

template <class T>
class Matrix {
public:
    Matrix() = default;
    Matrix(int rows, int cols, Uninitialized) : r_(rows), c_(cols) {
        if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
        v_.resize(static_cast<size_t>(rows) * cols);
    }
    Matrix(int rows, int cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows) * cols, T(0)) {
        if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
    }
    static Matrix Zero(int rows, int cols) { return Matrix(rows, cols); }
    static Matrix Identity(int rows, int cols) {
        Matrix m(rows, cols);
        for (int i = 0; i < std::min(rows, cols); ++i) m(i, i) = T(1);
        return m;
    }
    int rows() const { return r_; }
    int cols() const { return c_; }
    size_t size() const { return v_.size(); }
    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }
    T& operator()(int i, int j) { return v_[static_cast<size_t>(j) * r_ + i]; }
    const T& operator()(int i, int j) const { return v_[static_cast<size_t>(j) * r_ + i]; }
    T* col(int j) { return v_.data() + static_cast<size_t>(j) * r_; }
    const T* col(int j) const { return v_.data() + static_cast<size_t>(j) * r_; }
    void resize(int rows, int cols) {
        r_ = rows;
        c_ = cols;
        v_.assign(static_cast<size_t>(rows) * cols, T(0));
    }
    bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

private:
    int r_ = 0, c_ = 0;
    std::vector<T, DefaultInitAllocator<T>> v_;
};

template <class T>
class Vector {
public:
    Vector() = default;
    explicit Vector(int n) : v_(static_cast<size_t>(n), T(0)) {}
    static Vector Zero(int n) { return Vector(n); }
    int size() const { return static_cast<int>(v_.size()); }
    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }
    T& operator[](int i) { return v_[static_cast<size_t>(i)]; }
    const T& operator[](int i) const { return v_[static_cast<size_t>(i)]; }
    T& operator()(int i) { return v_[static_cast<size_t>(i)]; }
    const T& operator()(int i) const { return v_[static_cast<size_t>(i)]; }
    void resize(int n) { v_.assign(static_cast<size_t>(n), T(0)); }
    T maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
    bool operator==(const Vector& o) const { return v_ == o.v_; }
    bool operator!=(const Vector& o) const { return !(*this == o); }

private:
    std::vector<T> v_;
};

using MatrixXd = Matrix<double>;
using MatrixXcd = Matrix<std::complex<double>>;
using VectorXd = Vector<double>;

}  // namespace feastlab
