// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU ORACLE. Not product code.
//
// A line-by-line C++ restatement of the reference feastlab hot path
// (/root/reference/proj/src/{contour,filterop,ritz,drivers,matmodel}.cpp) with
// the reference's third-party dense kernels (Eigen3 >= 3.3, unpinned; absent
// from the container) replaced by their published algorithms on scipy's
// bundled OpenBLAS 0.3.30 LAPACK:
//   Eigen::PartialPivLU     -> blocked right-looking LU, partial pivoting on
//                              |a_ik| (Eigen scalar_score_coeff_op = abs),
//                              first index on ties; zgemm/ztrsm for the
//                              blocked updates; solve = P, unit-L, U (ztrsm)
//   SelfAdjointEigenSolver  -> dsyevd (ascending eigenvalues)
//   ColPivHouseholderQR     -> dgeqp3 (+ dorgqr), rank = #|R_ii| > thr*max|R_jj|
//   HouseholderQR           -> dgeqrf + dorgqr
//   triangularView::solve   -> dtrsm
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library. The product path (paper_1605_08771_b200) never does.
//
// Parity pin: the reference cannot be compiled here (Eigen absent), and it
// ships no golden vectors. This oracle is pinned against every analytic
// known-answer test and oracle-tolerance test of the reference suite
// (tests/test_ref_*.py re-express proj/tests/*.cpp and acceptance.cpp).
// Bit-level parity with Eigen is unpinned.
// =============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "lapack.hpp"

namespace orc {

// ----------------------------------------------------------------- errors
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CholeskyError : std::runtime_error {
    CholeskyError(double p, int i)
        : std::runtime_error("rayleigh_ritz: B' not numerically SPD, pivot " + std::to_string(p) +
                             " at index " + std::to_string(i)),
          pivot(p), index(i) {}
    double pivot;
    int index;
};
struct SingularNode : std::runtime_error {
    SingularNode(const std::string& m, int k, std::complex<double> z)
        : std::runtime_error(m), node(k), z(z) {}
    int node;
    std::complex<double> z;
};

// ----------------------------------------------------------------- matrix
template <class T>
struct Mat {
    int r = 0, c = 0;
    std::vector<T> v;
    Mat() = default;
    Mat(int r_, int c_) : r(r_), c(c_), v(static_cast<size_t>(r_) * c_, T(0)) {}
    T& operator()(int i, int j) { return v[static_cast<size_t>(j) * r + i]; }
    const T& operator()(int i, int j) const { return v[static_cast<size_t>(j) * r + i]; }
    T* col(int j) { return v.data() + static_cast<size_t>(j) * r; }
    const T* col(int j) const { return v.data() + static_cast<size_t>(j) * r; }
    T* data() { return v.data(); }
    const T* data() const { return v.data(); }
};
using MatD = Mat<double>;
using MatZ = Mat<std::complex<double>>;

static MatD gemm(char ta, char tb, const MatD& A, const MatD& B) {
    int m = (ta == 'N') ? A.r : A.c;
    int k = (ta == 'N') ? A.c : A.r;
    int n = (tb == 'N') ? B.c : B.r;
    MatD C(m, n);
    if (m == 0 || n == 0) return C;
    double one = 1.0, zero = 0.0;
    int lda = std::max(1, A.r), ldb = std::max(1, B.r), ldc = std::max(1, m);
    scipy_dgemm_(&ta, &tb, &m, &n, &k, &one, A.data(), &lda, B.data(), &ldb, &zero, C.data(),
                 &ldc, 1, 1);
    return C;
}

static void symmetrize(MatD& M) {  // M = 0.5*(M + M^T) as Eigen evaluates it
    MatD T = M;
    for (int j = 0; j < M.c; ++j)
        for (int i = 0; i < M.r; ++i) M(i, j) = 0.5 * (T(i, j) + T(j, i));
}

static double col_norm(const double* x, int n) {
    // Eigen's norm(): sqrt of squaredNorm (plain sum of squares)
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return std::sqrt(s);
}

// Ascending symmetric eigendecomposition (SelfAdjointEigenSolver stand-in).
static void sym_eig(const MatD& M, std::vector<double>& w, MatD& V) {
    int n = M.r;
    V = M;
    w.assign(n, 0.0);
    if (n == 0) return;
    char jobz = 'V', uplo = 'L';
    int lda = n, info = 0, lwork = -1, liwork = -1, iwq = 0;
    double wq = 0;
    scipy_dsyevd_(&jobz, &uplo, &n, V.data(), &lda, w.data(), &wq, &lwork, &iwq, &liwork, &info,
                  1, 1);
    lwork = static_cast<int>(wq);
    liwork = iwq;
    std::vector<double> work(std::max(1, lwork));
    std::vector<int> iwork(std::max(1, liwork));
    scipy_dsyevd_(&jobz, &uplo, &n, V.data(), &lda, w.data(), work.data(), &lwork, iwork.data(),
                  &liwork, &info, 1, 1);
    if (info != 0) throw std::runtime_error("dsyevd failed, info=" + std::to_string(info));
}

// Column-pivoted Householder QR (ColPivHouseholderQR stand-in). Returns rank
// under Eigen's rule and optionally the thin Q (first `rank` columns).
static int colpiv_qr_rank(const MatD& X, double threshold, MatD* Qout) {
    MatD F = X;
    int m = F.r, n = F.c, lda = std::max(1, m), info = 0, lwork = -1;
    std::vector<int> jpvt(n, 0);
    std::vector<double> tau(std::min(m, n));
    double wq;
    scipy_dgeqp3_(&m, &n, F.data(), &lda, jpvt.data(), tau.data(), &wq, &lwork, &info);
    lwork = static_cast<int>(wq);
    std::vector<double> work(std::max(1, lwork));
    scipy_dgeqp3_(&m, &n, F.data(), &lda, jpvt.data(), tau.data(), work.data(), &lwork, &info);
    int kmax = std::min(m, n);
    double maxpivot = 0.0;
    for (int i = 0; i < kmax; ++i) maxpivot = std::max(maxpivot, std::abs(F(i, i)));
    int rank = 0;
    for (int i = 0; i < kmax; ++i)
        if (std::abs(F(i, i)) > maxpivot * threshold) ++rank;
    if (Qout && rank > 0) {
        MatD Q(m, rank);
        for (int j = 0; j < rank; ++j) std::memcpy(Q.col(j), F.col(j), sizeof(double) * m);
        int k = rank;
        lwork = -1;
        scipy_dorgqr_(&m, &rank, &k, Q.data(), &lda, tau.data(), &wq, &lwork, &info);
        lwork = static_cast<int>(wq);
        work.assign(std::max(1, lwork), 0.0);
        scipy_dorgqr_(&m, &rank, &k, Q.data(), &lda, tau.data(), work.data(), &lwork, &info);
        *Qout = std::move(Q);
    }
    return rank;
}

// ================================================================= contour
// proj/src/contour.cpp:11-15
struct Interval {
    double lo, hi;
    Interval(double l, double h) : lo(l), hi(h) {
        if (!(lo < hi))
            throw InvalidArgument("SearchInterval: require lo < hi, got [" + std::to_string(lo) +
                                  ", " + std::to_string(hi) + "]");
    }
    double center() const { return 0.5 * (lo + hi); }
    double radius() const { return 0.5 * (hi - lo); }
    bool contains(double x) const { return x > lo && x < hi; }
};

// proj/src/contour.cpp:17-51 — Newton on the Legendre recurrence.
static void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
    if (n < 1 || n > 64)
        throw InvalidArgument("gauss_legendre: n must be in [1, 64], got " + std::to_string(n));
    nodes.assign(n, 0.0);
    weights.assign(n, 0.0);
    const double pi = std::acos(-1.0);
    const int half = (n + 1) / 2;
    for (int i = 1; i <= half; ++i) {
        double z = std::cos(pi * (i - 0.25) / (n + 0.5));
        double pp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p1 = 1.0, p2 = 0.0;
            for (int j = 1; j <= n; ++j) {
                double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            double z1 = z;
            z = z1 - p1 / pp;
            if (std::abs(z - z1) <= 1e-15) break;
        }
        nodes[i - 1] = -z;
        nodes[n - i] = z;
        double w = 2.0 / ((1.0 - z * z) * pp * pp);
        weights[i - 1] = w;
        weights[n - i] = w;
    }
    if (n % 2 == 1) nodes[n / 2] = 0.0;
}

struct Rule {
    std::vector<std::complex<double>> z, w;
    int nc() const { return static_cast<int>(z.size()); }
};

// proj/src/contour.cpp:53-69
static Rule build_rule(const Interval& I, int nc) {
    std::vector<double> g, gw;
    gauss_legendre(nc, g, gw);
    const double c = I.center(), r = I.radius(), pi = std::acos(-1.0);
    Rule rule;
    rule.z.resize(nc);
    rule.w.resize(nc);
    for (int k = 0; k < nc; ++k) {
        double theta = 0.5 * pi * (g[k] + 1.0);
        std::complex<double> e{std::cos(theta), std::sin(theta)};
        rule.z[k] = c + r * e;
        rule.w[k] = 0.5 * gw[k] * r * e;
    }
    return rule;
}

// proj/src/contour.cpp:83-88
static double filter_value(const Rule& rule, double lambda) {
    double sum = 0.0;
    for (int k = 0; k < rule.nc(); ++k) sum += std::real(rule.w[k] / (rule.z[k] - lambda));
    return sum;
}

// proj/src/contour.cpp:114-124
static double predicted_rate(const Rule& rule, const std::vector<double>& spectrum, int m0) {
    if (m0 < 1) throw InvalidArgument("predicted_rate: m0 must be >= 1");
    if (m0 >= static_cast<int>(spectrum.size()))
        throw InvalidArgument("predicted_rate: m0 must be < spectrum size");
    std::vector<double> rho(spectrum.size());
    for (size_t i = 0; i < spectrum.size(); ++i) rho[i] = filter_value(rule, spectrum[i]);
    std::sort(rho.begin(), rho.end(), std::greater<double>());
    return rho[m0] / rho[m0 - 1];
}

// ================================================================= matmodel
// proj/src/matmodel.cpp:10-19
static MatD symmetric_matrix(const MatD& E, double sym_tol) {
    if (E.r < 1 || E.r != E.c) throw InvalidArgument("SymmetricMatrix: matrix must be square, n >= 1");
    double scale = 1.0, asym = 0.0;
    for (double x : E.v) scale = std::max(scale, std::abs(x));
    for (int j = 0; j < E.c; ++j)
        for (int i = 0; i < E.r; ++i) asym = std::max(asym, std::abs(E(i, j) - E(j, i)));
    if (asym > sym_tol * scale)
        throw InvalidArgument("SymmetricMatrix: input not symmetric (max |A - A^T| = " +
                              std::to_string(asym) + ")");
    MatD S(E.r, E.c);
    for (int j = 0; j < E.c; ++j)
        for (int i = 0; i < E.r; ++i) S(i, j) = 0.5 * (E(i, j) + E(j, i));
    return S;
}

// Seeded column-major N(0,1) fill — proj/src/matmodel.cpp:93-97,
// proj/src/drivers.cpp:28-32, proj/tests/oracles.hpp:50-67.
static void gaussian_fill(double* out, size_t count, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (size_t i = 0; i < count; ++i) out[i] = gauss(rng);
}

// Householder Q of a seeded Gaussian n x n block with column-sign
// normalisation — proj/src/matmodel.cpp:93-104.
static MatD seeded_orthogonal(int n, std::uint64_t seed) {
    MatD G(n, n);
    gaussian_fill(G.data(), G.v.size(), seed);
    int lda = n, info = 0, lwork = -1;
    std::vector<double> tau(n);
    double wq;
    scipy_dgeqrf_(&n, &n, G.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = static_cast<int>(wq);
    std::vector<double> work(std::max(1, lwork));
    scipy_dgeqrf_(&n, &n, G.data(), &lda, tau.data(), work.data(), &lwork, &info);
    lwork = -1;
    scipy_dorgqr_(&n, &n, &n, G.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = static_cast<int>(wq);
    work.assign(std::max(1, lwork), 0.0);
    scipy_dorgqr_(&n, &n, &n, G.data(), &lda, tau.data(), work.data(), &lwork, &info);
    for (int j = 0; j < n; ++j) {
        int imax = 0;
        double best = -1.0;
        for (int i = 0; i < n; ++i)
            if (std::abs(G(i, j)) > best) { best = std::abs(G(i, j)); imax = i; }
        if (G(imax, j) < 0.0)
            for (int i = 0; i < n; ++i) G(i, j) = -G(i, j);
    }
    return G;
}

static void append_uniform(std::vector<double>& out, double lo, double hi, int count) {
    if (count == 1) { out.push_back(0.5 * (lo + hi)); return; }
    for (int i = 0; i < count; ++i) out.push_back(lo + (hi - lo) * i / (count - 1));
}

// proj/src/matmodel.cpp:20-110 (validate_layout + generate_spectrum values)
static std::vector<double> layout_values(int n, Interval in, int in_count, Interval out,
                                         int out_count, int clustered, int num_clusters,
                                         double cluster_width) {
    if (n < 1) throw InvalidArgument("SpectrumLayout: n must be >= 1");
    if (in_count < 1) throw InvalidArgument("SpectrumLayout: inside_count must be >= 1");
    if (out_count < 0) throw InvalidArgument("SpectrumLayout: outside_count must be >= 0");
    if (in_count + out_count != n)
        throw InvalidArgument("SpectrumLayout: inside_count + outside_count must equal n");
    if (out_count > 0 && !(in.hi <= out.lo || out.hi <= in.lo))
        throw InvalidArgument("SpectrumLayout: inside and outside intervals overlap");
    if (clustered) {
        if (num_clusters < 1) throw InvalidArgument("SpectrumLayout: num_clusters must be >= 1");
        if (!(cluster_width > 0.0)) throw InvalidArgument("SpectrumLayout: cluster_width must be > 0");
        if (num_clusters * cluster_width > out.hi - out.lo)
            throw InvalidArgument("SpectrumLayout: clusters do not fit in outside interval");
    }
    std::vector<double> values;
    values.reserve(n);
    append_uniform(values, in.lo, in.hi, in_count);
    if (out_count > 0) {
        if (!clustered) {
            append_uniform(values, out.lo, out.hi, out_count);
        } else {
            const int k = num_clusters;
            const double w = cluster_width;
            const double c_lo = out.lo + 0.5 * w, c_hi = out.hi - 0.5 * w;
            const int base = out_count / k, extra = out_count % k;
            for (int g = 0; g < k; ++g) {
                double center = (k == 1) ? 0.5 * (c_lo + c_hi) : c_lo + (c_hi - c_lo) * g / (k - 1);
                int count = base + (g < extra ? 1 : 0);
                if (count > 0) append_uniform(values, center - 0.5 * w, center + 0.5 * w, count);
            }
        }
    }
    std::sort(values.begin(), values.end());
    return values;
}

// proj/src/matmodel.cpp:112-119 — A = Q diag(values) Q^T, symmetrized.
static MatD assemble(const std::vector<double>& values, const MatD& Q) {
    int n = Q.r;
    MatD QL = Q;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) QL(i, j) *= values[j];
    MatD A = gemm('N', 'T', QL, Q);
    symmetrize(A);
    return symmetric_matrix(A, 1e-12);
}

// ================================================================= filterop
// proj/src/filterop.cpp:9-32 — NodeFactorization: S = zI - A, PartialPivLU.
struct NodeLU {
    MatZ lu;
    std::vector<int> perm;  // row transpositions: row k swapped with perm[k]
    std::complex<double> z;

    NodeLU(const MatD& A, std::complex<double> z_, int node_index) : lu(A.r, A.c), z(z_) {
        const int n = A.r;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) lu(i, j) = std::complex<double>(-A(i, j), 0.0);
        for (int i = 0; i < n; ++i) lu(i, i) += z;
        factor();
        for (int i = 0; i < n; ++i) {
            double d = std::abs(lu(i, i));
            if (!(d > 0.0) || !std::isfinite(d))
                throw SingularNode("factorize_node: singular factorization at node " +
                                       std::to_string(node_index) + " (z = " +
                                       std::to_string(z.real()) + "+" + std::to_string(z.imag()) +
                                       "i)",
                                   node_index, z);
        }
    }

    // Blocked right-looking partial-pivot LU, pivot = argmax |a_ik| (first on
    // ties), the algorithm of Eigen's PartialPivLU (blocked_lu/unblocked_lu).
    void factor() {
        const int n = lu.r;
        perm.assign(n, 0);
        const int nb = 64;
        for (int k0 = 0; k0 < n; k0 += nb) {
            const int kb = std::min(nb, n - k0);
            // unblocked panel on columns [k0, k0+kb), rows [k0, n)
            for (int k = k0; k < k0 + kb; ++k) {
                int piv = k;
                double best = std::abs(lu(k, k));
                for (int i = k + 1; i < n; ++i) {
                    double s = std::abs(lu(i, k));
                    if (s > best) { best = s; piv = i; }
                }
                perm[k] = piv;
                if (best != 0.0) {
                    if (piv != k)
                        for (int j = k0; j < k0 + kb; ++j) std::swap(lu(k, j), lu(piv, j));
                    const std::complex<double> inv = 1.0 / lu(k, k);
                    for (int i = k + 1; i < n; ++i) lu(i, k) *= inv;
                }
                for (int j = k + 1; j < k0 + kb; ++j) {
                    const std::complex<double> u = lu(k, j);
                    if (u == 0.0) continue;
                    for (int i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * u;
                }
            }
            // apply the panel's row swaps to the columns left and right of it
            for (int k = k0; k < k0 + kb; ++k) {
                int piv = perm[k];
                if (piv == k) continue;
                for (int j = 0; j < k0; ++j) std::swap(lu(k, j), lu(piv, j));
                for (int j = k0 + kb; j < n; ++j) std::swap(lu(k, j), lu(piv, j));
            }
            const int nr = n - k0 - kb;
            if (nr <= 0) continue;
            // U12 = L11^{-1} A12
            {
                char side = 'L', uplo = 'L', ta = 'N', diag = 'U';
                int m = kb, ncols = nr, lda = n, ldb = n;
                std::complex<double> one(1.0, 0.0);
                scipy_ztrsm_(&side, &uplo, &ta, &diag, &m, &ncols, &one, &lu(k0, k0), &lda,
                             &lu(k0, k0 + kb), &ldb, 1, 1, 1, 1);
            }
            // A22 -= L21 U12
            {
                char ta = 'N', tb = 'N';
                int m = nr, ncols = nr, k = kb, lda = n;
                std::complex<double> mone(-1.0, 0.0), one(1.0, 0.0);
                scipy_zgemm_(&ta, &tb, &m, &ncols, &k, &mone, &lu(k0 + kb, k0), &lda,
                             &lu(k0, k0 + kb), &lda, &one, &lu(k0 + kb, k0 + kb), &lda, 1, 1);
            }
        }
    }

    // W = (zI - A)^{-1} B  (PartialPivLU::solve: P, unit-lower L, upper U)
    MatZ solve(const MatZ& B) const {
        MatZ W = B;
        const int n = lu.r;
        for (int k = 0; k < n; ++k)
            if (perm[k] != k)
                for (int j = 0; j < W.c; ++j) std::swap(W(k, j), W(perm[k], j));
        char side = 'L', uplo = 'L', ta = 'N', diag = 'U';
        int m = n, ncols = W.c, lda = n, ldb = n;
        std::complex<double> one(1.0, 0.0);
        scipy_ztrsm_(&side, &uplo, &ta, &diag, &m, &ncols, &one, lu.data(), &lda, W.data(), &ldb,
                     1, 1, 1, 1);
        uplo = 'U';
        diag = 'N';
        scipy_ztrsm_(&side, &uplo, &ta, &diag, &m, &ncols, &one, lu.data(), &lda, W.data(), &ldb,
                     1, 1, 1, 1);
        return W;
    }
    MatZ solve(const MatD& X) const {  // proj/src/filterop.cpp:26-28: real -> complex cast
        MatZ B(X.r, X.c);
        for (size_t i = 0; i < X.v.size(); ++i) B.v[i] = std::complex<double>(X.v[i], 0.0);
        return solve(B);
    }
};

struct Accounting {
    long long rhs = 0, facts = 0;
};

// proj/src/filterop.cpp:56-84 — FilterApplier
struct Applier {
    const MatD& A;
    const Rule& rule;
    bool cache;
    std::vector<std::unique_ptr<NodeLU>> cached;
    Applier(const MatD& A_, const Rule& r, bool c) : A(A_), rule(r), cache(c) {
        if (cache) cached.resize(rule.nc());
    }
    MatD apply(const MatD& X, Accounting& acc) {
        if (X.r != A.r)
            throw InvalidArgument("apply_filter: block dimension " + std::to_string(X.r) +
                                  " != matrix dimension " + std::to_string(A.r));
        if (X.c < 1) throw InvalidArgument("apply_filter: block must have p >= 1");
        MatD Y(X.r, X.c);
        for (int k = 0; k < rule.nc(); ++k) {
            const NodeLU* f;
            std::unique_ptr<NodeLU> local;
            if (cache) {
                if (!cached[k]) {
                    cached[k] = std::make_unique<NodeLU>(A, rule.z[k], k);
                    ++acc.facts;
                }
                f = cached[k].get();
            } else {
                local = std::make_unique<NodeLU>(A, rule.z[k], k);
                ++acc.facts;
                f = local.get();
            }
            MatZ W = f->solve(X);
            const std::complex<double> w = rule.w[k];
            for (size_t i = 0; i < Y.v.size(); ++i) Y.v[i] += std::real(w * W.v[i]);
        }
        acc.rhs += static_cast<long long>(rule.nc()) * X.c;
        return Y;
    }
};

// ================================================================= ritz
struct Ritz {
    std::vector<double> values;
    MatD vectors;
    std::vector<double> norms;
    std::vector<char> inside;
    int size() const { return static_cast<int>(values.size()); }
};

// proj/src/ritz.cpp:17-59
static std::pair<MatD, int> orthonormalize(const MatD& X, double drop_tol, int method) {
    if (X.c < 1 || X.r < 1) throw InvalidArgument("orthonormalize: empty block");
    if (method == 1) {
        MatD Q;
        int rank = colpiv_qr_rank(X, drop_tol, &Q);
        if (rank == 0) throw std::runtime_error("orthonormalize: block is numerically zero");
        return {std::move(Q), rank};
    }
    MatD G = gemm('T', 'N', X, X);
    symmetrize(G);
    std::vector<double> ev;
    MatD V;
    sym_eig(G, ev, V);
    const int p = X.c;
    const double sigma_max = std::sqrt(std::max(0.0, ev[p - 1]));
    if (!(sigma_max > 0.0)) throw std::runtime_error("orthonormalize: block is numerically zero");
    const double ev_floor =
        std::max(drop_tol * drop_tol, std::numeric_limits<double>::epsilon() * p) * ev[p - 1];
    std::vector<int> keep;
    for (int i = p - 1; i >= 0; --i)
        if (ev[i] > ev_floor) keep.push_back(i);
    const int rank = static_cast<int>(keep.size());
    if (rank == 0) throw std::runtime_error("orthonormalize: block is numerically zero");
    MatD Vk(p, rank);
    for (int j = 0; j < rank; ++j) std::memcpy(Vk.col(j), V.col(keep[j]), sizeof(double) * p);
    MatD U = gemm('N', 'N', X, Vk);
    for (int j = 0; j < rank; ++j) {
        double sigma = std::sqrt(ev[keep[j]]);
        double* u = U.col(j);
        for (int i = 0; i < U.r; ++i) u[i] /= sigma;
    }
    return {std::move(U), rank};
}

// proj/src/ritz.cpp:64-79 (verbatim semantics)
static MatD cholesky_or_throw(const MatD& B) {
    const int p = B.r;
    MatD L(p, p);
    for (int j = 0; j < p; ++j) {
        double s = B(j, j);
        for (int k = 0; k < j; ++k) s -= L(j, k) * L(j, k);
        if (!(s > 0.0) || !std::isfinite(s)) throw CholeskyError(s, j);
        L(j, j) = std::sqrt(s);
        for (int i = j + 1; i < p; ++i) {
            double t = B(i, j);
            for (int k = 0; k < j; ++k) t -= L(i, k) * L(j, k);
            L(i, j) = t / L(j, j);
        }
    }
    return L;
}

static void trsm(char side, char uplo, char ta, const MatD& L, MatD& B) {
    char diag = 'N';
    int m = B.r, n = B.c, lda = std::max(1, L.r), ldb = std::max(1, B.r);
    double one = 1.0;
    scipy_dtrsm_(&side, &uplo, &ta, &diag, &m, &n, &one, L.data(), &lda, B.data(), &ldb, 1, 1, 1, 1);
}

static MatD residual_block(const MatD& A, const std::vector<double>& vals, const MatD& V) {
    MatD R = gemm('N', 'N', A, V);
    for (int k = 0; k < V.c; ++k)
        for (int i = 0; i < V.r; ++i) R(i, k) -= V(i, k) * vals[k];
    return R;
}

// proj/src/ritz.cpp:83-118
static Ritz rayleigh_ritz(const MatD& A, const MatD& X, const Interval& I) {
    if (X.r != A.r) throw InvalidArgument("rayleigh_ritz: block/matrix dimension mismatch");
    const int p = X.c;
    if (p < 1) throw InvalidArgument("rayleigh_ritz: empty block");
    MatD AX = gemm('N', 'N', A, X);
    MatD Ap = gemm('T', 'N', X, AX);
    MatD Bp = gemm('T', 'N', X, X);
    symmetrize(Ap);
    symmetrize(Bp);
    MatD L = cholesky_or_throw(Bp);
    MatD T = Ap;
    trsm('L', 'L', 'N', L, T);  // T = L^{-1} A'
    MatD C(p, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < p; ++i) C(i, j) = T(j, i);
    trsm('L', 'L', 'N', L, C);  // C = L^{-1} T^T
    symmetrize(C);
    Ritz out;
    MatD V;
    sym_eig(C, out.values, V);
    trsm('L', 'L', 'T', L, V);  // Q = L^{-T} V
    out.vectors = gemm('N', 'N', X, V);
    out.norms.assign(p, 0.0);
    out.inside.assign(p, 0);
    for (int k = 0; k < p; ++k) {
        double* v = out.vectors.col(k);
        double nrm = col_norm(v, X.r);
        for (int i = 0; i < X.r; ++i) v[i] /= nrm;
        out.inside[k] = I.contains(out.values[k]);
    }
    MatD R = residual_block(A, out.values, out.vectors);
    for (int k = 0; k < p; ++k) out.norms[k] = col_norm(R.col(k), R.r);
    return out;
}

// proj/src/ritz.cpp:124-151 — the chosen indices, in selection order
static std::vector<int> select_indices(const Ritz& ritz, int m0, const Interval& I) {
    if (ritz.size() == 0) throw InvalidArgument("select_pairs: empty RitzSet");
    const double c = I.center();
    auto by_residual = [&](int a, int b) {
        if (ritz.norms[a] != ritz.norms[b]) return ritz.norms[a] < ritz.norms[b];
        double da = std::abs(ritz.values[a] - c), db = std::abs(ritz.values[b] - c);
        if (da != db) return da < db;
        return a < b;
    };
    std::vector<int> inside, outside;
    for (int k = 0; k < ritz.size(); ++k) (ritz.inside[k] ? inside : outside).push_back(k);
    std::sort(inside.begin(), inside.end(), by_residual);
    std::sort(outside.begin(), outside.end(), by_residual);
    std::vector<int> chosen;
    for (int k : inside) { if (static_cast<int>(chosen.size()) >= m0) break; chosen.push_back(k); }
    for (int k : outside) { if (static_cast<int>(chosen.size()) >= m0) break; chosen.push_back(k); }
    return chosen;
}

// proj/src/ritz.cpp:153-166 — gather
static Ritz select_pairs(const Ritz& ritz, int m0, const Interval& I) {
    std::vector<int> chosen = select_indices(ritz, m0, I);
    Ritz out;
    const int sz = static_cast<int>(chosen.size());
    out.values.resize(sz);
    out.vectors = MatD(ritz.vectors.r, sz);
    out.norms.resize(sz);
    out.inside.resize(sz);
    for (int j = 0; j < sz; ++j) {
        out.values[j] = ritz.values[chosen[j]];
        std::memcpy(out.vectors.col(j), ritz.vectors.col(chosen[j]), sizeof(double) * ritz.vectors.r);
        out.norms[j] = ritz.norms[chosen[j]];
        out.inside[j] = ritz.inside[chosen[j]];
    }
    return out;
}

static int count_inside(const Ritz& r) {
    return static_cast<int>(std::count(r.inside.begin(), r.inside.end(), 1));
}

// ================================================================= drivers
struct Config {
    int m0 = 1, n_c = 8, s = 1;
    double tol = 1e-12;
    int max_iter = 50;
    std::uint64_t seed = 42;
    int orthogonalizer = 0;
    double drop_tol = 1e-10;
    int cache = 0, generalized_reduced = 0;
};
struct TraceRec {
    int iter, dim;
    long long rhs;
    double r;
    int m_found;
};
struct Solution {
    std::vector<double> values, norms;
    MatD vectors;
    int converged = 0, iterations = 0, recovery = 0;
    Accounting acc;
    std::vector<TraceRec> trace;
    MatD first_filtered;  // Y_1 (parity hook: first filtered subspace)
};

// proj/src/drivers.cpp:23-38
static MatD make_initial_guess(int n, int m0, std::uint64_t seed) {
    if (m0 < 1 || m0 > n) throw InvalidArgument("make_initial_guess: require 1 <= m0 <= n");
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
    std::normal_distribution<double> gauss(0.0, 1.0);
    MatD X(n, m0);
    for (int j = 0; j < m0; ++j)
        for (int i = 0; i < n; ++i) X(i, j) = gauss(rng);
    if (colpiv_qr_rank(X, 1e-10, nullptr) < m0)
        throw std::runtime_error("make_initial_guess: guess block is rank deficient");
    return X;
}

static void validate_config(int n, const Config& c) {
    if (c.m0 < 1 || c.m0 > n) throw InvalidArgument("SolverConfig: require 1 <= m0 <= n");
    if (c.s < 1) throw InvalidArgument("SolverConfig: require s >= 1");
    if (!(c.tol > 0.0)) throw InvalidArgument("SolverConfig: require tol > 0");
    if (c.max_iter < 1) throw InvalidArgument("SolverConfig: require max_iter >= 1");
}

static std::vector<int> inside_by_residual(const Ritz& rr) {
    std::vector<int> idx;
    for (int k = 0; k < rr.size(); ++k)
        if (rr.inside[k]) idx.push_back(k);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) {
        if (rr.norms[a] != rr.norms[b]) return rr.norms[a] < rr.norms[b];
        return a < b;
    });
    return idx;
}

static double max_residual(const Ritz& rr, const std::vector<int>& idx) {
    double r = 0.0;
    for (int k : idx) r = std::max(r, rr.norms[k]);
    return r;
}

static void fill_solution(Solution& sol, const Ritz& rr, std::vector<int> idx) {
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return rr.values[a] < rr.values[b]; });
    const int m = static_cast<int>(idx.size());
    sol.values.resize(m);
    sol.norms.resize(m);
    sol.vectors = MatD(rr.vectors.r, m);
    for (int j = 0; j < m; ++j) {
        sol.values[j] = rr.values[idx[j]];
        std::memcpy(sol.vectors.col(j), rr.vectors.col(idx[j]), sizeof(double) * rr.vectors.r);
        sol.norms[j] = rr.norms[idx[j]];
    }
}

static MatD hconcat(const std::deque<MatD>& blocks) {
    int cols = 0;
    for (const auto& b : blocks) cols += b.c;
    MatD out(blocks.front().r, cols);
    size_t at = 0;
    for (const auto& b : blocks) {
        std::memcpy(out.data() + at, b.data(), sizeof(double) * b.v.size());
        at += b.v.size();
    }
    return out;
}

// proj/src/drivers.cpp:98-139
static Solution feast_solve(const MatD& A, const Interval& I, const Config& cfg) {
    validate_config(A.r, cfg);
    const Rule rule = build_rule(I, cfg.n_c);
    Applier filt(A, rule, cfg.cache);
    Solution sol;
    MatD X = make_initial_guess(A.r, cfg.m0, cfg.seed);
    Ritz rr;
    int last_m_found = 0;
    for (int iter = 1; iter <= cfg.max_iter; ++iter) {
        MatD Y = filt.apply(X, sol.acc);
        if (iter == 1) sol.first_filtered = Y;
        int dim;
        if (cfg.generalized_reduced) {
            rr = rayleigh_ritz(A, Y, I);
            dim = Y.c;
        } else {
            auto [U, rank] = orthonormalize(Y, cfg.drop_tol, cfg.orthogonalizer);
            if (rank < last_m_found)
                throw std::runtime_error(
                    "feast_solve: filtered subspace rank collapsed below the inside "
                    "eigenpair count; m0 may be too small");
            rr = rayleigh_ritz(A, U, I);
            dim = rank;
        }
        std::vector<int> inside = inside_by_residual(rr);
        double r = max_residual(rr, inside);
        sol.trace.push_back({iter, dim, sol.acc.rhs, r, static_cast<int>(inside.size())});
        sol.iterations = iter;
        last_m_found = static_cast<int>(inside.size());
        if (r <= cfg.tol) {
            sol.converged = 1;
            fill_solution(sol, rr, inside);
            return sol;
        }
        X = rr.vectors;
    }
    fill_solution(sol, rr, inside_by_residual(rr));
    return sol;
}

// proj/src/drivers.cpp:141-186
static Solution xfeast_solve(const MatD& A, const Interval& I, const Config& cfg) {
    validate_config(A.r, cfg);
    if (static_cast<long>(cfg.s) * cfg.m0 > A.r)
        std::fprintf(stderr, "xfeast_solve: warning: s*m0 = %ld exceeds matrix dimension %d\n",
                     static_cast<long>(cfg.s) * cfg.m0, A.r);
    const Rule rule = build_rule(I, cfg.n_c);
    Applier filt(A, rule, cfg.cache);
    Solution sol;
    std::deque<MatD> window;
    window.push_back(make_initial_guess(A.r, cfg.m0, cfg.seed));
    for (int k = 2; k < cfg.s; ++k) {
        window.push_back(filt.apply(window.back(), sol.acc));
        if (sol.first_filtered.c == 0) sol.first_filtered = window.back();
    }
    MatD estimate = window.back();
    Ritz sel;
    for (int iter = 1; iter <= cfg.max_iter; ++iter) {
        window.push_back(filt.apply(estimate, sol.acc));
        if (sol.first_filtered.c == 0) sol.first_filtered = window.back();
        while (static_cast<int>(window.size()) > cfg.s) window.pop_front();
        auto [U, rank] = orthonormalize(hconcat(window), cfg.drop_tol, cfg.orthogonalizer);
        Ritz rr = rayleigh_ritz(A, U, I);
        sel = select_pairs(rr, cfg.m0, I);
        std::vector<int> inside = inside_by_residual(sel);
        double r = max_residual(sel, inside);
        sol.trace.push_back({iter, rank, sol.acc.rhs, r, static_cast<int>(inside.size())});
        sol.iterations = iter;
        if (r <= cfg.tol) {
            sol.converged = 1;
            fill_solution(sol, sel, inside);
            return sol;
        }
        estimate = sel.vectors;
    }
    fill_solution(sol, sel, inside_by_residual(sel));
    return sol;
}

// proj/src/drivers.cpp:188-252
static Solution rfeast_solve(const MatD& A, const Interval& I, const Config& cfg) {
    validate_config(A.r, cfg);
    if (static_cast<long>(cfg.s + 1) * cfg.m0 > A.r)
        std::fprintf(stderr, "rfeast_solve: warning: (s+1)*m0 = %ld exceeds matrix dimension %d\n",
                     static_cast<long>(cfg.s + 1) * cfg.m0, A.r);
    const Rule rule = build_rule(I, cfg.n_c);
    Applier filt(A, rule, cfg.cache);
    Solution sol;
    MatD X = make_initial_guess(A.r, cfg.m0, cfg.seed);
    Ritz sel;
    int m_expected = 0;
    for (int iter = 1; iter <= cfg.max_iter; ++iter) {
        MatD Xp = filt.apply(X, sol.acc);
        if (iter == 1) sol.first_filtered = Xp;
        int dim = Xp.c;
        for (int j = 1; j <= cfg.s; ++j) {
            Ritz rr;
            try {
                rr = rayleigh_ritz(A, Xp, I);
            } catch (const CholeskyError&) {
                ++sol.recovery;
                auto [U, rank] = orthonormalize(Xp, cfg.drop_tol, cfg.orthogonalizer);
                Xp = std::move(U);
                rr = rayleigh_ritz(A, Xp, I);
            }
            if (j == 1) m_expected = count_inside(rr);
            sel = select_pairs(rr, cfg.m0, I);
            if (j < cfg.s) {
                MatD R = residual_block(A, sel.values, sel.vectors);
                MatD ex(Xp.r, Xp.c + R.c);
                std::memcpy(ex.data(), Xp.data(), sizeof(double) * Xp.v.size());
                std::memcpy(ex.data() + Xp.v.size(), R.data(), sizeof(double) * R.v.size());
                Xp = std::move(ex);
                dim = Xp.c;
            }
        }
        std::vector<int> inside = inside_by_residual(sel);
        if (static_cast<int>(inside.size()) > m_expected) inside.resize(m_expected);
        double r = max_residual(sel, inside);
        sol.trace.push_back({iter, dim, sol.acc.rhs, r, m_expected});
        sol.iterations = iter;
        if (r <= cfg.tol) {
            sol.converged = 1;
            fill_solution(sol, sel, inside);
            return sol;
        }
        X = sel.vectors;
    }
    {
        std::vector<int> inside = inside_by_residual(sel);
        if (static_cast<int>(inside.size()) > m_expected) inside.resize(m_expected);
        fill_solution(sol, sel, inside);
    }
    return sol;
}

}  // namespace orc

// ================================================================= C ABI
// Error codes shared with the product ABI (include/feastlab_b200.h):
// 0 ok, 1 invalid_argument, 2 runtime_error, 3 CholeskyError, 4 singular node.
using namespace orc;

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

#define ORC_TRY try {
#define ORC_CATCH(e)                                                              \
    }                                                                             \
    catch (const CholeskyError& x) {                                              \
        if (e) { e->pivot = x.pivot; e->index = x.index; }                        \
        return fail(e, 3, x.what());                                              \
    }                                                                             \
    catch (const SingularNode& x) {                                               \
        if (e) { e->index = x.node; e->z_re = x.z.real(); e->z_im = x.z.imag(); } \
        return fail(e, 4, x.what());                                              \
    }                                                                             \
    catch (const std::invalid_argument& x) { return fail(e, 1, x.what()); }       \
    catch (const std::exception& x) { return fail(e, 2, x.what()); }              \
    return 0;

static MatD wrap(const double* p, int r, int c) {
    MatD M(r, c);
    if (static_cast<size_t>(r) * c > 0) std::memcpy(M.data(), p, sizeof(double) * (size_t)r * c);
    return M;
}
static Rule wrap_rule(int nc, const double* zr, const double* zi, const double* wr,
                      const double* wi) {
    Rule r;
    for (int k = 0; k < nc; ++k) {
        r.z.emplace_back(zr[k], zi[k]);
        r.w.emplace_back(wr[k], wi[k]);
    }
    return r;
}

void orc_set_threads(int t) { scipy_openblas_set_num_threads(t); }
int orc_get_threads(void) { return scipy_openblas_get_num_threads(); }

int orc_gauss_legendre(int n, double* nodes, double* weights, orc_err* e) {
    ORC_TRY
    std::vector<double> g, w;
    gauss_legendre(n, g, w);
    std::memcpy(nodes, g.data(), sizeof(double) * n);
    std::memcpy(weights, w.data(), sizeof(double) * n);
    ORC_CATCH(e)
}

int orc_build_contour_rule(double lo, double hi, int nc, double* zr, double* zi, double* wr,
                           double* wi, orc_err* e) {
    ORC_TRY
    Rule r = build_rule(Interval(lo, hi), nc);
    for (int k = 0; k < nc; ++k) {
        zr[k] = r.z[k].real(); zi[k] = r.z[k].imag();
        wr[k] = r.w[k].real(); wi[k] = r.w[k].imag();
    }
    ORC_CATCH(e)
}

double orc_filter_value(int nc, const double* zr, const double* zi, const double* wr,
                        const double* wi, double lambda) {
    return filter_value(wrap_rule(nc, zr, zi, wr, wi), lambda);
}

int orc_predicted_rate(int nc, const double* zr, const double* zi, const double* wr,
                       const double* wi, const double* spectrum, int ns, int m0, double* out,
                       orc_err* e) {
    ORC_TRY
    *out = predicted_rate(wrap_rule(nc, zr, zi, wr, wi), std::vector<double>(spectrum, spectrum + ns),
                          m0);
    ORC_CATCH(e)
}

int orc_symmetric_matrix(const double* M, int n, double sym_tol, double* out, orc_err* e) {
    ORC_TRY
    MatD S = symmetric_matrix(wrap(M, n, n), sym_tol);
    std::memcpy(out, S.data(), sizeof(double) * (size_t)n * n);
    ORC_CATCH(e)
}

void orc_gaussian_fill(double* out, long long count, unsigned long long seed) {
    gaussian_fill(out, static_cast<size_t>(count), seed);
}

void orc_uniform_fill(double* out, long long count, double lo, double hi,
                      unsigned long long seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(lo, hi);
    for (long long i = 0; i < count; ++i) out[i] = u(rng);
}

int orc_seeded_orthogonal(int n, unsigned long long seed, double* Q, orc_err* e) {
    ORC_TRY
    MatD M = seeded_orthogonal(n, seed);
    std::memcpy(Q, M.data(), sizeof(double) * (size_t)n * n);
    ORC_CATCH(e)
}

// generate_spectrum (proj/src/matmodel.cpp:60-110): values ascending + Q.
int orc_generate_spectrum(int n, double in_lo, double in_hi, int in_count, double out_lo,
                          double out_hi, int out_count, int clustered, int num_clusters,
                          double cluster_width, unsigned long long seed, double* values,
                          double* Q, orc_err* e) {
    ORC_TRY
    Interval in(in_lo, in_hi), out(out_lo, out_hi);
    auto v = layout_values(n, in, in_count, out, out_count, clustered, num_clusters, cluster_width);
    std::memcpy(values, v.data(), sizeof(double) * n);
    MatD M = seeded_orthogonal(n, seed);
    std::memcpy(Q, M.data(), sizeof(double) * (size_t)n * n);
    ORC_CATCH(e)
}

int orc_assemble_matrix(int n, const double* values, const double* Q, double* A, orc_err* e) {
    ORC_TRY
    MatD M = assemble(std::vector<double>(values, values + n), wrap(Q, n, n));
    std::memcpy(A, M.data(), sizeof(double) * (size_t)n * n);
    ORC_CATCH(e)
}

// Test hook: NodeFactorization(A, z).solve(B) with complex B (interleaved).
int orc_node_solve(const double* A, int n, double zr, double zi, const double* B, int p, double* W,
                   orc_err* e) {
    ORC_TRY
    MatD Am = wrap(A, n, n);
    NodeLU f(Am, {zr, zi}, -1);
    MatZ Bm(n, p);
    std::memcpy(static_cast<void*>(Bm.data()), B, sizeof(double) * 2 * (size_t)n * p);
    MatZ Wm = f.solve(Bm);
    std::memcpy(W, Wm.data(), sizeof(double) * 2 * (size_t)n * p);
    ORC_CATCH(e)
}

// Test hook: the packed LU factors and the row transpositions.
int orc_node_factor(const double* A, int n, double zr, double zi, double* LU, int* perm,
                    orc_err* e) {
    ORC_TRY
    NodeLU f(wrap(A, n, n), {zr, zi}, -1);
    std::memcpy(LU, f.lu.data(), sizeof(double) * 2 * (size_t)n * n);
    std::memcpy(perm, f.perm.data(), sizeof(int) * n);
    ORC_CATCH(e)
}

// apply_filter / FilterApplier::apply; `napply` repeated applications of one
// applier (cache=1 exercises the factor cache) — Y receives the last result.
int orc_apply_filter(const double* A, int n, int nc, const double* zr, const double* zi,
                     const double* wr, const double* wi, const double* X, int xr, int p,
                     int cache, int napply, double* Y, long long* rhs, long long* facts,
                     orc_err* e) {
    ORC_TRY
    MatD Am = wrap(A, n, n);
    Rule rule = wrap_rule(nc, zr, zi, wr, wi);
    Applier ap(Am, rule, cache != 0);
    Accounting acc{*rhs, *facts};
    MatD Xm = wrap(X, xr, p);
    MatD Ym;
    for (int i = 0; i < napply; ++i) Ym = ap.apply(Xm, acc);
    std::memcpy(Y, Ym.data(), sizeof(double) * (size_t)xr * p);
    *rhs = acc.rhs;
    *facts = acc.facts;
    ORC_CATCH(e)
}

int orc_orthonormalize(const double* X, int n, int p, double drop_tol, int method, double* U,
                       int* rank, orc_err* e) {
    ORC_TRY
    auto [Um, r] = orthonormalize(wrap(X, n, p), drop_tol, method);
    std::memcpy(U, Um.data(), sizeof(double) * (size_t)n * r);
    *rank = r;
    ORC_CATCH(e)
}

int orc_rayleigh_ritz(const double* A, int n, const double* X, int xr, int p, double lo, double hi,
                      double* vals, double* V, double* norms, unsigned char* inside, orc_err* e) {
    ORC_TRY
    Ritz r = rayleigh_ritz(wrap(A, n, n), wrap(X, xr, p), Interval(lo, hi));
    std::memcpy(vals, r.values.data(), sizeof(double) * p);
    std::memcpy(V, r.vectors.data(), sizeof(double) * (size_t)n * p);
    std::memcpy(norms, r.norms.data(), sizeof(double) * p);
    for (int k = 0; k < p; ++k) inside[k] = r.inside[k];
    ORC_CATCH(e)
}

int orc_residual_block(const double* A, int n, const double* vals, const double* V, int p,
                       double* R, orc_err* e) {
    ORC_TRY
    MatD Rm = residual_block(wrap(A, n, n), std::vector<double>(vals, vals + p), wrap(V, n, p));
    std::memcpy(R, Rm.data(), sizeof(double) * (size_t)n * p);
    ORC_CATCH(e)
}

// select_pairs: outputs the chosen indices (the column gather is the caller's)
int orc_select_pairs(const double* vals, const double* norms, const unsigned char* inside, int p,
                     int m0, double lo, double hi, int* chosen, int* nchosen, orc_err* e) {
    ORC_TRY
    Ritz r;
    r.values.assign(vals, vals + p);
    r.norms.assign(norms, norms + p);
    r.inside.assign(inside, inside + p);
    std::vector<int> idx = select_indices(r, m0, Interval(lo, hi));
    for (size_t j = 0; j < idx.size(); ++j) chosen[j] = idx[j];
    *nchosen = static_cast<int>(idx.size());
    ORC_CATCH(e)
}

int orc_make_initial_guess(int n, int m0, unsigned long long seed, double* X, orc_err* e) {
    ORC_TRY
    MatD M = make_initial_guess(n, m0, seed);
    std::memcpy(X, M.data(), sizeof(double) * (size_t)n * m0);
    ORC_CATCH(e)
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

// variant: 0 feast, 1 xfeast, 2 rfeast. Output capacities: values/norms m0,
// vectors n*m0, trace max_iter, first_filtered n*m0 (may be null).
int orc_solve(int variant, const double* A, int n, double lo, double hi, const orc_config* c,
              double* values, double* vectors, double* norms, int* m, int* converged,
              int* iterations, long long* rhs, long long* facts, int* recovery, orc_trace* trace,
              int* ntrace, double* first_filtered, orc_err* e) {
    ORC_TRY
    Config cfg;
    cfg.m0 = c->m0; cfg.n_c = c->n_c; cfg.s = c->s; cfg.tol = c->tol; cfg.max_iter = c->max_iter;
    cfg.seed = c->seed; cfg.orthogonalizer = c->orthogonalizer; cfg.drop_tol = c->drop_tol;
    cfg.cache = c->cache_factorizations; cfg.generalized_reduced = c->generalized_reduced;
    MatD Am = wrap(A, n, n);
    Interval I(lo, hi);
    Solution s = variant == 0 ? feast_solve(Am, I, cfg)
                 : variant == 1 ? xfeast_solve(Am, I, cfg)
                                : rfeast_solve(Am, I, cfg);
    *m = static_cast<int>(s.values.size());
    std::memcpy(values, s.values.data(), sizeof(double) * s.values.size());
    std::memcpy(norms, s.norms.data(), sizeof(double) * s.norms.size());
    std::memcpy(vectors, s.vectors.data(), sizeof(double) * s.vectors.v.size());
    *converged = s.converged;
    *iterations = s.iterations;
    *rhs = s.acc.rhs;
    *facts = s.acc.facts;
    *recovery = s.recovery;
    *ntrace = static_cast<int>(s.trace.size());
    for (size_t t = 0; t < s.trace.size(); ++t)
        trace[t] = {s.trace[t].iter, s.trace[t].dim, s.trace[t].rhs, s.trace[t].r, s.trace[t].m_found};
    if (first_filtered && s.first_filtered.c > 0)
        std::memcpy(first_filtered, s.first_filtered.data(),
                    sizeof(double) * s.first_filtered.v.size());
    ORC_CATCH(e)
}

}  // extern "C"
