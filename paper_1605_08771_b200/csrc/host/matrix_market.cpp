// Matrix Market reader / writer (proj/src/matrix_market.cpp:31-147), the
// input-side format of the filter path. Semantics follow the reference line
// by line -- banner and header checks in the same order with the same
// messages, '%' comment and blank lines skipped, entry tokens read as
// `long long double` with trailing text ignored, 1-based line numbers in
// every MatrixMarketError -- but the file is read once into memory and
// scanned in place, instead of an istringstream per line.
#include "feastlab/matrix_market.hpp"

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace feastlab {

namespace {

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// In-memory line scanner with the reference's next_data_line rule
// (matrix_market.cpp:18-27): skip lines that are blank (" \t\r") or whose
// first non-blank character is '%'.
struct Lines {
    const char* p;
    const char* end;
    int line = 0;
    const char* cur = nullptr;      // current line [cur, cur_end)
    const char* cur_end = nullptr;
    bool next_raw() {
        if (p >= end) return false;
        cur = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        cur_end = nl ? nl : end;
        p = nl ? nl + 1 : end;
        ++line;
        return true;
    }
    bool next_data() {
        while (next_raw()) {
            const char* q = cur;
            while (q < cur_end && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
            if (q == cur_end) continue;
            if (*q == '%') continue;
            return true;
        }
        return false;
    }
};

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// `istream >> long` on [q, e): skip blanks, optional sign, digits
bool read_long(const char*& q, const char* e, long long& v) {
    while (q < e && is_space(*q)) ++q;
    const char* s = q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    if (q >= e || !std::isdigit(static_cast<unsigned char>(*q))) return false;
    char buf[32];
    const char* d = q;
    while (q < e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
    const size_t len = static_cast<size_t>(q - s);
    if (len >= sizeof(buf)) return false;
    std::memcpy(buf, s, len);
    buf[len] = 0;
    (void)d;
    errno = 0;
    v = std::strtoll(buf, nullptr, 10);
    return errno == 0;
}

// `istream >> double` on [q, e): decimal floating point (no inf / nan / hex,
// which libstdc++'s num_get rejects too)
bool read_double(const char*& q, const char* e, double& v) {
    while (q < e && is_space(*q)) ++q;
    const char* s = q;
    const char* t = q;
    if (t < e && (*t == '+' || *t == '-')) ++t;
    bool digits = false;
    while (t < e && std::isdigit(static_cast<unsigned char>(*t))) ++t, digits = true;
    if (t < e && *t == '.') {
        ++t;
        while (t < e && std::isdigit(static_cast<unsigned char>(*t))) ++t, digits = true;
    }
    if (!digits) return false;
    if (t < e && (*t == 'e' || *t == 'E')) {
        const char* x = t + 1;
        if (x < e && (*x == '+' || *x == '-')) ++x;
        if (x < e && std::isdigit(static_cast<unsigned char>(*x))) {
            while (x < e && std::isdigit(static_cast<unsigned char>(*x))) ++x;
            t = x;
        }
    }
    char buf[128];
    const size_t len = static_cast<size_t>(t - s);
    if (len >= sizeof(buf)) return false;
    std::memcpy(buf, s, len);
    buf[len] = 0;
    v = std::strtod(buf, nullptr);
    q = t;
    return true;
}

std::vector<char> slurp(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("read_matrix_market: cannot open '" + path + "'");
    std::vector<char> data;
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long size = std::ftell(f);
        if (size > 0) data.resize(static_cast<size_t>(size));
        std::rewind(f);
    }
    size_t got = data.empty() ? 0 : std::fread(data.data(), 1, data.size(), f);
    data.resize(got);
    char chunk[1 << 16];  // streams whose size is unknown (pipes)
    while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.insert(data.end(), chunk, chunk + got);
    std::fclose(f);
    return data;
}

}  // namespace

int read_matrix_market_into(const std::string& path, double* A, long lda) {
    const std::vector<char> data = slurp(path);
    Lines in{data.data(), data.data() + data.size()};
    if (!in.next_raw()) throw MatrixMarketError("read_matrix_market: empty file", 1);
    // header tokens (istringstream >> banner >> object >> format >> field >> symmetry)
    std::string tok[5];
    {
        const char* q = in.cur;
        for (auto& t : tok) {
            while (q < in.cur_end && std::isspace(static_cast<unsigned char>(*q))) ++q;
            const char* s = q;
            while (q < in.cur_end && !std::isspace(static_cast<unsigned char>(*q))) ++q;
            t.assign(s, q);
        }
    }
    const std::string& banner = tok[0];
    const std::string object = lower(tok[1]), format = lower(tok[2]), field = lower(tok[3]),
                      symmetry = lower(tok[4]);
    if (banner != "%%MatrixMarket")
        throw MatrixMarketError("read_matrix_market: missing %%MatrixMarket banner", 1);
    if (object != "matrix")
        throw MatrixMarketError("read_matrix_market: unsupported object '" + object + "'", 1);
    if (format != "coordinate" && format != "array")
        throw MatrixMarketError("read_matrix_market: unsupported format '" + format + "'", 1);
    if (field != "real")
        throw MatrixMarketError("read_matrix_market: unsupported field '" + field + "'", 1);
    if (symmetry != "symmetric")
        throw NotSymmetricError("read_matrix_market: expected symmetry 'symmetric', got '" +
                                    symmetry + "'",
                                1);
    if (!in.next_data())
        throw MatrixMarketError("read_matrix_market: missing size line", in.line);

    const bool coord = format == "coordinate";
    long long rows = 0, cols = 0, nnz = 0;
    {
        const char* q = in.cur;
        if (!read_long(q, in.cur_end, rows) || !read_long(q, in.cur_end, cols) ||
            (coord && !read_long(q, in.cur_end, nnz)))
            throw MatrixMarketError("read_matrix_market: malformed size line", in.line);
        if (rows != cols || rows < 1)
            throw MatrixMarketError("read_matrix_market: matrix must be square", in.line);
        if (rows > 0x7fffffffLL) throw MatrixMarketError("read_matrix_market: matrix too large", in.line);
    }
    const int n = static_cast<int>(rows);
    if (!A) return n;
    if (lda < n) throw std::invalid_argument("read_matrix_market: lda < n");
    if (coord) {
        for (int j = 0; j < n; ++j) std::memset(A + (long)j * lda, 0, sizeof(double) * n);
        for (long long e = 0; e < nnz; ++e) {
            if (!in.next_data())
                throw MatrixMarketError("read_matrix_market: unexpected end of file", in.line);
            long long i, j;
            double v;
            const char* q = in.cur;
            if (!read_long(q, in.cur_end, i) || !read_long(q, in.cur_end, j) ||
                !read_double(q, in.cur_end, v))
                throw MatrixMarketError("read_matrix_market: malformed entry", in.line);
            if (i < 1 || i > rows || j < 1 || j > cols)
                throw MatrixMarketError("read_matrix_market: index out of range", in.line);
            if (j > i)
                throw MatrixMarketError(
                    "read_matrix_market: upper-triangle entry in symmetric file", in.line);
            A[(j - 1) * lda + (i - 1)] = v;
            A[(i - 1) * lda + (j - 1)] = v;
        }
        return n;
    }
    // array symmetric: packed lower triangle, column major
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) {
            if (!in.next_data())
                throw MatrixMarketError("read_matrix_market: unexpected end of file", in.line);
            double v;
            const char* q = in.cur;
            if (!read_double(q, in.cur_end, v))
                throw MatrixMarketError("read_matrix_market: malformed value", in.line);
            A[(long)j * lda + i] = v;
            A[(long)i * lda + j] = v;
        }
    }
    return n;
}

SymmetricMatrix read_matrix_market(const std::string& path) {
    const int n = read_matrix_market_into(path, nullptr, 0);
    MatrixXd M(n, n);
    read_matrix_market_into(path, M.data(), n);
    return SymmetricMatrix(std::move(M));
}

void write_matrix_market(const double* A, int n, long lda, const std::string& path,
                         MatrixMarketFormat format) {
    std::FILE* out = std::fopen(path.c_str(), "w");
    if (!out) throw std::runtime_error("write_matrix_market: cannot open '" + path + "'");
    bool ok = true;
    if (format == MatrixMarketFormat::coordinate) {
        ok &= std::fprintf(out, "%%%%MatrixMarket matrix coordinate real symmetric\n%d %d %ld\n", n,
                           n, static_cast<long>(n) * (n + 1) / 2) > 0;
        for (int j = 0; j < n && ok; ++j)
            for (int i = j; i < n; ++i)
                ok &= std::fprintf(out, "%d %d %.17g\n", i + 1, j + 1, A[(long)j * lda + i]) > 0;
    } else {
        ok &= std::fprintf(out, "%%%%MatrixMarket matrix array real symmetric\n%d %d\n", n, n) > 0;
        for (int j = 0; j < n && ok; ++j)
            for (int i = j; i < n; ++i) ok &= std::fprintf(out, "%.17g\n", A[(long)j * lda + i]) > 0;
    }
    ok &= std::fclose(out) == 0;
    if (!ok) throw std::runtime_error("write_matrix_market: write failed for '" + path + "'");
}

void write_matrix_market(const SymmetricMatrix& matrix, const std::string& path,
                         MatrixMarketFormat format) {
    write_matrix_market(matrix.mat().data(), matrix.dim(), matrix.dim(), path, format);
}

}  // namespace feastlab
