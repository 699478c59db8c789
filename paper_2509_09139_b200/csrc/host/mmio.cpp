// Matrix Market coordinate I/O and a binary CSR cache (host) — SURVEY.md §8f-2.
// Semantics follow the reference reader/writer (matrix_market.cpp:36-121):
//  * banner "%%MatrixMarket matrix coordinate <real|integer> <general|symmetric>"
//    (case-insensitive) on line 1;
//  * comment ('%') and blank lines may precede the size line and interleave
//    the entries; the size line is "rows cols nnz";
//  * entries are 1-based "i j value" (extra tokens ignored); symmetric files
//    mirror every off-diagonal entry;
//  * assembly = SparseMatrix::from_triplets (sparse_matrix.cpp:52-88): sort by
//    (row, col, bit pattern of the value), sum duplicates in that order from 0.0;
//  * every parse error names its 1-based line ("matrix market: line N: ...").
// The writer emits "real general" with %.17g values (exact round trip).
// The parser works on the whole file in memory with strtoll/strtod (no
// iostreams), which is what makes SuiteSparse-size files load quickly.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../hpbj_common.hpp"

namespace hpbj {

namespace {

struct Trip {
    int64_t r, c;
    double v;
};

[[noreturn]] void mm_error(long line, const std::string& what) {
    fail(HPBJ_EIO, "matrix market: line " + std::to_string(line) + ": " + what);
}

std::string lower(std::string s) {
    for (char& ch : s) ch = (char)std::tolower((unsigned char)ch);
    return s;
}

bool is_blank(const char* b, const char* e) {
    for (; b < e; ++b)
        if (!std::isspace((unsigned char)*b)) return false;
    return true;
}

std::string read_all(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(HPBJ_EIO, std::string("cannot open matrix file: ") + path);
    std::string buf;
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.append(chunk, got);
    std::fclose(f);
    return buf;
}

// Parse one integer / double token from [p, e); false if none.
bool next_i64(const char*& p, const char* e, int64_t& out) {
    while (p < e && std::isspace((unsigned char)*p)) ++p;
    if (p >= e) return false;
    std::string tok;
    const char* q = p;
    while (q < e && !std::isspace((unsigned char)*q)) ++q;
    tok.assign(p, q);
    char* end = nullptr;
    errno = 0;
    const long long v = std::strtoll(tok.c_str(), &end, 10);
    if (end == tok.c_str() || errno == ERANGE) return false;
    p += end - tok.c_str();  // like operator>>: stop at the first character that is not part of the number
    out = v;
    return true;
}

bool next_f64(const char*& p, const char* e, double& out) {
    while (p < e && std::isspace((unsigned char)*p)) ++p;
    if (p >= e) return false;
    std::string tok;
    const char* q = p;
    while (q < e && !std::isspace((unsigned char)*q)) ++q;
    tok.assign(p, q);
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str()) return false;
    if (errno == ERANGE && std::isinf(v)) return false;  // overflow: the stream extractor fails too
    p += end - tok.c_str();
    out = v;
    return true;
}

}  // namespace

// Assemble CSR from triplets with the reference's from_triplets semantics.
void assemble_csr(std::vector<Trip>& t, int64_t nrows, std::vector<int64_t>& rp, std::vector<int64_t>& ci,
                  std::vector<double>& val) {
    std::sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
        if (a.r != b.r) return a.r < b.r;
        if (a.c != b.c) return a.c < b.c;
        uint64_t ua, ub;
        std::memcpy(&ua, &a.v, 8);
        std::memcpy(&ub, &b.v, 8);
        return ua < ub;
    });
    rp.assign(nrows + 1, 0);
    ci.clear();
    val.clear();
    ci.reserve(t.size());
    val.reserve(t.size());
    for (size_t k = 0; k < t.size();) {
        const int64_t r = t[k].r, c = t[k].c;
        double sum = 0.0;
        while (k < t.size() && t[k].r == r && t[k].c == c) sum += t[k++].v;
        ci.push_back(c);
        val.push_back(sum);
        rp[r + 1] = (int64_t)ci.size();
    }
    for (int64_t i = 0; i < nrows; ++i) rp[i + 1] = std::max(rp[i + 1], rp[i]);
}

void mm_read(const char* path, int64_t& nrows, int64_t& ncols, std::vector<int64_t>& rp, std::vector<int64_t>& ci,
             std::vector<double>& val) {
    const std::string buf = read_all(path);
    const char* p = buf.data();
    const char* end = p + buf.size();
    long line = 0;
    auto next_line = [&](const char*& b, const char*& e) -> bool {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        ++line;
        return true;
    };
    const char *b, *e;
    if (!next_line(b, e)) mm_error(1, "empty stream");
    {
        std::vector<std::string> tok;
        const char* q = b;
        while (q < e) {
            while (q < e && std::isspace((unsigned char)*q)) ++q;
            const char* s = q;
            while (q < e && !std::isspace((unsigned char)*q)) ++q;
            if (q > s) tok.emplace_back(s, q);
        }
        tok.resize(5);
        if (lower(tok[0]) != "%%matrixmarket") mm_error(line, "missing %%MatrixMarket banner");
        if (lower(tok[1]) != "matrix") mm_error(line, "unsupported object '" + tok[1] + "'");
        if (lower(tok[2]) != "coordinate") mm_error(line, "unsupported format '" + tok[2] + "' (coordinate only)");
        const std::string field = lower(tok[3]);
        if (field != "real" && field != "integer")
            mm_error(line, "unsupported field '" + field + "' (real/integer only)");
        const std::string sym = lower(tok[4]);
        if (sym != "general" && sym != "symmetric")
            mm_error(line, "unsupported symmetry '" + sym + "' (general/symmetric only)");
        tok[4] = sym;
        nrows = ncols = -1;
        int64_t declared = -1;
        while (next_line(b, e)) {
            if (b < e && *b == '%') continue;
            if (is_blank(b, e)) continue;
            const char* q = b;
            int64_t r, c, z;
            if (!next_i64(q, e, r) || !next_i64(q, e, c) || !next_i64(q, e, z) || r < 0 || c < 0 || z < 0)
                mm_error(line, "malformed size line '" + std::string(b, e) + "'");
            nrows = r;
            ncols = c;
            declared = z;
            break;
        }
        if (declared < 0) mm_error(line, "missing size line");
        const bool symmetric = tok[4] == "symmetric";
        std::vector<Trip> t;
        t.reserve((size_t)(symmetric ? 2 * declared : declared));
        int64_t read = 0;
        while (read < declared) {
            if (!next_line(b, e))
                mm_error(line + 1, "unexpected end of file, expected " + std::to_string(declared) +
                                       " entries, got " + std::to_string(read));
            if (b < e && *b == '%') continue;
            if (is_blank(b, e)) continue;
            const char* q = b;
            int64_t i, j;
            double v;
            if (!next_i64(q, e, i) || !next_i64(q, e, j) || !next_f64(q, e, v))
                mm_error(line, "malformed entry '" + std::string(b, e) + "'");
            if (i < 1 || i > nrows || j < 1 || j > ncols)
                mm_error(line, "index (" + std::to_string(i) + ", " + std::to_string(j) + ") out of range");
            t.push_back({i - 1, j - 1, v});
            if (symmetric && i != j) t.push_back({j - 1, i - 1, v});
            ++read;
        }
        assemble_csr(t, nrows, rp, ci, val);
    }
}

void mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
              const double* val) {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(HPBJ_EIO, std::string("cannot open output file: ") + path);
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)nrows,
                 (long long)ncols, (long long)rp[nrows]);
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            std::fprintf(f, "%lld %lld %.17g\n", (long long)(i + 1), (long long)(ci[k] + 1), val[k]);
    if (std::fclose(f) != 0) fail(HPBJ_EIO, std::string("write failed: ") + path);
}

// Binary CSR cache: "HPBJCSR1", int64 n, int64 nnz, int64 rp[n+1], int64 ci[nnz], f64 val[nnz].
constexpr char kCsrMagic[8] = {'H', 'P', 'B', 'J', 'C', 'S', 'R', '1'};

void csr_write(const char* path, int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(HPBJ_EIO, std::string("cannot open output file: ") + path);
    const int64_t nnz = rp[n];
    bool ok = std::fwrite(kCsrMagic, 1, 8, f) == 8 && std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&nnz, 8, 1, f) == 1 &&
              std::fwrite(rp, 8, (size_t)n + 1, f) == (size_t)n + 1 && std::fwrite(ci, 8, (size_t)nnz, f) == (size_t)nnz &&
              std::fwrite(val, 8, (size_t)nnz, f) == (size_t)nnz;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) fail(HPBJ_EIO, std::string("write failed: ") + path);
}

void csr_read(const char* path, int64_t& n, std::vector<int64_t>& rp, std::vector<int64_t>& ci,
              std::vector<double>& val) {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(HPBJ_EIO, std::string("cannot open CSR cache: ") + path);
    char magic[8];
    int64_t nnz = -1;
    bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kCsrMagic, 8) == 0 &&
              std::fread(&n, 8, 1, f) == 1 && std::fread(&nnz, 8, 1, f) == 1 && n >= 0 && nnz >= 0;
    if (ok) {
        rp.resize(n + 1);
        ci.resize(nnz);
        val.resize(nnz);
        ok = std::fread(rp.data(), 8, (size_t)n + 1, f) == (size_t)n + 1 &&
             std::fread(ci.data(), 8, (size_t)nnz, f) == (size_t)nnz &&
             std::fread(val.data(), 8, (size_t)nnz, f) == (size_t)nnz && rp[0] == 0 && rp[n] == nnz;
    }
    std::fclose(f);
    if (!ok) fail(HPBJ_EIO, std::string("not a valid CSR cache: ") + path);
}

}  // namespace hpbj

using namespace hpbj;

namespace {
template <class T>
T* dup_array(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(1, v.size())));
    if (!p) fail(HPBJ_ENOMEM, "out of host memory");
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}
}  // namespace

extern "C" {

int hpbj_mm_read(const char* path, int64_t* nrows, int64_t* ncols, int64_t** row_ptr, int64_t** col,
                 double** val) {
    if (!path || !nrows || !ncols || !row_ptr || !col || !val) return HPBJ_EINVAL;
    return guard(nullptr, [&] {
        std::vector<int64_t> rp, ci;
        std::vector<double> v;
        mm_read(path, *nrows, *ncols, rp, ci, v);
        *row_ptr = dup_array(rp);
        *col = dup_array(ci);
        *val = dup_array(v);
    });
}

int hpbj_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int64_t* col,
                  const double* val) {
    if (!path || nrows < 0 || ncols < 0 || !row_ptr) return HPBJ_EINVAL;
    return guard(nullptr, [&] { mm_write(path, nrows, ncols, row_ptr, col, val); });
}

int hpbj_csr_cache_write(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* col,
                         const double* val) {
    if (!path || n < 0 || !row_ptr) return HPBJ_EINVAL;
    return guard(nullptr, [&] { csr_write(path, n, row_ptr, col, val); });
}

int hpbj_csr_cache_read(const char* path, int64_t* n, int64_t** row_ptr, int64_t** col, double** val) {
    if (!path || !n || !row_ptr || !col || !val) return HPBJ_EINVAL;
    return guard(nullptr, [&] {
        std::vector<int64_t> rp, ci;
        std::vector<double> v;
        csr_read(path, *n, rp, ci, v);
        *row_ptr = dup_array(rp);
        *col = dup_array(ci);
        *val = dup_array(v);
    });
}

void hpbj_free(void* p) { std::free(p); }

}  // extern "C"
