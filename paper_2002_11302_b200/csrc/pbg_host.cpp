// pbg_host.cpp — host input preparation (include/pbg_host.h). OpenMP C++,
// not on the timed hot path. Generators follow the reference's published
// algorithms (proj/src/generate.cpp:20-90, proj/include/spgemm/generate.hpp:
// 12-40) so the same seed gives the same matrix; conversions follow
// proj/src/convert.cpp:41-98 but run as parallel counting sorts.
#include "pbg_host.h"

#include <omp.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

namespace {

struct Sm64 {  // generate.hpp:12-36
    uint64_t s;
    explicit Sm64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t bound) {
        const uint64_t limit = bound * (~uint64_t{0} / bound);
        uint64_t x;
        do x = next();
        while (x >= limit);
        return x % bound;
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

uint64_t split(uint64_t seed, uint64_t stream) {
    return Sm64(seed ^ (stream * 0xD6E8FEB86659FD93ULL)).next();
}

// Parallel exclusive prefix over counts[0..n) into ptr[0..n].
void prefix(const std::vector<uint64_t>& counts, uint64_t* ptr) {
    ptr[0] = 0;
    for (size_t i = 0; i < counts.size(); ++i) ptr[i + 1] = ptr[i] + counts[i];
}

thread_local std::string g_host_err;

int host_fail(const std::string& msg) {
    g_host_err = msg;
    return 1;
}

// ---- Matrix Market (semantics of mm_read, proj/src/mmio.cpp:33-105) ----
struct MmParse {
    std::string err;
};

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

bool blank_or_comment(const char* b, const char* e) {
    for (const char* p = b; p < e; ++p) {
        if (*p == '%') return true;
        if (!std::isspace(static_cast<unsigned char>(*p))) return false;
    }
    return true;
}

// One whitespace-separated unsigned integer token like `istream >> uint64`
// (a leading '+' or '-' is accepted by istream; '-' wraps, as there).
bool take_u64(const char*& p, const char* e, uint64_t& v) {
    while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
    if (p >= e) return false;
    char buf[64];
    size_t n = 0;
    while (p < e && !std::isspace(static_cast<unsigned char>(*p)) && n < sizeof buf - 1) buf[n++] = *p++;
    buf[n] = 0;
    char* end = nullptr;
    errno = 0;
    const unsigned long long x = std::strtoull(buf, &end, 10);
    if (end == buf || errno) return false;
    v = x;
    p -= (buf + n) - end;  // give back an unparsed tail (e.g. "12abc")
    return true;
}

bool take_f64(const char*& p, const char* e, double& v) {
    while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
    if (p >= e) return false;
    char buf[128];
    size_t n = 0;
    while (p < e && !std::isspace(static_cast<unsigned char>(*p)) && n < sizeof buf - 1) buf[n++] = *p++;
    buf[n] = 0;
    // istream >> double (libstdc++ num_get) takes decimal numbers only and
    // fails on overflow; strtod would also take inf/nan/hex spellings
    const char* d = buf + (buf[0] == '+' || buf[0] == '-');
    if (!(std::isdigit(static_cast<unsigned char>(*d)) || *d == '.')) return false;
    if (d[0] == '0' && (d[1] == 'x' || d[1] == 'X')) {
        v = 0.0;  // num_get reads the "0" and stops at 'x'
        p -= (buf + n) - (d + 1);
        return true;
    }
    char* end = nullptr;
    errno = 0;
    const double x = std::strtod(buf, &end);
    if (end == buf || (errno == ERANGE && std::isinf(x))) return false;
    v = x;
    p -= (buf + n) - end;
    return true;
}

}  // namespace

struct pbgh_mm {
    uint32_t nrows = 0, ncols = 0;
    std::vector<uint32_t> rows, cols;
    std::vector<double> vals;
};

namespace {

int mm_parse(const std::string& name, const std::string& text, pbgh_mm& out) {
    const char* p = text.data();
    const char* end = p + text.size();
    uint64_t lineno = 0;
    auto next_line = [&](const char*& b, const char*& e) -> bool {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        if (e > b && e[-1] == '\r') --e;
        ++lineno;
        return true;
    };
    auto fail = [&](uint64_t ln, const std::string& msg) {
        return host_fail(name + ":" + std::to_string(ln) + ": " + msg);
    };
    const char *b, *e;
    if (!next_line(b, e)) return fail(1, "empty file");
    std::string tok[5];
    {
        const char* q = b;
        for (auto& t : tok) {
            while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
            while (q < e && !std::isspace(static_cast<unsigned char>(*q))) t += *q++;
        }
    }
    if (lower(tok[0]) != "%%matrixmarket") return fail(lineno, "missing %%MatrixMarket banner");
    if (lower(tok[1]) != "matrix") return fail(lineno, "unsupported object '" + tok[1] + "'");
    if (lower(tok[2]) != "coordinate") return fail(lineno, "unsupported format '" + tok[2] + "'");
    const std::string field = lower(tok[3]), symmetry = lower(tok[4]);
    if (field != "real" && field != "integer" && field != "pattern")
        return fail(lineno, "unsupported field '" + field + "'");
    if (symmetry != "general" && symmetry != "symmetric")
        return fail(lineno, "unsupported symmetry '" + symmetry + "'");
    const bool pattern = field == "pattern";
    const bool symmetric = symmetry == "symmetric";

    uint64_t nrows = 0, ncols = 0, nnz_decl = 0;
    for (;;) {
        if (!next_line(b, e)) return fail(lineno + 1, "missing size line");
        if (blank_or_comment(b, e)) continue;
        const char* q = b;
        if (!take_u64(q, e, nrows) || !take_u64(q, e, ncols) || !take_u64(q, e, nnz_decl))
            return fail(lineno, "malformed size line");
        break;
    }
    if (nrows < 1 || ncols < 1) return fail(lineno, "matrix dims must be at least 1x1");
    if (nrows > (uint64_t{1} << 31) || ncols > (uint64_t{1} << 31))
        return fail(lineno, "dims exceed 2^31 cap");
    out.nrows = static_cast<uint32_t>(nrows);
    out.ncols = static_cast<uint32_t>(ncols);
    const uint64_t cap = symmetric ? 2 * nnz_decl : nnz_decl;
    out.rows.reserve(cap);
    out.cols.reserve(cap);
    out.vals.reserve(cap);
    uint64_t seen = 0;
    while (seen < nnz_decl) {
        if (!next_line(b, e))
            return fail(lineno + 1, "expected " + std::to_string(nnz_decl) + " entries, got " +
                                        std::to_string(seen));
        if (blank_or_comment(b, e)) continue;
        const char* q = b;
        uint64_t r = 0, c = 0;
        double v = 1.0;
        if (!take_u64(q, e, r) || !take_u64(q, e, c)) return fail(lineno, "malformed entry");
        if (!pattern && !take_f64(q, e, v)) return fail(lineno, "entry missing value");
        if (r < 1 || r > nrows || c < 1 || c > ncols)
            return fail(lineno, "index (" + std::to_string(r) + "," + std::to_string(c) +
                                    ") outside declared " + std::to_string(nrows) + "x" +
                                    std::to_string(ncols));
        if (std::isnan(v)) return fail(lineno, "NaN value");
        const uint32_t row = static_cast<uint32_t>(r - 1), col = static_cast<uint32_t>(c - 1);
        out.rows.push_back(row);
        out.cols.push_back(col);
        out.vals.push_back(v);
        if (symmetric && row != col) {
            out.rows.push_back(col);
            out.cols.push_back(row);
            out.vals.push_back(v);
        }
        ++seen;
    }
    return 0;
}

}  // namespace

extern "C" {

const char* pbgh_last_error(void) { return g_host_err.c_str(); }

int pbgh_mm_open(const char* path, pbgh_mm** out, uint32_t* nrows, uint32_t* ncols,
                 uint64_t* nnz) {
    if (!path || !out) return host_fail("null argument");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) return host_fail(std::string(path) + ": cannot open");
    std::string text;
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, n);
    std::fclose(f);
    auto* h = new pbgh_mm;
    if (int rc = mm_parse(path, text, *h)) {
        delete h;
        return rc;
    }
    *out = h;
    if (nrows) *nrows = h->nrows;
    if (ncols) *ncols = h->ncols;
    if (nnz) *nnz = h->rows.size();
    return 0;
}

int pbgh_mm_fetch(const pbgh_mm* h, uint32_t* rows, uint32_t* cols, double* vals) {
    if (!h) return host_fail("null handle");
    if (rows) std::memcpy(rows, h->rows.data(), h->rows.size() * 4);
    if (cols) std::memcpy(cols, h->cols.data(), h->cols.size() * 4);
    if (vals) std::memcpy(vals, h->vals.data(), h->vals.size() * 8);
    return 0;
}

void pbgh_mm_free(pbgh_mm* h) { delete h; }

int pbgh_mm_write(const char* path, uint32_t nrows, uint32_t ncols, uint64_t nnz,
                  const uint32_t* rows, const uint32_t* cols, const double* vals) {
    for (uint64_t i = 0; i < nnz; ++i)  // validate (convert.cpp:8-37): indices in range
        if (rows[i] >= nrows || cols[i] >= ncols)
            return host_fail("entry " + std::to_string(i) + " outside " + std::to_string(nrows) +
                             "x" + std::to_string(ncols));
    FILE* f = std::fopen(path, "wb");
    if (!f) return host_fail(std::string(path) + ": cannot open for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%u %u %llu\n", nrows, ncols,
                 static_cast<unsigned long long>(nnz));
    for (uint64_t i = 0; i < nnz; ++i)
        std::fprintf(f, "%u %u %.17g\n", rows[i] + 1, cols[i] + 1, vals ? vals[i] : 1.0);
    return std::fclose(f) == 0 ? 0 : host_fail(std::string(path) + ": write failed");
}


uint64_t pbgh_split_seed(uint64_t seed, uint64_t stream) { return split(seed, stream); }

int pbgh_gen_er(int scale, uint32_t d, uint64_t seed, uint32_t* rows, uint32_t* cols) {
    if (scale < 1 || scale > 30 || d < 1) return 1;
    const uint32_t n = 1u << scale;
    if (d > n) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < static_cast<int64_t>(n); ++j) {
        Sm64 rng(split(seed, static_cast<uint64_t>(j)));
        uint32_t* col = rows + static_cast<uint64_t>(j) * d;
        uint32_t filled = 0;
        for (uint32_t t = n - d; t < n; ++t) {  // Floyd's sampling
            const uint32_t r = static_cast<uint32_t>(rng.below(static_cast<uint64_t>(t) + 1));
            bool seen = false;
            for (uint32_t s = 0; s < filled; ++s)
                if (col[s] == r) {
                    seen = true;
                    break;
                }
            cols[static_cast<uint64_t>(j) * d + filled] = static_cast<uint32_t>(j);
            col[filled++] = seen ? t : r;
        }
    }
    return 0;
}

int pbgh_gen_rmat(int scale, uint32_t ef, uint64_t seed, double a, double b, double c,
                  uint32_t* rows, uint32_t* cols) {
    if (scale < 1 || scale > 30 || ef < 1) return 1;
    const uint64_t nedges = static_cast<uint64_t>(ef) << scale;
    const double cut_a = a, cut_ab = a + b, cut_abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < static_cast<int64_t>(nedges); ++e) {
        Sm64 rng(split(seed, static_cast<uint64_t>(e)));
        uint32_t row = 0, col = 0;
        for (int level = scale - 1; level >= 0; --level) {
            const double u = rng.unit();
            if (u >= cut_ab) row |= 1u << level;
            if (u >= cut_abc || (u >= cut_a && u < cut_ab)) col |= 1u << level;
        }
        rows[e] = row;
        cols[e] = col;
    }
    return 0;
}

int pbgh_coo_to_csr(uint32_t nrows, uint32_t ncols, uint64_t nnz, const uint32_t* rows,
                    const uint32_t* cols, const double* vals, int combine, int drop_diag,
                    uint64_t* rowptr, uint32_t* colids, double* vals_out, uint64_t* nnz_out) {
    for (uint64_t i = 0; i < nnz; ++i)
        if (rows[i] >= nrows || cols[i] >= ncols) return 2;
    // counting sort by row (stable), then per-row sort by col + combine
    const int nt = omp_get_max_threads();
    std::vector<std::vector<uint64_t>> local(nt, std::vector<uint64_t>(nrows, 0));
#pragma omp parallel num_threads(nt)
    {
        auto& cnt = local[omp_get_thread_num()];
#pragma omp for schedule(static)
        for (int64_t i = 0; i < static_cast<int64_t>(nnz); ++i) ++cnt[rows[i]];
    }
    std::vector<uint64_t> start(static_cast<size_t>(nrows) + 1, 0);
    {
        uint64_t run = 0;
        for (uint32_t r = 0; r < nrows; ++r) {
            start[r] = run;
            for (int t = 0; t < nt; ++t) {
                const uint64_t c = local[t][r];
                local[t][r] = run;
                run += c;
            }
        }
        start[nrows] = run;
    }
    std::vector<uint32_t> tc(nnz);
    std::vector<double> tv(nnz);
#pragma omp parallel num_threads(nt)
    {
        auto& cur = local[omp_get_thread_num()];
#pragma omp for schedule(static)
        for (int64_t i = 0; i < static_cast<int64_t>(nnz); ++i) {
            const uint64_t at = cur[rows[i]]++;
            tc[at] = cols[i];
            tv[at] = vals ? vals[i] : 1.0;
        }
    }
    std::vector<uint64_t> kept(nrows, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < static_cast<int64_t>(nrows); ++r) {
        const uint64_t lo = start[r], hi = start[r + 1];
        // sort (col, val) pairs by col; stable keeps input order of duplicates
        std::vector<std::pair<uint32_t, double>> seg(hi - lo);
        for (uint64_t p = lo; p < hi; ++p) seg[p - lo] = {tc[p], tv[p]};
        std::stable_sort(seg.begin(), seg.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        uint64_t w = lo;
        for (size_t i = 0; i < seg.size(); ++i) {
            if (drop_diag && seg[i].first == static_cast<uint32_t>(r)) continue;
            if (w > lo && tc[w - 1] == seg[i].first) {
                if (!combine) tv[w - 1] += seg[i].second;
                continue;
            }
            tc[w] = seg[i].first;
            tv[w] = combine ? 1.0 : seg[i].second;
            ++w;
        }
        kept[r] = w - lo;
    }
    prefix(kept, rowptr);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < static_cast<int64_t>(nrows); ++r) {
        const uint64_t src = start[r], dst = rowptr[r], c = kept[r];
        std::memcpy(colids + dst, tc.data() + src, c * 4);
        std::memcpy(vals_out + dst, tv.data() + src, c * 8);
    }
    *nnz_out = rowptr[nrows];
    return 0;
}

int pbgh_csr_to_csc(uint32_t nrows, uint32_t ncols, const uint64_t* rowptr,
                    const uint32_t* colids, const double* vals, uint64_t* colptr,
                    uint32_t* rowids, double* vals_out) {
    const uint64_t nnz = rowptr[nrows];
    const int nt = omp_get_max_threads();
    // rows are split statically among threads in order, so a per-thread
    // cursor keeps rows ascending inside each column.
    std::vector<std::vector<uint64_t>> local(nt, std::vector<uint64_t>(ncols, 0));
    std::vector<uint32_t> rlo(nt + 1);
    for (int t = 0; t <= nt; ++t) rlo[t] = static_cast<uint32_t>(uint64_t(nrows) * t / nt);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        auto& cnt = local[t];
        for (uint32_t r = rlo[t]; r < rlo[t + 1]; ++r)
            for (uint64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) ++cnt[colids[p]];
    }
    uint64_t run = 0;
    for (uint32_t c = 0; c < ncols; ++c) {
        colptr[c] = run;
        for (int t = 0; t < nt; ++t) {
            const uint64_t k = local[t][c];
            local[t][c] = run;
            run += k;
        }
    }
    colptr[ncols] = run;
    if (run != nnz) return 3;
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        auto& cur = local[t];
        for (uint32_t r = rlo[t]; r < rlo[t + 1]; ++r)
            for (uint64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) {
                const uint64_t at = cur[colids[p]]++;
                rowids[at] = r;
                vals_out[at] = vals[p];
            }
    }
    return 0;
}

int pbgh_csr_fill_values(uint64_t vseed, uint32_t nrows, const uint64_t* rowptr,
                         const uint32_t* colids, double* vals) {
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < static_cast<int64_t>(nrows); ++r)
        for (uint64_t p = rowptr[r]; p < rowptr[r + 1]; ++p)
            vals[p] = Sm64(split(vseed, (static_cast<uint64_t>(r) << 32) | colids[p])).unit();
    return 0;
}

int pbgh_stencil27(uint32_t nx, uint32_t ny, uint32_t nz, uint64_t* rowptr, uint32_t* colids,
                   double* vals, uint64_t* nnz_out) {
    const uint64_t n = uint64_t(nx) * ny * nz;
    if (n > 0xffffffffull) return 1;
    auto deg1 = [](uint32_t i, uint32_t e) { return uint32_t((i > 0) + 1 + (i + 1 < e)); };
    std::vector<uint64_t> cnt(n);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) {
        const uint32_t x = r % nx, y = (r / nx) % ny, z = static_cast<uint32_t>(r / (uint64_t(nx) * ny));
        cnt[r] = uint64_t(deg1(x, nx)) * deg1(y, ny) * deg1(z, nz);
    }
    uint64_t total = 0;
    for (uint64_t r = 0; r < n; ++r) total += cnt[r];
    *nnz_out = total;
    if (!rowptr) return 0;
    prefix(cnt, rowptr);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < static_cast<int64_t>(n); ++r) {
        const int64_t x = r % nx, y = (r / nx) % ny, z = r / (int64_t(nx) * ny);
        uint64_t at = rowptr[r];
        for (int dz = -1; dz <= 1; ++dz)  // ascending column order: z, then y, then x
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t X = x + dx, Y = y + dy, Z = z + dz;
                    if (X < 0 || Y < 0 || Z < 0 || X >= nx || Y >= ny || Z >= nz) continue;
                    colids[at] = static_cast<uint32_t>((Z * ny + Y) * nx + X);
                    vals[at] = (dx == 0 && dy == 0 && dz == 0) ? 26.0 : -1.0;
                    ++at;
                }
    }
    return 0;
}

int pbgh_csc_row_band(uint32_t nrows, uint32_t ncols, const uint64_t* colptr,
                      const uint32_t* rowids, const double* vals, uint32_t r0, uint32_t r1,
                      uint64_t* colptr_out, uint32_t* rowids_out, double* vals_out,
                      uint64_t* nnz_out) {
    if (r0 > r1 || r1 > nrows) return 1;
    // row ids inside a column need not be sorted: filter, keeping their order
    std::vector<uint64_t> cnt(ncols);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < static_cast<int64_t>(ncols); ++j) {
        uint64_t c = 0;
        for (uint64_t q = colptr[j]; q < colptr[j + 1]; ++q) c += rowids[q] >= r0 && rowids[q] < r1;
        cnt[j] = c;
    }
    uint64_t total = 0;
    for (uint32_t j = 0; j < ncols; ++j) total += cnt[j];
    *nnz_out = total;
    if (!colptr_out) return 0;
    prefix(cnt, colptr_out);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < static_cast<int64_t>(ncols); ++j) {
        uint64_t o = colptr_out[j];
        for (uint64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
            const uint32_t r = rowids[q];
            if (r < r0 || r >= r1) continue;
            rowids_out[o] = r - r0;
            vals_out[o] = vals[q];
            ++o;
        }
    }
    return 0;
}

int pbgh_row_flop(uint32_t nrows, uint32_t ncols, const uint64_t* a_colptr,
                  const uint32_t* a_rowids, const uint64_t* b_rowptr, uint64_t* row_flop) {
    std::fill(row_flop, row_flop + nrows, 0);
    for (uint32_t j = 0; j < ncols; ++j) {
        const uint64_t lb = b_rowptr[j + 1] - b_rowptr[j];
        for (uint64_t p = a_colptr[j]; p < a_colptr[j + 1]; ++p) row_flop[a_rowids[p]] += lb;
    }
    return 0;
}

int pbgh_band_cuts(uint32_t nrows, const uint64_t* row_flop, uint32_t g, uint32_t* cuts) {
    if (g == 0) return 1;
    unsigned __int128 total = 0;
    for (uint32_t r = 0; r < nrows; ++r) total += row_flop[r];
    cuts[0] = 0;
    for (uint32_t j = 1; j <= g; ++j) cuts[j] = nrows;
    unsigned __int128 acc = 0;
    uint32_t j = 1;
    for (uint32_t r = 0; r < nrows && j < g; ++r) {
        acc += row_flop[r];
        while (j < g && acc * g >= total * j) cuts[j++] = r + 1;
    }
    return 0;
}

}  // extern "C"
