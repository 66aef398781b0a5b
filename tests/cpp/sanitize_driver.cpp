// sanitize_driver: small products that reach every kernel family of the
// C-ABI (expand, count, sort+merge with its TMA bulk loads/stores, the
// duplicate pre-merge, the LSD fallback, the heavy-row split + dense reduce,
// the column hash SpGEMM incl. hub columns, COO conversion, device
// generators, bounded-memory rounds and multi-context bands), run under
// compute-sanitizer (memcheck / racecheck / synccheck / initcheck) by
// tests/test_gpu_sanitize.py. No torch: the process holds only libpbg.
// Exit code 0 = every call returned PBG_OK and the conservation counters
// agree; the sanitizer's own --error-exitcode flags its findings.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pbg.h"
#include "pbg_host.h"

static int failures = 0;
#define CHECK(x)                                                                    \
    do {                                                                            \
        if (!(x)) {                                                                 \
            std::printf("CHECK failed %s:%d: %s (%s)\n", __FILE__, __LINE__, #x,    \
                        pbg_last_error());                                          \
            ++failures;                                                             \
        }                                                                           \
    } while (0)

struct Csx {
    uint32_t nrows = 0, ncols = 0;
    std::vector<uint64_t> ptr;
    std::vector<uint32_t> idx;
    std::vector<double> val;
    pbg_csx_view view() const {
        return pbg_csx_view{nrows, ncols, idx.size(), ptr.data(), idx.data(), val.data()};
    }
};

static bool fetch(pbg_handle* h, uint32_t nmajor, uint64_t nnz, Csx& m, pbg_report* rep) {
    m.ptr.assign(nmajor + 1, 0);
    m.idx.assign(nnz, 0);
    m.val.assign(nnz, 0.0);
    const int rc = pbg_multiply_fetch(h, m.ptr.data(), m.idx.data(), m.val.data(), rep);
    pbg_release(h);
    return rc == PBG_OK;
}

// kind 0 = ER (ef = d), 1 = RMAT; CSR or CSC of the same seeded matrix
static Csx generate(int kind, int scale, uint32_t ef, int to_csc) {
    pbg_config cfg;
    pbg_default_config(&cfg);
    pbg_handle* h = nullptr;
    uint64_t nnz = 0;
    Csx m;
    m.nrows = m.ncols = 1u << scale;
    CHECK(pbg_generate_begin(kind, scale, ef, 1, 2, to_csc, &cfg, &h, &nnz) == PBG_OK);
    if (h) CHECK(fetch(h, m.nrows, nnz, m, nullptr));
    return m;
}

static Csx csr_to_csc(const Csx& r) {
    Csx c;
    c.nrows = r.nrows;
    c.ncols = r.ncols;
    c.ptr.assign(r.ncols + 1, 0);
    for (uint32_t j : r.idx) ++c.ptr[j + 1];
    for (uint32_t j = 0; j < r.ncols; ++j) c.ptr[j + 1] += c.ptr[j];
    c.idx.resize(r.idx.size());
    c.val.resize(r.idx.size());
    std::vector<uint64_t> pos(c.ptr.begin(), c.ptr.end() - 1);
    for (uint32_t i = 0; i < r.nrows; ++i)
        for (uint64_t e = r.ptr[i]; e < r.ptr[i + 1]; ++e) {
            const uint64_t p = pos[r.idx[e]]++;
            c.idx[p] = i;
            c.val[p] = r.val[e];
        }
    return c;
}

static void multiply(const char* name, const Csx& a_csc, const Csx& b_csr, uint32_t bin_cap) {
    pbg_config cfg;
    pbg_default_config(&cfg);
    cfg.bin_cap = bin_cap;
    pbg_handle* h = nullptr;
    uint64_t nnz = 0;
    const pbg_csx_view av = a_csc.view(), bv = b_csr.view();
    CHECK(pbg_multiply_begin(&av, &bv, &cfg, &h, &nnz) == PBG_OK);
    if (!h) return;
    Csx c;
    pbg_report rep;
    CHECK(fetch(h, a_csc.nrows, nnz, c, &rep));
    CHECK(rep.tuples_into_sort == rep.flop && rep.merged_total == nnz);
    std::printf("%-28s flop=%llu nnz(C)=%llu heavy=%u lsd=%llu\n", name,
                (unsigned long long)rep.flop, (unsigned long long)nnz, rep.heavy_bins,
                (unsigned long long)rep.sort_fallbacks);
}

int main(int argc, char** argv) {
    const std::string only = argc > 1 ? argv[1] : "";
    auto want = [&](const char* c) { return only.empty() || only == c; };
    if (!pbg_device_available()) {
        std::printf("no CUDA device\n");
        return 2;
    }
    if (want("er")) {
        const Csx b = generate(0, 12, 8, 0), a = generate(0, 12, 8, 1);
        multiply("ER 2^12 d8", a, b, 0);
        multiply("ER 2^12 d8 bin_cap 512", a, b, 512);
        // bounded-memory rounds + two contexts on one device (row bands)
        pbg_config cfg;
        pbg_default_config(&cfg);
        cfg.ngpus = 2;
        cfg.flags = PBG_FLAG_WRAP_DEVICES;
        cfg.reserved[0] = 40000;  // tuples per round: several rounds per band
        const pbg_csx_view av = a.view(), bv = b.view();
        std::vector<uint64_t> rp(a.nrows + 1);
        const uint64_t cap = 1u << 20;
        std::vector<uint32_t> ci(cap);
        std::vector<double> cv(cap);
        uint64_t nnz = 0;
        pbg_report rep;
        CHECK(pbg_multiply_into(&av, &bv, &cfg, rp.data(), ci.data(), cv.data(), cap, &nnz, &rep) ==
              PBG_OK);
        std::printf("%-28s nnz(C)=%llu rounds=%u\n", "ER bands x2 + rounds",
                    (unsigned long long)nnz, rep.nrounds);
    }
    if (want("rmat")) {
        const Csx b = generate(1, 11, 8, 0), a = generate(1, 11, 8, 1);
        multiply("RMAT 2^11 ef8 bin_cap 256", a, b, 256);  // heavy split + dense reduce
        multiply("RMAT 2^11 ef8", a, b, 0);
    }
    if (want("stencil")) {  // duplicate-heavy bins: the shared-memory pre-merge
        uint64_t nnz = 0;
        CHECK(pbgh_stencil27(10, 10, 10, nullptr, nullptr, nullptr, &nnz) == 0);
        Csx s;
        s.nrows = s.ncols = 1000;
        s.ptr.resize(1001);
        s.idx.resize(nnz);
        s.val.resize(nnz);
        CHECK(pbgh_stencil27(10, 10, 10, s.ptr.data(), s.idx.data(), s.val.data(), &nnz) == 0);
        multiply("stencil 10^3", csr_to_csc(s), s, 0);
    }
    if (want("lsd")) {
        // 5 rows of 700 clustered columns in one bin: 23 key bits, MSD buckets of
        // 2048 columns, 700 keys in a bucket > SM_BMAX (512) -> LSD radix
        Csx a, b;
        a.nrows = b.ncols = 1u << 20;
        a.ncols = b.nrows = 1;
        a.ptr = {0, 5};
        a.idx = {0, 1, 2, 3, 4};
        a.val = {2.0, 3.0, 4.0, 5.0, 6.0};
        b.ptr = {0, 700};
        for (uint32_t j = 0; j < 700; ++j) {
            b.idx.push_back(699 - j);
            b.val.push_back(j + 1.0);
        }
        multiply("clustered rows (LSD)", a, b, 0);
    }
    if (want("hash")) {
        const Csx a = generate(1, 12, 8, 1);
        pbg_config cfg;
        pbg_default_config(&cfg);
        pbg_handle* h = nullptr;
        uint64_t nnz = 0;
        const pbg_csx_view av = a.view();
        CHECK(pbg_hash_multiply_begin(&av, &av, &cfg, &h, &nnz) == PBG_OK);
        Csx c;
        if (h) CHECK(fetch(h, a.ncols, nnz, c, nullptr));
        std::printf("%-28s nnz(C)=%llu\n", "hash RMAT 2^12 (hubs)", (unsigned long long)nnz);
    }
    if (want("coo")) {  // duplicates and exact-zero sums through the conversion
        std::vector<uint32_t> r = {3, 1, 3, 0, 1, 3}, c = {2, 0, 2, 1, 0, 2};
        std::vector<double> v = {1.0, 2.0, -1.0, 4.0, 5.0, 0.0};
        pbg_config cfg;
        pbg_default_config(&cfg);
        pbg_handle* h = nullptr;
        uint64_t nnz = 0;
        CHECK(pbg_coo_convert_begin(4, 3, r.size(), r.data(), c.data(), v.data(), 0, &cfg, &h,
                                    &nnz) == PBG_OK);
        Csx m;
        if (h) CHECK(fetch(h, 4, nnz, m, nullptr));
        CHECK(nnz == 3);
    }
    std::printf("sanitize_driver: %d failure(s)\n", failures);
    return failures ? 1 : 0;
}
