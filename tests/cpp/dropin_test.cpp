// Drop-in check: code written against the reference's C++ API
// (spgemm::pb_multiply, CscMatrix/CsrMatrix, PbConfig, parameter_error /
// internal_error — proj/include/spgemm/pb_spgemm.hpp:116, types.hpp:51-91)
// compiles unchanged against include/spgemm_b200/ and runs on the GPU.
//   ./dropin_test nodevice   -> parameter errors still thrown, compute throws runtime_error
//   ./dropin_test gpu        -> known answers of test_pb_spgemm.cpp on the B200
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "spgemm_b200/baseline.hpp"
#include "spgemm_b200/mmio.hpp"
#include "spgemm_b200/pb_spgemm.hpp"

using namespace spgemm;

static int failures = 0;
#define CHECK(x)                                                          \
    do {                                                                  \
        if (!(x)) {                                                       \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++failures;                                                   \
        }                                                                 \
    } while (0)

static CscMatrix csc_of(index_t n, std::vector<CooEntry> e) {
    CscMatrix m;
    m.dims = {n, n};
    m.colptr.assign(n + 1, 0);
    std::sort(e.begin(), e.end(), [](auto& a, auto& b) { return a.col == b.col ? a.row < b.row : a.col < b.col; });
    for (auto& x : e) ++m.colptr[x.col + 1];
    for (index_t j = 0; j < n; ++j) m.colptr[j + 1] += m.colptr[j];
    for (auto& x : e) {
        m.rowids.push_back(x.row);
        m.values.push_back(x.val);
    }
    return m;
}

static CsrMatrix csr_of(index_t n, std::vector<CooEntry> e) {
    CsrMatrix m;
    m.dims = {n, n};
    m.rowptr.assign(n + 1, 0);
    std::sort(e.begin(), e.end(), [](auto& a, auto& b) { return a.row == b.row ? a.col < b.col : a.row < b.row; });
    for (auto& x : e) ++m.rowptr[x.row + 1];
    for (index_t i = 0; i < n; ++i) m.rowptr[i + 1] += m.rowptr[i];
    for (auto& x : e) {
        m.colids.push_back(x.col);
        m.values.push_back(x.val);
    }
    return m;
}

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    // helpers that are pure header code (pb_spgemm.hpp:20-41 semantics)
    CHECK(pack_key(2049, 7, 2048, 20) == ((std::uint64_t{1} << 20) | 7));
    CHECK(unpack_key((std::uint64_t{1} << 20) | 7, 2048, 20).row == 2049);
    CHECK(choose_key_width(1 << 10, 1 << 20) == 32);
    CHECK(choose_key_width(1 << 13, 1 << 20) == 64);
    CHECK(choose_nbins(std::uint64_t{16} << 20, 1 << 20, PbConfig{}) == 512);

    CooMatrix dummy;
    CscMatrix a43;
    a43.dims = {4, 3};
    a43.colptr.assign(4, 0);
    CsrMatrix b44 = csr_of(4, {});
    CHECK(throws<parameter_error>([&] { pb_multiply(a43, b44); }));
    PbConfig bad;
    bad.nbins = 3;
    CHECK(throws<parameter_error>([&] { pb_multiply(csc_of(4, {}), b44, bad); }));
    PbConfig badl;
    badl.lbin_bytes = 24;
    CHECK(throws<parameter_error>([&] { pb_multiply(csc_of(4, {}), b44, badl); }));

    // Matrix Market round trip (mmio.hpp:15-21), host only
    {
        CooMatrix m;
        m.dims = {3, 4};
        m.entries = {{0, 0, 1.5}, {2, 3, -2e-3}, {1, 1, 0.0}};
        const char* path = "dropin_test_tmp.mtx";
        mm_write(m, path);
        CooMatrix r = mm_read(path);
        CHECK(r.dims == m.dims && r.entries == m.entries);
        std::remove(path);
        CHECK(throws<parse_error>([&] { mm_read("no/such/file.mtx"); }));
    }
    CHECK(throws<parameter_error>([&] { hash_multiply(a43, csc_of(4, {})); }));

    std::vector<CooEntry> eye;
    for (index_t i = 0; i < 4; ++i) eye.push_back({i, i, 1.0});
    if (!gpu) {
        CHECK(throws<std::runtime_error>([&] { pb_multiply(csc_of(4, eye), csr_of(4, eye)); }));
    } else {
        PbResult r = pb_multiply(csc_of(4, eye), csr_of(4, eye));
        CHECK(r.sym.flop == 4);
        CHECK(r.c.nnz() == 4);
        CHECK((r.sym.per_column_flop == std::vector<std::uint64_t>{1, 1, 1, 1}));
        std::vector<CooEntry> d2 = {{0, 0, 1.0}, {0, 1, 2.0}, {1, 0, 3.0}, {1, 1, 4.0}};
        PbResult q = pb_multiply(csc_of(2, d2), csr_of(2, d2));
        CHECK(q.sym.flop == 8);
        CHECK((q.c.values == std::vector<double>{7.0, 10.0, 15.0, 22.0}));
        CHECK(q.tuples_into_sort == 8 && q.merged_total == 4);
        // 64-bit key widening case (test_pb_spgemm.cpp:337-359)
        const index_t big = 1u << 21;
        CscMatrix wa = csc_of(big, {{0, 0, 2.0}, {5, big - 1, 3.0}, {big - 1, 5, 4.0}});
        CsrMatrix wb = csr_of(big, {{0, 7, 5.0}, {big - 1, 0, 6.0}, {5, 5, 7.0}});
        PbResult w = pb_multiply(wa, wb);
        CHECK(w.c.nnz() == 3);
        CHECK(w.c.rowptr[1] == 1 && w.c.colids[0] == 7 && w.c.values[0] == 10.0);
        CHECK(w.c.colids[1] == 0 && w.c.values[1] == 18.0);
        CHECK(w.c.colids[2] == 5 && w.c.values[2] == 28.0 && w.c.rowptr[big] == 3);
        // empty product (test_pb_spgemm.cpp:381-387)
        PbResult e = pb_multiply(csc_of(16, {}), csr_of(16, {}));
        CHECK(e.c.nnz() == 0 && e.sym.flop == 0);
        // cancellation keeps a structural zero (test_pb_spgemm.cpp:238-244)
        PbResult z = pb_multiply(csc_of(2, {{0, 0, 1.0}, {0, 1, -1.0}}),
                                 csr_of(2, {{0, 1, 1.0}, {1, 1, 1.0}}));
        CHECK(z.c.nnz() == 1 && z.c.values[0] == 0.0);
        // column hash SpGEMM (baseline.hpp:21-24): the 2x2 known answer in CSC
        CscMatrix hc = hash_multiply(csc_of(2, d2), csc_of(2, d2));
        CHECK((hc.colptr == std::vector<offset_t>{0, 2, 4}));
        CHECK((hc.rowids == std::vector<index_t>{0, 1, 0, 1}));
        CHECK((hc.values == std::vector<double>{7.0, 15.0, 10.0, 22.0}));
        CHECK(heap_multiply(csc_of(2, d2), csc_of(2, d2)).values == hc.values);
    }
    if (!gpu) {
        CHECK(throws<std::runtime_error>([&] { hash_multiply(csc_of(4, eye), csc_of(4, eye)); }));
    }
    std::printf("%s: %d failure(s)\n", gpu ? "gpu" : "nodevice", failures);
    return failures ? 1 : 0;
}
