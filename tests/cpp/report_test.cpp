// Drop-in check for the measurement headers: code in the style of the
// reference's callers — bench.cpp:84-93 (run_once), bench.cpp:149
// (rec.phases.derive(rec.stats, b)), spgemm_bench.cpp:121,148-151 — compiles
// against include/spgemm_b200 alone, and the roofline known answers of
// proj/tests/test_roofline.cpp:9-55 hold.
//   ./report_test nodevice   -> header KATs + validate(); the multiply throws runtime_error
//   ./report_test gpu        -> also a run_once on the B200 with derive()
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "spgemm_b200/pb_spgemm.hpp"
#include "spgemm_b200/report.hpp"
#include "spgemm_b200/roofline.hpp"

using namespace spgemm;

static int failures = 0;
#define CHECK(x)                                                             \
    do {                                                                     \
        if (!(x)) {                                                          \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static bool near(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::fabs(b); }

struct Record {  // bench.hpp BenchRecord fields the reference's bench fills
    MultiplyStats stats;
    PhaseReport phases;
    double cf = 0.0, ai_upper = 0.0, ai_outer_lower = 0.0, peak_mflops = 0.0;
};

// bench.cpp:84-93: one PB run, PhaseReport copied out of the result
static Record run_once(const CscMatrix& a, const CsrMatrix& b) {
    PbConfig cfg;
    cfg.nthreads = 0;
    WallTimer wall;
    PbResult res = pb_multiply(a, b, cfg);
    Record rec;
    rec.stats = {a.nnz(), b.nnz(), res.c.nnz(), res.sym.flop};
    rec.phases = res.phases;
    rec.phases.derive(rec.stats, 16.0);  // bench.cpp:149
    rec.cf = compression_factor(rec.stats);
    rec.ai_upper = ai_upper(rec.cf, 16.0);
    rec.ai_outer_lower = ai_outer_lower(rec.cf, 16.0);
    rec.peak_mflops = peak_flops(MachineModel{6.55e12, 16.0}, rec.ai_upper) / 1e6;
    CHECK(wall.seconds() >= rec.phases.t_total * 0.5);
    return rec;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    // test_roofline.cpp:9-16
    CHECK(near(compression_factor({0, 0, 9000000, 27500000}), 3.06, 0.01));
    CHECK(near(compression_factor({0, 0, 34200000, 562000000}), 16.41, 0.01));
    CHECK(compression_factor({0, 0, 100, 100}) == 1.0);
    CHECK(std::isnan(compression_factor({0, 0, 0, 0})));
    // :18-28
    CHECK(ai_upper(1.0, 16.0) == 0.0625);
    CHECK(ai_upper(8.0, 16.0) == 0.5);
    CHECK(near(ai_col_lower(1.0, 16.0), 1.0 / 48.0, 1e-15));
    CHECK(near(ai_col_lower(2.0, 16.0), 1.0 / 32.0, 1e-15));
    CHECK(ai_outer_lower(1.0, 16.0) == 0.0125);
    // :30-33
    CHECK(near(ai_col_lower(1e9, 16.0), 1.0 / 16.0, 1e-6));
    CHECK(near(ai_outer_lower(1e9, 16.0), 1.0 / 32.0, 1e-6));
    // :35-41
    CHECK(near(peak_flops(50e9, 1.0 / 16.0), 3.125e9, 1e-12));
    CHECK(near(peak_flops(40e9, 1.0 / 80.0), 500e6, 1e-12));
    CHECK(peak_flops(50e9, 0.0) == 0.0);
    MachineModel mm{50e9, 16.0};
    CHECK(near(peak_flops(mm, ai_upper(1.0, mm.b)), 3.125e9, 1e-12));
    // :43-55
    MultiplyStats s{1000, 1000, 4000, 5000};
    TrafficModel t = traffic_model(s, 16.0);
    CHECK(t.expand_read == 32000.0);
    CHECK(t.expand_write == 80000.0);
    CHECK(t.sort_read == 80000.0);
    CHECK(t.compress_write == 64000.0);
    CHECK(t.total() == 16.0 * (1000 + 1000 + 2 * 5000 + 4000));
    MultiplyStats id{4, 4, 4, 4};
    CHECK(traffic_model(id, 16.0).total() == 320.0);
    CHECK(crossover_cf() == 4.0);
    CHECK(near(ai_ratio_outer_over_col(1.0), 3.0 / 5.0, 1e-15));
    // PhaseReport::derive (report.hpp:42-51)
    PhaseReport ph;
    ph.t_expand = 2.0;
    ph.t_sort = 1.0;
    ph.t_total = 4.0;
    ph.derive(s, 16.0);
    CHECK(ph.bytes_expand == 112000.0);
    CHECK(ph.bytes_sort == 80000.0);
    CHECK(ph.bytes_compress == 64000.0);
    CHECK(ph.bw_expand == 56000.0);
    CHECK(ph.bw_sort == 80000.0);
    CHECK(ph.bw_compress == 0.0);
    CHECK(ph.mflops == 5000.0 / 4.0 / 1e6);
    WallTimer w;
    CHECK(w.lap() >= 0.0 && w.seconds() >= 0.0);

    // validate (convert.cpp:8-80) and the entry orders (types.hpp:35-42)
    CHECK(coo_order_row_major({0, 5, 1.0}, {1, 0, 1.0}));
    CHECK(!coo_order_col_major({0, 5, 1.0}, {1, 0, 1.0}));
    CooMatrix coo;
    coo.dims = {2, 2};
    coo.entries = {{0, 1, 1.0}, {1, 0, 2.0}};
    validate(coo);
    coo.entries.push_back({2, 0, 1.0});
    bool threw = false;
    try {
        validate(coo);
    } catch (const structural_error& e) {
        threw = std::strcmp(e.what(), "coo entry (2,0) out of 2x2") == 0;
    }
    CHECK(threw);
    CsrMatrix bad;
    bad.dims = {1, 3};
    bad.rowptr = {0, 2};
    bad.colids = {2, 1};
    bad.values = {1.0, 1.0};
    threw = false;
    try {
        validate(bad);
    } catch (const structural_error& e) {
        threw = std::strcmp(e.what(), "csr: ids not strictly increasing") == 0;
    }
    CHECK(threw);

    // identity squared (n = 4): every count is 4 -> model total 320 bytes
    CscMatrix a;
    a.dims = {4, 4};
    a.colptr = {0, 1, 2, 3, 4};
    a.rowids = {0, 1, 2, 3};
    a.values = {1, 1, 1, 1};
    CsrMatrix b;
    b.dims = {4, 4};
    b.rowptr = {0, 1, 2, 3, 4};
    b.colids = {0, 1, 2, 3};
    b.values = {1, 1, 1, 1};
    validate(a);
    validate(b);
    if (gpu) {
        Record rec = run_once(a, b);
        CHECK(rec.stats.flop == 4 && rec.stats.nnz_c == 4);
        CHECK(traffic_model(rec.stats, 16.0).total() == 320.0);
        CHECK(rec.phases.bytes_expand == 16.0 * (4 + 4 + 4));
        CHECK(rec.phases.t_total > 0.0 && rec.phases.mflops > 0.0);
        CHECK(rec.cf == 1.0);
    } else {
        bool rt = false;
        try {
            run_once(a, b);
        } catch (const std::runtime_error&) {
            rt = true;
        }
        CHECK(rt);
    }
    std::printf("%s: %d failure(s)\n", gpu ? "gpu" : "nodevice", failures);
    return failures ? 1 : 0;
}
