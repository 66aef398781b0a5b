// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/build_ref.sh into oracle/_ref/).
// It lets the Python tests and bench.py's reference/cpu_baseline arm call the
// reference's own entry points through ctypes:
//   spgemm::pb_multiply           proj/include/spgemm/pb_spgemm.hpp:116
//   spgemm::symbolic/make_bins/expand/sort_bins/compress_bins/convert_csr
//                                 proj/include/spgemm/pb_spgemm.hpp:59-108
//   spgemm::gen_er / gen_rmat     proj/include/spgemm/generate.hpp:65-69
//   spgemm::coo_to_csc/coo_to_csr proj/include/spgemm/convert.hpp:8-9
//   spgemm::reference_multiply    proj/include/spgemm/reference.hpp:12
//   spgemm::mm_read / mm_write    proj/include/spgemm/mmio.hpp:15-21
//   spgemm::hash_multiply         proj/include/spgemm/baseline.hpp:21-24
// Exceptions are turned into return codes: 1 parameter_error, 2 internal_error,
// 3 anything else; the message goes to ref_last_error().

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "spgemm/baseline.hpp"
#include "spgemm/convert.hpp"
#include "spgemm/generate.hpp"
#include "spgemm/mmio.hpp"
#include "spgemm/pb_spgemm.hpp"
#include "spgemm/reference.hpp"

using namespace spgemm;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const parameter_error& e) {
        g_err = e.what();
        return 1;
    } catch (const internal_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

CscMatrix make_csc(uint32_t nrows, uint32_t ncols, uint64_t nnz, const uint64_t* ptr,
                   const uint32_t* idx, const double* val) {
    CscMatrix m;
    m.dims = {nrows, ncols};
    m.colptr.assign(ptr, ptr + ncols + 1);
    m.rowids.assign(idx, idx + nnz);
    m.values.assign(val, val + nnz);
    return m;
}

CsrMatrix make_csr(uint32_t nrows, uint32_t ncols, uint64_t nnz, const uint64_t* ptr,
                   const uint32_t* idx, const double* val) {
    CsrMatrix m;
    m.dims = {nrows, ncols};
    m.rowptr.assign(ptr, ptr + nrows + 1);
    m.colids.assign(idx, idx + nnz);
    m.values.assign(val, val + nnz);
    return m;
}

PbConfig make_cfg(uint32_t nbins, uint32_t lbin, uint64_t l2, int nthreads, int balanced) {
    PbConfig c;
    c.nbins = nbins;
    c.lbin_bytes = lbin;
    c.l2_bytes = l2;
    c.nthreads = nthreads;
    c.balanced_bins = balanced != 0;
    return c;
}

struct RefResult {
    CsrMatrix c;
    SymbolicResult sym;
    PhaseReport phases;
    uint64_t tuples_into_sort = 0;
    uint64_t merged_total = 0;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- generators (values 1.0 as the reference emits them) ----
int ref_gen(int kind, int scale, uint32_t ef, uint64_t seed, void** out) {
    return guarded([&] {
        auto* m = new CooMatrix(kind == 0 ? gen_er(GenSpec::er(scale, ef, seed))
                                          : gen_rmat(GenSpec::rmat(scale, ef, seed)));
        *out = m;
    });
}

uint64_t ref_coo_nnz(void* h) { return static_cast<CooMatrix*>(h)->nnz(); }

void ref_coo_get(void* h, uint32_t* rows, uint32_t* cols, double* vals) {
    auto* m = static_cast<CooMatrix*>(h);
    for (size_t i = 0; i < m->entries.size(); ++i) {
        rows[i] = m->entries[i].row;
        cols[i] = m->entries[i].col;
        vals[i] = m->entries[i].val;
    }
}

void ref_coo_free(void* h) { delete static_cast<CooMatrix*>(h); }

// ---- column hash SpGEMM (CSC x CSC -> CSC) ----
int ref_hash_multiply(uint32_t a_nrows, uint32_t a_ncols, uint64_t a_nnz, const uint64_t* a_colptr,
                      const uint32_t* a_rowids, const double* a_vals, uint32_t b_nrows,
                      uint32_t b_ncols, uint64_t b_nnz, const uint64_t* b_colptr,
                      const uint32_t* b_rowids, const double* b_vals, int nthreads, void** out) {
    return guarded([&] {
        CscMatrix a, b;
        a.dims = {a_nrows, a_ncols};
        a.colptr.assign(a_colptr, a_colptr + a_ncols + 1);
        a.rowids.assign(a_rowids, a_rowids + a_nnz);
        a.values.assign(a_vals, a_vals + a_nnz);
        b.dims = {b_nrows, b_ncols};
        b.colptr.assign(b_colptr, b_colptr + b_ncols + 1);
        b.rowids.assign(b_rowids, b_rowids + b_nnz);
        b.values.assign(b_vals, b_vals + b_nnz);
        *out = new CscMatrix(hash_multiply(a, b, nthreads));
    });
}
uint64_t ref_csc_nnz(void* h) { return static_cast<CscMatrix*>(h)->rowids.size(); }
void ref_csc_get(void* h, uint64_t* colptr, uint32_t* rowids, double* vals) {
    auto* m = static_cast<CscMatrix*>(h);
    std::memcpy(colptr, m->colptr.data(), m->colptr.size() * 8);
    std::memcpy(rowids, m->rowids.data(), m->rowids.size() * 4);
    std::memcpy(vals, m->values.data(), m->values.size() * 8);
}
void ref_csc_free(void* h) { delete static_cast<CscMatrix*>(h); }

// ---- Matrix Market: mm_read into a COO handle (ref_coo_*), mm_write ----
int ref_mm_read(const char* path, void** out, uint32_t* nrows, uint32_t* ncols) {
    return guarded([&] {
        auto* m = new CooMatrix(mm_read(std::string(path)));
        *nrows = m->dims.nrows;
        *ncols = m->dims.ncols;
        *out = m;
    });
}

int ref_mm_write(const char* path, uint32_t nrows, uint32_t ncols, uint64_t nnz,
                 const uint32_t* rows, const uint32_t* cols, const double* vals) {
    return guarded([&] {
        CooMatrix m;
        m.dims = {nrows, ncols};
        for (uint64_t i = 0; i < nnz; ++i) m.entries.push_back({rows[i], cols[i], vals[i]});
        mm_write(m, std::string(path));
    });
}

// ---- conversion: COO -> CSC (major=col) or CSR (major=row) ----
// Caller gives ptr of size nmajor+1 and idx/val of size nnz (upper bound);
// *nnz_out gets the merged count.
int ref_coo_convert(int to_csr, uint32_t nrows, uint32_t ncols, uint64_t nnz,
                    const uint32_t* rows, const uint32_t* cols, const double* vals,
                    uint64_t* ptr, uint32_t* idx, double* val, uint64_t* nnz_out) {
    return guarded([&] {
        CooMatrix m;
        m.dims = {nrows, ncols};
        m.entries.resize(nnz);
        for (uint64_t i = 0; i < nnz; ++i) m.entries[i] = {rows[i], cols[i], vals[i]};
        if (to_csr) {
            CsrMatrix r = coo_to_csr(m);
            std::memcpy(ptr, r.rowptr.data(), r.rowptr.size() * 8);
            std::memcpy(idx, r.colids.data(), r.colids.size() * 4);
            std::memcpy(val, r.values.data(), r.values.size() * 8);
            *nnz_out = r.nnz();
        } else {
            CscMatrix c = coo_to_csc(m);
            std::memcpy(ptr, c.colptr.data(), c.colptr.size() * 8);
            std::memcpy(idx, c.rowids.data(), c.rowids.size() * 4);
            std::memcpy(val, c.values.data(), c.values.size() * 8);
            *nnz_out = c.nnz();
        }
    });
}

// ---- the hot path: pb_multiply (stepwise=1 runs the stepwise API to expose
// the conservation counters, as acceptance.cpp:46-58 does) ----
int ref_pb_multiply(uint32_t a_nrows, uint32_t a_ncols, uint64_t a_nnz, const uint64_t* a_colptr,
                    const uint32_t* a_rowids, const double* a_vals, uint32_t b_nrows,
                    uint32_t b_ncols, uint64_t b_nnz, const uint64_t* b_rowptr,
                    const uint32_t* b_colids, const double* b_vals, uint32_t nbins,
                    uint32_t lbin_bytes, uint64_t l2_bytes, int nthreads, int balanced,
                    int stepwise, void** out) {
    return guarded([&] {
        const CscMatrix a = make_csc(a_nrows, a_ncols, a_nnz, a_colptr, a_rowids, a_vals);
        const CsrMatrix b = make_csr(b_nrows, b_ncols, b_nnz, b_rowptr, b_colids, b_vals);
        const PbConfig cfg = make_cfg(nbins, lbin_bytes, l2_bytes, nthreads, balanced);
        auto* r = new RefResult;
        try {
            if (stepwise) {
                r->sym = symbolic(a, b, cfg);
                BinSet bins = make_bins(r->sym, {a.dims.nrows, b.dims.ncols});
                expand(a, b, bins, cfg);
                r->tuples_into_sort = bins.total_filled();
                sort_bins(bins, cfg);
                compress_bins(bins, cfg);
                r->merged_total = bins.total_merged();
                r->c = convert_csr(bins);
            } else {
                PbResult res = pb_multiply(a, b, cfg);
                r->c = std::move(res.c);
                r->sym = std::move(res.sym);
                r->phases = res.phases;
                r->tuples_into_sort = r->sym.flop;
                r->merged_total = r->c.nnz();
            }
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

uint64_t ref_res_nnz(void* h) { return static_cast<RefResult*>(h)->c.nnz(); }
uint32_t ref_res_nbins(void* h) { return static_cast<RefResult*>(h)->sym.nbins; }

void ref_res_get(void* h, uint64_t* rowptr, uint32_t* colids, double* vals) {
    auto* r = static_cast<RefResult*>(h);
    std::memcpy(rowptr, r->c.rowptr.data(), r->c.rowptr.size() * 8);
    std::memcpy(colids, r->c.colids.data(), r->c.colids.size() * 4);
    std::memcpy(vals, r->c.values.data(), r->c.values.size() * 8);
}

// counters[0..3] = flop, tuples_into_sort, merged_total, uniform_rows_per_bin
void ref_res_counters(void* h, uint64_t* counters) {
    auto* r = static_cast<RefResult*>(h);
    counters[0] = r->sym.flop;
    counters[1] = r->tuples_into_sort;
    counters[2] = r->merged_total;
    counters[3] = r->sym.uniform_rows_per_bin;
}

// per_column_flop[ncols(A)], per_bin_flop[nbins], bin_row_starts[nbins+1]
void ref_res_symbolic(void* h, uint64_t* per_column_flop, uint64_t* per_bin_flop,
                      uint32_t* bin_row_starts) {
    auto* r = static_cast<RefResult*>(h);
    std::memcpy(per_column_flop, r->sym.per_column_flop.data(),
                r->sym.per_column_flop.size() * 8);
    std::memcpy(per_bin_flop, r->sym.per_bin_flop.data(), r->sym.per_bin_flop.size() * 8);
    std::memcpy(bin_row_starts, r->sym.bin_row_starts.data(),
                r->sym.bin_row_starts.size() * 4);
}

// t_symbolic, t_expand, t_sort, t_compress, t_convert, t_total (seconds)
void ref_res_times(void* h, double* t) {
    auto* r = static_cast<RefResult*>(h);
    t[0] = r->phases.t_symbolic;
    t[1] = r->phases.t_expand;
    t[2] = r->phases.t_sort;
    t[3] = r->phases.t_compress;
    t[4] = r->phases.t_convert;
    t[5] = r->phases.t_total;
}

void ref_res_free(void* h) { delete static_cast<RefResult*>(h); }

// choose_nbins (pb_spgemm.cpp:10-18) for the KATs
uint32_t ref_choose_nbins(uint64_t flop, uint32_t nrows, uint64_t l2_bytes, uint32_t tuple_bytes) {
    PbConfig c;
    c.l2_bytes = l2_bytes;
    return choose_nbins(flop, nrows, c, tuple_bytes);
}

// dense oracle (reference.cpp:8-35) on COO input; output COO in a handle
int ref_dense_multiply(uint32_t m, uint32_t k, uint32_t n, uint64_t annz, const uint32_t* ar,
                       const uint32_t* ac, const double* av, uint64_t bnnz, const uint32_t* br,
                       const uint32_t* bc, const double* bv, void** out) {
    return guarded([&] {
        CooMatrix a, b;
        a.dims = {m, k};
        b.dims = {k, n};
        for (uint64_t i = 0; i < annz; ++i) a.entries.push_back({ar[i], ac[i], av[i]});
        for (uint64_t i = 0; i < bnnz; ++i) b.entries.push_back({br[i], bc[i], bv[i]});
        *out = new CooMatrix(reference_multiply(a, b));
    });
}

// ---- bench.py --impl reference: the benchmark configs built and multiplied
// with the reference library alone (nothing of the product is loaded). ----
//
// kind 0: gen_er (generate.cpp:20-54); kind 1: gen_rmat (generate.cpp:56-90,
// duplicates collapsed) minus self-loops; kind 2: the 27-point stencil on a
// scale^3 grid (26 on the diagonal, -1 off it; not a reference generator).
// Values U[0,1) = SplitMix64(split_seed(vseed, row << 32 | col)).next_unit()
// (generate.hpp:12-40) for kinds 0/1. A is kept as CSC (left operand) and
// CSR (right operand) converted by the reference's coo_to_csc / coo_to_csr
// (convert.cpp:82-98) — the reference bench's --matrix squaring path
// (spgemm_bench.cpp:55-58).
struct RefConfig {
    CscMatrix a;        // full left operand
    CsrMatrix b;        // right operand
    CscMatrix band;     // rows [0, r1) of a (same dims), when a band is chosen
    bool use_band = false;
    std::vector<std::uint64_t> row_flop;
    std::uint64_t flop = 0;
};

int ref_config_make(int kind, int scale, uint32_t ef, uint64_t seed, uint64_t vseed, void** out) {
    return guarded([&] {
        CooMatrix coo;
        if (kind == 0 || kind == 1) {
            coo = kind == 0 ? gen_er(GenSpec::er(scale, ef, seed))
                            : gen_rmat(GenSpec::rmat(scale, ef, seed));
            if (kind == 1) {
                std::size_t w = 0;
                for (std::size_t i = 0; i < coo.entries.size(); ++i)
                    if (coo.entries[i].row != coo.entries[i].col) coo.entries[w++] = coo.entries[i];
                coo.entries.resize(w);
            }
            for (auto& e : coo.entries)
                e.val = SplitMix64(split_seed(vseed, (std::uint64_t(e.row) << 32) | e.col)).next_unit();
        } else if (kind == 2) {
            const std::int64_t g = scale;
            const std::int64_t n = g * g * g;
            coo.dims = {static_cast<index_t>(n), static_cast<index_t>(n)};
            coo.entries.reserve(static_cast<std::size_t>(n) * 27);
            for (std::int64_t r = 0; r < n; ++r) {
                const std::int64_t x = r % g, y = (r / g) % g, z = r / (g * g);
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const std::int64_t X = x + dx, Y = y + dy, Z = z + dz;
                            if (X < 0 || Y < 0 || Z < 0 || X >= g || Y >= g || Z >= g) continue;
                            const bool diag = dx == 0 && dy == 0 && dz == 0;
                            coo.entries.push_back({static_cast<index_t>(r),
                                                   static_cast<index_t>((Z * g + Y) * g + X),
                                                   diag ? 26.0 : -1.0});
                        }
            }
        } else {
            throw parameter_error("ref_config_make: unknown kind");
        }
        auto* c = new RefConfig;
        c->a = coo_to_csc(coo);
        c->b = coo_to_csr(coo);
        // per-row flop of A*B (the quantity balanced_starts accumulates,
        // pb_spgemm.cpp:58-82) for band sampling
        c->row_flop.assign(c->a.dims.nrows, 0);
        for (index_t k = 0; k < c->a.dims.ncols; ++k) {
            const std::uint64_t bk = c->b.rowptr[k + 1] - c->b.rowptr[k];
            for (offset_t p = c->a.colptr[k]; p < c->a.colptr[k + 1]; ++p)
                c->row_flop[c->a.rowids[p]] += bk;
        }
        for (auto f : c->row_flop) c->flop += f;
        *out = c;
    });
}

// A Matrix Market file squared: mm_read (mmio.cpp:33-105) -> coo_to_csc /
// coo_to_csr, as the reference bench's --matrix path (spgemm_bench.cpp:55-58).
int ref_config_from_mtx(const char* path, void** out) {
    return guarded([&] {
        CooMatrix coo = mm_read(std::string(path));
        if (coo.dims.nrows != coo.dims.ncols) throw parameter_error("--matrix needs a square matrix");
        auto* c = new RefConfig;
        c->a = coo_to_csc(coo);
        c->b = coo_to_csr(coo);
        c->row_flop.assign(c->a.dims.nrows, 0);
        for (index_t k = 0; k < c->a.dims.ncols; ++k) {
            const std::uint64_t bk = c->b.rowptr[k + 1] - c->b.rowptr[k];
            for (offset_t p = c->a.colptr[k]; p < c->a.colptr[k + 1]; ++p)
                c->row_flop[c->a.rowids[p]] += bk;
        }
        for (auto f : c->row_flop) c->flop += f;
        *out = c;
    });
}

// stats[0..3] = nrows, nnz(A), flop(A*A), nnz(B)
void ref_config_stats(void* h, uint64_t* stats) {
    auto* c = static_cast<RefConfig*>(h);
    stats[0] = c->a.dims.nrows;
    stats[1] = c->a.nnz();
    stats[2] = c->flop;
    stats[3] = c->b.nnz();
}

// The CSC (left) and CSR (right) arrays, for the test that pins this builder
// to the product's input builder.
void ref_config_get(void* h, uint64_t* a_colptr, uint32_t* a_rowids, double* a_vals,
                    uint64_t* b_rowptr, uint32_t* b_colids, double* b_vals) {
    auto* c = static_cast<RefConfig*>(h);
    std::memcpy(a_colptr, c->a.colptr.data(), c->a.colptr.size() * 8);
    std::memcpy(a_rowids, c->a.rowids.data(), c->a.rowids.size() * 4);
    std::memcpy(a_vals, c->a.values.data(), c->a.values.size() * 8);
    std::memcpy(b_rowptr, c->b.rowptr.data(), c->b.rowptr.size() * 8);
    std::memcpy(b_colids, c->b.colids.data(), c->b.colids.size() * 4);
    std::memcpy(b_vals, c->b.values.data(), c->b.values.size() * 8);
}

// Restrict the left operand to the leading rows holding about frac of the
// flop (frac >= 1: the whole matrix). *r1 / *band_flop describe the band.
int ref_config_band(void* h, double frac, uint32_t* r1, uint64_t* band_flop) {
    return guarded([&] {
        auto* c = static_cast<RefConfig*>(h);
        const index_t m = c->a.dims.nrows;
        if (frac >= 1.0) {
            c->use_band = false;
            c->band = CscMatrix{};
            *r1 = m;
            *band_flop = c->flop;
            return;
        }
        const double target = frac * static_cast<double>(c->flop);
        index_t r = 0;
        std::uint64_t acc = 0;
        while (r < m && static_cast<double>(acc) < target) acc += c->row_flop[r++];
        CscMatrix& bd = c->band;
        bd.dims = c->a.dims;
        bd.colptr.assign(c->a.dims.ncols + 1, 0);
        bd.rowids.clear();
        bd.values.clear();
        for (index_t k = 0; k < c->a.dims.ncols; ++k) {
            for (offset_t p = c->a.colptr[k]; p < c->a.colptr[k + 1]; ++p)
                if (c->a.rowids[p] < r) {
                    bd.rowids.push_back(c->a.rowids[p]);
                    bd.values.push_back(c->a.values[p]);
                }
            bd.colptr[k + 1] = bd.rowids.size();
        }
        c->use_band = true;
        *r1 = r;
        *band_flop = acc;
    });
}

// One spgemm::pb_multiply (pb_spgemm.hpp:116) with the default PbConfig and
// nthreads threads, on the config (or its band). times[0..5] = the
// reference's own PhaseReport (t_symbolic, t_expand, t_sort, t_compress,
// t_convert, t_total: its WallTimer laps, pb_spgemm.cpp:330-361 — how
// bench.cpp:84-93,130-138 times a run). out[0..1] = flop, nnz(C).
int ref_config_multiply(void* h, int nthreads, double* times, uint64_t* out) {
    return guarded([&] {
        auto* c = static_cast<RefConfig*>(h);
        PbConfig cfg;
        cfg.nthreads = nthreads;
        PbResult res = pb_multiply(c->use_band ? c->band : c->a, c->b, cfg);
        times[0] = res.phases.t_symbolic;
        times[1] = res.phases.t_expand;
        times[2] = res.phases.t_sort;
        times[3] = res.phases.t_compress;
        times[4] = res.phases.t_convert;
        times[5] = res.phases.t_total;
        out[0] = res.sym.flop;
        out[1] = res.c.nnz();
    });
}

void ref_config_free(void* h) { delete static_cast<RefConfig*>(h); }

}  // extern "C"
