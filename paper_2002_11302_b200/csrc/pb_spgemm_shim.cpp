// pb_spgemm_shim.cpp — spgemm::pb_multiply re-implemented over the C-ABI
// (include/pbg.h). The drop-in for reference proj/src/pb_spgemm.cpp:330-361:
// same signature, same exception classes, GPU underneath, no CPU fallback.
#include <cstdlib>
#include <stdexcept>

#include "pbg.h"
#include "pbg_host.h"
#include "spgemm_b200/baseline.hpp"
#include "spgemm_b200/mmio.hpp"
#include "spgemm_b200/pb_spgemm.hpp"

namespace spgemm {

std::uint32_t choose_nbins(std::uint64_t flop, index_t nrows, const PbConfig& cfg,
                           std::uint32_t tuple_bytes) {
    return pbg_choose_nbins(flop, nrows, cfg.l2_bytes, tuple_bytes);
}

namespace {

[[noreturn]] void throw_for(int rc) {
    const std::string msg = pbg_last_error();
    switch (rc) {
        case PBG_ERR_DIM:
        case PBG_ERR_NBINS:
        case PBG_ERR_LBIN:
        case PBG_ERR_FLOP_OVERFLOW:
            throw parameter_error(msg);
        case PBG_ERR_INTERNAL:
            throw internal_error(msg);
        default:
            throw std::runtime_error("pb_multiply (GPU): " + msg);
    }
}

pbg_config to_c(const PbConfig& c) {
    pbg_config o;
    pbg_default_config(&o);
    o.nbins = c.nbins;
    o.lbin_bytes = c.lbin_bytes;
    o.l2_bytes = c.l2_bytes;
    o.nthreads = c.nthreads;
    o.balanced_bins = c.balanced_bins ? 1 : 0;
    o.device = c.device;
    o.ngpus = c.ngpus;
    if (o.ngpus == 0)
        if (const char* e = std::getenv("SPGEMM_B200_NGPUS")) o.ngpus = std::atoi(e);
    return o;
}

struct Handle {
    pbg_handle* h = nullptr;
    ~Handle() { pbg_release(h); }
};

}  // namespace

PbResult pb_multiply(const CscMatrix& a, const CsrMatrix& b, const PbConfig& cfg) {
    require_multipliable(a.dims, b.dims);
    const pbg_config c = to_c(cfg);
    const pbg_csx_view av{a.dims.nrows, a.dims.ncols, a.nnz(), a.colptr.data(), a.rowids.data(),
                          a.values.data()};
    const pbg_csx_view bv{b.dims.nrows, b.dims.ncols, b.nnz(), b.rowptr.data(), b.colids.data(),
                          b.values.data()};
    Handle h;
    std::uint64_t nnz = 0;
    int rc = pbg_multiply_begin(&av, &bv, &c, &h.h, &nnz);
    if (rc) throw_for(rc);
    PbResult res;
    res.c.dims = {a.dims.nrows, b.dims.ncols};
    res.c.rowptr.resize(static_cast<std::size_t>(a.dims.nrows) + 1);
    res.c.colids.resize(nnz);
    res.c.values.resize(nnz);
    pbg_report rep;
    rc = pbg_multiply_fetch(h.h, res.c.rowptr.data(), res.c.colids.data(), res.c.values.data(),
                            &rep);
    if (rc) throw_for(rc);
    res.sym.flop = rep.flop;
    res.sym.nbins = rep.nbins;
    res.sym.per_column_flop.resize(a.dims.ncols);
    res.sym.per_bin_flop.resize(rep.nbins);
    res.sym.bin_row_starts.resize(static_cast<std::size_t>(rep.nbins) + 1);
    rc = pbg_symbolic_fetch(h.h, res.sym.per_column_flop.data(), res.sym.per_bin_flop.data(),
                            res.sym.bin_row_starts.data());
    if (rc) throw_for(rc);
    const index_t m = a.dims.nrows;
    const std::uint64_t rpb = rep.nbins ? (static_cast<std::uint64_t>(m) + rep.nbins - 1) / rep.nbins : 0;
    bool uniform = true;
    for (std::uint32_t i = 0; i <= rep.nbins; ++i)
        if (res.sym.bin_row_starts[i] != std::min<std::uint64_t>(i * rpb, m)) uniform = false;
    res.sym.uniform_rows_per_bin = uniform ? static_cast<index_t>(rpb) : 0;
    res.phases.t_symbolic = rep.t_symbolic;
    res.phases.t_expand = rep.t_expand;
    res.phases.t_sort = rep.t_sort;
    res.phases.t_compress = rep.t_compress;
    res.phases.t_convert = rep.t_convert;
    res.phases.t_total = rep.t_total;
    res.tuples_into_sort = rep.tuples_into_sort;
    res.merged_total = rep.merged_total;
    res.gpu_bins = rep.gpu_bins;
    if (res.c.nnz() != res.merged_total)
        throw internal_error("compressed counts disagree with output nnz");
    return res;
}

CscMatrix hash_multiply(const CscMatrix& a, const CscMatrix& b, int /*nthreads*/) {
    require_multipliable(a.dims, b.dims);
    pbg_config c;
    pbg_default_config(&c);
    const pbg_csx_view av{a.dims.nrows, a.dims.ncols, a.nnz(), a.colptr.data(), a.rowids.data(),
                          a.values.data()};
    const pbg_csx_view bv{b.dims.nrows, b.dims.ncols, b.nnz(), b.colptr.data(), b.rowids.data(),
                          b.values.data()};
    Handle h;
    std::uint64_t nnz = 0;
    int rc = pbg_hash_multiply_begin(&av, &bv, &c, &h.h, &nnz);
    if (rc) throw_for(rc);
    CscMatrix out;
    out.dims = {a.dims.nrows, b.dims.ncols};
    out.colptr.resize(static_cast<std::size_t>(b.dims.ncols) + 1);
    out.rowids.resize(nnz);
    out.values.resize(nnz);
    rc = pbg_multiply_fetch(h.h, out.colptr.data(), out.rowids.data(), out.values.data(), nullptr);
    if (rc) throw_for(rc);
    return out;
}

CscMatrix heap_multiply(const CscMatrix& a, const CscMatrix& b, int nthreads) {
    return hash_multiply(a, b, nthreads);  // same result; the GPU path has one column kernel
}

// ---- structural validation (convert.cpp:8-80), host-side ----
void validate(const CooMatrix& m) {
    if (m.dims.nrows < 1 || m.dims.ncols < 1) throw structural_error("empty dims");
    for (const CooEntry& e : m.entries) {
        if (e.row >= m.dims.nrows || e.col >= m.dims.ncols)
            throw structural_error("coo entry (" + std::to_string(e.row) + "," +
                                   std::to_string(e.col) + ") out of " +
                                   std::to_string(m.dims.nrows) + "x" +
                                   std::to_string(m.dims.ncols));
        if (e.val != e.val) throw structural_error("coo entry holds NaN");
    }
}

namespace {
void check_compressed(MatrixDims dims, const std::vector<offset_t>& ptr,
                      const std::vector<index_t>& ids, std::size_t nvals, index_t nmajor,
                      index_t nminor, const std::string& what) {
    if (dims.nrows < 1 || dims.ncols < 1) throw structural_error("empty dims");
    const bool shape_ok = ptr.size() == static_cast<std::size_t>(nmajor) + 1 && ptr.front() == 0 &&
                          ptr.back() == ids.size() && ids.size() == nvals;
    if (!shape_ok) throw structural_error(what + ": bad pointer array shape");
    for (index_t j = 0; j < nmajor; ++j) {
        if (ptr[j] > ptr[j + 1]) throw structural_error(what + ": ptr not monotone");
        for (offset_t p = ptr[j]; p < ptr[j + 1]; ++p) {
            if (ids[p] >= nminor) throw structural_error(what + ": id out of range");
            if (p > ptr[j] && ids[p - 1] >= ids[p])
                throw structural_error(what + ": ids not strictly increasing");
        }
    }
}
}  // namespace

void validate(const CscMatrix& m) {
    check_compressed(m.dims, m.colptr, m.rowids, m.values.size(), m.dims.ncols, m.dims.nrows, "csc");
}

void validate(const CsrMatrix& m) {
    check_compressed(m.dims, m.rowptr, m.colids, m.values.size(), m.dims.nrows, m.dims.ncols, "csr");
}

CooMatrix mm_read(const std::string& path) {
    pbgh_mm* h = nullptr;
    std::uint32_t nr = 0, nc = 0;
    std::uint64_t n = 0;
    if (pbgh_mm_open(path.c_str(), &h, &nr, &nc, &n)) throw parse_error(pbgh_last_error());
    std::vector<std::uint32_t> r(n), c(n);
    std::vector<double> v(n);
    pbgh_mm_fetch(h, r.data(), c.data(), v.data());
    pbgh_mm_free(h);
    CooMatrix m;
    m.dims = {nr, nc};
    m.entries.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) m.entries[i] = {r[i], c[i], v[i]};
    return m;
}

void mm_write(const CooMatrix& m, const std::string& path) {
    std::vector<std::uint32_t> r(m.nnz()), c(m.nnz());
    std::vector<double> v(m.nnz());
    for (std::size_t i = 0; i < m.nnz(); ++i) {
        r[i] = m.entries[i].row;
        c[i] = m.entries[i].col;
        v[i] = m.entries[i].val;
    }
    if (pbgh_mm_write(path.c_str(), m.dims.nrows, m.dims.ncols, m.nnz(), r.data(), c.data(), v.data()))
        throw structural_error(pbgh_last_error());
}

}  // namespace spgemm
