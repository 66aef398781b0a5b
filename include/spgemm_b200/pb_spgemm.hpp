// spgemm_b200/pb_spgemm.hpp — drop-in declaration of the PB-SpGEMM entry
// point, implemented on the B200 by libspgemm_b200 over the C-ABI in pbg.h.
//
// Mirrors proj/include/spgemm/pb_spgemm.hpp: PbConfig (:11-17), the key
// helpers (:20-41), choose_nbins (:45-46), SymbolicResult (:48-55), PbResult
// and pb_multiply (:110-116); PhaseReport / WallTimer come from
// spgemm_b200/report.hpp (proj/include/spgemm/report.hpp:9-52). The reference's stepwise API (symbolic/make_bins/expand/
// sort_bins/compress_bins/convert_csr) exposes host BinSet internals and is
// not offered; the GPU returns its conservation counters in PbResult instead.
#pragma once

#include <bit>
#include <cstdint>

#include "spgemm_b200/report.hpp"
#include "spgemm_b200/types.hpp"

namespace spgemm {

struct PbConfig {
    std::uint32_t nbins = 0;         // 0 = auto; otherwise a power of two
    std::uint32_t lbin_bytes = 512;  // validated: positive multiple of 16
    std::uint64_t l2_bytes = 1 << 20;
    int nthreads = 0;                // no meaning on the GPU
    bool balanced_bins = false;
    // B200 extension (after the reference's fields, so the reference's
    // aggregate initialisations still compile): devices to split C's rows
    // over as flop-balanced bands (pbg_config.ngpus; 0 = the
    // SPGEMM_B200_NGPUS environment variable, else one; -1 = every visible
    // device), and the first device (-1 = the current one).
    int ngpus = 0;
    int device = -1;
};

inline int ceil_log2(std::uint64_t x) { return x <= 1 ? 0 : std::bit_width(x - 1); }

inline int choose_key_width(index_t max_bin_rows, index_t ncols) {
    return ceil_log2(max_bin_rows) + ceil_log2(ncols) <= 32 ? 32 : 64;
}

inline std::uint64_t pack_key(index_t rowid, index_t colid, index_t bin_base, int col_bits) {
    return (static_cast<std::uint64_t>(rowid - bin_base) << col_bits) | colid;
}

struct RowCol {
    index_t row;
    index_t col;
};

inline RowCol unpack_key(std::uint64_t key, index_t bin_base, int col_bits) {
    return {static_cast<index_t>(bin_base + (key >> col_bits)),
            static_cast<index_t>(key & ((std::uint64_t{1} << col_bits) - 1))};
}

std::uint32_t choose_nbins(std::uint64_t flop, index_t nrows, const PbConfig& cfg,
                           std::uint32_t tuple_bytes = 12);

// The reference-layout symbolic result (uniform or balanced row ranges as the
// CPU would choose them); the GPU's own shared-memory bins are reported in
// PbResult::gpu_bins.
struct SymbolicResult {
    std::uint64_t flop = 0;
    std::vector<std::uint64_t> per_column_flop;
    std::uint32_t nbins = 1;
    std::vector<std::uint64_t> per_bin_flop;
    std::vector<index_t> bin_row_starts;
    index_t uniform_rows_per_bin = 0;
};

struct PbResult {
    CsrMatrix c;
    SymbolicResult sym;
    PhaseReport phases;
    // GPU counters (acceptance.cpp:46-58 reads the same two from BinSet)
    std::uint64_t tuples_into_sort = 0;
    std::uint64_t merged_total = 0;
    std::uint32_t gpu_bins = 0;
};

// C = A * B on the GPU. Throws parameter_error / internal_error exactly where
// the reference does, std::runtime_error on CUDA failures or no device.
PbResult pb_multiply(const CscMatrix& a, const CsrMatrix& b, const PbConfig& cfg = {});

}  // namespace spgemm
