// pbg_bands.cuh — output row bands on the device.
//
// C(r0:r1, :) = A(r0:r1, :) · B, so a flop-balanced row band of A is a unit
// of work that needs nothing from the other bands: the multi-GPU split (one
// band per device) and the bounded-memory rounds (bands one after another
// on a device) are both built from the kernels here, with no host pass over
// the matrices.
//
//   k_cut_search  flop-balanced cuts from the row-flop prefix of symbolic
//                 (the rule of the reference's balanced_starts,
//                 pb_spgemm.cpp:58-82: cut j sits after the first row whose
//                 inclusive flop prefix reaches j/G of the total)
//   k_slab_bits / k_slab_colptr / k_slab_gather
//                 the CSC row slab A(r0:r1, :) with rows renumbered from 0
//                 (stable; entry-parallel: one selection bit per entry, a
//                 scan over the words' popcounts, column pointers by lookup)
//   k_csr_checksum
//                 nnz, row-count and column-id hashes and the value sum of a
//                 CSR band: the checksum-and-discard mode of products whose C
//                 does not fit anywhere (C5b), and a cheap band identity check
//   k_add_base    rowptr of a band shifted to its place in the global CSR
#pragma once

#include <cstdint>

#include "pbg_device.cuh"

namespace pbg {

// Cuts of the rows [lo, hi) into g flop-balanced bands: cuts[0] = lo,
// cuts[g] = hi, and for 0 < j < g the smallest t in (lo, hi] with
// (row_off[t] - row_off[lo]) * g >= (row_off[hi] - row_off[lo]) * j, i.e. the
// row after the first one whose inclusive flop prefix reaches j/g of the
// range (row_off = exclusive row-flop prefix). 128-bit products: exact.
// off[j] = row_off[cuts[j]] (the flop prefix at every cut).
__global__ void k_cut_search(const uint64_t* __restrict__ row_off, uint32_t lo, uint32_t hi,
                             uint32_t g, uint32_t* cuts, uint64_t* off) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > g) return;
    uint32_t c;
    if (j == 0 || lo == hi) {
        c = j == g ? hi : lo;
    } else if (j == g) {
        c = hi;
    } else {
        const uint64_t base = row_off[lo];
        const unsigned __int128 target = static_cast<unsigned __int128>(row_off[hi] - base) * j;
        uint64_t a = uint64_t(lo) + 1, b = hi;
        while (a < b) {
            const uint64_t mid = a + (b - a) / 2;
            if (static_cast<unsigned __int128>(row_off[mid] - base) * g >= target) b = mid;
            else a = mid + 1;
        }
        c = static_cast<uint32_t>(a);
    }
    cuts[j] = c;
    off[j] = row_off[c];
}

// Per-column flop nnz(A(:, i)) * nnz(B(i, :)) (the reference's
// per_column_flop, pb_spgemm.cpp:93-101).
__global__ void k_colflop_each(const uint64_t* __restrict__ a_colptr,
                               const uint64_t* __restrict__ b_rowptr, uint64_t k, uint64_t* out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < k) out[i] = (a_colptr[i + 1] - a_colptr[i]) * (b_rowptr[i + 1] - b_rowptr[i]);
}

// The reference's uniform bin layout (pb_spgemm.cpp:107-137: nbins ranges
// of ceil(m / nbins) rows) from the row-flop prefix the symbolic phase keeps
// on the device: starts[b] = min(b * rpb, m), per_bin_flop[b] = prefix
// difference. Replaces a host pass over all m row counters per report.
__global__ void k_ref_layout_uniform(const uint64_t* __restrict__ row_off, uint64_t m, uint32_t nb,
                                     uint64_t rpb, uint32_t* starts, uint64_t* pbf) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b > nb) return;
    const uint64_t s = b * rpb < m ? b * rpb : m;
    starts[b] = static_cast<uint32_t>(s);
    if (b < nb) {
        const uint64_t e = (b + 1) * rpb < m ? (b + 1) * rpb : m;
        pbf[b] = row_off[e] - row_off[s];
    }
}

// ---- CSC row slab A(r0:r1, :) on the device, entry-parallel ---------------
// One bit per entry of A (row in [r0, r1)?), one word per 32 entries; a scan
// of the words' popcounts gives every word's position in the slab, so the
// slab's column pointers are a lookup per column (prefix of the word holding
// colptr[j] + the bits below it) and the selected entries are gathered in
// order (stable) with coalesced loads. (The first version walked each column
// with one thread — a warp for long columns — in both a counting and a copying
// kernel: 12.3 ms per round at C5b's 1.3e8 entries, 12 % of every round;
// this one reads the row ids once.)
__global__ void k_slab_bits(const uint32_t* __restrict__ a_rowids, uint64_t nnz, uint32_t r0,
                            uint32_t r1, uint32_t* bits, uint32_t* wcnt) {
    // a warp takes 32 words (1024 entries) per trip: lane i keeps the ballot of
    // the trip's i-th word, so the words leave as coalesced 128-byte stores
    const int lane = threadIdx.x & 31;
    const uint64_t nwords = (nnz + 31) >> 5;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w0 = warp * 32; w0 < nwords; w0 += nwarps * 32) {
        uint32_t mine = 0;
        for (int i = 0; i < 32; ++i) {
            const uint64_t p = (w0 + i) * 32 + lane;
            bool in = false;
            if (p < nnz) {
                const uint32_t r = __ldcs(a_rowids + p);
                in = r >= r0 && r < r1;
            }
            const uint32_t b = __ballot_sync(FULL, in);
            if (lane == i) mine = b;
        }
        if (w0 + lane < nwords) {
            bits[w0 + lane] = mine;
            wcnt[w0 + lane] = __popc(mine);
        }
    }
}

// s_colptr[j] = selected entries before entry a_colptr[j] (j = 0 .. k)
__global__ void k_slab_colptr(const uint64_t* __restrict__ a_colptr, uint64_t k, uint64_t nnz,
                              const uint32_t* __restrict__ bits, const uint64_t* __restrict__ wpre,
                              uint64_t* s_colptr) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j > k) return;
    const uint64_t p = a_colptr[j];
    const uint64_t nwords = (nnz + 31) >> 5;
    if (p >= nnz) {
        s_colptr[j] = wpre[nwords];
        return;
    }
    const uint32_t below = bits[p >> 5] & ((1u << (p & 31u)) - 1u);
    s_colptr[j] = wpre[p >> 5] + __popc(below);
}

// the slab's rowids (renumbered, r - r0) and values, in A's order
__global__ void k_slab_gather(const uint32_t* __restrict__ a_rowids, const double* __restrict__ a_vals,
                              uint64_t nnz, uint32_t r0, const uint32_t* __restrict__ bits,
                              const uint64_t* __restrict__ wpre, uint32_t* s_rowids, double* s_vals) {
    const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    const uint32_t b = bits[p >> 5];
    const int lane = threadIdx.x & 31;
    if ((b >> lane) & 1u) {
        const uint64_t at = wpre[p >> 5] + __popc(b & lanemask_lt());
        s_rowids[at] = a_rowids[p] - r0;
        s_vals[at] = a_vals[p];
    }
}

// Band checksum: out[0] += nnz, out[1] += sum over rows of (row count x
// row hash), out[2] += sum of the mixed (row, col) words — sums, so the
// checksums of the bands of a product add up to the product's; *vsum += the
// value sum (f64 atomics: an identity check within rounding, not exact).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_csr_checksum(const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ colids,
                               const double* __restrict__ vals, uint64_t m, uint64_t row_base,
                               unsigned long long* out, double* vsum) {
    uint64_t h_rows = 0, h_cols = 0;
    double vs = 0.0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < m;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p0 = rowptr[r], p1 = rowptr[r + 1];
        h_rows += (p1 - p0) * mix64(row_base + r + 1);
        for (uint64_t p = p0; p < p1; ++p) {
            h_cols += mix64((static_cast<uint64_t>(row_base + r) << 32) | colids[p]);
            vs += vals[p];
        }
    }
    h_rows = warp_sum(h_rows);
    h_cols = warp_sum(h_cols);
    vs = warp_sum(vs);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[1], static_cast<unsigned long long>(h_rows));
        atomicAdd(&out[2], static_cast<unsigned long long>(h_cols));
        atomicAdd(vsum, vs);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&out[0], static_cast<unsigned long long>(rowptr[m] - rowptr[0]));
}

__global__ void k_add_base(uint64_t* __restrict__ p, uint64_t n, uint64_t base) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] += base;
}

}  // namespace pbg
