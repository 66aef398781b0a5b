// pbg_hash.cuh — column hash SpGEMM: the reference's
// spgemm::hash_multiply (proj/src/baseline.cpp:141-200, baseline.hpp:21-24),
// C = A·B with A, B and C in CSC, on the GPU.
//
// The paper compares PB-SpGEMM against this column (Gustavson) algorithm and
// finds hashing wins above a compression factor of ~4: the
// duplicates are summed as they are produced instead of being written out,
// re-read and sorted. Per output column j (column_symbolic, baseline.cpp:
// 73-85, gives its product count f_j and its scratch range):
//   * the products A(:, i)·B(i, j) for every B(i, j) are accumulated in a
//     shared-memory open-addressing table keyed by row id (linear probing,
//     bit_ceil(f_j + 1) slots, exact zeros kept);
//   * the occupied slots are compacted, sorted by row id (rank counting for
//     short columns, a bitonic network otherwise) and written to the column's
//     scratch range at bound_start[j] (ScratchOutput, baseline.cpp:16-50);
//   * a scan of the per-column counts and a copy kernel give the tight CSC.
// One CTA per column; each CTA walks columns in order, so consecutive
// columns' A columns (banded matrices) come from L2. Columns up to
// HASH_BIG_F products use the large-table kernel; beyond that the path
// reports PBG_ERR_UNIMPLEMENTED (RMAT hub columns: use pb_multiply).
#pragma once

#include <cstdint>

#include "pbg_device.cuh"

namespace pbg {

constexpr uint32_t HASH_EMPTY = 0xffffffffu;
constexpr uint64_t HASH_SMALL_F = 1024;  // small kernel: 128 threads, 2048-slot table
constexpr uint64_t HASH_BIG_F = 4096;    // large kernel: 512 threads, 8192-slot table

// f_j = sum over B(i, j) of nnz(A(:, i))   (column_symbolic, baseline.cpp:73-85)
__global__ void k_hash_colflop(const uint64_t* __restrict__ a_colptr,
                               const uint64_t* __restrict__ b_colptr,
                               const uint32_t* __restrict__ b_rowids, uint64_t ncols,
                               uint64_t* __restrict__ flop) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= ncols) return;
    uint64_t f = 0;
    for (uint64_t p = b_colptr[j]; p < b_colptr[j + 1]; ++p) {
        const uint32_t i = b_rowids[p];
        f += a_colptr[i + 1] - a_colptr[i];
    }
    flop[j] = f;
}

struct HashArgs {
    const uint64_t* a_colptr;
    const uint32_t* a_rowids;
    const double* a_vals;
    const uint64_t* b_colptr;
    const uint32_t* b_rowids;
    const double* b_vals;
    uint64_t ncols;
    const uint64_t* flop;   // per column
    const uint64_t* bound;  // scratch start per column (scan of flop)
    uint32_t* s_rows;       // scratch output (flop-bound sized)
    double* s_vals;
    uint64_t* count;        // merged entries per column
    unsigned int* err;      // bit0: a column above HASH_BIG_F
};

template <int NT, int TMAX, int MMAX>
struct HashSmem {
    uint32_t key[TMAX];
    double val[TMAX];
    uint32_t skey[MMAX];
    double sval[MMAX];
    uint32_t warp[NT / 32 + 1];
};

// One column per iteration, columns with flop in (lo_f, hi_f].
template <int NT, int TMAX, int MMAX>
__global__ void __launch_bounds__(NT) k_hash_cols(HashArgs a, uint64_t lo_f, uint64_t hi_f) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& sm = *reinterpret_cast<HashSmem<NT, TMAX, MMAX>*>(smem_raw);
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (uint64_t j = blockIdx.x; j < a.ncols; j += gridDim.x) {
        const uint64_t f = a.flop[j];
        if (f <= lo_f || f > hi_f) continue;
        // bit_ceil(f + 1) slots: the distinct row ids never exceed f, so the
        // table cannot fill; half the reference's bit_ceil(2 f) halves the
        // clear and compaction scans (C4 42 -> 34 ms; C2 22 -> 24 ms)
#ifdef PBG_HASH_LOAD2
        uint32_t T = 32;
        while (T < 2 * f) T <<= 1;
#else
        uint32_t T = 32;
        while (T < f + 1) T <<= 1;
#endif
        for (uint32_t s = tid; s < T; s += NT) {
            sm.key[s] = HASH_EMPTY;
            sm.val[s] = 0.0;
        }
        __syncthreads();
        // ---- accumulate: warp w takes B entries w, w + NW, ...; lanes walk A(:, i)
        const uint64_t b0 = a.b_colptr[j], b1 = a.b_colptr[j + 1];
        for (uint64_t p = b0 + w; p < b1; p += NW) {
            const uint32_t i = a.b_rowids[p];
            const double bv = a.b_vals[p];
            const uint64_t q1 = a.a_colptr[i + 1];
            for (uint64_t q = a.a_colptr[i] + lane; q < q1; q += 32) {
                const uint32_t r = a.a_rowids[q];
                const double v = a.a_vals[q] * bv;
                uint32_t h = static_cast<uint32_t>((r * 0x9E3779B97F4A7C15ull) >> 32) & (T - 1);
                while (true) {
                    const uint32_t old = atomicCAS(&sm.key[h], HASH_EMPTY, r);
                    if (old == HASH_EMPTY || old == r) {
                        atomicAdd(&sm.val[h], v);
                        break;
                    }
                    h = (h + 1) & (T - 1);
                }
            }
        }
        __syncthreads();
        // ---- compact the occupied slots (slot order) into skey/sval
        constexpr int SPT = TMAX / NT;
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < SPT; ++q) {
            const uint32_t s = tid * SPT + q;
            c += s < T && sm.key[s] != HASH_EMPTY;
        }
        uint32_t m;
        uint32_t o = block_exclusive_scan<NT>(c, sm.warp, m);
#pragma unroll
        for (int q = 0; q < SPT; ++q) {
            const uint32_t s = tid * SPT + q;
            if (s < T && sm.key[s] != HASH_EMPTY) {
                sm.skey[o] = sm.key[s];
                sm.sval[o] = sm.val[s];
                ++o;
            }
        }
        __syncthreads();
        // ---- sort the m distinct row ids
        const uint32_t* ok;
        const double* ov;
        if (m <= 2 * NT) {
            // rank = number of smaller row ids (all distinct); result in key/val
            for (uint32_t e = tid; e < m; e += NT) {
                const uint32_t k = sm.skey[e];
                uint32_t r = 0;
                for (uint32_t t = 0; t < m; ++t) r += sm.skey[t] < k;
                sm.key[r] = k;
                sm.val[r] = sm.sval[e];
            }
            ok = sm.key;
            ov = sm.val;
        } else {
            // bitonic network on the next power of two, padded with HASH_EMPTY
            uint32_t P = 1;
            while (P < m) P <<= 1;
            for (uint32_t e = m + tid; e < P; e += NT) sm.skey[e] = HASH_EMPTY;
            __syncthreads();
            for (uint32_t k = 2; k <= P; k <<= 1) {
                for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
                    for (uint32_t e = tid; e < P; e += NT) {
                        const uint32_t x = e ^ jj;
                        if (x > e) {
                            const bool up = (e & k) == 0;
                            const uint32_t ke = sm.skey[e], kx = sm.skey[x];
                            if ((ke > kx) == up) {
                                sm.skey[e] = kx;
                                sm.skey[x] = ke;
                                const double t2 = sm.sval[e];
                                sm.sval[e] = sm.sval[x];
                                sm.sval[x] = t2;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            ok = sm.skey;
            ov = sm.sval;
        }
        __syncthreads();
        // ---- the column's scratch range (baseline.cpp:186-197)
        const uint64_t base = a.bound[j];
        for (uint32_t e = tid; e < m; e += NT) {
            a.s_rows[base + e] = ok[e];
            a.s_vals[base + e] = ov[e];
        }
        if (tid == 0) a.count[j] = m;
        __syncthreads();
    }
    (void)lane;
}

// Columns above the large-table capacity: flag them (the host reports
// PBG_ERR_UNIMPLEMENTED).
__global__ void k_hash_check(const uint64_t* __restrict__ flop, uint64_t ncols, uint64_t hi_f,
                             unsigned int* err) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < ncols && flop[j] > hi_f) atomicOr(err, 1u);
}

// Tight CSC from the scratch ranges (ScratchOutput::compact, baseline.cpp:
// 34-50): one warp per column.
__global__ void k_hash_compact(const uint64_t* __restrict__ bound,
                               const uint64_t* __restrict__ colptr, uint64_t ncols,
                               const uint32_t* __restrict__ s_rows,
                               const double* __restrict__ s_vals, uint32_t* __restrict__ rows,
                               double* __restrict__ vals) {
    const uint64_t wgl = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wgl >= ncols) return;
    const uint64_t src = bound[wgl], dst = colptr[wgl], n = colptr[wgl + 1] - dst;
    for (uint64_t e = lane; e < n; e += 32) {
        rows[dst + e] = s_rows[src + e];
        vals[dst + e] = s_vals[src + e];
    }
}

}  // namespace pbg
