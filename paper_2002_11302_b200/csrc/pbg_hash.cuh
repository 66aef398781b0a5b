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
// HASH_BIG_F products use the large-table kernel; hub columns beyond that
// (RMAT) a dense per-CTA accumulator in global memory (k_hash_hub).
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
    unsigned int* err;      // reserved (no error is raised by the column kernels)
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
            sm.val[s] = -0.0;  // the additive identity: a lone -0.0 product keeps its sign
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

// Short columns, one WARP per column (no block barriers): a TW-slot table
// per warp in shared memory; products flattened over the warp (a B chunk's
// A-column lengths are scanned across lanes, each lane finds its product's
// B entry by a shuffle search); in-place compaction of the occupied slots
// in slot order (a warp's chunk is read before any write lands at or below
// it); a bitonic network in the table's front; then the scratch range.
template <int TW, int NWARP>
struct HashWarpSmem {
    uint32_t key[NWARP][TW];
    double val[NWARP][TW];
};

template <int TW, int NWARP>
__global__ void __launch_bounds__(NWARP * 32) k_hash_warp(HashArgs a, uint64_t lo_f, uint64_t hi_f) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& sm = *reinterpret_cast<HashWarpSmem<TW, NWARP>*>(smem_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* K = sm.key[w];
    double* V = sm.val[w];
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * NWARP + w;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * NWARP;
    for (uint64_t j = gw; j < a.ncols; j += nwarps) {
        const uint64_t f = a.flop[j];
        if (f <= lo_f || f > hi_f) continue;
        uint32_t T = 32;
        while (T < f + 1) T <<= 1;
        for (uint32_t s2 = lane; s2 < T; s2 += 32) {
            K[s2] = HASH_EMPTY;
            V[s2] = -0.0;  // as k_hash_cols / k_hash_hub
        }
        __syncwarp();
        // ---- products, 32 B entries per chunk, flattened over the lanes
        const uint64_t b0 = a.b_colptr[j], b1 = a.b_colptr[j + 1];
        for (uint64_t c0 = b0; c0 < b1; c0 += 32) {
            const uint64_t p = c0 + lane;
            uint64_t qs = 0;
            uint32_t len = 0;
            double bv = 0.0;
            if (p < b1) {
                const uint32_t i = a.b_rowids[p];
                bv = a.b_vals[p];
                qs = a.a_colptr[i];
                len = static_cast<uint32_t>(a.a_colptr[i + 1] - qs);
            }
            const uint32_t incl = warp_inclusive_scan(len);
            const uint32_t tot = __shfl_sync(FULL, incl, 31);
            const uint32_t excl = incl - len;
            for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
                const uint32_t t = t0 + lane;
                // owner: the number of lanes whose inclusive prefix is <= t
                int lo = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const uint32_t v = __shfl_sync(FULL, incl, lo + st - 1);
                    if (v <= t) lo += st;
                }
                const uint64_t oqs = __shfl_sync(FULL, qs, lo);
                const double obv = __shfl_sync(FULL, bv, lo);
                const uint32_t oex = __shfl_sync(FULL, excl, lo);
                if (t < tot) {
                    const uint64_t q = oqs + (t - oex);
                    const uint32_t r = a.a_rowids[q];
                    const double v = a.a_vals[q] * obv;
                    uint32_t h = static_cast<uint32_t>((r * 0x9E3779B97F4A7C15ull) >> 32) & (T - 1);
                    while (true) {
                        const uint32_t old = atomicCAS(&K[h], HASH_EMPTY, r);
                        if (old == HASH_EMPTY || old == r) {
                            atomicAdd(&V[h], v);
                            break;
                        }
                        h = (h + 1) & (T - 1);
                    }
                }
            }
        }
        __syncwarp();
        // ---- in-place compaction in slot order
        uint32_t m = 0;
        for (uint32_t s0 = 0; s0 < T; s0 += 32) {
            const uint32_t s2 = s0 + lane;
            const uint32_t k = K[s2];
            const double v = V[s2];
            const bool occ = k != HASH_EMPTY;
            const uint32_t bal = __ballot_sync(FULL, occ);
            __syncwarp();
            if (occ) {
                const uint32_t o = m + __popc(bal & lanemask_lt());
                K[o] = k;
                V[o] = v;
            }
            m += __popc(bal);
            __syncwarp();
        }
        // ---- bitonic sort of K/V[0, P), P = bit_ceil(m), padded with EMPTY
        uint32_t P = 1;
        while (P < m) P <<= 1;
        for (uint32_t e = m + lane; e < P; e += 32) K[e] = HASH_EMPTY;
        __syncwarp();
        for (uint32_t k2 = 2; k2 <= P; k2 <<= 1) {
            for (uint32_t jj = k2 >> 1; jj > 0; jj >>= 1) {
                for (uint32_t e0 = 0; e0 < P / 2; e0 += 32) {
                    const uint32_t c = e0 + lane;  // compare-exchange index
                    if (c < P / 2) {
                        const uint32_t e = 2 * c - (c & (jj - 1));  // lower element of the pair
                        const uint32_t x = e + jj;
                        const bool up = (e & k2) == 0;
                        const uint32_t ke = K[e], kx = K[x];
                        if ((ke > kx) == up) {
                            K[e] = kx;
                            K[x] = ke;
                            const double t2 = V[e];
                            V[e] = V[x];
                            V[x] = t2;
                        }
                    }
                }
                __syncwarp();
            }
        }
        const uint64_t base = a.bound[j];
        for (uint32_t e = lane; e < m; e += 32) {
            a.s_rows[base + e] = K[e];
            a.s_vals[base + e] = V[e];
        }
        if (lane == 0) a.count[j] = m;
        __syncwarp();
    }
}

// Hub columns (f_j > HASH_BIG_F: RMAT hubs, more products than a shared-memory
// table holds). Each CTA owns a dense accumulator in global memory — nrows f64
// sums and a presence bitmap (exact-zero sums kept, as the reference's table
// keeps them) — and walks the hub columns j = blockIdx.x, +gridDim.x, ...
// One warp per B(i, j) entry, lanes over A(:, i): the products are added with
// native f64 L2 atomics and their rows marked with atomicOr. Walking the
// bitmap in word order (block scan of the popcounts) yields the column's rows
// already sorted, so no sort follows; the walk resets the touched sums and
// words for the next column. The sums start at -0.0, the exact additive
// identity, so a single product keeps its sign as in the reference's
// first-insert. The order of the f64 additions is not the reference's (its
// table visits products in B-entry order), so values agree within rounding.
template <int NT>
__global__ void __launch_bounds__(NT) k_hash_hub(HashArgs a, uint64_t lo_f, uint32_t nrows,
                                                 double* __restrict__ dense,
                                                 uint32_t* __restrict__ bits) {
    __shared__ uint32_t s_warp[NT / 32 + 1];
    // 64-bit word / row arithmetic: nrows up to 2^32 - 1 (the host sizes the
    // bitmap with the same 64-bit count)
    const uint64_t nw = (uint64_t(nrows) + 31) / 32;
    double* dv = dense + uint64_t(blockIdx.x) * nrows;
    uint32_t* bm = bits + uint64_t(blockIdx.x) * nw;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (uint64_t r = threadIdx.x; r < nrows; r += NT) dv[r] = -0.0;
    for (uint64_t w = threadIdx.x; w < nw; w += NT) bm[w] = 0u;
    __syncthreads();
    for (uint64_t j = blockIdx.x; j < a.ncols; j += gridDim.x) {
        if (a.flop[j] <= lo_f) continue;  // uniform over the CTA
        const uint64_t b1 = a.b_colptr[j + 1];
        for (uint64_t p = a.b_colptr[j] + wp; p < b1; p += NT / 32) {
            const uint32_t i = a.b_rowids[p];
            const double bv = a.b_vals[p];
            const uint64_t q1 = a.a_colptr[i + 1];
            for (uint64_t q = a.a_colptr[i] + lane; q < q1; q += 32) {
                const uint32_t r = a.a_rowids[q];
                atomicAdd(&dv[r], a.a_vals[q] * bv);
                atomicOr(&bm[r >> 5], 1u << (r & 31));
            }
        }
        __syncthreads();
        const uint64_t base = a.bound[j];
        uint32_t done = 0;
        for (uint64_t w0 = 0; w0 < nw; w0 += NT) {
            const uint64_t w = w0 + threadIdx.x;
            const uint32_t word = w < nw ? __ldcg(bm + w) : 0u;
            uint32_t tot;
            uint32_t k = done + block_exclusive_scan<NT>(uint32_t(__popc(word)), s_warp, tot);
            for (uint32_t x = word; x; x &= x - 1) {
                const uint32_t r = static_cast<uint32_t>(w * 32 + (__ffs(x) - 1));
                a.s_rows[base + k] = r;
                a.s_vals[base + k] = __ldcg(dv + r);
                dv[r] = -0.0;
                ++k;
            }
            if (word) bm[w] = 0u;
            done += tot;
        }
        if (threadIdx.x == 0) a.count[j] = done;
        __syncthreads();
    }
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
