// pbg_kernels.cuh — the sm_100a kernels of the PB-SpGEMM hot path.
//
//   symbolic  : k_colflop_total, k_scan<ColFlop>, k_rowflop, k_scan<RowFlop>,
//               k_binflags, k_scan<Flags>, k_binrows, k_binsizes, k_scan<Pad>
//               (reference symbolic + make_bins, pb_spgemm.cpp:86-176)
//   expand    : k_chunks, k_expand           (expand_impl, pb_spgemm.cpp:180-246)
//   sort/merge: k_sortmerge — per-bin smem radix sort, duplicate merge, CSR
//               rows written at look-back offsets (sort_bins + compress_bins +
//               convert_csr, pb_spgemm.cpp:260-328, pb_spgemm.hpp:118-216)
//
// Tuple layout (the reference BinSet's keys32 + values SoA, pb_spgemm.hpp:
// 84-86): key = (row - bin_row_start) << col_bits | col as u32, value f64.
// GPU bins are contiguous row ranges sized to one CTA's shared memory.
#pragma once

#include <cstdint>

#include "pbg_device.cuh"

namespace pbg {

// ---------------------------------------------------------------- scans --
constexpr int SCAN_NT = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_NT * SCAN_ITEMS;

// Exclusive scan out[0..n) of in(i), out[n] = total, single pass with
// decoupled look-back. n may live in device memory (n_dev) when the host does
// not know it; tiles at or beyond n exit. Optional max of the inputs.
template <class In>
__global__ void __launch_bounds__(SCAN_NT)
k_scan(In in, uint64_t* out, uint64_t n_host, const uint64_t* n_dev, unsigned long long* status,
       unsigned int* ticket, unsigned long long* total_out, unsigned long long* max_out) {
    __shared__ uint64_t s_items[SCAN_TILE];
    __shared__ uint64_t s_warp[SCAN_NT / 32 + 1];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_prefix;
    const int tid = threadIdx.x;
    const uint64_t n = n_dev ? *n_dev : n_host;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * SCAN_TILE;
    if (base >= n && !(base == 0)) return;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const uint64_t i = base + j * SCAN_NT + tid;
        s_items[j * SCAN_NT + tid] = i < n ? in(i) : 0;
    }
    __syncthreads();
    uint64_t loc[SCAN_ITEMS];
    uint64_t sum = 0, mx = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        loc[j] = s_items[tid * SCAN_ITEMS + j];
        sum += loc[j];
        mx = loc[j] > mx ? loc[j] : mx;
    }
    uint64_t total;
    const uint64_t excl = block_exclusive_scan<SCAN_NT>(sum, s_warp, total);
    if (tid < 32) {
        const uint64_t p = lookback_warp(status, tile, total);
        if (tid == 0) s_prefix = p;
    }
    if (max_out) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(FULL, mx, o);
            mx = y > mx ? y : mx;
        }
        if ((tid & 31) == 0) atomicMax(max_out, static_cast<unsigned long long>(mx));
    }
    __syncthreads();
    uint64_t run = s_prefix + excl;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        s_items[tid * SCAN_ITEMS + j] = run;
        run += loc[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const uint64_t i = base + j * SCAN_NT + tid;
        if (i < n) out[i] = s_items[j * SCAN_NT + tid];
    }
    if (base + SCAN_TILE >= n && tid == 0) {
        out[n] = s_prefix + total;
        if (total_out) *total_out = s_prefix + total;
    }
}

// per_column_flop[i] = nnz(A(:,i)) * nnz(B(i,:))   (pb_spgemm.cpp:98-101)
struct ColFlopIn {
    const uint64_t* a_colptr;
    const uint64_t* b_rowptr;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        return (a_colptr[i + 1] - a_colptr[i]) * (b_rowptr[i + 1] - b_rowptr[i]);
    }
};

// 1 for a bin above the shared-memory capacity (heavy row), else 0
struct HeavyFlagIn {
    const uint64_t* bin_cnt;
    uint64_t cap;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        return bin_cnt[i] > cap ? 1u : 0u;
    }
};

// padded tuple count of a heavy bin (its scratch size), 0 for other bins
struct HeavyPadIn {
    const uint64_t* bin_cnt;
    uint64_t cap;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        const uint64_t n = bin_cnt[i];
        return n > cap ? ((n + 3) & ~3ull) : 0u;
    }
};

struct ArrayIn {
    const uint64_t* a;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};
struct ArrayIn32 {
    const uint32_t* a;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return a[i]; }
};

// 128-bit accumulation of the per-column flop so an overflow of the 64-bit
// total is detected exactly (pb_spgemm.cpp:103-105). also rejects totals the
// 62-bit look-back cannot carry.
__global__ void k_colflop_total(const uint64_t* __restrict__ a_colptr,
                                const uint64_t* __restrict__ b_rowptr, uint64_t k,
                                unsigned long long* lo_out, unsigned long long* hi_out) {
    uint64_t lo = 0, hi = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t la = a_colptr[i + 1] - a_colptr[i];
        const uint64_t lb = b_rowptr[i + 1] - b_rowptr[i];
        const uint64_t f = la * lb;
        hi += __umul64hi(la, lb);
        const uint64_t s = lo + f;
        hi += s < lo;
        lo = s;
    }
    // warp reduce lo with carries
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t olo = __shfl_xor_sync(FULL, lo, o);
        const uint64_t ohi = __shfl_xor_sync(FULL, hi, o);
        const uint64_t s = lo + olo;
        hi += ohi + (s < lo);
        lo = s;
    }
    if ((threadIdx.x & 31) == 0) {
        const unsigned long long old = atomicAdd(lo_out, static_cast<unsigned long long>(lo));
        if (old + lo < old) hi += 1;
        if (hi) atomicAdd(hi_out, static_cast<unsigned long long>(hi));
    }
}

// row_flop[r] += nnz(B(k,:)) for every A(r,k)  (bin_flop / balanced_starts,
// pb_spgemm.cpp:36-82, at row granularity). Thread per column; long columns
// are walked by the whole warp. Counters are 32-bit whenever nnz(B) < 2^32
// (a row's flop never exceeds nnz(B)): half the scattered-RED footprint, so
// the m counters stay L2-resident for larger m.
template <typename T>
__global__ void k_rowflop(const uint64_t* __restrict__ a_colptr,
                          const uint32_t* __restrict__ a_rowids,
                          const uint64_t* __restrict__ b_rowptr, uint64_t k,
                          T* row_flop) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint64_t p0 = 0, p1 = 0, lb = 0;
    if (i < k) {
        lb = b_rowptr[i + 1] - b_rowptr[i];
        if (lb) {
            p0 = a_colptr[i];
            p1 = a_colptr[i + 1];
        }
    }
    const bool longcol = (p1 - p0) > 64;
    if (!longcol)
        for (uint64_t p = p0; p < p1; ++p) atomicAdd(&row_flop[a_rowids[p]], static_cast<T>(lb));
    uint32_t lm = __ballot_sync(FULL, longcol);
    while (lm) {
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint64_t q0 = __shfl_sync(FULL, p0, src), q1 = __shfl_sync(FULL, p1, src);
        const uint64_t qb = __shfl_sync(FULL, lb, src);
        for (uint64_t p = q0 + lane; p < q1; p += 32)
            atomicAdd(&row_flop[a_rowids[p]], static_cast<T>(qb));
    }
}

// Bin boundaries (GPU bin layout). A row starts a bin when its
// flop prefix enters a new window of T tuples, at every MAXR-aligned row,
// and around every row heavier than H (those become single-row bins). All
// non-heavy bins then hold < T + H = cap tuples and <= MAXR rows.
struct BinParams {
    uint64_t cap;   // tuples per bin (smem capacity)
    uint32_t maxr;  // rows per bin (2^(32-col_bits), <= 1024)
};

template <typename T>
__global__ void k_binflags(const T* __restrict__ row_flop,
                           const uint64_t* __restrict__ row_off, uint64_t m, BinParams bp,
                           const unsigned long long* max_row_flop, uint64_t* flags) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint64_t mx = *max_row_flop;
    const uint64_t h = mx < bp.cap / 4 ? mx : bp.cap / 4;
    const uint64_t t = bp.cap - h;
    uint64_t f;
    if (r == 0 || (r % bp.maxr) == 0) {
        f = 1;
    } else {
        const bool heavy = row_flop[r] > h, heavy_prev = row_flop[r - 1] > h;
        f = heavy || heavy_prev || (row_off[r] / t != row_off[r - 1] / t);
    }
    flags[r] = f;
}

// row -> bin id, bin -> first row.
__global__ void k_binrows(const uint64_t* __restrict__ flag_excl, uint64_t m, uint32_t* row_bin,
                          uint32_t* bin_rs) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint64_t e = flag_excl[r], e1 = flag_excl[r + 1];
    const uint32_t b = static_cast<uint32_t>(e1 - 1);  // inclusive - 1
    row_bin[r] = b;
    if (e1 != e) bin_rs[b] = static_cast<uint32_t>(r);
    if (r == m - 1) bin_rs[e1] = static_cast<uint32_t>(m);
}

// row -> bin << lbits | (row - bin row start): the expand's single dependent
// lookup per run (u32 when nbins < 2^(32 - lbits), else u64).
template <typename P>
__global__ void k_rowpack(const uint32_t* __restrict__ row_bin,
                          const uint32_t* __restrict__ bin_rs, uint64_t m, int lbits, P* pack) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const uint32_t b = row_bin[r];
    pack[r] = (static_cast<P>(b) << lbits) | static_cast<P>(r - bin_rs[b]);
}

// Per-bin tuple count, 4-tuple padded capacity (16-B aligned key runs),
// heavy-bin count.
__global__ void k_binsizes(const uint32_t* __restrict__ bin_rs,
                           const uint64_t* __restrict__ row_off, const uint64_t* nb_dev,
                           uint64_t cap, uint64_t* bin_cnt, uint64_t* bin_pad,
                           unsigned long long* heavy,
                           unsigned long long* maxbin) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t c = 0;
    if (b < *nb_dev) {
        c = row_off[bin_rs[b + 1]] - row_off[bin_rs[b]];
        bin_cnt[b] = c;
        bin_pad[b] = (c + 3) & ~3ull;
    }
    // warp-aggregated: one atomic per warp instead of one per bin
    const uint32_t nh = __popc(__ballot_sync(FULL, c > cap));
    uint64_t mx = c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(FULL, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (nh) atomicAdd(heavy, static_cast<unsigned long long>(nh));
        if (mx) atomicMax(maxbin, static_cast<unsigned long long>(mx));
    }
}

// ---------------------------------------------------------------- expand --
// Chunk c owns the runs (A entries) whose tuple range starts in
// [c*CH, (c+1)*CH); chunk_p0[c] is its first A entry.
// With row-banded expand (k_band_*), A's columns are virtual: v = band * kb
// + j, and B's row for v is j = v % kb (kb = A's real column count).
__global__ void k_chunks(const uint64_t* __restrict__ colflop_off,
                         const uint64_t* __restrict__ a_colptr,
                         const uint64_t* __restrict__ b_rowptr, uint64_t k, uint64_t kb,
                         uint64_t nnz_a, uint64_t ch, uint64_t nchunks, uint64_t* chunk_p0,
                         uint64_t* chunk_col, const unsigned long long* abort) {
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (c > nchunks) return;
    if (abort && *abort) {  // speculative launch rejected: every chunk empty
        chunk_p0[c] = 0;
        return;
    }
    if (c == nchunks) {
        chunk_p0[c] = nnz_a;
        chunk_col[c] = k;
        return;
    }
    const uint64_t t0 = c * ch;
    const uint64_t col = last_le(colflop_off, 0, k, t0);  // off[col] <= t0 < off[col+1]
    const uint64_t bj = col % kb;
    const uint64_t lb = b_rowptr[bj + 1] - b_rowptr[bj];
    const uint64_t rel = t0 - colflop_off[col];
    const uint64_t i = (rel + lb - 1) / lb;
    chunk_p0[c] = a_colptr[col] + i;
    // a lower bound on the column of run chunk_p0[c] (the expand starts its
    // column search there instead of searching colptr from 0: C1 expand
    // 0.053 -> 0.029 ms)
    chunk_col[c] = i < a_colptr[col + 1] - a_colptr[col] ? col : col + 1;
}

struct ExpandArgs {
    const uint64_t* a_colptr;
    const uint32_t* a_rowids;
    const double* a_vals;
    const uint64_t* b_rowptr;
    const uint32_t* b_colids;
    const double* b_vals;
    uint64_t a_ncols;   // (virtual) columns of A
    uint64_t b_rows;    // real columns of A = rows of B (virtual column v reads B row v % b_rows)
    const uint64_t* chunk_p0;
    const uint64_t* chunk_col;  // lower bound on the column of each chunk's first run
    uint64_t nchunks;
    const void* row_pack;          // per row: bin << lbits | (row - bin row start), u32 or u64
    int lbits;
    unsigned long long* cursor;    // per bin: next free tuple slot (absolute)
    uint32_t* keys;
    double* vals;
    int col_bits;
    const uint64_t* bin_off;  // bin tuple offsets (PBG_CHECKED: reservations stay inside the bin)
};

constexpr int EXP_NT = 256;
#ifndef PBG_EXP_U
#define PBG_EXP_U 4
#endif
#ifndef PBG_EXP_LONG_U
#define PBG_EXP_LONG_U 8  // long-run fast path: tuple steps in flight (4: C5b band expand 15.9 vs 15.0 ms)
#endif
#ifndef PBG_EXP_EVICT_LAST
#define PBG_EXP_EVICT_LAST 1
#endif

// Tuple stores. With PBG_EXP_EVICT_LAST the lines carry an L2 evict_last
// policy: a bin's partially written frontier line then survives the
// streaming input reads until its neighbours complete it, instead of being
// written back half-full (read-modify-write of the missing bytes).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_tuple_key(uint32_t* p, uint32_t v, uint64_t pol) {
#if PBG_EXP_EVICT_LAST
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol)
                 : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_tuple_val(double* p, double v, uint64_t pol) {
#if PBG_EXP_EVICT_LAST
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
                 : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_tuple_key2(uint32_t* p, uint32_t v0, uint32_t v1, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v0), "r"(v1), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_tuple_val2(double* p, double v0, double v1, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v0), "d"(v1), "l"(pol)
                 : "memory");
}
constexpr int EXP_NW = EXP_NT / 32;

// Outer-product expansion (expand_impl, pb_spgemm.cpp:180-246). One warp per
// chunk. Runs are processed 32 at a time, one per lane: the lane resolves the
// run's column k (shuffle search over 32 colptr boundaries), its bin, and
// reserves nnz(B(k,:)) slots in the bin with one atomicAdd on the bin cursor
// (the GPU version of the reference's `omp atomic capture` range
// reservation). The batch's tuples are then streamed flat, 32 per step, each
// lane finding its run with a redux.or over run-start bits, so stores of a
// run are coalesced and no lane idles on short runs. The 126 MB L2 plays the
// role of the reference's thread-private local bins: each bin's write
// frontier stays resident until its lines are full.
#ifndef PBG_EXP_MINB
#define PBG_EXP_MINB 2
#endif
// MINB: resident CTAs per SM the register budget is sized for — 2 for short
// runs (ER, stencil: 128 registers, deeper batch pipeline), 4 for long runs
// (RMAT: more warps streaming B rows).
// EXP_U: tuple steps of 32 a lane keeps in flight (loads issued before their
// stores): 8 for very short runs (C5a's 8-tuple runs: expand 16.3 -> 15.1 ms),
// 4 otherwise (C4 loses 2 % with 8).
template <typename P, int MINB, int EXP_U = PBG_EXP_U>
__global__ void __launch_bounds__(EXP_NT, MINB) k_expand(ExpandArgs a) {
    __shared__ uint64_t s_dst[EXP_NW][32];
    __shared__ uint64_t s_bst[EXP_NW][32];
    __shared__ double s_av[EXP_NW][32];
    __shared__ uint64_t s_st[EXP_NW][32];
    __shared__ uint32_t s_rp[EXP_NW][32];
#ifdef PBG_EXP_PAIRS
    __shared__ uint32_t s_lb[EXP_NW][32];
#endif
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lt = lanemask_lt();
    const int cb = a.col_bits;
    const uint64_t pol = l2_evict_last_policy();

    for (uint64_t c = gw; c < a.nchunks; c += nw) {
        uint64_t p = a.chunk_p0[c];
#ifdef PBG_DIAG_SEQSTORE
        uint64_t tpos = c * 8192;  // timing experiment only (wrong output)
#endif
        const uint64_t pend = a.chunk_p0[c + 1];
        if (p >= pend) continue;
        // the column of run p: at most a few columns past the chunk's bound
        uint64_t kcur = a.chunk_col[c];
        if (a.a_colptr[kcur + 1] <= p) kcur = warp_last_le(a.a_colptr, kcur, a.a_ncols, p);
        // Software pipeline over batches of 32 runs: batch t+1's loads (row
        // id, value, column window, then packed bin and B row bounds) are
        // issued while batch t's tuples stream out, so only the bin-cursor
        // atomic's round trip remains exposed per batch.
        double av_n = 0.0;
        uint32_t rid_n = 0;
        uint64_t bnd_n;
        {
            const uint64_t pl = p + lane;
            if (pl < pend) {
                av_n = a.a_vals[pl];
                rid_n = a.a_rowids[pl];
            }
            const uint64_t bi = kcur + 1 + lane;
            bnd_n = bi <= a.a_ncols ? a.a_colptr[bi] : ~0ull;
        }
        P pack_n = 0;
        uint64_t kl_n = 0, bst_n = 0, bend_n = 0;
        bool staged = false;  // pack_n / kl_n / bst_n hold the batch at p
        while (p < pend) {
            const uint64_t pl = p + lane;
            const bool valid = pl < pend;
            // ---- stage 2 of this batch (unless done during the last tuple loop)
            if (!staged) {
                if (valid) pack_n = static_cast<const P*>(a.row_pack)[rid_n];
                int cnt = 0;
#pragma unroll
                for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                    const uint64_t v = __shfl_sync(FULL, bnd_n, cnt + s2 - 1);
                    if (v <= pl) cnt += s2;
                }
                {
                    const uint64_t v = __shfl_sync(FULL, bnd_n, cnt & 31);
                    if (cnt == 31 && v <= pl) cnt = 32;
                }
                kl_n = kcur + cnt;
                if (valid && cnt == 32) kl_n = last_le(a.a_colptr, kcur, a.a_ncols, pl);
                if (valid) {
                    const uint64_t bj = kl_n < a.b_rows ? kl_n : kl_n % a.b_rows;
                    bst_n = a.b_rowptr[bj];
                    bend_n = a.b_rowptr[bj + 1];
                }
            }
            const double av = av_n;
            const P pack = pack_n;
            const uint64_t kl = kl_n;
            uint64_t lb = 0, bst = 0, dst = 0;
            uint32_t rp = 0;
            if (valid) {
                bst = bst_n;
                lb = bend_n - bst;
                if (lb) {
                    const P bin = pack >> a.lbits;
                    dst = atomicAdd(&a.cursor[bin], (unsigned long long)lb);
                    PBG_DCHECK(dst >= a.bin_off[bin] && dst + lb <= a.bin_off[bin + 1]);
                    rp = static_cast<uint32_t>(pack & ((P(1) << a.lbits) - 1)) << cb;
                }
            }
            // ---- stage 1 of the next batch
            const int last = (pend - p) < 32 ? static_cast<int>(pend - p) - 1 : 31;
            const uint64_t knext = __shfl_sync(FULL, kl, last);
            const uint64_t pn = p + 32;
            const bool has_next = pn < pend;
            if (has_next) {
                const uint64_t pln = pn + lane;
                if (pln < pend) {
                    av_n = a.a_vals[pln];
                    rid_n = a.a_rowids[pln];
                }
                const uint64_t bi = knext + 1 + lane;
                bnd_n = bi <= a.a_ncols ? a.a_colptr[bi] : ~0ull;
            }
            staged = false;
            // Long runs (RMAT hub rows of B): the warp streams one run at a
            // time, 32 consecutive tuples per step, with none of the flat
            // stream's per-step run lookup (85 warp instructions per 32 tuples
            // on a C3 round, 61 % issue-active). Only with the long-run
            // register budget (MINB >= 4): short-run inputs never take it.
            if (MINB >= 4) {
                constexpr uint64_t EXP_LONG = 256;
                uint32_t longm = __ballot_sync(FULL, lb >= EXP_LONG);
                const bool is_long = lb >= EXP_LONG;
                while (longm) {
                    const int L = __ffs(longm) - 1;
                    longm &= longm - 1;
                    const uint64_t n0 = __shfl_sync(FULL, lb, L);
                    const uint32_t* bc = a.b_colids + __shfl_sync(FULL, bst, L);
                    const double* bv = a.b_vals + __shfl_sync(FULL, bst, L);
                    uint32_t* kd = a.keys + __shfl_sync(FULL, dst, L);
                    double* vd = a.vals + __shfl_sync(FULL, dst, L);
                    const double a0 = __shfl_sync(FULL, av, L);
                    const uint32_t r0 = __shfl_sync(FULL, rp, L);
                    constexpr int LU = PBG_EXP_LONG_U;  // steps of 32 tuples in flight
                    for (uint64_t q0 = 0; q0 < n0; q0 += 32 * LU) {
                        uint32_t kq[LU];
                        double vq[LU];
#pragma unroll
                        for (int u = 0; u < LU; ++u) {
                            const uint64_t q = q0 + 32 * u + lane;
                            kq[u] = q < n0 ? __ldg(bc + q) : 0u;
                            vq[u] = q < n0 ? __ldg(bv + q) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < LU; ++u) {
                            const uint64_t q = q0 + 32 * u + lane;
                            if (q < n0) {
                                st_tuple_key(kd + q, r0 | kq[u], pol);
                                st_tuple_val(vd + q, a0 * vq[u], pol);
                            }
                        }
                    }
                }
                if (is_long) lb = 0;  // done: not part of the flat stream below
            }
            const bool ne = lb != 0;
            const uint32_t nemask = __ballot_sync(FULL, ne);
            const int rank = __popc(nemask & lt);
#ifdef PBG_EXP_PAIRS
            // a run is cut into pieces of 2 tuples at even slots (one 8-byte
            // key store + one 16-byte value store each) plus an odd head/tail
            const uint64_t hd = lb ? (dst & 1u) : 0u;
            const uint64_t units = hd + (lb - hd + 1) / 2;
#else
            const uint64_t units = lb;
#endif
            uint64_t incl = warp_inclusive_scan(units);
            const uint64_t start = incl - units;
            const uint64_t total = __shfl_sync(FULL, incl, 31);
            if (ne) {
                s_dst[w][rank] = dst;
                s_bst[w][rank] = bst;
                s_av[w][rank] = av;
                s_st[w][rank] = start;
                s_rp[w][rank] = rp;
#ifdef PBG_EXP_PAIRS
                s_lb[w][rank] = static_cast<uint32_t>(lb);
#endif
            }
            __syncwarp();
            // tuples, EXP_U steps of 32 per iteration: all B loads of the
            // group are issued before any store so their latencies overlap
            uint32_t before = 0;
#ifdef PBG_EXP_PAIRS
            for (uint64_t s0 = 0; s0 < total; s0 += 32 * EXP_U) {
                uint32_t kv[EXP_U], kv1[EXP_U];
                double bv[EXP_U], bv1[EXP_U], avv[EXP_U];
                uint32_t rpv[EXP_U];
                uint64_t dv[EXP_U];
                int cntv[EXP_U];
#pragma unroll
                for (int u = 0; u < EXP_U; ++u) {
                    const uint64_t s = s0 + 32 * u;
                    const uint32_t bit =
                        (ne && start >= s && start < s + 32) ? (1u << (start - s)) : 0u;
                    const uint32_t mk = __reduce_or_sync(FULL, bit);
                    const uint64_t t = s + lane;
                    const bool ok = t < total;
                    const uint32_t upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
                    int ri = static_cast<int>(before + __popc(mk & upto)) - 1;
                    ri = ok ? ri : 0;
                    const uint64_t q = t - s_st[w][ri];  // piece of the run
                    const uint64_t d0 = s_dst[w][ri];
                    const uint32_t h = static_cast<uint32_t>(d0 & 1u);
                    const uint32_t off = q == 0 ? 0u : static_cast<uint32_t>(2 * q - h);
                    const uint32_t L = s_lb[w][ri];
                    cntv[u] = !ok ? 0 : ((h && q == 0) || off + 1 >= L) ? 1 : 2;
                    const uint64_t src = s_bst[w][ri] + off;
                    kv[u] = cntv[u] ? __ldg(a.b_colids + src) : 0u;
                    bv[u] = cntv[u] ? __ldg(a.b_vals + src) : 0.0;
                    kv1[u] = cntv[u] == 2 ? __ldg(a.b_colids + src + 1) : 0u;
                    bv1[u] = cntv[u] == 2 ? __ldg(a.b_vals + src + 1) : 0.0;
                    rpv[u] = s_rp[w][ri];
                    avv[u] = s_av[w][ri];
                    dv[u] = d0 + off;
                    before += __popc(mk);
                }
#pragma unroll
                for (int u = 0; u < EXP_U; ++u) {
                    if (cntv[u] == 2) {
                        st_tuple_key2(a.keys + dv[u], rpv[u] | kv[u], rpv[u] | kv1[u], pol);
                        st_tuple_val2(a.vals + dv[u], avv[u] * bv[u], avv[u] * bv1[u], pol);
                    } else if (cntv[u] == 1) {
                        st_tuple_key(a.keys + dv[u], rpv[u] | kv[u], pol);
                        st_tuple_val(a.vals + dv[u], avv[u] * bv[u], pol);
                    }
                }
#else
            for (uint64_t s0 = 0; s0 < total; s0 += 32 * EXP_U) {
                uint32_t kv[EXP_U];
                double bv[EXP_U], avv[EXP_U];
                uint32_t rpv[EXP_U];
                uint64_t dv[EXP_U];
                bool ok[EXP_U];
#pragma unroll
                for (int u = 0; u < EXP_U; ++u) {
                    const uint64_t s = s0 + 32 * u;
                    const uint32_t bit =
                        (ne && start >= s && start < s + 32) ? (1u << (start - s)) : 0u;
                    const uint32_t mk = __reduce_or_sync(FULL, bit);
                    const uint64_t t = s + lane;
                    ok[u] = t < total;
                    const uint32_t upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
                    int ri = static_cast<int>(before + __popc(mk & upto)) - 1;
                    ri = ok[u] ? ri : 0;
                    const uint64_t q = t - s_st[w][ri];
                    const uint64_t src = s_bst[w][ri] + q;
#ifdef PBG_DIAG_NOBLOAD  // timing experiment: no B gathers (wrong output)
                    kv[u] = static_cast<uint32_t>(src) & 0xfffffu;
                    bv[u] = 1.0;
#else
                    kv[u] = ok[u] ? __ldg(a.b_colids + src) : 0u;
                    bv[u] = ok[u] ? __ldg(a.b_vals + src) : 0.0;
#endif
                    rpv[u] = s_rp[w][ri];
                    avv[u] = s_av[w][ri];
#ifdef PBG_DIAG_SEQSTORE
                    dv[u] = (tpos + t) % (1ull << 28);
#elif defined(PBG_DIAG_REGION)  // timing experiment: the same scatter folded into 2^R tuples
                    dv[u] = (s_dst[w][ri] + q) & ((1ull << PBG_DIAG_REGION) - 1);
#else
                    dv[u] = s_dst[w][ri] + q;
#endif
                    before += __popc(mk);
                }
#pragma unroll
                for (int u = 0; u < EXP_U; ++u) {
#ifdef PBG_DIAG_NOSTORE
                    if (ok[u] && (rpv[u] | kv[u]) == 0xfffffffeu && avv[u] * bv[u] == 1.2345)
#else
                    if (ok[u])
#endif
                    {
#ifdef PBG_DIAG_AOS16  // timing experiment: 16-byte AoS tuples, one vector store each
                        {
                            uint32_t* T = reinterpret_cast<uint32_t*>(a.vals) + dv[u] * 4;
                            const double vv = avv[u] * bv[u];
                            const unsigned long long bits = __double_as_longlong(vv);
                            asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(T),
                                         "r"(rpv[u] | kv[u]), "r"(0u), "r"(static_cast<uint32_t>(bits)),
                                         "r"(static_cast<uint32_t>(bits >> 32)), "l"(pol)
                                         : "memory");
                        }
                        continue;
#endif
#ifdef PBG_DIAG_AOS12  // timing experiment: 12-byte AoS tuples (one store segment per run)
                        {
                            uint32_t* T = reinterpret_cast<uint32_t*>(a.vals) + dv[u] * 3;
                            const double vv = avv[u] * bv[u];
                            const unsigned long long bits = __double_as_longlong(vv);
                            st_tuple_key(T, rpv[u] | kv[u], pol);
                            st_tuple_key(T + 1, static_cast<uint32_t>(bits), pol);
                            st_tuple_key(T + 2, static_cast<uint32_t>(bits >> 32), pol);
                        }
                        continue;
#endif
#ifndef PBG_DIAG_NOKEYST
                        st_tuple_key(a.keys + dv[u], rpv[u] | kv[u], pol);
#endif
#ifndef PBG_DIAG_NOVALST
                        st_tuple_val(a.vals + dv[u], avv[u] * bv[u], pol);
#endif
                    }
                }
#endif  // PBG_EXP_PAIRS
                // ---- stage 2 of the next batch, once its stage-1 loads landed
                if (s0 == 0 && has_next) {
                    const uint64_t pln = pn + lane;
                    const bool vn = pln < pend;
                    if (vn) pack_n = static_cast<const P*>(a.row_pack)[rid_n];
                    int cnt = 0;
#pragma unroll
                    for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                        const uint64_t v = __shfl_sync(FULL, bnd_n, cnt + s2 - 1);
                        if (v <= pln) cnt += s2;
                    }
                    {
                        const uint64_t v = __shfl_sync(FULL, bnd_n, cnt & 31);
                        if (cnt == 31 && v <= pln) cnt = 32;
                    }
                    kl_n = knext + cnt;
                    if (vn && cnt == 32) kl_n = last_le(a.a_colptr, knext, a.a_ncols, pln);
                    if (vn) {
                        const uint64_t bj = kl_n < a.b_rows ? kl_n : kl_n % a.b_rows;
                        bst_n = a.b_rowptr[bj];
                        bend_n = a.b_rowptr[bj + 1];
                    }
                    staged = true;
                }
            }
            __syncwarp();
            kcur = knext;
            p = pn;
#ifdef PBG_DIAG_SEQSTORE
            tpos += total;
#endif
        }
    }
}


// ------------------------------------------------------- row-banded expand --
// The expand's write frontier is one partially filled line per bin array;
// with ~10^5 bins it no longer fits the 126 MB L2 and half-written sectors are
// evicted (DRAM read-modify-write). Expanding G row bands one after another
// (A re-ordered band-major: virtual column v = band * k + j holds A(band
// rows, j)) keeps only nbins/G bins active at a time. Bands are unions of
// whole bins, so bins, offsets and cursors are unchanged.
struct VColFlopIn {
    const uint64_t* va_colptr;
    const uint64_t* b_rowptr;
    uint64_t kb;
    __device__ __forceinline__ uint64_t operator()(uint64_t v) const {
        const uint64_t j = v % kb;
        return (va_colptr[v + 1] - va_colptr[v]) * (b_rowptr[j + 1] - b_rowptr[j]);
    }
};

// count[v = s*k + j] = #A(:,j) entries with rows in band s
__device__ __forceinline__ int band_of(uint32_t r, const uint32_t* __restrict__ cuts, int g) {
    int s = 0;
    while (s + 1 < g && r >= cuts[s + 1]) ++s;
    return s;
}

constexpr int BAND_MAX = 16;

// Band-major re-ordering of A (virtual column v = band * k + j), entry-
// parallel like the row slabs of pbg_bands.cuh: per band one selection bit per
// entry (one word per 32 entries), ONE scan over the band-major sequence of
// word popcounts (so a word's prefix is its place in the re-ordered arrays),
// the virtual column pointers by lookup, a stable coalesced gather. (The
// first version walked every column with one thread in a counting and a
// copying kernel, with a scan over all G * k virtual columns between them:
// 2.2 ms of C5a's expand phase.)
__global__ void k_band_bits(const uint32_t* __restrict__ a_rowids, uint64_t nnz, uint64_t nwords,
                            const uint32_t* __restrict__ cuts, int g, uint32_t* bits, uint32_t* wcnt) {
    __shared__ uint32_t s_cuts[BAND_MAX + 1];
    if (threadIdx.x <= g) s_cuts[threadIdx.x] = cuts[threadIdx.x];
    __syncthreads();
    // a warp takes 32 words (1024 entries) per trip: lane i keeps the ballots
    // of the trip's i-th word, so the words leave as coalesced 128-byte stores
    // (one 4-byte store per word and band by lane 0 ran at 0.7 TB/s)
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w0 = warp * 32; w0 < nwords; w0 += nwarps * 32) {
        uint32_t mine[BAND_MAX];
#pragma unroll
        for (int s = 0; s < BAND_MAX; ++s) mine[s] = 0;
        for (int i = 0; i < 32; ++i) {
            const uint64_t p = (w0 + i) * 32 + lane;
            const int bnd = p < nnz ? band_of(__ldcs(a_rowids + p), s_cuts, g) : -1;
#pragma unroll
            for (int s = 0; s < BAND_MAX; ++s) {
                if (s < g) {
                    const uint32_t b = __ballot_sync(FULL, bnd == s);
                    if (lane == i) mine[s] = b;
                }
            }
        }
        if (w0 + lane < nwords) {
#pragma unroll
            for (int s = 0; s < BAND_MAX; ++s) {
                if (s < g) {
                    bits[static_cast<uint64_t>(s) * nwords + w0 + lane] = mine[s];
                    wcnt[static_cast<uint64_t>(s) * nwords + w0 + lane] = __popc(mine[s]);
                }
            }
        }
    }
}

// va_colptr[v] for v = band * k + j (v = 0 .. g*k): entries of the bands before
// `band` plus the band's entries before a_colptr[j]
__global__ void k_band_colptr(const uint64_t* __restrict__ a_colptr, uint64_t k, uint64_t nnz,
                              uint64_t nwords, int g, const uint32_t* __restrict__ bits,
                              const uint64_t* __restrict__ wpre, uint64_t* va_colptr) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t kv = k * static_cast<uint64_t>(g);
    if (v > kv) return;
    if (v == kv) {
        va_colptr[v] = wpre[static_cast<uint64_t>(g) * nwords];
        return;
    }
    const uint64_t s = v / k, j = v - s * k;
    const uint64_t p = a_colptr[j];
    if (p >= nnz) {
        va_colptr[v] = wpre[(s + 1) * nwords];  // the band's end
        return;
    }
    const uint64_t w = s * nwords + (p >> 5);
    va_colptr[v] = wpre[w] + __popc(bits[w] & ((1u << (p & 31u)) - 1u));
}

__global__ void k_band_gather(const uint32_t* __restrict__ a_rowids, const double* __restrict__ a_vals,
                              uint64_t nnz, uint64_t nwords, const uint32_t* __restrict__ cuts, int g,
                              const uint32_t* __restrict__ bits, const uint64_t* __restrict__ wpre,
                              uint32_t* va_rowids, double* va_vals) {
    __shared__ uint32_t s_cuts[BAND_MAX + 1];
    if (threadIdx.x <= g) s_cuts[threadIdx.x] = cuts[threadIdx.x];
    __syncthreads();
    const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p >= nnz) return;
    const uint32_t r = a_rowids[p];
    const uint64_t w = static_cast<uint64_t>(band_of(r, s_cuts, g)) * nwords + (p >> 5);
    const uint64_t at = wpre[w] + __popc(bits[w] & lanemask_lt());
    va_rowids[at] = r;
    va_vals[at] = a_vals[p];
}

__global__ void k_band_cuts(const uint32_t* __restrict__ bin_rs, const uint64_t* nb_dev, int g,
                            uint32_t* cuts) {
    const int s = threadIdx.x;
    if (s > g) return;
    const uint64_t nb = *nb_dev;
    cuts[s] = bin_rs[(nb * static_cast<uint64_t>(s)) / g];
}


__global__ void k_zero_u64(uint64_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = 0;
}

// ---------------------------------------------------- COO -> CSR / CSC --
// The conversion runs as the product A.B with A(major(e), e) = 1 (a CSC with
// one entry per column) and B(e, minor(e)) = val(e) (a CSR with one entry
// per row): the expand emits one tuple per entry, the sort+merge sums
// duplicates and orders minors, the CSR assembly builds the pointer array.
__global__ void k_coo_views(uint64_t nnz, uint64_t* iota_a, uint64_t* iota_b, double* ones,
                            const uint32_t* __restrict__ major, const uint32_t* __restrict__ minor,
                            unsigned long long* maxes) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t mj = 0, mn = 0;
    if (e <= nnz) {
        iota_a[e] = e;
        iota_b[e] = e;
    }
    if (e < nnz) {
        ones[e] = 1.0;
        mj = major[e];
        mn = minor[e];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mj = max(mj, __shfl_xor_sync(FULL, mj, o));
        mn = max(mn, __shfl_xor_sync(FULL, mn, o));
    }
    if ((threadIdx.x & 31) == 0 && e < nnz + 32) {
        atomicMax(maxes, static_cast<unsigned long long>(mj));
        atomicMax(maxes + 1, static_cast<unsigned long long>(mn));
    }
}

// ------------------------------------------------ benchmark generators --
// The reference's generators (generate.hpp:12-40, generate.cpp:20-90) as
// device streams: SplitMix64 per column (ER, Floyd sampling) or per edge
// (RMAT quadrant descent), the same seeds giving the same draws.
struct DSm64 {
    uint64_t s;
    __device__ explicit DSm64(uint64_t seed) : s(seed) {}
    __device__ uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    __device__ uint64_t below(uint64_t bound) {
        const uint64_t limit = bound * (~uint64_t{0} / bound);
        uint64_t x;
        do x = next();
        while (x >= limit);
        return x % bound;
    }
    __device__ double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
__device__ __forceinline__ uint64_t dsplit(uint64_t seed, uint64_t stream) {
    return DSm64(seed ^ (stream * 0xD6E8FEB86659FD93ULL)).next();
}

// gen_er: column j holds d distinct rows (Floyd's sampling); entry j*d + f
__global__ void k_gen_er(int scale, uint32_t d, uint64_t seed, uint32_t* rows, uint32_t* cols) {
    const uint32_t n = 1u << scale;
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    DSm64 rng(dsplit(seed, j));
    uint32_t* col = rows + j * d;
    uint32_t filled = 0;
    for (uint32_t t = n - d; t < n; ++t) {
        const uint32_t r = static_cast<uint32_t>(rng.below(static_cast<uint64_t>(t) + 1));
        bool seen = false;
        for (uint32_t q = 0; q < filled; ++q) seen |= col[q] == r;
        cols[j * d + filled] = static_cast<uint32_t>(j);
        col[filled++] = seen ? t : r;
    }
}

// gen_rmat: edge e descends `scale` quadrant levels with cuts a, a+b, a+b+c
__global__ void k_gen_rmat(int scale, uint64_t nedges, uint64_t seed, double a, double b, double c,
                           uint32_t* rows, uint32_t* cols) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= nedges) return;
    DSm64 rng(dsplit(seed, e));
    const double cut_a = a, cut_ab = a + b, cut_abc = a + b + c;
    uint32_t row = 0, col = 0;
    for (int level = scale - 1; level >= 0; --level) {
        const double u = rng.unit();
        if (u >= cut_ab) row |= 1u << level;
        if (u >= cut_abc || (u >= cut_a && u < cut_ab)) col |= 1u << level;
    }
    rows[e] = row;
    cols[e] = col;
}

struct OffDiagIn {  // 1 for an entry off the diagonal (self-loops dropped)
    const uint32_t* r;
    const uint32_t* c;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return r[i] != c[i]; }
};
__global__ void k_compact_offdiag(const uint32_t* __restrict__ r, const uint32_t* __restrict__ c,
                                  const uint64_t* __restrict__ pos, uint64_t n, uint32_t* r2,
                                  uint32_t* c2) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n || r[i] == c[i]) return;
    r2[pos[i]] = r[i];
    c2[pos[i]] = c[i];
}

// U[0,1) value of (row, col): SplitMix64(split_seed(vseed, row << 32 | col))
// (generate.hpp:35-40), over a compressed matrix (major = row for CSR).
__global__ void k_fill_values(uint64_t vseed, uint64_t nmajor, const uint64_t* __restrict__ ptr,
                              const uint32_t* __restrict__ idx, double* vals, int major_is_col) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nmajor) return;
    for (uint64_t p = ptr[i]; p < ptr[i + 1]; ++p) {
        const uint64_t r = major_is_col ? idx[p] : i, c = major_is_col ? i : idx[p];
        vals[p] = DSm64(dsplit(vseed, (r << 32) | c)).unit();
    }
}

}  // namespace pbg
