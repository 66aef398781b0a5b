// pbg_sort.cuh — per-bin sort + duplicate merge + CSR assembly (one kernel).
//
// Replaces sort_bins -> sort_bin_records (American-flag MSD radix with an
// insertion-sort cutoff, pb_spgemm.hpp:118-197), compress_bins ->
// compress_bin_records (two-pointer merge, pb_spgemm.hpp:202-216) and
// convert_csr (pb_spgemm.cpp:288-328).
//
// Persistent CTAs take work bins (a GPU bin, or one key range of a heavy
// row, pbg_heavy.cuh) in ticket order. A work bin holds <= SM_CAP tuples
// (u32 key = local_row << col_bits | col, f64 value) with keys in
// [keylo, keylo + 2^keybits). Per work bin:
//   0. the bin arrives in one shared-memory buffer by two TMA bulk copies
//      (cp.async.bulk, mbarrier completion) issued while the CTA was still
//      busy with the previous bin;
//   1. it is sorted IN PLACE with every tuple staged in registers (8 per
//      thread): an MSD bucket pass on the top used key bits (SM_NB buckets ~
//      1 tuple each; the smem histogram atomic returns the tuple's slot in its
//      bucket), a scan, the keys scattered to their buckets, a rank inside
//      the bucket (smaller keys + earlier equal keys) and the tuple written at
//      its sorted position — the reference's first radix level wide enough
//      that the insertion-sort cutoff is a 1-2 element compare loop. A bucket
//      above SM_BMAX (clustered keys) switches the bin to a stable LSD radix;
//   2. duplicate keys are summed (two-pointer merge semantics: exact zeros
//      are kept) and compacted in place;
//   3. the merged count U_b is published at once; one warp of the grid scans
//      the counts in work-bin order (single-pass chained scan,
//      status_scanner). The bin itself stays in its buffer while the CTA
//      sorts its NEXT bin, and is written out (cols, values, rowptr) one bin
//      later, when its prefix is long known. The output offset therefore
//      needs no separate distinct-count pass over the tuples, and CTAs never
//      wait on slower neighbours (an undelayed look-back was measured 2-3x
//      slower).
// Duplicate-heavy bins (the 27-point stencil squared, cf ~ 6) are detected
// from the bucket histogram and pre-merged in a shared-memory hash first.
#pragma once

#include <cstdint>

#include "pbg_device.cuh"
#include "pbg_heavy.cuh"

namespace pbg {

#ifndef PBG_SM_CAP
#define PBG_SM_CAP 4096
#endif
#ifndef PBG_SM_NT
#define PBG_SM_NT 512
#endif
#ifndef PBG_SM_LAG
#define PBG_SM_LAG 1
#endif
#ifndef PBG_SM_PF
#define PBG_SM_PF 0
#endif

constexpr int SM_NT = PBG_SM_NT;
constexpr int SM_NW = SM_NT / 32;
constexpr int SM_CAP = PBG_SM_CAP;            // max tuples per smem bin
constexpr int SM_NB = 2 * SM_CAP;             // buckets of the MSD pass (u16 counters, 2 per word)
constexpr int SM_NB_BITS = __builtin_ctz(SM_NB);
constexpr int SM_NBW = SM_NB / 2;             // counter words
#ifndef PBG_SM_BMAX
#define PBG_SM_BMAX 128
#endif
constexpr int SM_BMAX = PBG_SM_BMAX;          // largest bucket ranked in place
#ifndef PBG_SM_BMAX_PM
#define PBG_SM_BMAX_PM 128
#endif
// after a hash pre-merge the distinct keys of banded rows cluster in a few
// buckets (stencil: 25 columns within +-258 of each other): LSD radix instead
constexpr int SM_BMAX_PM = PBG_SM_BMAX_PM;
constexpr int SM_ITEMS = SM_CAP / SM_NT;      // tuples per thread
constexpr int SM_PER_WARP = SM_CAP / SM_NW;   // warp-contiguous element layout
constexpr int SM_WPT = SM_NBW / SM_NT;        // counter words per thread in the scan
static_assert(SM_WPT % 4 == 0, "counter words per thread: whole uint4s");
// LSD fallback digits: per-(warp, digit) counters must fit the counter words
constexpr int LSD_BITS = SM_NW * 256 <= SM_NBW ? 8 : 7;
constexpr int LSD_ND = 1 << LSD_BITS;
static_assert(SM_NW * LSD_ND <= SM_NBW, "LSD counters fit the bucket counter words");
// Buffer ring: the bin being sorted, LAG sorted bins whose output is still
// pending (their prefixes need all earlier bins sorted) and PF bins whose TMA
// copy is in flight.
constexpr int SM_LAG = PBG_SM_LAG;
constexpr int SM_PF = PBG_SM_PF;
constexpr int SM_NBUF = 1 + SM_LAG + SM_PF;
constexpr int SM_NMETA = SM_NBUF + 1;         // descriptors: pending .. next to fetch

struct SortArgs {
    WorkBins w;
    const uint64_t* nw_dev;   // number of work bins
    unsigned long long* status;  // look-back status word per work bin (zeroed)
    unsigned int* ticket;
    uint32_t* keys;           // tuples (main buffer); a parked bin is stored back here
    double* vals;
    uint32_t* skeys;          // tuples (heavy-row scratch buffer)
    double* svals;
    uint32_t* ccol;           // C colids
    double* cval;             // C values
    uint64_t* rowptr;
    uint64_t m;
    int col_bits;
    unsigned long long* merged_total;
    unsigned int* err;  // bit1 work bin above capacity
    unsigned long long* fallbacks;
    unsigned long long* premerged;
    unsigned long long* parked;
    int force_park;            // test hook: park whenever the ring has room
    unsigned long long* prof;  // PBG_SORT_PROF builds: cycles per phase (thread 0 of each CTA)
};

#ifdef PBG_SORT_PROF
#define PROF_MARK(i)                                                       \
    do {                                                                   \
        if (threadIdx.x == 0) {                                            \
            const long long t_ = clock64();                                \
            atomicAdd(&a.prof[i], (unsigned long long)(t_ - prof_t));      \
            prof_t = t_;                                                   \
        }                                                                  \
    } while (0)
#else
#define PROF_MARK(i) \
    do {             \
    } while (0)
#endif

constexpr int SM_NHMAX = 32;  // non-head duplicates merged without a compaction pass

// Work-bin descriptor staged in shared memory (cp.async by thread 0, one bin
// ahead, so no thread waits on these loads).
struct BinMeta {
    uint64_t n, off;
    uint32_t flags, keybits, keylo, rs, span, pad;
};

// A sorted bin whose output offset was not yet known when its buffer was
// needed: stored back into its own (consumed) tuple range, written to C a
// few bins later by the same CTA (still L2-resident).
constexpr int PK_MAX = 6;
struct Parked {
    BinMeta m;
    uint64_t bin;
    uint32_t U, pad;
};

struct SortSmem {
    uint32_t k[SM_NBUF][SM_CAP];
    double v[SM_NBUF][SM_CAP];
    uint32_t cnt[SM_NBW];  // bucket histogram -> bucket starts (u16 pairs); LSD per-warp counters
    uint32_t s_warp32[SM_NW + 1];
    uint16_t nh_pos[SM_NHMAX];
    uint32_t nh_cnt;
    uint32_t s_dupheavy;  // the previous bin of this CTA was duplicate-heavy
    unsigned long long mbar[SM_NBUF];  // TMA completion, one per buffer
    uint32_t pend_U[SM_NBUF];          // merged count of the sorted bin in each buffer
    uint64_t s_bin[SM_NMETA];
    BinMeta meta[SM_NMETA];            // descriptor ring (CTA-local bin sequence)
    Parked pk[PK_MAX];    // parked bins (ring, oldest first)
    uint64_t pk_P[PK_MAX];
    uint64_t s_pbP;
    uint32_t pk_head, pk_count, s_nres, s_park;
};

// ---- TMA bulk copy (global -> shared) with mbarrier completion ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// ---- work-bin descriptors: cp.async into shared memory one bin ahead ----
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// Thread 0: work bin b becomes ring slot `slot` (its descriptor arrives
// asynchronously; cp_async_wait_all + a barrier make it visible).
__device__ __forceinline__ void meta_fetch(const SortArgs& a, SortSmem& sm, int slot, uint64_t b,
                                           uint64_t nw) {
    sm.s_bin[slot] = b;
    if (b >= nw) return;
    BinMeta& m = sm.meta[slot];
    cp_async8(&m.n, a.w.n + b);
    cp_async8(&m.off, a.w.off + b);
    cp_async4(&m.flags, a.w.flags + b);
    cp_async4(&m.keybits, a.w.keybits + b);
    cp_async4(&m.keylo, a.w.keylo + b);
    cp_async4(&m.rs, a.w.rs + b);
    cp_async4(&m.span, a.w.span + b);
}

// How a work bin reaches shared memory: 1 = TMA bulk copy, 2 = plain loads
// (unaligned heavy sub-bin), 0 = nothing to load (empty / merged / error).
__device__ __forceinline__ uint32_t bin_kind(const BinMeta& m) {
    if (m.n == 0 || m.n > SM_CAP || (m.flags & 2u)) return 0;
    return (m.off & 3u) ? 2 : 1;
}

// Thread 0: start the TMA copy of a kind-1 bin into buffer `buf` (generic-
// proxy accesses to it are finished: caller syncs).
__device__ __forceinline__ void issue_tma(const SortArgs& a, SortSmem& sm, int buf,
                                          const BinMeta& m) {
    const uint32_t* ks = (m.flags & 1u) ? a.skeys : a.keys;
    const double* vs = (m.flags & 1u) ? a.svals : a.vals;
    const uint32_t kb = static_cast<uint32_t>((m.n * 4 + 15) & ~15ull);
    const uint32_t vb = static_cast<uint32_t>((m.n * 8 + 15) & ~15ull);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&sm.mbar[buf], kb + vb);
    bulk_g2s(sm.k[buf], ks + m.off, kb, &sm.mbar[buf]);
    bulk_g2s(sm.v[buf], vs + m.off, vb, &sm.mbar[buf]);
}

__device__ __forceinline__ uint32_t elem_idx(int it) {
    return (threadIdx.x >> 5) * SM_PER_WARP + it * 32 + (threadIdx.x & 31);
}

// Exclusive scan of the SM_NB u16 counters (two per word, 16 per thread) in
// index order. Returns the number of tuples sitting 4th or later in their
// bucket (< 1 % of a bin of distinct uniform keys, most of a duplicate-heavy
// one).
__device__ __forceinline__ uint32_t scan_cnt(SortSmem& sm) {
    const int tid = threadIdx.x;
    uint4* c4 = reinterpret_cast<uint4*>(sm.cnt) + (SM_WPT / 4) * tid;
    uint32_t w8[SM_WPT];
#pragma unroll
    for (int q = 0; q < SM_WPT / 4; ++q) {
        const uint4 x = c4[q];
        w8[4 * q] = x.x;
        w8[4 * q + 1] = x.y;
        w8[4 * q + 2] = x.z;
        w8[4 * q + 3] = x.w;
    }
    uint32_t s = 0, crowd = 0;
#pragma unroll
    for (int j = 0; j < SM_WPT; ++j) {
        const uint32_t c0 = w8[j] & 0xffffu, c1 = w8[j] >> 16;
        s += c0 + c1;
        crowd += (c0 > 3 ? c0 - 3 : 0) + (c1 > 3 ? c1 - 3 : 0);
    }
    uint32_t tot;  // counts <= SM_CAP < 2^16: both sums in one scan
    uint32_t run = block_exclusive_scan<SM_NT>(crowd << 16 | s, sm.s_warp32, tot) & 0xffffu;
    uint32_t o[SM_WPT];
#pragma unroll
    for (int j = 0; j < SM_WPT; ++j) {
        const uint32_t c0 = w8[j] & 0xffffu, c1 = w8[j] >> 16;
        o[j] = run | (run + c0) << 16;
        run += c0 + c1;
    }
#pragma unroll
    for (int q = 0; q < SM_WPT / 4; ++q) c4[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    return tot >> 16;
}

// u16 counter d of the packed bucket array
__device__ __forceinline__ uint32_t cnt_get(const SortSmem& sm, uint32_t d) {
    return (sm.cnt[d >> 1] >> ((d & 1) * 16)) & 0xffffu;
}
__device__ __forceinline__ uint32_t cnt_inc(SortSmem& sm, uint32_t d) {
    const uint32_t sh = (d & 1) * 16;
    return (atomicAdd(&sm.cnt[d >> 1], 1u << sh) >> sh) & 0xffffu;
}

__device__ __forceinline__ void zero_cnt(SortSmem& sm) {
    uint4* c4 = reinterpret_cast<uint4*>(sm.cnt) + (SM_WPT / 4) * threadIdx.x;
#pragma unroll
    for (int q = 0; q < SM_WPT / 4; ++q) c4[q] = make_uint4(0, 0, 0, 0);
}

// Stable LSD radix sort of K/V[0, n) in place (the tuples are staged in
// registers, element layout elem_idx) over `bits` key bits, LSD_BITS-bit
// digits. Ranks from match.any per warp in element order, per-(warp, digit)
// counters cnt[w*LSD_ND+d] scanned digit-major.
__device__ __noinline__ void lsd_sort(SortSmem& sm, uint32_t* K, double* V, uint32_t n, int bits,
                                      uint32_t keylo) {
    const int tid = threadIdx.x, w = tid >> 5;
    const uint32_t lt = lanemask_lt();
    uint32_t kr[SM_ITEMS];
    double vr[SM_ITEMS];
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t idx = elem_idx(it);
        kr[it] = idx < n ? K[idx] : 0u;
        vr[it] = idx < n ? V[idx] : 0.0;
    }
    for (int shift = 0; shift < bits; shift += LSD_BITS) {
        zero_cnt(sm);
        __syncthreads();
        uint32_t rd[SM_ITEMS];  // rank << 9 | digit
        uint32_t* wc = sm.cnt + w * LSD_ND;
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const bool valid = elem_idx(it) < n;
            const uint32_t d = valid ? (((kr[it] - keylo) >> shift) & (LSD_ND - 1)) : 0x100u;
            const uint32_t peers = __match_any_sync(FULL, d);
            const uint32_t old = valid ? wc[d] : 0;
            rd[it] = (old + __popc(peers & lt)) << 9 | d;
            __syncwarp();
            if (valid && (peers & lt) == 0) wc[d] = old + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {  // digit-major exclusive scan over (digit, warp)
            constexpr int PER = SM_NW * LSD_ND / SM_NT;  // counters per thread
            constexpr int TPD = SM_NW / PER;             // threads per digit
            const int d = tid / TPD, w0 = (tid % TPD) * PER;
            uint32_t c[PER], s = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                c[j] = sm.cnt[(w0 + j) * LSD_ND + d];
                s += c[j];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan<SM_NT>(s, sm.s_warp32, tot);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                sm.cnt[(w0 + j) * LSD_ND + d] = run;
                run += c[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            if (elem_idx(it) < n) {
                const uint32_t pos = wc[rd[it] & 0x1ffu] + (rd[it] >> 9);
                K[pos] = kr[it];
                V[pos] = vr[it];
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = elem_idx(it);
            if (idx < n) {
                kr[it] = K[idx];
                vr[it] = V[idx];
            }
        }
    }
}

// Sum equal-key runs of the sorted K/V[0, n) and compact them in place.
// Returns the merged count.
__device__ __noinline__ uint32_t merge_dups_inplace(SortSmem& sm, uint32_t* K, double* V,
                                                       uint32_t n) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    uint32_t masks[SM_ITEMS];
    uint32_t heads = 0;
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t i = elem_idx(it);
        bool h = false;
        if (i < n) {
            const uint32_t key = K[i];
            h = i == 0 || K[i - 1] != key;
            if (h && i + 1 < n && K[i + 1] == key) {
                // a head sums its run into its own slot (only it reads it)
                double s = V[i];
                for (uint32_t e = i + 1; e < n && K[e] == key; ++e) s += V[e];
                V[i] = s;
            }
        }
        masks[it] = __ballot_sync(FULL, h);
        heads += __popc(masks[it]);
    }
    uint32_t tot;
    uint32_t base = block_exclusive_scan<SM_NT>(lane == 0 ? heads : 0u, sm.s_warp32, tot);
    base = __shfl_sync(FULL, base, 0);
    // (block_exclusive_scan ends with a barrier: every run sum is in place)
    uint32_t hk[SM_ITEMS];
    double hv[SM_ITEMS];
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t i = elem_idx(it);
        if ((masks[it] >> lane) & 1u) {
            hk[it] = K[i];
            hv[it] = V[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        if ((masks[it] >> lane) & 1u) {
            const uint32_t u = base + __popc(masks[it] & lt);
            K[u] = hk[it];
            V[u] = hv[it];
        }
        base += __popc(masks[it]);
    }
    __syncthreads();
    return tot;
}

// Duplicate-heavy bin: sum duplicates in a shared-memory hash built in the
// bin's own buffer (the tuples are in registers), then compact the distinct
// (key, sum) pairs back to K/V[0, distinct). Returns the distinct count.
__device__ __noinline__ uint32_t hash_premerge(SortSmem& sm, uint32_t* K, double* V, uint32_t n) {
    const int tid = threadIdx.x;
    uint32_t kr[SM_ITEMS];
    double vr[SM_ITEMS];
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t idx = elem_idx(it);
        kr[it] = idx < n ? K[idx] : 0u;
        vr[it] = idx < n ? V[idx] : 0.0;
    }
    __syncthreads();  // every thread holds its tuples: the buffer becomes the table
    for (uint32_t i = tid; i < SM_CAP; i += SM_NT) {
        K[i] = 0xffffffffu;
        V[i] = 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        if (elem_idx(it) < n) {
            const uint32_t key = kr[it];
            uint32_t h = (key * 0x9E3779B1u) >> (32 - __builtin_ctz(SM_CAP));
            while (true) {
                const uint32_t old = atomicCAS(&K[h], 0xffffffffu, key);
                if (old == 0xffffffffu || old == key) {
                    atomicAdd(&V[h], vr[it]);
                    break;
                }
                h = (h + 1) & (SM_CAP - 1);
            }
        }
    }
    __syncthreads();
    // compact occupied slots (SM_ITEMS consecutive slots per thread)
    uint32_t hk[SM_ITEMS];
    double hv[SM_ITEMS];
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < SM_ITEMS; ++j) {
        hk[j] = K[tid * SM_ITEMS + j];
        hv[j] = V[tid * SM_ITEMS + j];
        c += hk[j] != 0xffffffffu;
    }
    uint32_t tot;
    uint32_t o = block_exclusive_scan<SM_NT>(c, sm.s_warp32, tot);  // ends with a barrier
#pragma unroll
    for (int j = 0; j < SM_ITEMS; ++j) {
        if (hk[j] != 0xffffffffu) {
            K[o] = hk[j];
            V[o] = hv[j];
            ++o;
        }
    }
    __syncthreads();
    return tot;
}

__device__ __forceinline__ bool st_inc(uint64_t s) { return (s >> 62) == 2; }

// The previous bin of an iteration and what happens to it: its output goes
// to C if its prefix is known, else it is parked (see Parked).
struct OutHook {
    bool have_prev;
    bool decided;   // thread 0 decided inside the sort (before its last barrier)
    uint32_t pU;
    uint64_t pb;
    uint64_t pst;   // thread 0: status word of pb (loaded early)
    uint64_t pk0, pk1;  // thread 0: status words of the two oldest parked bins
    uint32_t tk;        // thread 0: ticket of the CTA's next work bin
    int mn;             // its descriptor slot
    bool fetched;       // its descriptor fetch was issued inside the sort
};

// Thread 0: decide the output phase from the status words. Parked bins whose
// prefixes arrived are resolved (oldest first); the previous bin is written
// or parked (waiting only when the ring is full). With `drain`, waits until
// everything resolves (kernel end). The decision lands in shared memory.
__device__ void decide_output(const SortArgs& a, SortSmem& sm, const OutHook& h, bool drain) {
    const uint32_t cnt = sm.pk_count, head = sm.pk_head;
    // the two oldest parked bins (statuses loaded early; they resolve in order)
    uint32_t nres = 0;
    if (cnt > 0 && st_inc(h.pk0)) {
        sm.pk_P[0] = (h.pk0 & ST_VAL) - sm.pk[head].U;
        nres = 1;
        if (cnt > 1 && st_inc(h.pk1)) {
            sm.pk_P[1] = (h.pk1 & ST_VAL) - sm.pk[(head + 1) % PK_MAX].U;
            nres = 2;
        }
    }
    uint32_t park = 0;
    if (h.have_prev) {
        uint64_t s = h.pst;
#ifdef PBG_DIAG_NOWAIT  // timing experiment only: output at the tuple offset (wrong CSR)
        s = ST_INC | (sm.meta[0].n * 0 + h.pU + a.w.off[h.pb]);
#endif
        if (a.force_park && !drain && cnt - nres < PK_MAX) s = 0;
        if (st_inc(s) || drain) {
            while (!st_inc(s)) {
                __nanosleep(64);
                s = ld_relaxed_gpu(&a.status[h.pb]);
            }
            sm.s_pbP = (s & ST_VAL) - h.pU;
        } else {
            park = 1;
            if (cnt - nres == PK_MAX) {  // ring full: wait for the oldest
                const Parked& e = sm.pk[head % PK_MAX];
                uint64_t so = ld_relaxed_gpu(&a.status[e.bin]);
                while (!st_inc(so)) {
                    __nanosleep(64);
                    so = ld_relaxed_gpu(&a.status[e.bin]);
                }
                sm.pk_P[0] = (so & ST_VAL) - e.U;
                nres = 1;
            }
        }
    }
    if (drain) {  // every parked bin (they resolve in order)
        for (uint32_t i = nres; i < cnt; ++i) {
            const Parked& e = sm.pk[(head + i) % PK_MAX];
            uint64_t so = ld_relaxed_gpu(&a.status[e.bin]);
            while (!st_inc(so)) {
                __nanosleep(64);
                so = ld_relaxed_gpu(&a.status[e.bin]);
            }
            sm.pk_P[i] = (so & ST_VAL) - e.U;
        }
        nres = cnt;
    }
    sm.s_nres = nres;
    sm.s_park = park;
}

// Sort + merge the n tuples of buffer `buf` in place. Returns the merged count.
__device__ uint32_t sort_merge_bin(const SortArgs& a, SortSmem& sm, int buf, uint32_t n,
                                   int bits, uint32_t keylo, OutHook& hk, long long& prof_t) {
    const int tid = threadIdx.x;
    uint32_t* K = sm.k[buf];
    double* V = sm.v[buf];
    const int sh = bits > SM_NB_BITS ? bits - SM_NB_BITS : 0;
#if defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 1  // timing experiments only (wrong output)
    return n;
#endif
    // keys live in registers through the sort; values are read just before
    // the final write (V keeps the input order until then)
    uint32_t kr[SM_ITEMS];
    double vr[SM_ITEMS];
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t idx = elem_idx(it);
        kr[it] = idx < n ? K[idx] : 0u;
    }
    // ---- duplicate-heavy bins (CTA-local guess from its previous bin) ----
    bool pm = false;
    if (sm.s_dupheavy && n >= 64) {
        pm = true;
        const uint32_t u = hash_premerge(sm, K, V, n);
        if (tid == 0) atomicAdd(a.premerged, 1ull);
        // keep the guess while the pre-merge removes at least half the tuples
        const bool heavy = u * 2 <= n;
        n = u;
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = elem_idx(it);
            kr[it] = idx < n ? K[idx] : 0u;
        }
        __syncthreads();
        if (tid == 0) sm.s_dupheavy = heavy;
    }
    // ---- 1. bucket histogram; the atomic returns the tuple's bucket slot ----
    uint32_t slot[SM_ITEMS];
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        slot[it] = 0;
        if (elem_idx(it) < n) slot[it] = cnt_inc(sm, (kr[it] - keylo) >> sh);
    }
    __syncthreads();
    uint32_t crowded = scan_cnt(sm);  // counter d = start of bucket d
    PROF_MARK(1);
    if (crowded * 4 >= n && n >= 256 && !pm) {
        // duplicate-heavy: pre-merge, then start over on the distinct keys
        __syncthreads();
        pm = true;
        const uint32_t u = hash_premerge(sm, K, V, n);
        if (tid == 0) {
            atomicAdd(a.premerged, 1ull);
            sm.s_dupheavy = u * 2 <= n;
        }
        n = u;
        zero_cnt(sm);
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = elem_idx(it);
            kr[it] = idx < n ? K[idx] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            slot[it] = 0;
            if (elem_idx(it) < n) slot[it] = cnt_inc(sm, (kr[it] - keylo) >> sh);
        }
        __syncthreads();
        scan_cnt(sm);
    }
    // values of this thread's tuples (input order) before anything moves
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t idx = elem_idx(it);
        vr[it] = idx < n ? V[idx] : 0.0;
    }
    __syncthreads();
#if defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 2
    return n;
#endif
    // ---- 2. tuples to their buckets ----
    bool dz = false;
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        if (elem_idx(it) < n) {
            dz |= slot[it] != 0;
            const uint32_t p = slot[it] + cnt_get(sm, (kr[it] - keylo) >> sh);
            K[p] = kr[it];
            V[p] = vr[it];
        }
    }
    if (sh == 0) {
        // a bucket is a single key: bucket order is sorted order, nothing to
        // rank (duplicate-heavy key ranges, e.g. RMAT heavy-row pieces)
        if (__syncthreads_or(dz)) return merge_dups_inplace(sm, K, V, n);
        return n;
    }
    __syncthreads();
#if defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 3
    return n;
#endif
    if (tid == 0) meta_fetch(a, sm, hk.mn, hk.tk, *a.nw_dev);  // lands while this bin sorts
    hk.fetched = true;
    PROF_MARK(2);
    // previous bin's status, fresh (consumed by decide_output below)
    if (tid == 0) {
        if (hk.have_prev && !st_inc(hk.pst)) hk.pst = ld_relaxed_gpu(&a.status[hk.pb]);
        const uint32_t c = sm.pk_count;
        if (c > 0) hk.pk0 = ld_relaxed_gpu(&a.status[sm.pk[sm.pk_head].bin]);
        if (c > 1) hk.pk1 = ld_relaxed_gpu(&a.status[sm.pk[(sm.pk_head + 1) % PK_MAX].bin]);
    }
    // ---- 3. rank inside the bucket, by position ----
    // Thread-owned positions p (bank-conflict free); the bucket of K[p] is a
    // few positions around p, so the compare loop and the final write stay
    // near p too. f = lo + (smaller keys) + (equal keys earlier in the
    // bucket) is the sorted position; eqb > 0 marks a duplicate that is not
    // the first of its key (a "non-head"). Non-heads are rare (C2: one in
    // ~9000 tuples): their sorted positions go to a short list, every head
    // computes its merged position u = f - (non-heads before f) and each
    // non-head adds its value into its head's slot — the two-pointer merge
    // (pb_spgemm.hpp:202-216) without a compaction pass. A tuple alone in its
    // bucket (~60 %) is already in place.
    bool big = false;
    uint32_t moved = 0;  // bit it: tuple it changes position
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t p = elem_idx(it);
        slot[it] = p;
        if (p < n) {
            const uint32_t key = K[p];
            kr[it] = key;
            const uint32_t d = (key - keylo) >> sh;
            const uint32_t w = sm.cnt[d >> 1];
            const uint32_t lo = (w >> ((d & 1) * 16)) & 0xffffu;
            const uint32_t hi = (d & 1) ? (d + 1 < SM_NB ? (sm.cnt[(d + 1) >> 1] & 0xffffu) : n) : (w >> 16);
            if (hi - lo > 1) {
                vr[it] = V[p];
                if (hi - lo > (pm ? SM_BMAX_PM : SM_BMAX)) {
                    big = true;
                } else {
                    uint32_t lt = 0, eqb = 0;
#pragma unroll 1
                    for (uint32_t j = lo; j < hi; ++j) {
                        const uint32_t kj = K[j];
                        lt += kj < key;
                        eqb += (kj == key) & (j < p);
                    }
                    const uint32_t f = lo + lt + eqb;
                    slot[it] = f | eqb << 16;
                    moved |= (f != p) << it;
                    if (eqb) {
                        moved |= 1u << it;
                        const uint32_t q = atomicAdd(&sm.nh_cnt, 1u);
                        if (q < SM_NHMAX) sm.nh_pos[q] = static_cast<uint16_t>(f);
                    }
                }
            }
        }
    }
    PROF_MARK(7);
    // the output decision for the previous bin rides on this barrier
    if (tid == 0) decide_output(a, sm, hk, false);
    hk.decided = true;
    const bool any_big = __syncthreads_or(big);
    PROF_MARK(3);
#if defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 4
    if (slot[0] == 0xfffffff && vr[0] == 1.2345) K[0] = 7;  // keep the rank live
    return n;
#endif
    if (any_big) {
        // clustered keys: stable LSD radix sort of the bucket-ordered bin
        lsd_sort(sm, K, V, n, bits, keylo);
        if (tid == 0) atomicAdd(a.fallbacks, 1ull);
        bool d2 = false;
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t i = elem_idx(it);
            d2 |= i > 0 && i < n && K[i] == K[i - 1];
        }
        if (__syncthreads_or(d2)) return merge_dups_inplace(sm, K, V, n);
        return n;
    }
    const uint32_t nh = sm.nh_cnt;
    if (nh == 0) {
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            if ((moved >> it) & 1u) {
                K[slot[it]] = kr[it];
                V[slot[it]] = vr[it];
            }
        }
        return n;
    }
    // tuples that stay in place need their value for the merged write
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t p = elem_idx(it);
        if (p < n && !((moved >> it) & 1u)) vr[it] = V[p];
    }
    if (nh > SM_NHMAX) {  // many duplicates: sorted write, then a merge pass
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            if (elem_idx(it) < n) {
                K[slot[it] & 0xffffu] = kr[it];
                V[slot[it] & 0xffffu] = vr[it];
            }
        }
        __syncthreads();
        return merge_dups_inplace(sm, K, V, n);
    }
    // heads at their merged positions, then non-heads add into their head
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        if (elem_idx(it) < n && (slot[it] >> 16) == 0) {
            const uint32_t f = slot[it];
            uint32_t before = 0;
            for (uint32_t q = 0; q < nh; ++q) before += sm.nh_pos[q] < f;
            K[f - before] = kr[it];
            V[f - before] = vr[it];
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        if (elem_idx(it) < n && (slot[it] >> 16) != 0) {
            const uint32_t fh = (slot[it] & 0xffffu) - (slot[it] >> 16);  // the head's sorted position
            uint32_t before = 0;
            for (uint32_t q = 0; q < nh; ++q) before += sm.nh_pos[q] < fh;
            atomicAdd(&V[fh - before], vr[it]);
        }
    }
    return n - nh;
}

// Write a work bin: colids / values at P, rowptr of the rows it starts.
__device__ __forceinline__ void write_bin(const SortArgs& a, const SortSmem& sm, int buf,
                                          uint64_t b, uint64_t nw, uint32_t rs, uint32_t span,
                                          uint32_t U, uint64_t P) {
    const int tid = threadIdx.x;
    const int cb = a.col_bits;
    const uint32_t colmask = cb >= 32 ? 0xffffffffu : ((1u << cb) - 1u);
    const uint32_t* K = sm.k[buf];
    const double* V = sm.v[buf];
    uint32_t* okeys = a.ccol + P;
    double* ovals = a.cval + P;
#if !(defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 5)
    for (uint32_t u = tid; u < U; u += SM_NT) {
#ifdef PBG_PLAIN_ST
        okeys[u] = K[u] & colmask;
        ovals[u] = V[u];
#else
        __stcs(okeys + u, K[u] & colmask);
        __stcs(ovals + u, V[u]);
#endif
    }
#endif
    // rowptr[rs + r] = P + first merged entry of local row r (binary search)
#if defined(PBG_DIAG_SORT) && PBG_DIAG_SORT == 6
    span = 0;
#endif
    for (uint32_t r = tid; r < span; r += SM_NT) {
        const uint64_t target = static_cast<uint64_t>(r) << cb;
        uint32_t lo = 0, hi = U;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (static_cast<uint64_t>(K[mid]) < target) lo = mid + 1;
            else hi = mid;
        }
        a.rowptr[rs + r] = P + lo;
    }
    if (tid == 0 && b == nw - 1) a.rowptr[a.m] = P + U;
}

// A MERGED heavy sub-bin (k_hv_dense: already sorted, duplicates summed, may
// exceed SM_CAP): copied from global memory straight to C.
__device__ void write_merged(const SortArgs& a, const BinMeta& m, uint64_t b, uint64_t nw,
                             uint64_t P, uint32_t U) {
    const int tid = threadIdx.x;
    const int cb = a.col_bits;
    const uint32_t colmask = cb >= 32 ? 0xffffffffu : ((1u << cb) - 1u);
    const uint32_t* K = ((m.flags & 1u) ? a.skeys : a.keys) + m.off;
    const double* V = ((m.flags & 1u) ? a.svals : a.vals) + m.off;
    for (uint32_t u = tid; u < U; u += SM_NT) {
        __stcs(a.ccol + P + u, K[u] & colmask);
        __stcs(a.cval + P + u, V[u]);
    }
    if (tid == 0) {
        if (m.span) a.rowptr[m.rs] = P;  // single-row sub-bin owning the row start
        if (b == nw - 1) a.rowptr[a.m] = P + U;
    }
}

// The scan over work bins: one warp of the grid's last CTA turns the
// published merged counts (ST_AGG) into inclusive prefixes (ST_INC) in work
// bin order, 256 bins per step. Sorting CTAs publish a count as soon as the
// bin is sorted (never waiting on anything), so the scan only ever waits for
// bins that are still being sorted; a CTA writing bin b one bin later finds
// its prefix already there. (Every CTA walking back to the nearest inclusive
// prefix itself — a decoupled look-back — cost ~25 % of the kernel: with
// one-bin lag the nearest inclusive prefix is ~one grid of bins back.)
#ifndef PBG_SCAN_T
#define PBG_SCAN_T 8
#endif
constexpr int SCAN_T = PBG_SCAN_T;  // bins per lane per step
__device__ void status_scanner(unsigned long long* status, uint64_t nw) {
    const int lane = threadIdx.x & 31;
    uint64_t base = 0, run = 0;
    while (base < nw) {
        uint64_t st[SCAN_T];
#pragma unroll
        for (int t = 0; t < SCAN_T; ++t) {
            const uint64_t tile = base + t * 32 + lane;
            st[t] = tile < nw ? ld_relaxed_gpu(&status[tile]) : ST_INC;
        }
        // bins ready in order: up to the first unpublished one
        int ready = 0;
        bool stop = false;
#pragma unroll
        for (int t = 0; t < SCAN_T; ++t) {
            if (!stop) {
                const uint32_t nr = __ballot_sync(FULL, (st[t] >> 62) == 0);
                if (nr) {
                    ready += __ffs(nr) - 1;
                    stop = true;
                } else {
                    ready += 32;
                }
            }
        }
        if (ready == 0) {
#ifndef PBG_SCAN_SLEEP
#define PBG_SCAN_SLEEP 128
#endif
            __nanosleep(PBG_SCAN_SLEEP);
            continue;
        }
#pragma unroll
        for (int t = 0; t < SCAN_T; ++t) {
            if (t * 32 < ready) {
                const int idx = t * 32 + lane;
                const uint64_t tile = base + idx;
                const bool mine = idx < ready && tile < nw;
                const uint64_t v = mine ? (st[t] & ST_VAL) : 0;
                const uint64_t incl = run + warp_inclusive_scan(v);
                // bin 0 publishes its own inclusive value (= its count)
                if (mine && (st[t] >> 62) == 1) st_relaxed_gpu(&status[tile], ST_INC | incl);
                run = __shfl_sync(FULL, incl, 31);
            }
        }
        base += static_cast<uint64_t>(ready);
    }
}

// Write a parked bin from its tuple range to C at P.
__device__ void write_parked(const SortArgs& a, const Parked& e, uint64_t nw, uint64_t P) {
    const BinMeta& m = e.m;
    if (m.flags & 2u) {
        write_merged(a, m, e.bin, nw, P, e.U);
        return;
    }
    const int tid = threadIdx.x;
    const int cb = a.col_bits;
    const uint32_t colmask = cb >= 32 ? 0xffffffffu : ((1u << cb) - 1u);
    const uint32_t* K = ((m.flags & 1u) ? a.skeys : a.keys) + m.off;
    const double* V = ((m.flags & 1u) ? a.svals : a.vals) + m.off;
    const uint32_t U = e.U;
    for (uint32_t u = tid; u < U; u += SM_NT) {
        __stcs(a.ccol + P + u, __ldcg(K + u) & colmask);
        __stcs(a.cval + P + u, __ldcg(V + u));
    }
    // rowptr holds the bin-local row starts written at park time
    for (uint32_t r = tid; r < m.span; r += SM_NT) a.rowptr[m.rs + r] += P;
    if (tid == 0 && e.bin == nw - 1) a.rowptr[a.m] = P + U;
}

// Output phase of one iteration (all threads): acts on thread 0's decision
// (made inside the sort when possible, else here behind one barrier): writes
// the resolved parked bins and the previous bin (buffer `buf`) to C, or
// parks the previous bin in its own tuple range. Ends with a barrier.
__device__ void output_phase(const SortArgs& a, SortSmem& sm, const OutHook& h, int mp, int buf,
                             uint64_t nw, bool drain) {
    const int tid = threadIdx.x;
    if (!h.decided) {
        if (tid == 0) decide_output(a, sm, h, drain);
        __syncthreads();
    }
    const uint32_t nres = sm.s_nres;
    for (uint32_t i = 0; i < nres; ++i)
        write_parked(a, sm.pk[(sm.pk_head + i) % PK_MAX], nw, sm.pk_P[i]);
    const uint64_t pb = h.pb;
    const uint32_t pU = h.pU;
    if (h.have_prev) {
        const BinMeta& m = sm.meta[mp];
        if (!sm.s_park) {
            if (m.flags & 2u) write_merged(a, m, pb, nw, sm.s_pbP, pU);
            else write_bin(a, sm, buf, pb, nw, m.rs, m.span, pU, sm.s_pbP);
        } else if (!(m.flags & 2u)) {
            // store the sorted bin into its own tuple range (it stays in L2
            // until written out) and its bin-local row starts into rowptr
            uint32_t* K = ((m.flags & 1u) ? a.skeys : a.keys) + m.off;
            double* V = ((m.flags & 1u) ? a.svals : a.vals) + m.off;
            for (uint32_t u = tid; u < pU; u += SM_NT) {
                __stcg(K + u, sm.k[buf][u]);
                __stcg(V + u, sm.v[buf][u]);
            }
            const int cb = a.col_bits;
            for (uint32_t r = tid; r < m.span; r += SM_NT) {
                const uint64_t target = static_cast<uint64_t>(r) << cb;
                uint32_t lo = 0, hi = pU;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (static_cast<uint64_t>(sm.k[buf][mid]) < target) lo = mid + 1;
                    else hi = mid;
                }
                a.rowptr[m.rs + r] = lo;
            }
        }
    }
    if (tid == 0) cp_async_wait_all();
    __syncthreads();  // buffer `buf` and the resolved ring slots are free
    if (tid == 0) {
        uint32_t head = (sm.pk_head + nres) % PK_MAX, cnt = sm.pk_count - nres;
        if (h.have_prev && sm.s_park) {
            Parked& e = sm.pk[(head + cnt) % PK_MAX];
            e.m = sm.meta[mp];
            e.bin = pb;
            e.U = pU;
            ++cnt;
            atomicAdd(a.parked, 1ull);
        }
        sm.pk_head = head;
        sm.pk_count = cnt;
    }
}

#ifndef PBG_SM_MINB
#define PBG_SM_MINB (SM_NT >= 1024 ? 1 : 1024 / SM_NT)
#endif
__global__ void __launch_bounds__(SM_NT, PBG_SM_MINB) k_sortmerge(SortArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint64_t nw = *a.nw_dev;
    if (blockIdx.x == gridDim.x - 1) {  // the work-bin scan (the grid is co-resident)
        if (tid < 32) status_scanner(a.status, nw);
        return;
    }
    // CTA-local bin sequence j = 0, 1, ...: bin j lives in buffer j % SM_NBUF
    // and descriptor slot j % SM_NMETA. Iteration i sorts bin i, writes bin
    // i - SM_LAG and starts the copy of bin i + SM_PF + 1 into the buffer
    // that frees up.
    if (tid == 0) {
        for (int q = 0; q < SM_NBUF; ++q) mbar_init(&sm.mbar[q], 1);
        sm.s_dupheavy = 0;
        sm.pk_head = 0;
        sm.pk_count = 0;
        for (int j = 0; j <= SM_PF; ++j) meta_fetch(a, sm, j, atomicAdd(a.ticket, 1u), nw);
        cp_async_wait_all();
        for (int j = 0; j <= SM_PF; ++j)
            if (sm.s_bin[j] < nw && bin_kind(sm.meta[j]) == 1) issue_tma(a, sm, j, sm.meta[j]);
    }
    __syncthreads();
    long long prof_t = clock64();
    (void)prof_t;
    uint32_t phase_bits = 0;  // mbarrier parity per buffer
    uint32_t i = 0;
    for (;; ++i) {
        const int cur = i % SM_NBUF, mc = i % SM_NMETA;
        const uint64_t b = sm.s_bin[mc];
        if (b >= nw) break;
        const BinMeta& M = sm.meta[mc];
        const uint32_t kind = bin_kind(M);
        const bool have_prev = i >= SM_LAG;
        const int pbuf = (i + SM_NBUF - SM_LAG) % SM_NBUF;   // buffer of bin i - LAG
        const int pm = (i + SM_NMETA - SM_LAG) % SM_NMETA;   // its descriptor
        const uint64_t pb = have_prev ? sm.s_bin[pm] : 0;
        const uint32_t pU = have_prev ? sm.pend_U[pbuf] : 0;
        // bin i - LAG's status (its prefix is usually there by now) and the
        // ticket of bin i + PF + 1, both consumed later
        OutHook hk{have_prev, false, pU, pb,
                   (have_prev && tid == 0) ? ld_relaxed_gpu(&a.status[pb]) : 0, 0, 0,
                   tid == 0 ? atomicAdd(a.ticket, 1u) : 0u, static_cast<int>((i + SM_PF + 1) % SM_NMETA),
                   false};
        if (tid == 0 && M.n > SM_CAP && !(M.flags & 2u)) atomicOr(a.err, 2u);
        uint32_t U = 0;
        if (kind) {
            const uint32_t n = static_cast<uint32_t>(M.n);
            zero_cnt(sm);
            if (tid == 0) sm.nh_cnt = 0;
            if (kind == 1) {
                mbar_wait(&sm.mbar[cur], (phase_bits >> cur) & 1u);
                phase_bits ^= 1u << cur;
            } else {  // unaligned heavy sub-bin: plain coalesced loads
                const uint32_t* ks = ((M.flags & 1u) ? a.skeys : a.keys) + M.off;
                const double* vs = ((M.flags & 1u) ? a.svals : a.vals) + M.off;
                for (uint32_t e = tid; e < n; e += SM_NT) {
                    sm.k[cur][e] = ks[e];
                    sm.v[cur][e] = vs[e];
                }
            }
            __syncthreads();
            PROF_MARK(0);
            U = sort_merge_bin(a, sm, cur, n, static_cast<int>(M.keybits), M.keylo, hk, prof_t);
#ifdef PBG_SORT_PROF
            __syncthreads();  // (profile builds: the final write's barrier wait)
#endif
            PROF_MARK(4);
        } else if (M.flags & 2u) {
            U = static_cast<uint32_t>(M.n);
        }
        PROF_MARK(9);
        if (tid == 0) {
            // publish this bin's count now (a count needs no ordering with
            // other memory: relaxed); its output goes out SM_LAG bins later
            st_relaxed_gpu(&a.status[b], (b == 0 ? ST_INC : ST_AGG) | (U & ST_VAL));
            atomicAdd(a.merged_total, (unsigned long long)U);
            sm.pend_U[cur] = U;
            if (!hk.fetched) meta_fetch(a, sm, hk.mn, hk.tk, nw);
        }
        output_phase(a, sm, hk, pm, pbuf, nw, false);
        PROF_MARK(5);
        // the buffer just written out receives bin i + PF + 1
        if (tid == 0 && sm.s_bin[hk.mn] < nw && bin_kind(sm.meta[hk.mn]) == 1)
            issue_tma(a, sm, pbuf, sm.meta[hk.mn]);
    }
    // drain: the last SM_LAG sorted bins, then every parked bin
    for (int q = SM_LAG; q >= 1; --q) {
        if (i < static_cast<uint32_t>(q)) continue;
        const uint32_t j = i - q;
        const int pbuf = j % SM_NBUF, pm = j % SM_NMETA;
        OutHook hk{true, false, sm.pend_U[pbuf], sm.s_bin[pm], 0, 0, 0, 0, 0, true};
        output_phase(a, sm, hk, pm, pbuf, nw, q == 1);
    }
    if (i == 0 || SM_LAG == 0) {
        OutHook hk{false, false, 0, 0, 0, 0, 0, 0, 0, true};
        output_phase(a, sm, hk, 0, 0, nw, true);
    }
}

}  // namespace pbg
