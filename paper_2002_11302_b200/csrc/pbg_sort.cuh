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
//   0. the bin arrives in shared memory by two TMA bulk copies
//      (cp.async.bulk, mbarrier completion) issued while the CTA was still
//      busy with the previous bin;
//   1. MSD bucket pass: SM_CAP buckets on the top used key bits (smem
//      histogram -> scan -> scatter) — the reference's first radix level,
//      wide enough that buckets hold ~1 tuple;
//   2. rank inside the bucket (smaller keys, ties by position): every tuple
//      lands at its sorted position. A bucket above SM_BMAX (clustered or
//      duplicate-heavy keys) switches the bin to a stable LSD radix sort;
//   3. duplicate keys are summed (two-pointer merge semantics: exact zeros
//      are kept) and compacted;
//   4. colids / values / rowptr are written at the bin's output offset P_b,
//      known before the kernel starts (k_bincount counts each bin's
//      distinct keys, a scan turns them into offsets), so bins are fully
//      independent: no look-back chain, no waiting on slower neighbours.
//      (A single-pass decoupled look-back over U_b was measured 2-3x slower:
//      per-bin work is long and uneven, so every CTA ended up waiting on the
//      slowest in-flight predecessor; a one-bin-lagged variant tied.)
//      A bin the count found duplicate-free skips the duplicate check, is
//      ranked in final form (masked column ids at a shared-memory offset
//      congruent to its place in C modulo 16 B) and leaves through TMA bulk
//      stores (cp.async.bulk shared -> global); its row starts come from
//      the MSD bucket ends. Work-bin descriptors are staged by cp.async one
//      bin ahead.
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

constexpr int SM_NT = PBG_SM_NT;
constexpr int SM_NW = SM_NT / 32;
constexpr int SM_CAP = PBG_SM_CAP;            // max tuples per smem bin
#ifndef PBG_SM_NB
#define PBG_SM_NB PBG_SM_CAP
#endif
constexpr int SM_NB = PBG_SM_NB;              // buckets of the MSD pass (u16 counters)
constexpr int SM_CQ = SM_NB * 2 / 16 / SM_NT; // uint4s of counters per thread
constexpr int SM_NB_BITS = __builtin_ctz(SM_NB);
#ifndef PBG_SM_BMAX
#define PBG_SM_BMAX 512
#endif
// largest bucket ranked in place (its rank loop is quadratic; beyond it the bin
// takes the LSD radix, whose match.any ranking is far slower per key: with 128
// a C5b band sent 30.8 K heavy sub-bins there — hot columns repeated > 128
// times — and its sort took 27.4 instead of 26.2 ms)
constexpr int SM_BMAX = PBG_SM_BMAX;
// hash pre-merge of a bin when distinct * NUM <= tuples * DEN (tuning hook)
#ifndef PBG_PM_NUM
#define PBG_PM_NUM 4
#endif
#ifndef PBG_PM_DEN
#define PBG_PM_DEN 3
#endif
#ifndef PBG_RANK_UNROLL
#define PBG_RANK_UNROLL 1
#endif
#ifndef PBG_HIST_UNROLL
#define PBG_HIST_UNROLL 1
#endif
#ifndef PBG_SCAT_UNROLL
#define PBG_SCAT_UNROLL 1
#endif
constexpr int RANK_UNROLL = PBG_RANK_UNROLL;  // tuning hooks (A/B)
constexpr int SCAT_UNROLL = PBG_SCAT_UNROLL;
constexpr int HIST_UNROLL = PBG_HIST_UNROLL;
constexpr int SM_ITEMS = SM_CAP / SM_NT;      // 8
constexpr int SM_PER_WARP = SM_CAP / SM_NW;
constexpr int SM_NBUF = 2;                    // ping, pong
static_assert(SM_ITEMS == 8, "one uint4 of u16 counters per thread");
static_assert(SM_CQ >= 1 && SM_CQ * 16 * SM_NT == SM_NB * 2, "counter scan layout");

struct SortArgs {
    WorkBins w;
    const uint64_t* nw_dev;   // number of work bins
    const uint64_t* wb_out;   // output offset of every work bin (scan of k_bincount)
    const uint64_t* wb_nnz;   // distinct keys per work bin (k_bincount), cross-checked
    unsigned int* ticket;
    const uint32_t* keys;     // tuples (main buffer)
    const double* vals;
    const uint32_t* skeys;    // tuples (heavy-row scratch buffer)
    const double* svals;
    uint32_t* ccol;           // C colids
    double* cval;             // C values
    uint64_t* rowptr;
    uint64_t m;
    uint64_t c_cap;           // entries the C arrays hold (PBG_CHECKED bound)
    int col_bits;
    unsigned long long* merged_total;
    unsigned int* err;  // bit1 work bin above capacity, bit2 merged != distinct count
    unsigned long long* fallbacks;
    unsigned long long* prof;  // PBG_SORT_PROF builds: cycles per phase (thread 0 of each CTA)
};

#ifdef PBG_SORT_PROF
#define PROF_MARK(i)                                                  \
    do {                                                              \
        if (threadIdx.x == 0) {                                       \
            const long long t_ = clock64();                           \
            atomicAdd(&a.prof[i], (unsigned long long)(t_ - prof_t)); \
            prof_t = t_;                                              \
        }                                                             \
    } while (0)
#else
#define PROF_MARK(i) \
    do {             \
    } while (0)
#endif

// Work-bin descriptor staged in shared memory by thread 0 (cp.async, one bin
// ahead: no warp waits on these loads).
struct BinMeta {
    uint64_t n, off, out, nnz;
    uint32_t flags, keybits, keylo, rs, span, pad;
};

struct SortSmem {
    // +4 / +2 slack: a duplicate-free bin is written sorted at an offset that
    // aligns it with its 16-byte-aligned place in C (TMA bulk store)
    uint32_t k[SM_NBUF][SM_CAP + 4];
    double v[SM_NBUF][SM_CAP + 2];
    uint16_t cnt[SM_NB];  // bucket histogram -> bucket ends; LSD per-warp counters
    uint32_t s_warp32[SM_NW + 1];
    unsigned long long mbar;
    uint64_t s_bin[2];
    BinMeta meta[2];  // current / next work bin (descriptors staged by cp.async)
};

// Thread 0: work bin b (its ticket taken a while ago) becomes descriptor
// slot `slot`; it arrives asynchronously (cp_async_wait_all + a barrier).
__device__ __forceinline__ void meta_fetch(const SortArgs& a, SortSmem& sm, int slot, uint64_t b,
                                           uint64_t nw) {
    sm.s_bin[slot] = b;
    if (b >= nw) return;
    BinMeta& m = sm.meta[slot];
    cp_async8(&m.n, a.w.n + b);
    cp_async8(&m.off, a.w.off + b);
    cp_async8(&m.out, a.wb_out + b);
    cp_async8(&m.nnz, a.wb_nnz + b);
    cp_async4(&m.flags, a.w.flags + b);
    cp_async4(&m.keybits, a.w.keybits + b);
    cp_async4(&m.keylo, a.w.keylo + b);
    cp_async4(&m.rs, a.w.rs + b);
    cp_async4(&m.span, a.w.span + b);
}

// How a work bin reaches shared memory: 1 = TMA bulk copy, 0 = nothing to
// load (empty / merged / error). A heavy sub-bin may start at any tuple: its
// copy starts at the 16-byte boundary below, so the bin sits (off & 3) keys /
// (off & 1) values into the buffer (the buffers' slack covers the shift).
// A MERGED sub-bin (k_hv_dense: sorted, duplicates summed, <= 4096 entries)
// takes the same route and is written out unsorted-path-free.
__device__ __forceinline__ uint32_t bin_kind(const BinMeta& m) {
    if (m.n == 0 || m.n > SM_CAP) return 0;
    return 1;
}

// Thread 0: start the TMA copy of a kind-1 bin into buffer `buf` (generic-
// proxy accesses to it are finished: caller syncs).
__device__ __forceinline__ void issue_tma(const SortArgs& a, SortSmem& sm, int buf,
                                          const BinMeta& m) {
    const uint32_t* ks = (m.flags & 1u) ? a.skeys : a.keys;
    const double* vs = (m.flags & 1u) ? a.svals : a.vals;
    const uint64_t sk = m.off & 3u, sv = m.off & 1u;
    const uint32_t kb = static_cast<uint32_t>(((m.n + sk) * 4 + 15) & ~15ull);
    const uint32_t vb = static_cast<uint32_t>(((m.n + sv) * 8 + 15) & ~15ull);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&sm.mbar, kb + vb);
    bulk_g2s(sm.k[buf], ks + (m.off - sk), kb, &sm.mbar);
    bulk_g2s(sm.v[buf], vs + (m.off - sv), vb, &sm.mbar);
}

// Exclusive scan of the SM_NB u16 counters in index order (8 per thread).
__device__ __forceinline__ void scan_cnt(SortSmem& sm) {
    const int tid = threadIdx.x;
    uint4* c4 = reinterpret_cast<uint4*>(sm.cnt) + SM_CQ * tid;
    uint32_t rw[4 * SM_CQ];
#pragma unroll
    for (int q = 0; q < SM_CQ; ++q) {
        const uint4 raw = c4[q];
        rw[4 * q] = raw.x;
        rw[4 * q + 1] = raw.y;
        rw[4 * q + 2] = raw.z;
        rw[4 * q + 3] = raw.w;
    }
    uint32_t s8 = 0;
#pragma unroll
    for (int j = 0; j < 4 * SM_CQ; ++j) s8 += (rw[j] & 0xffffu) + (rw[j] >> 16);
    uint32_t tot;
    // (the caller's barrier after scan_cnt protects s_warp32)
    uint32_t run = block_exclusive_scan<SM_NT, uint32_t, false>(s8, sm.s_warp32, tot);
#pragma unroll
    for (int j = 0; j < 4 * SM_CQ; ++j) {
        const uint32_t lo = run;
        run += rw[j] & 0xffffu;
        const uint32_t hi = run;
        run += rw[j] >> 16;
        rw[j] = lo | (hi << 16);
    }
#pragma unroll
    for (int q = 0; q < SM_CQ; ++q)
        c4[q] = make_uint4(rw[4 * q], rw[4 * q + 1], rw[4 * q + 2], rw[4 * q + 3]);
}

__device__ __forceinline__ void zero_cnt(SortSmem& sm) {
    uint4* c4 = reinterpret_cast<uint4*>(sm.cnt) + SM_CQ * threadIdx.x;
#pragma unroll
    for (int q = 0; q < SM_CQ; ++q) c4[q] = make_uint4(0, 0, 0, 0);
}

// Stable LSD radix sort of buffer `x` (n <= SM_CAP) over `bits` key bits,
// 8-bit digits, ping-ponging with buffer `y`. Ranks from match.any per warp in
// element order, per-(warp, digit) counters cnt[w*256+d] scanned digit-major.
// Returns the buffer holding the result.
__device__ int lsd_sort(SortSmem& sm, int x, int y, uint32_t n, int bits, uint32_t keylo) {
    static_assert(SM_NW * 256 <= SM_NB, "LSD counters fit the bucket counters");
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t lt = lanemask_lt();
    int cur = x, nxt = y;
    uint32_t kr[SM_ITEMS];
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t idx = w * SM_PER_WARP + it * 32 + lane;
        kr[it] = idx < n ? sm.k[cur][idx] : 0u;
    }
    for (int shift = 0; shift < bits; shift += 8) {
        zero_cnt(sm);
        __syncthreads();
        uint16_t rank[SM_ITEMS];
        uint32_t dig[SM_ITEMS];
        uint16_t* wc = sm.cnt + w * 256;
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = w * SM_PER_WARP + it * 32 + lane;
            const bool valid = idx < n;
            const uint32_t d = valid ? (((kr[it] - keylo) >> shift) & 0xffu) : 0x100u;
            const uint32_t peers = __match_any_sync(FULL, d);
            const uint16_t old = valid ? wc[d] : 0;
            rank[it] = old + __popc(peers & lt);
            dig[it] = d;
            __syncwarp();
            if (valid && (peers & lt) == 0) wc[d] = old + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {  // digit-major exclusive scan over (digit, warp)
            constexpr int PER = SM_NW * 256 / SM_NT;  // counters per thread
            constexpr int TPD = SM_NW / PER;          // threads per digit
            const int d = tid / TPD, w0 = (tid % TPD) * PER;
            uint32_t c[PER], s = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                c[j] = sm.cnt[(w0 + j) * 256 + d];
                s += c[j];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan<SM_NT>(s, sm.s_warp32, tot);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                sm.cnt[(w0 + j) * 256 + d] = static_cast<uint16_t>(run);
                run += c[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = w * SM_PER_WARP + it * 32 + lane;
            if (idx < n) {
                const uint32_t pos = wc[dig[it]] + rank[it];
                sm.k[nxt][pos] = kr[it];
                sm.v[nxt][pos] = sm.v[cur][idx];
            }
        }
        __syncthreads();
        const int t = cur;
        cur = nxt;
        nxt = t;
#pragma unroll
        for (int it = 0; it < SM_ITEMS; ++it) {
            const uint32_t idx = w * SM_PER_WARP + it * 32 + lane;
            if (idx < n) kr[it] = sm.k[cur][idx];
        }
    }
    return cur;
}

// Sum equal-key runs of sorted buffer `x` into buffer `y`, compacted.
// Warp w owns elements [w*PER_WARP, +PER_WARP), lane-striped in windows of 32.
// A warp-shuffle segmented reduction sums each run's part inside a window
// into the window's first lane of that run (written back in place); the
// thread of a run's head then adds the leading partial of every following
// window the run covers: a key repeated r times costs its head r/32 adds
// instead of r (RMAT's hot columns repeat hundreds of times; the serial
// per-head loop was 29 % of the sort kernel on a C3 round).
// HV = false (no heavy rows in the product: duplicates are rare and short)
// keeps the plain per-head loop.
template <bool HV>
__device__ __forceinline__ uint32_t merge_dups(SortSmem& sm, int x, int y, uint32_t n) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t lt = lanemask_lt();
    const uint32_t* K = sm.k[x];
    double* V = sm.v[x];
    uint32_t* KO = sm.k[y];
    double* VO = sm.v[y];
    uint32_t masks[SM_ITEMS];
    uint32_t heads = 0;
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t i = w * SM_PER_WARP + it * 32 + lane;
        const bool in = i < n;
        const bool h = in && (i == 0 || K[i] != K[i - 1]);
        masks[it] = __ballot_sync(FULL, h);
        heads += __popc(masks[it]);
        if (!HV) continue;
        if (masks[it] == __ballot_sync(FULL, in)) continue;  // no duplicate inside this window
        // segment starts of the window: run heads and lane 0
        const uint32_t seg = masks[it] | 1u;
        double v = in ? V[i] : 0.0;
        const uint32_t above = seg >> 1 >> lane;  // bit j: lane + 1 + j starts a segment
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_down_sync(FULL, v, o);
            if (lane + o < 32 && (above & ((1u << o) - 1u)) == 0) v += t;
        }
        if (in && ((seg >> lane) & 1u)) V[i] = v;
    }
    uint32_t tot;
    // (the scan's barriers publish the windows' partial sums)
    uint32_t base = block_exclusive_scan<SM_NT>(lane == 0 ? heads : 0u, sm.s_warp32, tot);
    base = __shfl_sync(FULL, base, 0);
#pragma unroll
    for (int it = 0; it < SM_ITEMS; ++it) {
        const uint32_t i = w * SM_PER_WARP + it * 32 + lane;
        if ((masks[it] >> lane) & 1u) {
            const uint32_t u = base + __popc(masks[it] & lt);
            const uint32_t key = K[i];
            double s = V[i];
            if (HV) {
                for (uint32_t e = (i | 31u) + 1; e < n && K[e] == key; e += 32) s += V[e];
            } else {
                for (uint32_t e = i + 1; e < n && K[e] == key; ++e) s += V[e];
            }
            KO[u] = key;
            VO[u] = s;
        }
        base += __popc(masks[it]);
    }
    return tot;
}

// Duplicate-heavy bin (its distinct count from k_bincount is <= n/2, e.g.
// the 27-point stencil squared, cf ~ 6): group duplicates first through a
// shared-memory hash set (keys in buffer `scr`, load <= 1/2), then compact
// the distinct (key, sum) pairs back into `in`. Returns the distinct count.
// No floating-point atomics (an f64 atomicAdd on shared memory is a CAS spin
// loop): a tuple takes a rank in its slot with a u16 counter add, a scan
// turns the slot counts into group starts, values are scattered into their
// groups and each group is summed by the thread owning its slot.
template <bool HV>
__device__ uint32_t hash_premerge(const SortArgs& a, SortSmem& sm, int in, int scr, uint32_t n,
                                  const uint32_t* Kin, const double* Vin, long long& prof_t) {
    const int tid = threadIdx.x;
    constexpr uint32_t EMPTY = 0xffffffffu;
    uint32_t* HK = sm.k[scr];
    uint32_t* cntw = reinterpret_cast<uint32_t*>(sm.cnt);  // per-slot u16 counts -> starts
    for (uint32_t i = tid; i < SM_CAP; i += SM_NT) HK[i] = EMPTY;
    zero_cnt(sm);
    __syncthreads();
    PROF_MARK(8);
    uint32_t hr[SM_ITEMS];  // slot << 16 | rank of the tuple within its slot
#pragma unroll
    for (int j = 0; j < SM_ITEMS; ++j) {
        const uint32_t i = tid + j * SM_NT;
        hr[j] = EMPTY;
        if (i < n) {
            const uint32_t key = Kin[i];
            uint32_t h = (key * 0x9E3779B1u) >> (32 - __builtin_ctz(SM_CAP));
            while (true) {
                const uint32_t old = atomicCAS(&HK[h], EMPTY, key);
                if (old == EMPTY || old == key) break;
                h = (h + 1) & (SM_CAP - 1);
            }
            const uint32_t sh16 = (h & 1u) * 16;
            const uint32_t old = atomicAdd(&cntw[h >> 1], 1u << sh16);
            hr[j] = h << 16 | ((old >> sh16) & 0xffffu);
        }
    }
    __syncthreads();
    PROF_MARK(9);
    // this thread's slots [tid*8, tid*8+8): one uint4 of u16 counts
    static_assert(SM_NB == SM_CAP, "one u16 counter per hash slot");
    const uint4 raw = reinterpret_cast<const uint4*>(sm.cnt)[tid];
    const uint32_t cw[4] = {raw.x, raw.y, raw.z, raw.w};
    uint32_t occ = 0, tsum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t c = (cw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        occ += c != 0;
        tsum += c;
    }
    uint32_t tot;
    // (distinct, tuples) prefixes in one scan: both <= SM_CAP < 2^16. The
    // scan's barriers also end every read of the counters.
    const uint32_t ex = block_exclusive_scan<SM_NT>(occ << 16 | tsum, sm.s_warp32, tot);
    // per occupied slot: its group start replaces its key in HK (own slots
    // only), the key moves to in[d] and (start, count) to grp[d]
    // (d < n/2 <= SM_CAP/2: fits the counter array as u32)
    uint32_t* grp = reinterpret_cast<uint32_t*>(sm.cnt);
    {
        uint32_t d = ex >> 16, p = ex & 0xffffu;
        uint4* hk4 = reinterpret_cast<uint4*>(HK) + tid * 2;  // own 8 slots, 2 x 16 B
        const uint4 ka = hk4[0], kb = hk4[1];
        const uint32_t kk[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
        uint32_t st[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t c = (cw[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
            st[j] = p;
            if (c) {
                sm.k[in][d] = kk[j];
                grp[d] = p << 16 | c;
                ++d;
            }
            p += c;
        }
        hk4[0] = make_uint4(st[0], st[1], st[2], st[3]);
        hk4[1] = make_uint4(st[4], st[5], st[6], st[7]);
    }
    __syncthreads();
    PROF_MARK(10);
#pragma unroll
    for (int j = 0; j < SM_ITEMS; ++j) {
        if (hr[j] != EMPTY)
            sm.v[scr][HK[hr[j] >> 16] + (hr[j] & 0xffffu)] = Vin[tid + j * SM_NT];
    }
    __syncthreads();
    PROF_MARK(11);
    const uint32_t D = tot >> 16;
    if (!HV) {
        // one thread per distinct key sums its group
        for (uint32_t d = tid; d < D; d += SM_NT) {
            const uint32_t g = grp[d], p = g >> 16, c = g & 0xffffu;
            double s = sm.v[scr][p];
            for (uint32_t t = 1; t < c; ++t) s += sm.v[scr][p + t];
            sm.v[in][d] = s;
        }
        __syncthreads();
        return D;
    }
    // heavy rows: a group of PM_BIG or more (RMAT's hot columns repeat
    // hundreds of times in a bin, and the thread owning one kept the whole
    // CTA waiting) is queued and summed by a warp afterwards
    constexpr uint32_t PM_BIG = 64;
    uint32_t* bigq = sm.k[scr];  // the hash keys are dead: queue of big groups (index d)
    if (tid == 0) sm.s_warp32[0] = 0;
    __syncthreads();
    for (uint32_t d = tid; d < D; d += SM_NT) {
        const uint32_t g = grp[d], p = g >> 16, c = g & 0xffffu;
        if (c >= PM_BIG) {
            bigq[atomicAdd(&sm.s_warp32[0], 1u)] = d;
            continue;
        }
        double s = sm.v[scr][p];
        for (uint32_t t = 1; t < c; ++t) s += sm.v[scr][p + t];
        sm.v[in][d] = s;
    }
    __syncthreads();
    const uint32_t nbig = sm.s_warp32[0];
    for (uint32_t q = tid >> 5; q < nbig; q += SM_NW) {
        const uint32_t d = bigq[q];
        const uint32_t g = grp[d], p = g >> 16, c = g & 0xffffu;
        double s = -0.0;
        for (uint32_t t = tid & 31; t < c; t += 32) s += sm.v[scr][p + t];
        s = warp_sum(s);
        if ((tid & 31) == 0) sm.v[in][d] = s;
    }
    __syncthreads();
    return tot >> 16;
}

// (out of line: inlined, its queue pass pushed k_sortmerge<true> into spills)
__device__ __noinline__ uint32_t hash_premerge_heavy(const SortArgs& a, SortSmem& sm, int in, int scr,
                                                     uint32_t n, const uint32_t* Kin, const double* Vin,
                                                     long long& prof_t) {
    return hash_premerge<true>(a, sm, in, scr, n, Kin, Vin, prof_t);
}

// Sort + merge the bin in buffer `in` using scratch buffer `scr`. Returns the
// merged count; *res gets the buffer holding the merged output.
template <bool HV>
__device__ uint32_t sort_merge_bin(const SortArgs& a, SortSmem& sm, int in, int scr, uint32_t n,
                                   int bits, uint32_t keylo, uint32_t distinct, int* res,
                                   int* rshift, uint64_t P, int* bulk,
                                   int next_slot, uint64_t next_bin, uint32_t insk, uint32_t insv,
                                   long long& prof_t) {
    const int tid = threadIdx.x;
    *bulk = 0;
    // the bin as it arrived: insk keys / insv values into buffer `in`
    // (heavy sub-bins only: bins of the main buffer are 16-byte aligned)
    const uint32_t* Kin = sm.k[in] + (HV ? insk : 0u);
    const double* Vin = sm.v[in] + (HV ? insv : 0u);
    // the previous bin's bulk store reads buffer `scr`: done before it is written
    if (tid == 0) bulk_wait_read();
    // pre-merge threshold: distinct <= n/2 (the stencil: cf 5.8); heavy rows'
    // sub-bins (cf ~1.9, hot keys) gain from distinct <= 3n/4 (C3 sort -8 %)
    const bool premerge = HV ? (distinct * PBG_PM_NUM <= n * PBG_PM_DEN && distinct <= SM_CAP / 2)
                             : (distinct * 2 <= n);
    if (premerge && n >= 64) {
        __syncthreads();  // thread 0's bulk_wait_read before anyone writes `scr`
        // now n distinct keys, no duplicates
        n = HV ? hash_premerge_heavy(a, sm, in, scr, n, Kin, Vin, prof_t)
               : hash_premerge<false>(a, sm, in, scr, n, Kin, Vin, prof_t);
        Kin = sm.k[in];  // the distinct pairs sit at the buffer's start
        Vin = sm.v[in];
        zero_cnt(sm);
        __syncthreads();
        PROF_MARK(7);
    }
    uint32_t* cntw = reinterpret_cast<uint32_t*>(sm.cnt);
    const int sh = bits > SM_NB_BITS ? bits - SM_NB_BITS : 0;
    // ---- 1. bucket histogram / scan / scatter in -> scr ----
    // (keeping the histogram's returned slot in registers to save the second
    // atomic was measured slower: register pressure at 64 regs spills. Two
    // duplicate-free fast paths were built and measured slower at C2, both
    // writing every tuple at bucket start + the histogram atomic's arrival
    // rank in final form, then ordering buckets of 2+ tuples per owning
    // thread: an 8x8 register rank network 2.3 -> 3.4 ms, an in-place
    // insertion sort 2.4 -> 2.8 ms — per-thread bucket work is uneven, so
    // warps wait at the next barrier, and bank conflicts rise.)
#pragma unroll HIST_UNROLL
    for (uint32_t i = tid; i < n; i += SM_NT) {
        const uint32_t d = (Kin[i] - keylo) >> sh;
        atomicAdd(&cntw[d >> 1], 1u << ((d & 1) * 16));
    }
    __syncthreads();
    scan_cnt(sm);  // cnt[d] = start of bucket d
    __syncthreads();
    PROF_MARK(1);
    // the next bin's descriptor (its ticket was taken at the loop top)
    if (threadIdx.x == 0) meta_fetch(a, sm, next_slot, next_bin, *a.nw_dev);
#pragma unroll SCAT_UNROLL
    for (uint32_t i = tid; i < n; i += SM_NT) {
        const uint32_t key = Kin[i];
        const uint32_t d = (key - keylo) >> sh;
        const uint32_t old = atomicAdd(&cntw[d >> 1], 1u << ((d & 1) * 16));
        const uint32_t pos = (old >> ((d & 1) * 16)) & 0xffffu;
        PBG_DCHECK(pos < n);
        sm.k[scr][pos] = key;
        sm.v[scr][pos] = Vin[i];
    }
    __syncthreads();
    PROF_MARK(2);
    // cnt[d] is now the END of bucket d
    // ---- 2. rank inside buckets scr -> in ----
    // (a fixed +-3 neighbour window without loops was measured slower: the
    // loop runs ~2 trips for buckets of ~1 tuple)
    bool big = false;
    if (sh == 0) {
        // a bucket is a single key: bucket order is sorted order, nothing to
        // rank (duplicate-heavy keys, e.g. RMAT heavy-row pieces)
        __syncthreads();
        *res = scr;
        *rshift = 0;  // row starts from the bucket ends if nothing merges
        if (distinct < n) {  // exact count: duplicates present
            *res = in;
            *rshift = -1;
            return merge_dups<HV>(sm, scr, in, n);
        }
        return n;
    }
    const bool nodup = distinct >= n;
    const uint32_t shK = static_cast<uint32_t>(P & 3), shV = static_cast<uint32_t>(P & 1);
    const uint32_t colmask = a.col_bits >= 32 ? 0xffffffffu : ((1u << a.col_bits) - 1u);
#pragma unroll RANK_UNROLL
    for (uint32_t i = tid; i < n; i += SM_NT) {
        const uint32_t key = sm.k[scr][i];
        const uint32_t d = (key - keylo) >> sh;
        const uint32_t lo = d ? sm.cnt[d - 1] : 0u, hi = sm.cnt[d];
        if (hi - lo > SM_BMAX) {
            big = true;
            continue;
        }
        uint32_t r = 0;
        if (distinct < n) {
            // duplicates present: ties by position. Four keys per trip (heavy
            // sub-bins' clustered hot columns make long buckets), then a
            // predicated tail of 0..3 keys
            uint32_t j = lo;
#pragma unroll 1
            for (; j + 4 <= hi; j += 4) {
                const uint32_t k0 = sm.k[scr][j], k1 = sm.k[scr][j + 1], k2 = sm.k[scr][j + 2],
                               k3 = sm.k[scr][j + 3];
                r += ((k0 < key) | ((k0 == key) & (j < i))) + ((k1 < key) | ((k1 == key) & (j + 1 < i))) +
                     ((k2 < key) | ((k2 == key) & (j + 2 < i))) + ((k3 < key) | ((k3 == key) & (j + 3 < i)));
            }
            const uint32_t left = hi - j;
            if (left > 0) {
                const uint32_t kj = sm.k[scr][j];
                r += (kj < key) | ((kj == key) & (j < i));
            }
            if (left > 1) {
                const uint32_t kj = sm.k[scr][j + 1];
                r += (kj < key) | ((kj == key) & (j + 1 < i));
            }
            if (left > 2) {
                const uint32_t kj = sm.k[scr][j + 2];
                r += (kj < key) | ((kj == key) & (j + 2 < i));
            }
        } else {  // all keys distinct
            // clustered keys (the stencil after its premerge: ~25 per bucket)
            // run long loops: four independent loads per trip
            uint32_t j = lo;
#pragma unroll 1
            for (; j + 4 <= hi; j += 4) {
                const uint32_t k0 = sm.k[scr][j], k1 = sm.k[scr][j + 1], k2 = sm.k[scr][j + 2],
                               k3 = sm.k[scr][j + 3];
                r += (k0 < key) + (k1 < key) + (k2 < key) + (k3 < key);
            }
            // 0..3 keys left: predicated, no loop (the scalar tail loop was the
            // kernel's hottest line at C2: 12.5 % of its instructions)
            const uint32_t left = hi - j;
            if (left > 0) r += sm.k[scr][j] < key;
            if (left > 1) r += sm.k[scr][j + 1] < key;
            if (left > 2) r += sm.k[scr][j + 2] < key;
        }
        if (nodup) {  // final form: masked column ids, C-aligned offsets
            sm.k[in][lo + r + shK] = key & colmask;
            sm.v[in][lo + r + shV] = sm.v[scr][i];
        } else {
            sm.k[in][lo + r] = key;
            sm.v[in][lo + r] = sm.v[scr][i];
        }
    }
    const bool any_big = __syncthreads_or(big);
    PROF_MARK(3);
    int sorted, other;
    if (any_big) {
        // clustered keys: stable LSD radix on scr (a permutation of the bin)
        sorted = lsd_sort(sm, scr, in, n, bits, keylo);
        other = sorted == scr ? in : scr;
        if (tid == 0) atomicAdd(a.fallbacks, 1ull);
    } else {
        sorted = in;
        other = scr;
    }
    // ---- 3. merge duplicates. The count kernel's distinct count is exact:
    // fewer distinct keys than tuples means there are duplicates, so no
    // adjacent-key check pass is needed to find out (a third of C2's bins
    // hold one duplicate pair)
    if (distinct < n) {
        __syncthreads();  // the rank pass's writes of `sorted`
        *res = other;
        return merge_dups<HV>(sm, sorted, other, n);
    }
    *res = sorted;
    *rshift = any_big ? -1 : sh;  // sorted positions = bucket ends: row starts from them
    *bulk = !any_big && nodup && sh <= a.col_bits;
    if (*bulk) fence_proxy_async_smem();  // this thread's smem writes -> the TMA store
    return n;
}

// Write a work bin: colids / values at P, rowptr of the rows it starts.
__device__ __forceinline__ void write_bin(const SortArgs& a, const SortSmem& sm, int buf,
                                          uint64_t b, uint64_t nw, uint32_t rs, uint32_t span,
                                          uint32_t U, uint64_t P, int rshift, uint32_t kofs = 0,
                                          uint32_t vofs = 0) {
    const int tid = threadIdx.x;
    const int cb = a.col_bits;
    const uint32_t colmask = cb >= 32 ? 0xffffffffu : ((1u << cb) - 1u);
    const uint32_t* K = sm.k[buf] + kofs;
    const double* V = sm.v[buf] + vofs;
    PBG_DCHECK(P + U <= a.c_cap && rs + span <= a.m);
    uint32_t* okeys = a.ccol + P;
    double* ovals = a.cval + P;
    for (uint32_t u = tid; u < U; u += SM_NT) {
        __stcs(okeys + u, K[u] & colmask);
        __stcs(ovals + u, V[u]);
    }
    if (rshift >= 0 && rshift <= cb) {
        // nothing merged: row r starts where its first MSD bucket starts
        // (cnt[d] holds the end of bucket d after the scatter)
        for (uint32_t r = tid; r < span; r += SM_NT) {
            const uint32_t d = (r << cb) >> rshift;
            a.rowptr[rs + r] = P + (d ? sm.cnt[d - 1] : 0u);
        }
        if (tid == 0 && b == nw - 1) a.rowptr[a.m] = P + U;
        return;
    }
    // rowptr[rs + r] = P + first merged entry of local row r (binary search)
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

// Output of a duplicate-free bin sorted in final form (masked column ids at
// smem index u + (P & 3), values at u + (P & 1), so smem and C agree modulo
// 16 bytes): thread 0 hands the 16-byte-aligned middles to the TMA engine
// (cp.async.bulk shared -> global, one bulk group) and a few threads store
// the unaligned head/tail elements; row starts come from the bucket ends.
// The buffer may be overwritten only after bulk_wait_read().
__device__ __forceinline__ void write_bin_bulk(const SortArgs& a, SortSmem& sm, int buf, uint64_t b,
                                               uint64_t nw, uint32_t rs, uint32_t span, uint32_t U,
                                               uint64_t P, int rshift) {
    const int tid = threadIdx.x;
    const uint32_t shK = static_cast<uint32_t>(P & 3), shV = static_cast<uint32_t>(P & 1);
    const uint32_t* K = sm.k[buf] + shK;
    const double* V = sm.v[buf] + shV;
    uint32_t ka = (4u - shK) & 3u, va = shV;
    if (ka > U) ka = U;
    if (va > U) va = U;
    const uint32_t kb = ka + ((U - ka) & ~3u), vb = va + ((U - va) & ~1u);
    PBG_DCHECK(P + U <= a.c_cap && rs + span <= a.m && U <= SM_CAP);
    if (tid < ka) a.ccol[P + tid] = K[tid];
    if (tid < U - kb) a.ccol[P + kb + tid] = K[kb + tid];
    if (tid < va) a.cval[P + tid] = V[tid];
    if (tid < U - vb) a.cval[P + vb + tid] = V[vb + tid];
    if (tid == 0) {
        fence_proxy_async_smem();  // the whole CTA's smem writes (barrier before) to the async proxy
        if (kb > ka) bulk_s2g(a.ccol + P + ka, K + ka, (kb - ka) * 4);
        if (vb > va) bulk_s2g(a.cval + P + va, V + va, (vb - va) * 8);
        bulk_commit();
    }
    const int cb = a.col_bits;
    for (uint32_t r = tid; r < span; r += SM_NT) {
        const uint32_t d = (r << cb) >> rshift;
        a.rowptr[rs + r] = P + (d ? sm.cnt[d - 1] : 0u);
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
    PBG_DCHECK(P + U <= a.c_cap && m.rs < a.m);
    for (uint32_t u = tid; u < U; u += SM_NT) {
        __stcs(a.ccol + P + u, K[u] & colmask);
        __stcs(a.cval + P + u, V[u]);
    }
    if (tid == 0) {
        if (m.span) a.rowptr[m.rs] = P;  // single-row sub-bin owning the row start
        if (b == nw - 1) a.rowptr[a.m] = P + U;
    }
}

// HV: the product has heavy rows (work bins may be unaligned heavy sub-bins or
// merged pieces, duplicates are frequent and hot). HV = false is the plain
// path of ER / stencil products.
template <bool HV>
__global__ void __launch_bounds__(SM_NT, 1024 / SM_NT) k_sortmerge(SortArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const uint64_t nw = *a.nw_dev;

    if (tid == 0) {
        mbar_init(&sm.mbar, 1);
        meta_fetch(a, sm, 0, atomicAdd(a.ticket, 1u), nw);
        cp_async_wait_all();
        if (sm.s_bin[0] < nw && bin_kind(sm.meta[0]) == 1) issue_tma(a, sm, 0, sm.meta[0]);
    }
    __syncthreads();
    uint32_t parity = 0;
    long long prof_t = clock64();
    (void)prof_t;
    int inb = 0;  // buffer the current work bin is copied into
    int mc = 0;   // its descriptor slot

    while (true) {
        const uint64_t b = sm.s_bin[mc];
        if (b >= nw) break;
        const BinMeta& M = sm.meta[mc];
        const uint32_t loaded = bin_kind(M);
        // the ticket of this CTA's next bin: consumed after the histogram
        const uint32_t tk = tid == 0 ? atomicAdd(a.ticket, 1u) : 0u;
        if (tid == 0 && M.n > SM_CAP && !(M.flags & 2u)) atomicOr(a.err, 2u);
        int res = inb;
        int rshift = -1, bulk = 0;
        uint32_t U = 0;
        bool merged = false, fetched = false;
        uint32_t wk = 0, wv = 0;  // where the output starts in buffer `res`
        if (HV && loaded && (M.flags & 2u)) {
            // merged sub-bin: already sorted and distinct, copied as it arrived
            mbar_wait(&sm.mbar, parity);
            parity ^= 1;
            U = static_cast<uint32_t>(M.n);
            wk = static_cast<uint32_t>(M.off & 3u);
            wv = static_cast<uint32_t>(M.off & 1u);
            PROF_MARK(0);
        } else if (loaded) {
            const uint32_t n = static_cast<uint32_t>(M.n);
            zero_cnt(sm);
            mbar_wait(&sm.mbar, parity);
            parity ^= 1;
            __syncthreads();
            PROF_MARK(0);
            U = sort_merge_bin<HV>(a, sm, inb, inb ^ 1, n, static_cast<int>(M.keybits), M.keylo,
                               static_cast<uint32_t>(M.nnz), &res, &rshift, M.out, &bulk, mc ^ 1,
                               tk, static_cast<uint32_t>(M.off & 3u),
                               static_cast<uint32_t>(M.off & 1u), prof_t);
            fetched = true;
#ifdef PBG_SORT_PROF
            __syncthreads();
#endif
            PROF_MARK(4);
        } else if (M.flags & 2u) {
            U = static_cast<uint32_t>(M.n);
            merged = true;
        }
        if (tid == 0) {
            if (!fetched) meta_fetch(a, sm, mc ^ 1, tk, nw);
            if (U != M.nnz) atomicOr(a.err, 4u);
            atomicAdd(a.merged_total, (unsigned long long)U);
            cp_async_wait_all();
        }
        __syncthreads();
        // next work bin's copy into the free buffer overlaps this one's output
        if (tid == 0 && sm.s_bin[mc ^ 1] < nw && bin_kind(sm.meta[mc ^ 1]) == 1) {
            bulk_wait_read();  // a previous bulk store may still read that buffer
            issue_tma(a, sm, res ^ 1, sm.meta[mc ^ 1]);
        }
        if (merged) write_merged(a, M, b, nw, M.out, U);
        else if (bulk) write_bin_bulk(a, sm, res, b, nw, M.rs, M.span, U, M.out, rshift);
        else write_bin(a, sm, res, b, nw, M.rs, M.span, U, M.out, rshift, wk, wv);
        PROF_MARK(5);
        inb = res ^ 1;
        mc ^= 1;
        __syncthreads();
        PROF_MARK(6);
    }
    if (tid == 0) bulk_wait_all();  // the last bins' C stores are complete
}

}  // namespace pbg
