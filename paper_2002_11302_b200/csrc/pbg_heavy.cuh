// pbg_heavy.cuh — bins larger than one CTA's shared memory ("heavy" rows).
//
// A GPU bin only exceeds SM_CAP tuples when it is a single output row whose
// flop exceeds the capacity (k_binflags makes every row above CAP/4 its own
// bin). RMAT inputs have many such rows (77-83% of the flop
// sits in rows above 65,536 tuples). The reference never has this problem —
// its bins live in DRAM and its sort recurses (pb_spgemm.hpp:139-175) — so
// this is the GPU's own MSD level above the per-bin sort:
//
//   split pass (one per key level, usually one in total): every SPLIT item
//         (a key range of one heavy row) is cut into tiles spread over all
//         CTAs; tile histograms on the next d key bits are summed per item,
//         consecutive buckets are grouped into children of <= SM_CAP tuples,
//         and each tile reserves one range per (tile, bucket) and writes its
//         tuples into those bucket segments of the other buffer
//         (main <-> scratch). d is chosen so that a child still above SM_CAP
//         (one bucket) spans <= 4096 columns.
//   dense reduce: such a child is summed in a 4096-slot shared-memory
//         accumulator and written back sorted and merged (MERGED): a column
//         hit millions of times costs one pass, not more splits.
//   The item list stays ordered by (row, key) across passes (children are
//   placed by a scan of per-item child counts), so afterwards the heavy rows
//   are sequences of sortable or merged sub-bins in key order.
// The work-bin list then replaces each heavy bin by its sub-bins; the count
// and sort+merge kernels run over work bins.
#pragma once

#include <cstdint>

#include "pbg_device.cuh"

namespace pbg {

constexpr int HV_NT = 512;
#ifndef PBG_HV_TILE
#define PBG_HV_TILE 8192
#endif
constexpr int HV_TILE = PBG_HV_TILE; // tuples per split tile (4096 or 8192)
constexpr int HV_DENSE_BITS = 12;    // key range of a dense-reduced item (4096 columns)
constexpr int HV_MAXD = 10;          // digit bits per split pass (<= 1024 buckets)
#ifndef PBG_HV_GREEDY
#define PBG_HV_GREEDY 1              // child grouping rule, see hv_plan_item
#endif
#ifndef PBG_DENSE_MIN
#define PBG_DENSE_MIN 0              // tuning hook, see k_hv_children
#endif

// SORT: <= cap tuples, a work bin of the sort kernel. SPLIT: split on the
// next key bits. DENSE: > cap tuples in a key range <= 2^HV_DENSE_BITS,
// reduced by k_hv_dense into MERGED (sorted, duplicates summed).
enum ItemKind : uint32_t { IT_SORT = 0, IT_SPLIT = 1, IT_DENSE = 2, IT_MERGED = 3 };

// Items (SoA). A heavy row h owns tuples [0, n_h) at main + bin_off[hbin[h]]
// or scratch + hoff[h]; an item is a contiguous key-ordered piece of it.
struct Items {
    uint64_t* loc;     // offset inside the heavy row's tuple range
    uint64_t* n;       // tuples
    uint32_t* h;       // heavy row index
    uint32_t* buf;     // 0 main, 1 scratch
    uint32_t* sh;      // keys agree above bit sh (bits still to split)
    uint32_t* kind;    // ItemKind
    uint32_t* keylo;   // smallest possible key
    uint32_t* keybits; // key range of the item = [keylo, keylo + 2^keybits)
};

struct HeavyCtx {
    const uint32_t* hbin;    // heavy row -> bin
    const uint64_t* bin_off; // main tuple offsets of bins
    const uint64_t* hoff;    // scratch tuple offsets of heavy rows
    uint32_t* keys;          // main tuples
    double* vals;
    uint32_t* skeys;         // scratch tuples
    double* svals;
    uint64_t cap;
};

__device__ __forceinline__ uint64_t item_base(const HeavyCtx& c, uint32_t h, uint32_t buf) {
    return buf ? c.hoff[h] : c.bin_off[c.hbin[h]];
}

// Heavy bins -> the initial item list (one SPLIT item per heavy row, in bin
// order) + the heavy row index of every bin (-1 if regular).
__global__ void k_heavy_init(const uint64_t* __restrict__ bin_cnt, const uint64_t* nb_dev,
                             const uint64_t* __restrict__ heavy_excl,
                             const uint64_t* __restrict__ hpad_excl, uint64_t cap, int col_bits,
                             uint32_t* hbin, uint64_t* hoff, uint32_t* bin_hidx, Items it) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= *nb_dev) return;
    const uint64_t n = bin_cnt[b];
    if (n <= cap) {
        bin_hidx[b] = 0xffffffffu;
        return;
    }
    const uint32_t h = static_cast<uint32_t>(heavy_excl[b]);
    hbin[h] = static_cast<uint32_t>(b);
    hoff[h] = hpad_excl[b];
    bin_hidx[b] = h;
    it.loc[h] = 0;
    it.n[h] = n;
    it.h[h] = h;
    it.buf[h] = 0;
    it.sh[h] = static_cast<uint32_t>(col_bits);
    it.kind[h] = col_bits <= HV_DENSE_BITS ? IT_DENSE : IT_SPLIT;
    it.keylo[h] = 0;
    it.keybits[h] = static_cast<uint32_t>(col_bits);
}

// ---- one split pass over all SPLIT items (they share `sh` at a level) ----
// d = hv_digit(sh) key bits below bit sh become 2^d buckets per item.
// Tiles of HV_TILE tuples are the unit of work, so one heavy row is spread
// over many CTAs:
//   k_hv_hist    tile histograms, piled up in shared memory over a CTA's
//                contiguous tiles and added to the item's bucket counters
//   k_hv_plan    per item: bucket starts (-> scatter cursors) and children
//                (consecutive buckets grouped greedily to <= cap tuples);
//                child counts are scanned on the host side
//   k_hv_scatter2 tile (staged by a TMA producer warp): ranks by bucket (one
//                warp-aggregated shared atomic per run of equal buckets), one
//                global reservation per (tile, bucket), tuples written into
//                their bucket segment of the other buffer
//   k_hv_children child descriptors at the scanned positions
// A child above cap is one bucket; if its key range is <= 2^HV_DENSE_BITS
// it is reduced by k_hv_dense, else split again on the next level.
// The remaining sh - 12 bits are cut into the fewest levels of at most 8 bits,
// evenly: 2^24 columns split 6 + 6 bits, not 10 + 2. A tile's tuples spread
// over 2^d bucket segments that start at any tuple: short unaligned segments
// leave partly written sectors behind (DRAM read-modify-write;
// scripts/micro/scatter_segments.cu: 8-tuple segments 0.74 TB/s, 128-tuple
// 2.3 TB/s, aligned or L2-resident 5.1 TB/s), so two passes with 128-tuple
// segments cost no more than one with 8-tuple segments (C5b band: -3 %).
__host__ __device__ inline int hv_digit(int sh) {
    const int rem = sh - HV_DENSE_BITS;
    if (rem < 1) return 1;
#ifdef PBG_HV_DIGIT_MAX  // A/B hook: as many bits as fit per level (10 + 2 for 2^24 columns)
    return rem > HV_MAXD ? HV_MAXD : rem;
#endif
    const int levels = (rem + 7) / 8;
    return (rem + levels - 1) / levels;
}

// tile counts of SPLIT items (scan input)
struct SplitTilesIn {
    const uint64_t* n;
    const uint32_t* kind;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        return kind[i] == IT_SPLIT ? (n[i] + HV_TILE - 1) / HV_TILE : 0u;
    }
};

// tile -> item (one warp per item)
__global__ void k_hv_tilemap(const uint64_t* __restrict__ tile_pos, uint64_t nitems,
                             uint32_t* tile_item) {
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nitems) return;
    const uint64_t t0 = tile_pos[i], t1 = tile_pos[i + 1];
    for (uint64_t t = t0 + lane; t < t1; t += 32) tile_item[t] = static_cast<uint32_t>(i);
}

struct HvTile {
    uint32_t i;       // item
    uint64_t start;   // first tuple of the tile inside the item
    uint32_t m;       // tuples in the tile
};
__device__ __forceinline__ HvTile hv_tile(const Items& it, const uint64_t* tile_pos,
                                          const uint32_t* tile_item, uint64_t t) {
    HvTile r;
    r.i = tile_item[t];
    r.start = (t - tile_pos[r.i]) * HV_TILE;
    const uint64_t left = it.n[r.i] - r.start;
    r.m = static_cast<uint32_t>(left < HV_TILE ? left : HV_TILE);
    return r;
}

// Warp-aggregated shared-memory histogram increment. Lanes hold consecutive
// tuples of a run-ordered stream (a B row's columns are sorted), so equal
// buckets come in runs of adjacent lanes: the first lane of each run adds
// the run's length once and the others derive their rank from its old
// count. RMAT's skewed columns made the one-atomic-per-tuple version
// serialise on a few hot buckets (ncu: 2.6 G shared bank conflicts in
// k_hv_scatter for 3.8 G tuples). Returns the tuple's rank in its bucket.
__device__ __forceinline__ uint32_t warp_bucket_rank(uint32_t* cnt, uint32_t bk, bool valid) {
    const int lane = threadIdx.x & 31;
    const uint32_t prev = __shfl_up_sync(FULL, bk, 1);
    const uint32_t vm = __ballot_sync(FULL, valid);
    const uint32_t heads = __ballot_sync(FULL, valid && (lane == 0 || bk != prev));
    const uint32_t upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const uint32_t above = heads & ~upto;
    const int end = above ? __ffs(above) - 1 : 32 - __clz(vm);  // one past this run
    uint32_t base = 0;
    if (valid && ((heads >> lane) & 1u)) base = atomicAdd(&cnt[bk], static_cast<uint32_t>(end - lane));
    const int head = 31 - __clz(heads & upto);
    const uint32_t hb = __shfl_sync(FULL, base, head < 0 ? 0 : head);
    return hb + static_cast<uint32_t>(lane - head);
}

// Tile histograms. A CTA takes a contiguous range of tiles, so consecutive
// tiles mostly belong to the same item: their counts pile up in shared memory
// and reach the item's global counters once per item and CTA (one global
// atomic per bucket and TILE serialised on the few hundred counters of the
// heaviest rows), with no barrier between tiles of one item. A thread takes 8
// CONSECUTIVE keys per 4096-key chunk (two 16-byte loads from the 16-byte
// boundary below the tile; the stream is run-ordered, so they mostly share a
// bucket) and adds each run of equal buckets once. (The lane-striped version
// with warp_bucket_rank spent ~45 instructions per tuple on ballots and
// shuffles and ran issue-bound at 2.1 TB/s.)
__global__ void __launch_bounds__(HV_NT) k_hv_hist(HeavyCtx c, Items it, uint64_t nitems,
                                                   const uint64_t* __restrict__ tile_pos,
                                                   const uint32_t* __restrict__ tile_item,
                                                   uint32_t sh, uint32_t d, uint32_t* hist) {
    __shared__ uint32_t cnt[1 << HV_MAXD];
    const int tid = threadIdx.x;
    const uint64_t ntiles = tile_pos[nitems];
    const uint32_t nbk = 1u << d, s2 = sh - d, mask = nbk - 1u;
    constexpr int CHUNKS = HV_TILE / (8 * HV_NT);  // 4096-key chunks per tile
    static_assert(CHUNKS >= 1 && CHUNKS * 8 * HV_NT == HV_TILE, "8 keys per thread and chunk");
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = blockIdx.x * per;
    const uint64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
    if (t0 >= t1) return;
    for (uint32_t q = tid; q < nbk; q += HV_NT) cnt[q] = 0;
    uint32_t item = tile_item[t0];
    __syncthreads();
    for (uint64_t t = t0; t < t1; ++t) {
        const HvTile tl = hv_tile(it, tile_pos, tile_item, t);
        if (tl.i != item) {  // (CTA-uniform) flush the finished item's counts
            __syncthreads();
            uint32_t* h = hist + static_cast<uint64_t>(item) * nbk;
            for (uint32_t q = tid; q < nbk; q += HV_NT) {
                const uint32_t v = cnt[q];
                if (v) atomicAdd(h + q, v);
                cnt[q] = 0;
            }
            item = tl.i;
            __syncthreads();
        }
        const uint32_t buf = it.buf[tl.i];
        const uint64_t abs0 = item_base(c, it.h[tl.i], buf) + it.loc[tl.i] + tl.start;
        const uint32_t sk = static_cast<uint32_t>(abs0 & 3u);
        const uint32_t* K = (buf ? c.skeys : c.keys) + (abs0 - sk);  // 16-byte aligned
        const uint32_t end = sk + tl.m;                               // valid: [sk, end)
        uint4 q0[CHUNKS], q1[CHUNKS];
#pragma unroll
        for (int ch = 0; ch < CHUNKS; ++ch) {
            const uint32_t e0 = 8u * (tid + ch * HV_NT);
            q0[ch] = make_uint4(0, 0, 0, 0);
            q1[ch] = q0[ch];
            if (e0 < end) q0[ch] = __ldcs(reinterpret_cast<const uint4*>(K + e0));
            if (e0 + 4 < end) q1[ch] = __ldcs(reinterpret_cast<const uint4*>(K + e0 + 4));
        }
        // the shift can push up to 3 keys past the HV_TILE covered above
        uint32_t xk = 0;
        const bool xv = tid < 3 && HV_TILE + tid < end;
        if (xv) xk = __ldcs(K + HV_TILE + tid);
#pragma unroll
        for (int ch = 0; ch < CHUNKS; ++ch) {
            const uint32_t e0 = 8u * (tid + ch * HV_NT);
            const uint32_t kk[8] = {q0[ch].x, q0[ch].y, q0[ch].z, q0[ch].w,
                                    q1[ch].x, q1[ch].y, q1[ch].z, q1[ch].w};
            uint32_t cur = 0xffffffffu, len = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t e = e0 + j;
                const bool valid = e >= sk && e < end;
                const uint32_t bk = (kk[j] >> s2) & mask;
                if (valid && bk == cur) {
                    ++len;
                } else {
                    if (len) atomicAdd(&cnt[cur], len);
                    cur = valid ? bk : 0xffffffffu;
                    len = valid ? 1u : 0u;
                }
            }
            if (len) atomicAdd(&cnt[cur], len);
        }
        if (xv) atomicAdd(&cnt[(xk >> s2) & mask], 1u);
    }
    __syncthreads();
    uint32_t* h = hist + static_cast<uint64_t>(item) * nbk;
    for (uint32_t q = tid; q < nbk; q += HV_NT) {
        const uint32_t v = cnt[q];
        if (v) atomicAdd(h + q, v);
    }
}

// Children of a SPLIT item from its bucket counts (block of HV_PT threads,
// HV_PB buckets each). start flag of bucket q: non-empty and either big, or
// after a big bucket, or its prefix enters a new window of T = cap/2.
constexpr int HV_PT = 256;
constexpr int HV_PB = (1 << HV_MAXD) / HV_PT;  // 4
struct PlanSmem {
    uint32_t st[(1 << HV_MAXD) + 1];  // bucket starts (exclusive), st[nbk] = n
    uint32_t fl[1 << HV_MAXD];        // child index << 1 | starts-a-child
    uint16_t nx[1 << HV_MAXD];        // greedy grouping: the bucket starting the next child
    uint32_t s_warp[HV_PT / 32 + 1];
};
__device__ uint32_t hv_plan_item(PlanSmem& sm, const uint32_t* cnt_g, uint32_t nbk, uint64_t cap) {
    const int tid = threadIdx.x;
    uint32_t v[HV_PB], s = 0;
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        v[j] = q < nbk ? cnt_g[q] : 0u;
        s += v[j];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<HV_PT>(s, sm.s_warp, tot);
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        if (q < nbk) sm.st[q] = run;
        run += v[j];
    }
    if (tid == 0) sm.st[nbk] = tot;
    __syncthreads();
#if PBG_HV_GREEDY
    // greedy grouping: a child takes consecutive buckets while their sum stays
    // <= cap (children ~cap/2 on average under the window rule below; fuller
    // children mean fewer work bins for the count and sort kernels). Every
    // non-empty bucket finds by two binary searches over the prefix where a
    // child starting at it would end and which non-empty bucket starts the
    // next one; one thread then follows these links from the first non-empty
    // bucket (one step per CHILD; walking all <= 1024 buckets serially cost
    // 2.8 % of C3's late rounds in k_hv_plan + k_hv_children).
    for (uint32_t q = tid; q < nbk; q += HV_PT) sm.fl[q] = 0;
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        if (q >= nbk || !v[j]) continue;
        const uint64_t limit = static_cast<uint64_t>(sm.st[q]) + cap;
        // e = largest index in (q, nbk] with st[e] <= limit, at least q + 1
        uint32_t lo = q + 1, hi = nbk;  // invariant: answer in [lo, hi]
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (sm.st[mid] <= limit) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t e = lo;
        // next start: the first non-empty bucket >= e, i.e. one below the first
        // prefix above st[e]; nbk if none
        const uint32_t se = sm.st[e];
        uint32_t a = e + 1, b = nbk + 1;  // first index in [e + 1, nbk] with st > se, else nbk + 1
        while (a < b) {
            const uint32_t mid = (a + b) >> 1;
            if (sm.st[mid] > se) b = mid;
            else a = mid + 1;
        }
        sm.nx[q] = static_cast<uint16_t>(a <= nbk ? a - 1 : nbk);
    }
    __syncthreads();
    if (tid == 0) {
        // first non-empty bucket: one below the first prefix above 0
        uint32_t a = 1, b = nbk + 1;
        while (a < b) {
            const uint32_t mid = (a + b) >> 1;
            if (sm.st[mid] > 0) b = mid;
            else a = mid + 1;
        }
        for (uint32_t q = a <= nbk ? a - 1 : nbk; q < nbk; q = sm.nx[q]) sm.fl[q] = 1;
    }
    __syncthreads();
    uint32_t starts = 0, f[HV_PB];
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        f[j] = q < nbk ? sm.fl[q] : 0u;
        starts += f[j];
    }
    uint32_t nchild;
    uint32_t ci = block_exclusive_scan<HV_PT>(starts, sm.s_warp, nchild);
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        if (q < nbk) sm.fl[q] = (ci << 1) | f[j];
        ci += f[j];
    }
    __syncthreads();
    return nchild;
#else
    const uint32_t T = static_cast<uint32_t>(cap / 2);
    uint32_t starts = 0, f[HV_PB];
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        f[j] = 0;
        if (q >= nbk || !v[j]) continue;
        int p = static_cast<int>(q) - 1;
        while (p >= 0 && sm.st[p] == sm.st[q]) --p;  // previous non-empty bucket
        bool start = true;
        if (p >= 0) {
            const uint32_t psize = sm.st[q] - sm.st[p];
            start = v[j] > T || psize > T || (sm.st[q] / T != sm.st[p] / T);
        }
        f[j] = start;
        starts += start;
    }
    uint32_t nchild;
    uint32_t ci = block_exclusive_scan<HV_PT>(starts, sm.s_warp, nchild);
#pragma unroll
    for (int j = 0; j < HV_PB; ++j) {
        const uint32_t q = tid * HV_PB + j;
        if (q < nbk) sm.fl[q] = (ci << 1) | f[j];
        ci += f[j];
    }
    __syncthreads();
    return nchild;
#endif
}

// per item: bucket counts -> scatter cursors (bucket starts), child count
__global__ void __launch_bounds__(HV_PT) k_hv_plan(Items it, uint64_t nitems, uint32_t d,
                                                   uint64_t cap, uint32_t* hist,
                                                   uint64_t* child_cnt) {
    __shared__ PlanSmem sm;
    const uint32_t nbk = 1u << d;
    for (uint64_t i = blockIdx.x; i < nitems; i += gridDim.x) {
        if (it.kind[i] != IT_SPLIT) {
            if (threadIdx.x == 0) child_cnt[i] = 1;
            continue;
        }
        uint32_t* h = hist + i * nbk;
        const uint32_t nc = hv_plan_item(sm, h, nbk, cap);
        for (uint32_t q = threadIdx.x; q < nbk; q += HV_PT) h[q] = sm.st[q];
        if (threadIdx.x == 0) child_cnt[i] = nc;
        __syncthreads();
    }
}

// k_hv_scatter2: the split pass with its tiles staged by TMA. A producer warp
// (warp HV_NT/32, one elected lane) walks the CTA's tiles one ahead of the 512
// consumer threads: it resolves the tile descriptor (tile -> item -> buffer
// addresses: three dependent global round trips that every thread of the
// first version, k_hv_scatter, paid per tile), publishes it in shared memory and starts two
// bulk copies (keys, values; from the 16-byte boundary below the tile) into
// the free one of two buffers, completion on that buffer's `full` mbarrier.
// Consumers rank the tile's keys from shared memory (no tuple registers held
// across the reservation round trip), reserve, store, and hand the buffer
// back through its `empty` mbarrier. ncu on a C3 round had k_hv_scatter at
// 50 % long-scoreboard stalls, 28 % issue, 3.1 TB/s. Measured and not kept:
// two consumer groups of 480 threads, each bound to one buffer and working on
// every other tile out of phase (+1.8 ms per C3 round: a group's buffer is
// refilled only after the group releases it); segment starts from per-tile
// bucket counts and a scan over each item's tiles instead of reservations
// (deterministic, no returning atomics, one barrier less per tile): the split
// kernel took 24.3 ms with grid-strided tiles and 20.9 ms with a contiguous
// tile range per CTA against 18.1 ms — the atomics hand out a bucket's
// positions in ARRIVAL order, so concurrently written segments are neighbours
// and their partly written sectors meet in L2; precomputed positions scatter
// them — and the per-tile histogram (4.1 vs 2.8 ms) and the scan (1.2 ms)
// come on top.
struct HvDesc {
    uint32_t* dk;      // destination of the item's tuples (other buffer)
    double* dv;
    uint32_t* cursor;  // the item's bucket cursors
    uint64_t n;        // tuples of the item (PBG_CHECKED bound)
    uint32_t m;        // tuples in the tile
    uint32_t sk, sv;   // the tile starts sk keys / sv values into the buffer
    uint32_t pad;
};
struct HvScatter2Smem {
    uint32_t k[2][HV_TILE + 4];
    double v[2][HV_TILE + 2];
    uint32_t cnt[1 << HV_MAXD];
    uint32_t gb[1 << HV_MAXD];
    HvDesc desc[2];
    unsigned long long full[2], empty[2];
};
constexpr int HV2_NC = HV_TILE <= 4096 ? HV_TILE / 8 : 960;  // consumer threads (a CTA holds <= 1024)
constexpr int HV2_NT = HV2_NC + 32;  // consumers + the producer warp

__global__ void __launch_bounds__(HV2_NT, HV_TILE <= 4096 ? 2 : 1) k_hv_scatter2(HeavyCtx c, Items it, uint64_t nitems,
                                                           const uint64_t* __restrict__ tile_pos,
                                                           const uint32_t* __restrict__ tile_item,
                                                           uint32_t sh, uint32_t d, uint32_t* cursor) {
    extern __shared__ __align__(16) unsigned char hv2_raw[];
    HvScatter2Smem& sm = *reinterpret_cast<HvScatter2Smem*>(hv2_raw);
    const int tid = threadIdx.x;
    const uint64_t ntiles = tile_pos[nitems];
    const uint32_t nbk = 1u << d, s2 = sh - d, mask = nbk - 1u;
    if (tid == 0) {
        mbar_init(&sm.full[0], 1);
        mbar_init(&sm.full[1], 1);
        mbar_init(&sm.empty[0], 1);
        mbar_init(&sm.empty[1], 1);
    }
    __syncthreads();
    if (tid >= HV2_NC) {  // ---- producer warp
        if (tid != HV2_NC) return;
        uint32_t i = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int s = i & 1;
            if (i >= 2) mbar_wait(&sm.empty[s], ((i >> 1) - 1) & 1);
            const HvTile tl = hv_tile(it, tile_pos, tile_item, t);
            const uint32_t buf = it.buf[tl.i], h = it.h[tl.i];
            const uint64_t loc = it.loc[tl.i];
            const uint64_t sbase = item_base(c, h, buf) + loc + tl.start;
            const uint64_t dbase = item_base(c, h, buf ^ 1u) + loc;
            const uint64_t sk = sbase & 3u, sv = sbase & 1u;
            HvDesc& D = sm.desc[s];
            D.dk = (buf ? c.keys : c.skeys) + dbase;
            D.dv = (buf ? c.vals : c.svals) + dbase;
            D.cursor = cursor + static_cast<uint64_t>(tl.i) * nbk;
            D.n = it.n[tl.i];
            D.m = tl.m;
            D.sk = static_cast<uint32_t>(sk);
            D.sv = static_cast<uint32_t>(sv);
            const uint32_t kb = static_cast<uint32_t>(((tl.m + sk) * 4 + 15) & ~15ull);
            const uint32_t vb = static_cast<uint32_t>(((tl.m + sv) * 8 + 15) & ~15ull);
            mbar_expect_tx(&sm.full[s], kb + vb);
            bulk_g2s(sm.k[s], (buf ? c.skeys : c.keys) + (sbase - sk), kb, &sm.full[s]);
            bulk_g2s(sm.v[s], (buf ? c.svals : c.vals) + (sbase - sv), vb, &sm.full[s]);
        }
        return;
    }
    // ---- consumers (threads 0 .. HV2_NC-1; barriers are named: the producer
    // warp takes no part)
    constexpr int TPT = (HV_TILE + HV2_NC - 1) / HV2_NC;  // 8 (9 for 8192-tuple tiles)
    uint32_t i = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i & 1;
        for (uint32_t q = tid; q < nbk; q += HV2_NC) sm.cnt[q] = 0;
        mbar_wait(&sm.full[s], (i >> 1) & 1);
        named_barrier<1, HV2_NC>();
        const HvDesc& D = sm.desc[s];
        const uint32_t m = D.m;
        const uint32_t* K = sm.k[s] + D.sk;
        const double* V = sm.v[s] + D.sv;
        uint32_t rb[TPT];
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            const uint32_t q = tid + j * HV2_NC;
            const bool valid = q < m;
            const uint32_t bk = valid ? ((K[q] >> s2) & mask) : 0u;
            const uint32_t r = warp_bucket_rank(sm.cnt, bk, valid);
            rb[j] = r | (bk << 16);
        }
        named_barrier<1, HV2_NC>();
        {  // one global reservation per non-empty bucket
            uint32_t* cur = D.cursor;
            for (uint32_t q = tid; q < nbk; q += HV2_NC) {
                const uint32_t v = sm.cnt[q];
                if (v) sm.gb[q] = atomicAdd(cur + q, v);
            }
        }
        named_barrier<1, HV2_NC>();
        uint32_t* DK = D.dk;
        double* DV = D.dv;
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            const uint32_t q = tid + j * HV2_NC;
            if (q < m) {
                const uint64_t dst = static_cast<uint64_t>(sm.gb[rb[j] >> 16]) + (rb[j] & 0xffffu);
                PBG_DCHECK(dst < D.n);
                DK[dst] = K[q];
                DV[dst] = V[q];
            }
        }
        named_barrier<1, HV2_NC>();  // buffer s, cnt and gb are free again
        if (tid == 0) mbar_arrive(&sm.empty[s]);
    }
}

// Child descriptors of every item at child_pos (non-SPLIT items are copied).
// `starts` holds the bucket starts again after the scatter (cursor - count
// is not needed: the plan is recomputed from the cursors' final values,
// which are the bucket ends, and the item size).
__global__ void __launch_bounds__(HV_PT) k_hv_children(HeavyCtx c, Items in, uint64_t nitems,
                                                       uint32_t sh, uint32_t d,
                                                       const uint32_t* __restrict__ ends,
                                                       const uint64_t* __restrict__ child_pos,
                                                       Items out) {
    __shared__ PlanSmem sm;
    __shared__ uint32_t cntb[1 << HV_MAXD];
    const int tid = threadIdx.x;
    const uint32_t nbk = 1u << d, s2 = sh - d;
    for (uint64_t i = blockIdx.x; i < nitems; i += gridDim.x) {
        const uint64_t o = child_pos[i];
        if (in.kind[i] != IT_SPLIT) {
            if (tid == 0) {
                out.loc[o] = in.loc[i];
                out.n[o] = in.n[i];
                out.h[o] = in.h[i];
                out.buf[o] = in.buf[i];
                out.sh[o] = in.sh[i];
                out.kind[o] = in.kind[i];
                out.keylo[o] = in.keylo[i];
                out.keybits[o] = in.keybits[i];
            }
            continue;
        }
        // bucket counts from the ends (cursor after the scatter = bucket end)
        const uint32_t* e = ends + i * nbk;
        for (uint32_t q = tid; q < nbk; q += HV_PT) cntb[q] = e[q] - (q ? e[q - 1] : 0u);
        __syncthreads();
        hv_plan_item(sm, cntb, nbk, c.cap);
        const uint64_t n = in.n[i], loc = in.loc[i];
        for (uint32_t q = tid; q < nbk; q += HV_PT) {
            if (!(sm.fl[q] & 1u)) continue;
            const uint32_t ci = sm.fl[q] >> 1;
            uint32_t e2 = q + 1;
            while (e2 < nbk && !(sm.fl[e2] & 1u)) ++e2;
            const uint64_t cs = sm.st[q];
            const uint64_t ce = e2 < nbk ? sm.st[e2] : n;
            const uint64_t cn = ce - cs;
            uint32_t last = e2 - 1;
            while (last > q && sm.st[last] == ce) --last;  // last non-empty bucket
            const uint32_t nb = last - q + 1;
            const uint32_t rbits = (nb > 1 ? 32 - __clz(nb - 1) : 0) + s2;
            const uint64_t oo = o + ci;
            out.loc[oo] = loc + cs;
            out.n[oo] = cn;
            out.h[oo] = in.h[i];
            out.buf[oo] = in.buf[i] ^ 1u;
            out.sh[oo] = s2;
            // a single-bucket child within the dense key range is summed by
            // k_hv_dense from PBG_DENSE_MIN tuples on (0 = only above cap)
            const bool dense_ok = s2 <= HV_DENSE_BITS && nb == 1;
            out.kind[oo] = cn <= c.cap ? ((PBG_DENSE_MIN && dense_ok && cn >= PBG_DENSE_MIN) ? IT_DENSE : IT_SORT)
                                       : (s2 <= HV_DENSE_BITS ? IT_DENSE : IT_SPLIT);
            out.keylo[oo] = in.keylo[i] + (q << s2);
            out.keybits[oo] = rbits;
        }
        __syncthreads();
    }
}

// A DENSE item (> cap tuples, key range <= 2^HV_DENSE_BITS): its duplicates
// are summed in a dense shared-memory accumulator indexed by key, and the
// distinct (key, sum) pairs are written back in key order over its own tuple
// range, so it becomes a MERGED work bin (already sorted and merged) that the
// count and sort kernels just copy. Exact-zero sums are kept (presence
// flags). (A global-memory accumulator with native L2 f64 reductions was
// measured 1.5x slower: these items are popular columns, and L2 atomics
// serialise per address. An atomic-free version — 32-bit rank atomics per
// slot, a scan, values grouped in shared memory, a warp-shuffle segmented sum
// and owner threads keeping their 8 slots' sums in registers — was built,
// parity-green, and measured slower: 20.2 vs 13.1 ms on a C3 round, eight
// barriers per 4096-tuple batch against none here.)
constexpr int HV_DENSE = 1 << HV_DENSE_BITS;
#ifndef PBG_DENSE_DU
#define PBG_DENSE_DU 4  // tuples a thread loads before their adds (8: +0.4 ms, 16: +2.6 ms per C3 round)
#endif
#ifndef PBG_DENSE_COPIES
#define PBG_DENSE_COPIES 2
#endif
// DC accumulator copies, lane l adding into copy l % DC (equal popular
// columns in one instruction's lanes retry each other's CAS; copies per WARP
// were measured useless: the contention is within the warp); summed into
// copy 0 before the write-back
constexpr int HV_DC = PBG_DENSE_COPIES;
__global__ void __launch_bounds__(HV_NT) k_hv_dense(HeavyCtx c, Items it, uint64_t nitems) {
    extern __shared__ __align__(16) unsigned char dn_raw[];
    double* acc_all = reinterpret_cast<double*>(dn_raw);                       // HV_DC x HV_DENSE
    uint8_t* seen = reinterpret_cast<uint8_t*>(acc_all + HV_DC * HV_DENSE);    // HV_DENSE
    __shared__ uint32_t s_warp[HV_NT / 32 + 1];
    constexpr int PER = HV_DENSE / HV_NT;  // 8
    const int tid = threadIdx.x;
    double* acc = acc_all + (tid % HV_DC) * HV_DENSE;
    for (uint64_t i = blockIdx.x; i < nitems; i += gridDim.x) {
        if (it.kind[i] != IT_DENSE) continue;
        const uint32_t buf = it.buf[i];
        const uint64_t base = item_base(c, it.h[i], buf) + it.loc[i];
        uint32_t* K = (buf ? c.skeys : c.keys) + base;
        double* V = (buf ? c.svals : c.vals) + base;
        const uint64_t n = it.n[i];
        const uint32_t keylo = it.keylo[i];
        // -0.0 is the exact additive identity: a column whose only product is
        // -0.0 keeps its sign, as the reference's first-insert does
        for (int q = tid; q < HV_DC * HV_DENSE; q += HV_NT) acc_all[q] = -0.0;
        for (int q = tid; q < HV_DENSE; q += HV_NT) seen[q] = 0;
        __syncthreads();
        // DU tuples per thread in flight: the loads of a batch are issued
        // before its shared-memory adds
        constexpr int DU = PBG_DENSE_DU;
        for (uint64_t q0 = 0; q0 < n; q0 += static_cast<uint64_t>(DU) * HV_NT) {
            uint32_t ks[DU];
            double vs[DU];
#pragma unroll
            for (int u = 0; u < DU; ++u) {
                const uint64_t q = q0 + tid + static_cast<uint64_t>(u) * HV_NT;
                ks[u] = q < n ? __ldcs(K + q) : 0xffffffffu;
                vs[u] = q < n ? __ldcs(V + q) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < DU; ++u) {
                if (ks[u] == 0xffffffffu) continue;
                const uint32_t slot = ks[u] - keylo;
                atomicAdd(&acc[slot], vs[u]);
                seen[slot] = 1;
            }
        }
        __syncthreads();
        if (HV_DC > 1) {
            for (int q = tid; q < HV_DENSE; q += HV_NT) {
                double sum = acc_all[q];
#pragma unroll
                for (int cpy = 1; cpy < HV_DC; ++cpy) sum += acc_all[cpy * HV_DENSE + q];
                acc_all[q] = sum;
            }
            __syncthreads();
        }
        uint32_t cnt = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) cnt += seen[tid * PER + j];
        uint32_t tot;
        uint32_t o = block_exclusive_scan<HV_NT>(cnt, s_warp, tot);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t slot = tid * PER + j;
            if (seen[slot]) {
                K[o] = keylo + slot;
                V[o] = acc_all[slot];
                ++o;
            }
        }
        if (tid == 0) {
            it.n[i] = tot;
            it.kind[i] = IT_MERGED;
        }
        __syncthreads();
    }
}

// First final item of every heavy row (items are ordered by row).
__global__ void k_heavy_heads(const uint32_t* __restrict__ item_h, uint64_t nitems,
                              uint32_t* head, uint32_t* count) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nitems) return;
    const uint32_t h = item_h[i];
    if (i == 0 || item_h[i - 1] != h) head[h] = static_cast<uint32_t>(i);
    atomicAdd(&count[h], 1u);
}

// Work bins per bin: 1 for a regular bin, the heavy row's items otherwise.
// Also the expand conservation check (pb_spgemm.cpp:241-245): every bin's
// fill cursor must equal its symbolic size; their sum is tuples_into_sort.
__global__ void k_work_count(const uint64_t* nb_dev, const uint32_t* __restrict__ bin_hidx,
                             const uint32_t* __restrict__ hcount,
                             const unsigned long long* __restrict__ cursor,
                             const uint64_t* __restrict__ bin_off,
                             const uint64_t* __restrict__ bin_cnt, uint64_t* wcnt,
                             unsigned long long* tuples_total, unsigned int* err) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t cur = 0;
    if (b < *nb_dev) {
        const uint32_t h = bin_hidx[b];
        wcnt[b] = h == 0xffffffffu ? 1 : hcount[h];
        cur = cursor[b] - bin_off[b];  // cursors start at the bin's offset
        if (cur != bin_cnt[b]) atomicOr(err, 1u);
    }
    cur = warp_sum(cur);
    if ((threadIdx.x & 31) == 0 && cur) atomicAdd(tuples_total, (unsigned long long)cur);
}

// Work-bin list (SoA): the sort/count kernels' unit of work.
struct WorkBins {
    uint64_t* off;     // tuple offset (in the buffer below)
    uint64_t* n;       // tuples
    uint32_t* rs;      // first output row
    uint32_t* span;    // rows (0 for a heavy sub-bin that does not own its row start)
    uint32_t* keylo;   // key range [keylo, keylo + 2^keybits)
    uint32_t* keybits;
    uint32_t* flags;   // bit0 scratch buffer, bit1 merged (sorted + distinct already), bit2 heavy sub-bin
};

__global__ void k_work_fill(const uint64_t* nb_dev, const uint32_t* __restrict__ bin_rs,
                            const uint64_t* __restrict__ bin_cnt,
                            const uint64_t* __restrict__ bin_off,
                            const uint32_t* __restrict__ bin_hidx,
                            const uint64_t* __restrict__ wpos, const uint32_t* __restrict__ head,
                            const uint32_t* __restrict__ hcount, HeavyCtx c, Items fin,
                            int col_bits, WorkBins w) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= *nb_dev) return;
    const uint32_t h = bin_hidx[b];
    const uint64_t p = wpos[b];
    const uint32_t rs = bin_rs[b], re = bin_rs[b + 1];
    if (h == 0xffffffffu) {
        const uint32_t span = re - rs;
        w.off[p] = bin_off[b];
        w.n[p] = bin_cnt[b];
        w.rs[p] = rs;
        w.span[p] = span;
        w.keylo[p] = 0;
        w.keybits[p] = (span > 1 ? 32 - __clz(span - 1) : 0) + col_bits;
        w.flags[p] = 0;
        return;
    }
    // heavy row: its items are filled by k_work_fill_items (one thread each)
}

// No heavy rows: every bin is one work bin (work bin b = bin b). Replaces
// k_heavy_init + k_work_count + scan + k_work_fill (four launches, the
// latency floor of small products) with one; also the expand conservation
// check and the tuples_into_sort total.
__global__ void k_work_direct(const uint64_t* nb_dev, const uint32_t* __restrict__ bin_rs,
                              const uint64_t* __restrict__ bin_cnt,
                              const uint64_t* __restrict__ bin_off,
                              const unsigned long long* __restrict__ cursor, int col_bits,
                              WorkBins w, unsigned long long* nw_out,
                              unsigned long long* tuples_total, unsigned int* err) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nb = *nb_dev;
    if (b == 0) *nw_out = nb;
    uint64_t cur = 0;
    if (b < nb) {
        const uint32_t rs = bin_rs[b], span = bin_rs[b + 1] - rs;
        const uint64_t off = bin_off[b], n = bin_cnt[b];
        w.off[b] = off;
        w.n[b] = n;
        w.rs[b] = rs;
        w.span[b] = span;
        w.keylo[b] = 0;
        w.keybits[b] = (span > 1 ? 32 - __clz(span - 1) : 0) + col_bits;
        w.flags[b] = 0;
        cur = cursor[b] - off;  // cursors start at the bin's offset
        if (cur != n) atomicOr(err, 1u);
    }
    cur = warp_sum(cur);
    if ((threadIdx.x & 31) == 0 && cur) atomicAdd(tuples_total, (unsigned long long)cur);
}

// Work bins of heavy-row items: item `it` of row h lands at wpos[bin] + (it - head[h]).
__global__ void k_work_fill_items(const uint64_t* __restrict__ wpos,
                                  const uint32_t* __restrict__ bin_rs,
                                  const uint32_t* __restrict__ head, HeavyCtx c, Items fin,
                                  uint64_t nitems, WorkBins w) {
    const uint64_t it = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (it >= nitems) return;
    const uint32_t h = fin.h[it];
    const uint32_t b = c.hbin[h];
    const uint32_t j = static_cast<uint32_t>(it) - head[h];
    const uint64_t q = wpos[b] + j;
    w.off[q] = item_base(c, h, fin.buf[it]) + fin.loc[it];
    w.n[q] = fin.n[it];
    w.rs[q] = bin_rs[b];
    w.span[q] = j == 0 ? 1u : 0u;
    w.keylo[q] = fin.keylo[it];
    w.keybits[q] = fin.keybits[it];
    w.flags[q] = (fin.buf[it] ? 1u : 0u) | (fin.kind[it] == IT_MERGED ? 2u : 0u) | 4u;
}

// ------------------------------------------------------ work-bin counts --
// Distinct keys per work bin = its merged count (its share of nnz(C)),
// counted from the keys alone with a shared-memory hash set (load <= 1/8 for
// a full bin, so probe chains stay short and warps rarely diverge). A scan of
// these counts gives every work bin its output offset before the sort+merge
// kernel runs, so bins never wait on each other. Uniform-key items count 1.
// Two shapes (template): 512 threads with a 16 K-slot table (3 CTAs/SM) and
// 1024 threads with a 27 K-slot table (2 CTAs/SM, 64 warps). The large table
// (load ~1/7) cuts the probe chains of distinct-key bins (C2 count 1.30 ->
// 1.15 ms, C5a 5.4 -> 4.9 ms); duplicate-heavy inputs (the stencil, RMAT)
// gain nothing from it and lose the third CTA per SM (C4 3.4 -> 4.2 ms), so
// the host picks the shape from the bin statistics (CountShape below).
constexpr uint32_t CNT_EMPTY = 0xffffffffu;

// Pipelined count k_bincount2 (same result as the round-1 kernel k_bincount, C2 1.15 -> 1.01
// ms). The per-bin critical path of k_bincount held two dependent global
// round trips (descriptor -> key address -> keys), every thread's probes ran
// one after another behind a branch per key, and one thread summed the warp
// counts serially. Here keys (16-byte vector loads) are in flight two bins
// ahead and descriptors four; a thread issues the first-probe CAS of all its
// keys back to back (a lane without a key CASes its own dummy slot, so no
// CAS is predicated) and only collided keys probe on; every key's final slot
// is reset unconditionally; warp counts go to one shared counter.
struct CntDesc {
    uint64_t off;
    uint64_t merged;  // tuples of a merged item (already distinct), else ~0
    uint32_t n;       // keys to count (0: merged / above capacity / past the end)
    uint32_t flags;   // bit0 scratch buffer
};

__device__ __forceinline__ CntDesc cnt_desc(const WorkBins& w, uint64_t b, uint64_t nw, uint64_t cap) {
    CntDesc d{0, ~0ull, 0, 0};
    if (b >= nw) return d;
    const uint32_t fl = w.flags[b];
    const uint64_t nn = w.n[b];
    d.off = w.off[b];
    d.flags = fl;
    d.merged = (fl & 2u) ? nn : ~0ull;
    d.n = ((fl & 2u) || nn > cap) ? 0u : static_cast<uint32_t>(nn);
    return d;
}

template <int NT>
__device__ __forceinline__ void cnt_keys(const uint32_t* __restrict__ keys,
                                         const uint32_t* __restrict__ skeys, const CntDesc& d,
                                         uint32_t (&kk)[4096 / NT]) {
    constexpr int PER = 4096 / NT;
    static_assert(PER % 4 == 0, "uint4 key loads");
    const uint32_t* kb = ((d.flags & 1u) ? skeys : keys) + d.off;
    if (!(d.flags & 1u) && (d.off & 3u) == 0) {
        // main-buffer bins start 16-byte aligned and are padded to 4 tuples
#pragma unroll
        for (int q = 0; q < PER / 4; ++q) {
            const uint32_t i = 4u * (threadIdx.x + q * NT);
            uint4 v = make_uint4(CNT_EMPTY, CNT_EMPTY, CNT_EMPTY, CNT_EMPTY);
            if (i < d.n) v = __ldcs(reinterpret_cast<const uint4*>(kb + i));
            kk[4 * q] = v.x;
            kk[4 * q + 1] = i + 1 < d.n ? v.y : CNT_EMPTY;
            kk[4 * q + 2] = i + 2 < d.n ? v.z : CNT_EMPTY;
            kk[4 * q + 3] = i + 3 < d.n ? v.w : CNT_EMPTY;
        }
    } else {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t i = threadIdx.x + j * NT;
            kk[j] = i < d.n ? __ldcs(kb + i) : CNT_EMPTY;
        }
    }
}

// resident CTAs per SM: shared memory (table + dummies) and 64 warps bound it
constexpr int cnt_ctas(int nt, int slots) {
    return (225 * 1024 / ((slots + 32) * 4)) < (2048 / nt) ? (225 * 1024 / ((slots + 32) * 4))
                                                         : (2048 / nt);
}
// Work-bin descriptors are staged in shared memory: thread 0 copies bin
// b + 4G's (n, off, flags) with cp.async while the CTA counts bin b, so the
// loop reads three shared words per bin instead of issuing three dependent
// global loads and their 64-bit address arithmetic per thread (a version
// loading them per thread, two bins ahead: C2 1.08 ms; this one 1.01).
struct RawDesc {
    uint64_t n, off;
    uint32_t flags, keybits;
};

__device__ __forceinline__ void stage_desc(RawDesc& d, const WorkBins& w, uint64_t b, uint64_t nw) {
    if (b < nw) {
        cp_async8(&d.n, w.n + b);
        cp_async8(&d.off, w.off + b);
        cp_async4(&d.flags, w.flags + b);
        cp_async4(&d.keybits, w.keybits + b);
    } else {
        d.n = 0;
        d.flags = 0;
        d.keybits = 0;
    }
    cp_async_commit();
}

__device__ __forceinline__ CntDesc cnt_desc_smem(const RawDesc& r, uint64_t cap) {
    CntDesc d;
    const uint64_t nn = r.n;
    d.off = r.off;
    d.flags = r.flags;
    d.merged = (r.flags & 2u) ? nn : ~0ull;
    d.n = ((r.flags & 2u) || nn > cap) ? 0u : static_cast<uint32_t>(nn);
    return d;
}

template <int NT, int SLOTS>
__global__ void __launch_bounds__(NT, cnt_ctas(NT, SLOTS)) k_bincount2(const uint32_t* __restrict__ keys,
                                                  const uint32_t* __restrict__ skeys, WorkBins w,
                                                  const uint64_t* nw_dev, uint64_t cap,
                                                  uint64_t* wb_nnz) {
    constexpr int PER = 4096 / NT;
    static_assert(SLOTS % 4 == 0, "table cleared in uint4s");
    extern __shared__ __align__(16) uint32_t table[];  // SLOTS + 32 per-lane dummies
    __shared__ RawDesc s_d[4];
    __shared__ uint32_t s_cnt;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint64_t nw = *nw_dev;
    const uint64_t G = gridDim.x;
    for (int i = tid; i < (SLOTS + 32) / 4; i += NT)
        reinterpret_cast<uint4*>(table)[i] = make_uint4(CNT_EMPTY, CNT_EMPTY, CNT_EMPTY, CNT_EMPTY);
    uint64_t b = blockIdx.x;
    if (tid == 0) {
        s_cnt = 0;
        for (int q = 0; q < 4; ++q) stage_desc(s_d[q], w, b + q * G, nw);
        cp_async_wait_all();
    }
    __syncthreads();
    uint32_t k0[PER], k1[PER], k2[PER];
    cnt_keys<NT>(keys, skeys, cnt_desc_smem(s_d[0], cap), k0);
    cnt_keys<NT>(keys, skeys, cnt_desc_smem(s_d[1], cap), k1);
    for (uint32_t it = 0; b < nw; b += G, ++it) {
        cnt_keys<NT>(keys, skeys, cnt_desc_smem(s_d[(it + 2) & 3], cap), k2);  // bin b + 2G
        uint32_t h[PER], old[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t hk =
                static_cast<uint32_t>((static_cast<uint64_t>(k0[j] * 0x9E3779B1u) * SLOTS) >> 32);
            h[j] = k0[j] == CNT_EMPTY ? SLOTS + lane : hk;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) old[j] = atomicCAS(&table[h[j]], CNT_EMPTY, k0[j]);
        uint32_t fresh = 0, pend = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            fresh += (old[j] == CNT_EMPTY) & (k0[j] != CNT_EMPTY);
            pend |= static_cast<uint32_t>(old[j] != CNT_EMPTY && old[j] != k0[j]) << j;
        }
        while (pend) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                if (!((pend >> j) & 1u)) continue;
                const uint32_t s = h[j] + 1 == SLOTS ? 0u : h[j] + 1;
                const uint32_t o = atomicCAS(&table[s], CNT_EMPTY, k0[j]);
                h[j] = s;
                if (o == CNT_EMPTY) fresh += 1;
                if (o == CNT_EMPTY || o == k0[j]) pend &= ~(1u << j);
            }
        }
        fresh = __reduce_add_sync(FULL, fresh);
        if (lane == 0) atomicAdd(&s_cnt, fresh);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) table[h[j]] = CNT_EMPTY;
        if (tid == 0) {
            RawDesc& dm = s_d[it & 3];
            // merged items are already distinct; a valid list has no other
            // bin above the capacity
            wb_nnz[b] = (dm.flags & 2u) ? dm.n : s_cnt;
            s_cnt = 0;
            stage_desc(dm, w, b + 4 * G, nw);  // slot of bin b is free: bin b + 4G
            cp_async_wait_group<1>();          // bin b + 3G's descriptor has landed
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            k0[j] = k1[j];
            k1[j] = k2[j];
        }
    }
}


}  // namespace pbg
