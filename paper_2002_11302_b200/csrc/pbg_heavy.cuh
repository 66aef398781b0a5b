// pbg_heavy.cuh — bins larger than one CTA's shared memory ("heavy" rows).
//
// A GPU bin only exceeds SM_CAP tuples when it is a single output row whose
// flop exceeds the capacity (k_binflags makes every row above CAP/4 its own
// bin). RMAT inputs have many such rows (77-83% of the flop
// sits in rows above 65,536 tuples). The reference never has this problem —
// its bins live in DRAM and its sort recurses (pb_spgemm.hpp:139-175) — so
// this is the GPU's own MSD level above the per-bin sort:
//
//   pass: every "split" item (a key range of one heavy row) is histogrammed
//         on its next 12 key bits (4096 buckets, smem), consecutive buckets
//         are grouped into children of <= SM_CAP tuples, and the tuples are
//         scattered in bucket order into the other buffer (main <-> scratch).
//         A child that is still too large is split again on the next bits;
//         one that is a single key (a column hit more than SM_CAP times) is a
//         "uniform" item the sort kernel reduces directly.
//   The item list stays ordered by (row, key) across passes (children are
//   placed by a scan of per-item child counts), so after <= 3 passes the
//   heavy rows are sequences of sortable sub-bins in key order.
// The work-bin list then replaces each heavy bin by its sub-bins; the count
// and sort+merge kernels run over work bins.
#pragma once

#include <cstdint>

#include "pbg_device.cuh"

namespace pbg {

constexpr int HV_NT = 512;
constexpr int HV_DBITS = 12;
constexpr int HV_NB = 1 << HV_DBITS;

enum ItemKind : uint32_t { IT_SORT = 0, IT_SPLIT = 1, IT_UNIFORM = 2 };

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
    it.kind[h] = IT_SPLIT;
    it.keylo[h] = 0;
    it.keybits[h] = static_cast<uint32_t>(col_bits);
}

struct SplitSmem {
    uint32_t cnt[HV_NB];    // histogram -> bucket start -> cursor
    uint32_t gstart[HV_NB]; // 1 where a bucket starts a child
    uint32_t s_warp[HV_NT / 32 + 1];
};

// Histogram of the item's next digit + grouping into children. Leaves cnt =
// exclusive bucket starts, gstart = child-start flags; returns #children.
__device__ uint32_t split_plan(const HeavyCtx& c, SplitSmem& sm, const uint32_t* keys,
                               uint64_t n, uint32_t sh, uint32_t d) {
    const int tid = threadIdx.x;
    for (int i = tid; i < HV_NB; i += HV_NT) sm.cnt[i] = 0;
    __syncthreads();
    const uint32_t mask = (1u << d) - 1u;
    const uint32_t s2 = sh - d;
    for (uint64_t i = tid; i < n; i += HV_NT) atomicAdd(&sm.cnt[(keys[i] >> s2) & mask], 1u);
    __syncthreads();
    // exclusive scan of 4096 counters, 8 per thread
    constexpr int PER = HV_NB / HV_NT;
    uint32_t v[PER], s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        v[j] = sm.cnt[tid * PER + j];
        s += v[j];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan<HV_NT>(s, sm.s_warp, tot);
    // grouping: a bucket starts a child when it is non-empty and either it or
    // its predecessor group would overflow: window rule on the prefix like
    // k_binflags (window T = cap/2, buckets above T stand alone)
    const uint32_t T = static_cast<uint32_t>(c.cap / 2);
    uint32_t starts = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = tid * PER + j;
        sm.cnt[i] = run;
        const bool nonempty = v[j] != 0;
        sm.gstart[i] = nonempty ? 1u : 0u;  // provisional, refined below
        run += v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = tid * PER + j;
        if (!v[j]) continue;
        // previous non-empty bucket's start (scan backwards; buckets are few-ish)
        int p = static_cast<int>(i) - 1;
        while (p >= 0 && sm.cnt[p] == sm.cnt[i]) --p;  // empty buckets share the start
        bool start = true;
        if (p >= 0) {
            const uint32_t psize = sm.cnt[i] - sm.cnt[p];
            const bool big = v[j] > T || psize > T;
            start = big || (sm.cnt[i] / T != sm.cnt[p] / T);
        }
        sm.gstart[i] = start ? 1u : 0u;
        starts += start;
    }
    uint32_t nchild;
    block_exclusive_scan<HV_NT>(starts, sm.s_warp, nchild);
    return nchild;
}

__global__ void __launch_bounds__(HV_NT) k_split_count(HeavyCtx c, Items in, uint64_t nitems,
                                                       uint64_t* child_cnt) {
    __shared__ SplitSmem sm;
    for (uint64_t i = blockIdx.x; i < nitems; i += gridDim.x) {
        if (in.kind[i] != IT_SPLIT) {
            if (threadIdx.x == 0) child_cnt[i] = 1;
            continue;
        }
        const uint32_t h = in.h[i], buf = in.buf[i], sh = in.sh[i];
        const uint32_t d = sh < HV_DBITS ? sh : HV_DBITS;
        const uint64_t base = item_base(c, h, buf) + in.loc[i];
        const uint32_t* keys = (buf ? c.skeys : c.keys) + base;
        const uint32_t nc = split_plan(c, sm, keys, in.n[i], sh, d);
        if (threadIdx.x == 0) child_cnt[i] = nc;
        __syncthreads();
    }
}

// Child counts were scanned into child_pos. Final items are copied; split
// items scatter their tuples (bucket order) into the other buffer and emit
// their children at child_pos[i]...
__global__ void __launch_bounds__(HV_NT) k_split_scatter(HeavyCtx c, Items in, uint64_t nitems,
                                                         const uint64_t* child_pos, Items out) {
    __shared__ SplitSmem sm;
    const int tid = threadIdx.x;
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
        const uint32_t h = in.h[i], buf = in.buf[i], sh = in.sh[i];
        const uint32_t d = sh < HV_DBITS ? sh : HV_DBITS;
        const uint32_t s2 = sh - d, mask = (1u << d) - 1u;
        const uint64_t n = in.n[i], loc = in.loc[i];
        const uint64_t sbase = item_base(c, h, buf) + loc;
        const uint64_t dbase = item_base(c, h, buf ^ 1u) + loc;
        const uint32_t* sk = (buf ? c.skeys : c.keys) + sbase;
        const double* sv = (buf ? c.svals : c.vals) + sbase;
        uint32_t* dk = (buf ? c.keys : c.skeys) + dbase;
        double* dv = (buf ? c.vals : c.svals) + dbase;
        split_plan(c, sm, sk, n, sh, d);
        // gstart[i] = child index << 1 | starts-a-child flag
        {
            constexpr int PER = HV_NB / HV_NT;
            uint32_t g[PER], s = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                g[j] = sm.gstart[tid * PER + j];
                s += g[j];
            }
            uint32_t tot;
            uint32_t run = block_exclusive_scan<HV_NT>(s, sm.s_warp, tot);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                run += g[j];
                sm.gstart[tid * PER + j] = ((run - 1) << 1) | g[j];
            }
        }
        __syncthreads();
        // child descriptors: one per child-start bucket
        for (int bkt = tid; bkt < HV_NB; bkt += HV_NT) {
            if (!(sm.gstart[bkt] & 1u)) continue;
            const uint32_t ci = sm.gstart[bkt] >> 1;
            // child ends where the next child starts
            int e = bkt + 1;
            while (e < HV_NB && !(sm.gstart[e] & 1u)) ++e;
            const uint64_t cstart = sm.cnt[bkt];
            const uint64_t cend = e < HV_NB ? sm.cnt[e] : n;
            const uint64_t cn = cend - cstart;
            // key range: buckets [bkt, last non-empty bucket before e]
            int last = e - 1;
            while (last > bkt && sm.cnt[last] == cend) --last;
            const uint32_t kb = in.keylo[i] + (static_cast<uint32_t>(bkt) << s2);
            const uint32_t nb = static_cast<uint32_t>(last - bkt + 1);
            const uint32_t rbits = (nb > 1 ? 32 - __clz(nb - 1) : 0) + s2;
            const uint64_t oo = o + ci;
            out.loc[oo] = loc + cstart;
            out.n[oo] = cn;
            out.h[oo] = h;
            out.buf[oo] = buf ^ 1u;
            out.sh[oo] = s2;
            out.kind[oo] = cn <= c.cap ? IT_SORT : (s2 == 0 ? IT_UNIFORM : IT_SPLIT);
            out.keylo[oo] = kb;
            out.keybits[oo] = rbits;
        }
        __syncthreads();
        // scatter tuples in bucket order (cursor = bucket start)
        for (uint64_t t = tid; t < n; t += HV_NT) {
            const uint32_t key = sk[t];
            const uint32_t pos = atomicAdd(&sm.cnt[(key >> s2) & mask], 1u);
            dk[pos] = key;
            dv[pos] = sv[t];
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
    uint32_t* flags;   // bit0 scratch buffer, bit1 uniform-key reduce, bit2 heavy sub-bin
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
    w.flags[q] = (fin.buf[it] ? 1u : 0u) | (fin.kind[it] == IT_UNIFORM ? 2u : 0u) | 4u;
}

// ------------------------------------------------------ work-bin counts --
// Distinct keys per work bin = its merged count (its share of nnz(C)),
// counted from the keys alone with a shared-memory hash set (load <= 1/8 for
// a full bin, so probe chains stay short and warps rarely diverge). A scan of
// these counts gives every work bin its output offset before the sort+merge
// kernel runs, so bins never wait on each other. Uniform-key items count 1.
constexpr int CNT_NT = 512;
#ifndef PBG_CNT_SLOTS_LOG
#define PBG_CNT_SLOTS_LOG 14
#endif
constexpr int CNT_SLOTS_LOG = PBG_CNT_SLOTS_LOG;
constexpr int CNT_SLOTS = 1 << CNT_SLOTS_LOG;
constexpr uint32_t CNT_EMPTY = 0xffffffffu;
constexpr int CNT_PER = 8;  // keys per thread: bins of up to CNT_NT*CNT_PER tuples

__device__ __forceinline__ void cnt_load(const uint32_t* __restrict__ keys,
                                         const uint32_t* __restrict__ skeys, const WorkBins& w,
                                         uint64_t b, uint64_t nw, uint64_t cap, uint32_t (&kk)[CNT_PER],
                                         uint32_t& n) {
    n = 0;
    if (b >= nw) return;
    const uint32_t fl = w.flags[b];
    const uint64_t nn = w.n[b];
    if ((fl & 2u) || nn > cap) return;
    n = static_cast<uint32_t>(nn);
    const uint32_t* kb = ((fl & 1u) ? skeys : keys) + w.off[b];
#pragma unroll
    for (int j = 0; j < CNT_PER; ++j) {
        const uint32_t i = threadIdx.x + j * CNT_NT;
        kk[j] = i < n ? __ldcs(kb + i) : CNT_EMPTY;
    }
}

__global__ void __launch_bounds__(CNT_NT) k_bincount(const uint32_t* __restrict__ keys,
                                                   const uint32_t* __restrict__ skeys,
                                                   WorkBins w, const uint64_t* nw_dev,
                                                   uint64_t cap, uint64_t* wb_nnz) {
    extern __shared__ __align__(16) uint32_t table[];  // CNT_SLOTS
    __shared__ uint32_t s_red[2][CNT_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const uint64_t nw = *nw_dev;
    for (int i = tid; i < CNT_SLOTS / 4; i += CNT_NT)
        reinterpret_cast<uint4*>(table)[i] = make_uint4(CNT_EMPTY, CNT_EMPTY, CNT_EMPTY, CNT_EMPTY);
    __syncthreads();
    int par = 0;
    uint32_t kk[CNT_PER], n;
    uint64_t b = blockIdx.x;
    cnt_load(keys, skeys, w, b, nw, cap, kk, n);  // software pipeline: keys of bin b
    for (; b < nw; b += gridDim.x) {
        uint32_t cur[CNT_PER];
#pragma unroll
        for (int j = 0; j < CNT_PER; ++j) cur[j] = kk[j];
        const uint32_t ncur = n;
        const uint32_t fl = w.flags[b];
        cnt_load(keys, skeys, w, b + gridDim.x, nw, cap, kk, n);  // next bin's keys in flight
        uint32_t slot[CNT_PER];
        uint32_t fresh = 0;
#pragma unroll
        for (int j = 0; j < CNT_PER; ++j) {
            slot[j] = CNT_SLOTS;  // none
            if (tid + j * CNT_NT < ncur) {
                const uint32_t key = cur[j];
                uint32_t h = (key * 0x9E3779B1u) >> (32 - CNT_SLOTS_LOG);
                while (true) {
                    const uint32_t old = atomicCAS(&table[h], CNT_EMPTY, key);
                    if (old == CNT_EMPTY) {
                        ++fresh;
                        slot[j] = h;
                        break;
                    }
                    if (old == key) break;
                    h = (h + 1) & (CNT_SLOTS - 1);
                }
            }
        }
        fresh = warp_sum(fresh);
        if (lane == 0) s_red[par][wp] = fresh;
        __syncthreads();
        // reset only the slots this thread claimed: the table is clean for the
        // next bin without a full clear
#pragma unroll
        for (int j = 0; j < CNT_PER; ++j)
            if (slot[j] < CNT_SLOTS) table[slot[j]] = CNT_EMPTY;
        if (tid == 0) {
            uint32_t t = 0;
            for (int i = 0; i < CNT_NT / 32; ++i) t += s_red[par][i];
            // uniform-key items merge to one entry; a valid list has no other
            // bin above the capacity
            wb_nnz[b] = (fl & 2u) ? 1u : t;
        }
        par ^= 1;
        __syncthreads();
    }
}

}  // namespace pbg
