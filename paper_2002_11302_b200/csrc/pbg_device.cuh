// pbg_device.cuh — device building blocks shared by the PB-SpGEMM kernels:
// warp/block scans, the decoupled look-back used by every single-pass scan
// and by the sort+merge kernel's output offsets, and small search helpers.
#pragma once

#include <cstdint>
#include <cstdio>

namespace pbg {

constexpr unsigned FULL = 0xffffffffu;

// PBG_CHECKED builds (libpbg_checked.so, tests/test_gpu_checked.py) trap on
// an out-of-range shared or global index at the kernels' store sites — the
// stand-in for compute-sanitizer memcheck, which the GPU pool does not run.
#ifdef PBG_CHECKED
#define PBG_DCHECK(cond)                                                                  \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("PBG_CHECKED failure %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define PBG_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// Look-back status word: 2 flag bits + 62-bit value.
constexpr uint64_t ST_AGG = 1ull << 62;
constexpr uint64_t ST_INC = 2ull << 62;
constexpr uint64_t ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned long long* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// Block-wide exclusive scan of one value per thread. s_warp needs NT/32+1
// slots. Returns the exclusive prefix and the block total. Ends with a
// __syncthreads so s_warp can be reused immediately (TRAIL = false: the
// caller guarantees a barrier before s_warp's next use).
template <int NT, typename T, bool TRAIL = true>
__device__ __forceinline__ T block_exclusive_scan(T v, T* s_warp, T& total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = warp_inclusive_scan(v);
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        T t = lane < NW ? s_warp[lane] : T(0);
        T inc = warp_inclusive_scan(t);
        if (lane < NW) s_warp[lane] = inc - t;
        if (lane == NW - 1) s_warp[NW] = inc;
    }
    __syncthreads();
    T excl = s_warp[w] + x - v;
    total = s_warp[NW];
    if (TRAIL) __syncthreads();
    return excl;
}

// Decoupled look-back (single-pass chained scan). Called by one full warp of
// the CTA owning `tile`; publishes `aggregate`, walks predecessors 32 at a
// time, publishes the inclusive prefix and returns the exclusive prefix
// (same value in every lane). Predecessors always hold an earlier ticket, so
// they are resident or finished: no deadlock.
__device__ __forceinline__ uint64_t lookback_warp(unsigned long long* status, uint64_t tile,
                                                  uint64_t aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_release_gpu(&status[0], ST_INC | (aggregate & ST_VAL));
        return 0;
    }
    if (lane == 0) st_release_gpu(&status[tile], ST_AGG | (aggregate & ST_VAL));
    uint64_t prefix = 0;
    int64_t idx = static_cast<int64_t>(tile) - 1;
    while (true) {
        const int64_t j = idx - lane;
        uint64_t s = j >= 0 ? ld_relaxed_gpu(&status[j]) : ST_INC;
        // wait for the contiguous run of published predecessors that reaches an
        // inclusive prefix (only lanes up to the first INC matter)
        while (true) {
            const uint32_t inc = __ballot_sync(FULL, (s >> 62) == 2);
            const uint32_t zero = __ballot_sync(FULL, (s >> 62) == 0);
            const uint32_t need = inc ? ((inc & (0u - inc)) << 1) - 1u : FULL;  // lanes <= first INC
            if ((zero & need) == 0) break;
            __nanosleep(64);
            if ((s >> 62) == 0) s = ld_relaxed_gpu(&status[j]);
        }
        const uint32_t inc = __ballot_sync(FULL, (s >> 62) == 2);
        if (inc) {
            const int first = __ffs(inc) - 1;
            uint64_t v = lane <= first ? (s & ST_VAL) : 0;
            prefix += warp_sum(v);
            break;
        }
        prefix += warp_sum(s & ST_VAL);
        idx -= 32;
    }
    if (lane == 0) st_release_gpu(&status[tile], ST_INC | ((prefix + aggregate) & ST_VAL));
    fence_acq_rel_gpu();
    return prefix;
}

// Largest i in [lo, hi) with a[i] <= x, assuming a[lo] <= x and a nondecreasing.
__device__ __forceinline__ uint64_t last_le(const uint64_t* __restrict__ a, uint64_t lo,
                                            uint64_t hi, uint64_t x) {
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Warp-cooperative version of last_le: 32 probes per round. Every lane gets
// the same answer.
__device__ __forceinline__ uint64_t warp_last_le(const uint64_t* __restrict__ a, uint64_t lo,
                                                 uint64_t hi, uint64_t x) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 1) {
        const uint64_t span = hi - lo;
        const uint64_t step = (span + 31) / 32;
        const uint64_t probe = lo + static_cast<uint64_t>(lane) * step;
        const bool ok = probe < hi && a[probe] <= x;
        const uint32_t m = __ballot_sync(FULL, ok);
        // m is a prefix of lanes (a is sorted); at least lane 0 holds.
        const int cnt = __popc(m);
        const uint64_t nlo = lo + static_cast<uint64_t>(cnt - 1) * step;
        uint64_t nhi = nlo + step;
        if (nhi > hi) nhi = hi;
        lo = nlo;
        hi = nhi;
        if (step == 1) break;
    }
    return lo;
}

// ---- shared-memory addresses and cp.async (global -> shared, L1-allocating)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion
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
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_addr(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the bulk stores issued so far have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// barrier over the first `nthreads` threads of the CTA (whole warps), id 1..15
template <int ID, int NTHREADS>
__device__ __forceinline__ void named_barrier() {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NTHREADS) : "memory");
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



}  // namespace pbg
