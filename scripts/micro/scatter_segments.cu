// scatter_segments.cu — how fast the memory system takes short scattered
// tuple segments (a u32 key stream + an f64 value stream, like the expand's
// runs and the heavy split's bucket segments): N tuples written as segments
// of s consecutive tuples at pseudo-random offsets, unaligned or aligned to
// the segment length, over a window of W tuples (W small: L2-resident).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scatter_segments scatter_segments.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// one warp step = 32 consecutive tuples of the flat stream; tuple t belongs
// to segment t / s, position t % s
// (s and the window are powers of two: shifts and masks only, so the kernel's
// own arithmetic stays off the critical path)
__global__ void k_scatter(uint32_t* keys, double* vals, uint64_t ntuples, uint32_t ls, uint64_t window,
                          int aligned, uint64_t seed) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t s = 1ull << ls;
#pragma unroll 4
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntuples; t += stride) {
        const uint64_t seg = t >> ls, pos = t & (s - 1);
        uint64_t off = mix(seg ^ seed) & (window - 1);
        if (off + s > window) off = window - s;
        if (aligned) off &= ~(s - 1);
        __stcs(keys + off + pos, (uint32_t)t);
        __stcs(vals + off + pos, (double)t);
    }
}

int main(int argc, char** argv) {
    const uint64_t ntuples = 1ull << 28;
    const uint64_t cap = 1ull << 28;
    uint32_t* keys;
    double* vals;
    cudaMalloc(&keys, cap * 4 + 4096);
    cudaMalloc(&vals, cap * 8 + 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("%8s %8s %10s %10s %12s %10s\n", "seg", "aligned", "window", "ms", "Gseg/s", "GB/s");
    for (uint64_t window : {cap, (uint64_t)1 << 20}) {
        for (int aligned = 0; aligned < 2; ++aligned) {
            for (uint32_t s : {4u, 8u, 16u, 32u, 64u, 128u, 512u, 4096u}) {
                float best = 1e30f;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaEventRecord(e0);
                    k_scatter<<<148 * 8, 256>>>(keys, vals, ntuples, __builtin_ctz(s), window, aligned, 1234 + rep);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (rep && ms < best) best = ms;
                }
                printf("%8u %8d %10llu %10.3f %12.2f %10.1f\n", s, aligned, (unsigned long long)window, best,
                       ntuples / (double)s / best * 1e-6, ntuples * 12.0 / best * 1e-6);
            }
        }
    }
    return 0;
}
