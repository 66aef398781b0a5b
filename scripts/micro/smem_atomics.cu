// Microbenchmark: shared-memory op throughput on the B200 (cycles per lane per SM)
// for the ranking primitives a per-bin sort/count can use.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 512, ITERS = 8192, SLOTS = 8192;

template <int MODE>
__global__ void k(uint32_t* out, uint32_t seed, long long* cyc) {
    __shared__ uint32_t t[SLOTS];
    for (int i = threadIdx.x; i < SLOTS; i += NT) t[i] = 0xffffffffu * (MODE == 2 || MODE == 8);
    __syncthreads();
    uint32_t x = seed ^ (threadIdx.x * 0x9E3779B1u) ^ (blockIdx.x * 0x85ebca6bu), acc = 0;
    long long c0 = clock64();
    #pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
        x = x * 1664525u + 1013904223u;
        uint32_t h = x >> 19;  // 13 bits
        if (MODE == 0) acc += atomicAdd(&t[h], 1u);                    // ATOMS.ADD with return
        else if (MODE == 1) atomicAdd(&t[h], 1u);                      // no return (RED-like)
        else if (MODE == 2) acc += atomicCAS(&t[h], 0xffffffffu, x);   // CAS
        else if (MODE == 3) { uint32_t v = t[h]; t[h ^ 1] = v + x; acc += v; }  // LDS + STS random
        else if (MODE == 4) acc += __popc(__match_any_sync(0xffffffffu, h >> 8));  // MATCH.ANY
        else if (MODE == 5) { uint32_t v = t[h]; acc += v; }            // LDS random
        else if (MODE == 6) atomicAdd(&t[h >> 1], 1u << ((h & 1) * 16));  // variable add, no return (histogram)
        else if (MODE == 7) acc += atomicAdd(&t[h >> 1], 1u << ((h & 1) * 16));  // variable add with return (scatter)
        else if (MODE == 8) acc += atomicCAS(&t[h], 0xffffffffu, x) == 0xffffffffu;  // CAS, insert-style
        else if (MODE == 9) atomicAdd(reinterpret_cast<double*>(t) + (h >> 1), 1.0 + x);  // f64 add (CAS loop), 4096 slots
        else if (MODE == 10) {  // f64 add through per-slot 32-bit locks (2048 slots + 2048 locks)
            const uint32_t sl = h >> 2;
            double* a = reinterpret_cast<double*>(t) + sl;  // doubles in t[0..4096)
            uint32_t* lock = t + 4096 + sl;
            bool done = false;
            while (!done) {
                if (atomicExch(lock, 1u) == 0u) {
                    *reinterpret_cast<volatile double*>(a) += 1.0 + x;
                    __threadfence_block();
                    *reinterpret_cast<volatile uint32_t*>(lock) = 0u;
                    done = true;
                }
            }
        }
        else if (MODE == 11) {  // f64 add as two u32 halves? no: 64-bit integer atomicAdd (native?)
            atomicAdd(reinterpret_cast<unsigned long long*>(t) + (h >> 1), (unsigned long long)x);
        }
    }
    __syncthreads();
    long long c1 = clock64();
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(c1 - c0));
    if (acc == 0x12345) out[0] = acc + t[x & (SLOTS - 1)];
}

template <int MODE>
void run(const char* name, int blocks_per_sm) {
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, 4); cudaMalloc(&cyc, 8); cudaMemset(cyc, 0, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int grid = sms * blocks_per_sm;
    k<MODE><<<grid, NT>>>(out, 1, cyc);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<grid, NT>>>(out, 2, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double lanes_per_sm = double(NT) * ITERS * blocks_per_sm;
    double avg_cyc = double(c) / grid;  // per CTA (all CTAs of an SM overlap)
    printf("%-28s blocks/SM=%d  %.3f ms  %.3f cycles/lane/SM (clock64)  %.3f ns/lane/SM (event)\n",
           name, blocks_per_sm, ms, avg_cyc / lanes_per_sm, ms * 1e6 / lanes_per_sm);
}

int main() {
    for (int b : {2, 4}) {
        run<0>("ATOMS.ADD (return)", b);
        run<1>("atomicAdd no return", b);
        run<2>("ATOMS.CAS", b);
        run<3>("LDS+STS random", b);
        run<4>("MATCH.ANY", b);
        run<5>("LDS random", b);
        run<6>("ATOMS var add, no return", b);
        run<7>("ATOMS var add, return", b);
        run<8>("ATOMS.CAS insert", b);
        run<9>("f64 atomicAdd (CAS loop)", b);
        run<10>("f64 add under u32 lock", b);
        run<11>("u64 atomicAdd", b);
    }
    return 0;
}
