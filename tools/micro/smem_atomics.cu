// microbenchmark: shared-memory marking costs on B200 (random targets per lane)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int MODE>
__global__ void k(int iters, uint32_t range_bits, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t words[16][256];   // 1 KB per warp
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = threadIdx.x; q < 16 * 256; q += blockDim.x) (&words[0][0])[q] = 0;
    __syncthreads();
    uint32_t* w = words[wid];
    uint8_t* b = reinterpret_cast<uint8_t*>(w);
    uint32_t h = hash32(threadIdx.x * 7919 + blockIdx.x);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        h = hash32(h + i);
        const uint32_t r = h & ((1u << range_bits) - 1);   // rank in [0, 2^range_bits)
        if (MODE == 0) b[r & 1023] = 1;                       // byte flag
        if (MODE == 1) atomicOr(&w[(r >> 5) & 255], 1u << (r & 31));   // bitmap atomic
        if (MODE == 2) { uint32_t pe = __match_any_sync(0xffffffffu, (r >> 5) & 255); if ((pe & ((1u << lane) - 1)) == 0) w[(r >> 5) & 255] |= 1u << (r & 31); }
    }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, t1 - t0);
    if (w[lane] == 12345) sink[0] = 1;
}

int main() {
    unsigned long long* d; uint32_t* s;
    cudaMalloc(&d, 8); cudaMalloc(&s, 4);
    const int iters = 4096, blocks = 148 * 1;
    for (int mode = 0; mode < 3; ++mode) for (int rb = 10; rb <= 12; rb += 2) {
        cudaMemset(d, 0, 8);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<blocks, 512>>>(iters, rb, d, s);
        if (mode == 1) k<1><<<blocks, 512>>>(iters, rb, d, s);
        if (mode == 2) k<2><<<blocks, 512>>>(iters, rb, d, s);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * 512 * iters;
        printf("mode %d (%s) range 2^%d: %.3f ms, %.2f lane-ops/cycle/SM (at 1.965 GHz)\n", mode,
               mode == 0 ? "STS.U8 flag" : mode == 1 ? "ATOMS.OR" : "match+STS", rb, ms,
               ops / (ms * 1e-3 * 1.965e9) / 148);
    }
    return 0;
}
