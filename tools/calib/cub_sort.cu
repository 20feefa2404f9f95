// Calibration only (not product code): how fast does the CUDA toolkit's own
// CUB onesweep radix sort order N (u64 key, u32 value) pairs on this B200?
// Gives the achievable per-pass bandwidth that libvrb's hand-written
// k_onesweep (radix_sort.cu) is measured against.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/calib/cub_sort.cu -o /tmp/cub_sort
//   /tmp/cub_sort 200000000
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__global__ void init(uint64_t* k, uint32_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull;
        z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
        k[i] = 0x4000000000000000ull | (z >> 9);   // 55 varying bits, like C5A's length keys
        v[i] = (uint32_t)i;
    }
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 200000000;
    uint64_t *k0, *k1; uint32_t *v0, *v1;
    cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bits : {32, 24, 64}) {
        const int begin = 64 - bits;
        size_t tmp = 0; void* t = nullptr;
        cub::DoubleBuffer<uint64_t> dk(k0, k1); cub::DoubleBuffer<uint32_t> dv(v0, v1);
        cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, n, begin, 64);
        cudaMalloc(&t, tmp);
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            init<<<2048, 256>>>(k0, v0, n);
            cub::DoubleBuffer<uint64_t> ek(k0, k1); cub::DoubleBuffer<uint32_t> ev(v0, v1);
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortPairs(t, tmp, ek, ev, n, begin, 64);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (rep && ms < best) best = ms;
        }
        const double passes = (bits + 7) / 8;
        printf("cub SortPairs n=%lld key bits [%d,64): %.3f ms = %g passes x %.3f ms, %.0f GB/s per pass (24 B/item)\n",
               (long long)n, begin, best, passes, best / passes, 24.0 * n / (best / passes * 1e-3) / 1e9);
        cudaFree(t);
    }
    return 0;
}
