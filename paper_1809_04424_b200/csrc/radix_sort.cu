// radix_sort.cu -- stable LSD radix sort of (u64 key, u32 value) pairs.
//
// One pass per 8-bit digit that actually varies across the keys (digits with
// no varying bit are skipped; see varying_bits()).  Each pass is
//   k_digit_hist  : per-tile 256-bin histogram          (reads keys)
//   exclusive_scan: digit-major offsets over all tiles   (tiny)
//   k_scatter     : stable in-tile ranking (warp match_any + per-warp digit
//                   counters, warps combined in order) and scatter
// Stability: items of a tile are ranked in index order (round, warp, lane),
// tiles in index order via the digit-major scan.  This is the sort behind the
// edge ranking (paper sec. 4.5: sortperm over the distance entries
// on the GPU) and behind the CSR builds.
#include "vrb_internal.cuh"

namespace vrb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kBins = 256;

__global__ void __launch_bounds__(kThreads) k_digit_hist(const uint64_t* __restrict__ keys, int64_t n,
                                                         int shift, int64_t ntiles,
                                                         uint32_t* __restrict__ counts) {
    __shared__ uint32_t hist[kWarps][kBins];
    for (int q = threadIdx.x; q < kWarps * kBins; q += kThreads) (&hist[0][0])[q] = 0;
    __syncthreads();
    const int wid = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int it = 0; it < kItems; ++it) {
        int64_t i = base + (int64_t)it * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&hist[wid][(keys[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    const int d = threadIdx.x;   // kThreads == kBins
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += hist[w][d];
    counts[(int64_t)d * ntiles + blockIdx.x] = t;
}

__global__ void __launch_bounds__(kThreads) k_scatter(const uint64_t* __restrict__ keys_in,
                                                      const uint32_t* __restrict__ vals_in,
                                                      uint64_t* __restrict__ keys_out,
                                                      uint32_t* __restrict__ vals_out, int64_t n,
                                                      int shift, int64_t ntiles,
                                                      const uint64_t* __restrict__ offsets) {
    __shared__ uint64_t run[kBins];            // running global offset per digit
    __shared__ uint64_t wcnt[kWarps][kBins];   // per-warp digit counts -> offsets
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    run[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int it = 0; it < kItems; ++it) {
        for (int q = threadIdx.x; q < kWarps * kBins; q += kThreads) (&wcnt[0][0])[q] = 0;
        __syncthreads();
        const int64_t i = base + (int64_t)it * kThreads + threadIdx.x;
        const bool valid = i < n;
        uint64_t key = valid ? keys_in[i] : 0;
        uint32_t val = valid ? vals_in[i] : 0;
        const uint32_t digit = valid ? (uint32_t)((key >> shift) & 0xFF) : (uint32_t)(kBins + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, digit);
        const uint32_t rank = __popc(peers & lt_mask);
        if (valid && rank == 0) wcnt[wid][digit] = __popc(peers);
        __syncthreads();
        {   // combine warps in order, per digit
            const int d = threadIdx.x;
            uint64_t r = run[d];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                uint64_t c = wcnt[w][d];
                wcnt[w][d] = r;
                r += c;
            }
            run[d] = r;
        }
        __syncthreads();
        if (valid) {
            const uint64_t dst = wcnt[wid][digit] + rank;
            keys_out[dst] = key;
            vals_out[dst] = val;
        }
        __syncthreads();
    }
}

}  // namespace

bool radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                      int64_t n, uint64_t varying, cudaStream_t s) {
    if (n <= 1 || varying == 0) return false;
    const int64_t ntiles = ceil_div(n, kTile);
    DBuf<uint32_t> counts((size_t)kBins * ntiles, s);
    DBuf<uint64_t> offsets((size_t)kBins * ntiles + 1, s);
    bool alt = false;
    for (int digit = 0; digit < 8; ++digit) {
        const int shift = 8 * digit;
        if (((varying >> shift) & 0xFFull) == 0) continue;
        uint64_t* kin = alt ? keys_alt : keys;
        uint64_t* kout = alt ? keys : keys_alt;
        uint32_t* vin = alt ? vals_alt : vals;
        uint32_t* vout = alt ? vals : vals_alt;
        k_digit_hist<<<(unsigned)ntiles, kThreads, 0, s>>>(kin, n, shift, ntiles, counts.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(counts.get(), offsets.get(), (int64_t)kBins * ntiles, s);
        k_scatter<<<(unsigned)ntiles, kThreads, 0, s>>>(kin, vin, kout, vout, n, shift, ntiles,
                                                       offsets.get());
        VRB_LAUNCH_CHECK();
        alt = !alt;
    }
    return alt;
}

}  // namespace vrb
