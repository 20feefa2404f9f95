// radix_sort.cu -- stable LSD radix sort of (u64 key, u32 value) pairs,
// onesweep style (one kernel per 8-bit digit pass).
//
//   k_histograms : ONE read of the keys builds the 256-bin histogram of every
//                  digit that varies (per-CTA shared histograms, atomics)
//   k_scan_bins  : exclusive scan per digit pass (256 entries each, tiny)
//   k_onesweep   : per pass; CTAs take tiles in order (atomic tile counter);
//                  stable in-tile ranking (warps own contiguous item runs,
//                  match_any per round); per-digit global offsets by decoupled
//                  look-back over earlier tiles; a shared-memory exchange turns
//                  the scatter into contiguous per-digit runs.
// Digits with no varying bit (varying_bits()) are skipped.  Stability: items
// of a tile are ranked in index order, tiles in index order.  This sort is
// the GPU sortperm of the edge lengths (paper sec. 4.5) and the
// grouping step of the neighbourhood-list builds.
#include <vector>

#include "vrb_internal.cuh"

namespace vrb {
namespace {

#ifndef VRB_SORT_THREADS
#define VRB_SORT_THREADS 256
#endif
constexpr int kThreads = VRB_SORT_THREADS;   // >= 256, a multiple of 32
constexpr int kWarps = kThreads / 32;
#ifndef VRB_SORT_MINB
#define VRB_SORT_MINB 4
#endif
#ifndef VRB_SORT_BALLOT
#define VRB_SORT_BALLOT 0
#endif
#ifndef VRB_SORT_MINB_KEYS
#define VRB_SORT_MINB_KEYS 4
#endif
#ifndef VRB_SORT_LOOK
#define VRB_SORT_LOOK 4
#endif
constexpr int kLook = VRB_SORT_LOOK;         // tiles read per look-back step
// items per thread: (key, value) pairs 8, keys only 20 (B200 sweep: the
// C5A edge sort 12.7 -> 12.4 ms at 8 instead of 12; HIV's keys-only tie
// sort 14.5 -> 13.5 / 12.7 ms at 16 / 20)
#ifndef VRB_SORT_ITEMS_PAIRS
#define VRB_SORT_ITEMS_PAIRS 8
#endif
#ifndef VRB_SORT_ITEMS_KEYS
#define VRB_SORT_ITEMS_KEYS 20
#endif
template <bool kVals>
__host__ __device__ constexpr int items_per_thread() { return kVals ? VRB_SORT_ITEMS_PAIRS : VRB_SORT_ITEMS_KEYS; }
template <bool kVals>
__host__ __device__ constexpr int tile_items() { return kThreads * items_per_thread<kVals>(); }
constexpr int kBins = 256;

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kThreads) k_histograms(const uint64_t* __restrict__ keys, int64_t n,
                                                         uint32_t digit_mask, unsigned long long* __restrict__ hist,
                                                         uint64_t bias) {
    __shared__ uint32_t h[8][kBins];
    for (int q = threadIdx.x; q < 8 * kBins; q += kThreads) (&h[0][0])[q] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i] - bias;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            if ((digit_mask >> d) & 1u) atomicAdd(&h[d][(k >> (8 * d)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 8 * kBins; q += kThreads) {
        const int d = q / kBins;
        if (((digit_mask >> d) & 1u) && (&h[0][0])[q]) atomicAdd(&hist[q], (unsigned long long)(&h[0][0])[q]);
    }
}

// exclusive scan of each digit's 256 bins (one warp per digit)
__global__ void k_scan_bins(unsigned long long* __restrict__ hist) {
    const int d = blockIdx.x, lane = threadIdx.x;
    unsigned long long* h = hist + d * kBins;
    unsigned long long carry = 0;
    for (int b0 = 0; b0 < kBins; b0 += 32) {
        const unsigned long long v = h[b0 + lane];
        unsigned long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        h[b0 + lane] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

template <bool kVals>
struct SweepSmem {
    uint64_t key[tile_items<kVals>()];
    uint32_t val[kVals ? tile_items<kVals>() : 1];
    uint32_t woff[kWarps][kBins];   // per-warp digit counts -> tile-local start per warp
    uint32_t tstart[kBins];         // tile-local start of each digit
    unsigned long long gstart[kBins];   // global position of the tile's run of each digit
    uint32_t wsum[kWarps];
    uint32_t tile_id;
};

// kVals = false: keys only (vals_in / vals_out unused)
template <bool kVals>
__global__ void __launch_bounds__(kThreads, kVals ? VRB_SORT_MINB : VRB_SORT_MINB_KEYS) k_onesweep(const uint64_t* __restrict__ keys_in,
                                                       const uint32_t* __restrict__ vals_in,
                                                       uint64_t* __restrict__ keys_out,
                                                       uint32_t* __restrict__ vals_out, int64_t n, int shift,
                                                       const unsigned long long* __restrict__ pass_base,
                                                       unsigned long long* __restrict__ status,
                                                       unsigned* __restrict__ tile_counter, uint64_t bias) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SweepSmem<kVals>& S = *reinterpret_cast<SweepSmem<kVals>*>(smem_raw);
    constexpr int kItems = items_per_thread<kVals>();
    constexpr int kTile = tile_items<kVals>();
    constexpr int kWarpItems = 32 * kItems;   // contiguous items per warp
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) S.tile_id = atomicAdd(tile_counter, 1u);
    for (int q = threadIdx.x; q < kWarps * kBins; q += kThreads) (&S.woff[0][0])[q] = 0;
    __syncthreads();
    const uint32_t tile = S.tile_id;
    const int64_t tile_base = (int64_t)tile * kTile;
    const int64_t base = tile_base + (int64_t)wid * kWarpItems;
    const int tile_n = (int)min((int64_t)kTile, n - tile_base);
    // ---- load: warp w owns items [base, base + 512) in rounds of 32 lanes
    uint64_t k[kItems];
    uint32_t v[kItems], rk[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t i = base + r * 32 + lane;
        k[r] = i < n ? keys_in[i] - bias : 0ull;
        v[r] = (kVals && i < n) ? vals_in[i] : 0u;
    }
    // ---- stable warp-local ranks (rounds in order, lanes in order)
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t i = base + r * 32 + lane;
        const bool ok = i < n;
        const uint32_t dg = ok ? (uint32_t)((k[r] >> shift) & 0xFF) : (uint32_t)(kBins + lane);
#if VRB_SORT_BALLOT
        // experiment (VRB_SORT_BALLOT=1): peers by one ballot per digit bit
        // (and one for the past-the-end lanes, whose digits are unique)
        // instead of match.any -- measured slower for the edge sort (C5A
        // edge rank 12.7 -> 13.6 ms), slightly faster for HIV's keys-only
        // tie sort with 3 CTAs per SM (14.5 -> 14.0 ms)
        uint32_t peers = __ballot_sync(0xffffffffu, ok);
        if (!ok) peers = ~peers;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const bool bit = (dg >> b) & 1u;
            const uint32_t vote = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? vote : ~vote;
        }
#else
        const uint32_t peers = __match_any_sync(0xffffffffu, dg);
#endif
        const uint32_t before = ok ? S.woff[wid][dg] : 0u;
        __syncwarp();
        rk[r] = before + __popc(peers & lt);
        if (ok && (peers & lt) == 0) S.woff[wid][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // ---- digit d (thread d < 256): warps in order -> per-warp starts; tile count
    const int d = threadIdx.x;
    const bool has_digit = d < kBins;
    uint32_t cnt = 0;
    if (has_digit) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = S.woff[w][d];
            S.woff[w][d] = cnt;
            cnt += c;
        }
        // publish the tile aggregate early, then look back over earlier tiles
        unsigned long long* st = status + (int64_t)tile * kBins + d;
        unsigned long long excl = 0;
        if (tile == 0) {
            atomicExch(st, kFlagPre | cnt);
        } else {
            atomicExch(st, kFlagAgg | cnt);
            // look back kLook tiles per step: their status words are read
            // together, so a walk over aggregate-only tiles is not a chain of
            // single dependent L2 reads
            bool done = false;
            for (int64_t j = (int64_t)tile - 1; !done; j -= kLook) {
                unsigned long long sv[kLook];
#pragma unroll
                for (int u = 0; u < kLook; ++u)
                    sv[u] = j - u >= 0 ? *(const volatile unsigned long long*)(status + (j - u) * kBins + d)
                                       : kFlagPre;
#pragma unroll
                for (int u = 0; u < kLook; ++u) {
                    if (done) break;
                    unsigned long long s = sv[u];
                    while ((s & (kFlagAgg | kFlagPre)) == 0)
                        s = *(const volatile unsigned long long*)(status + (j - u) * kBins + d);
                    excl += s & kValMask;
                    if (s & kFlagPre) done = true;
                }
            }
            atomicExch(st, kFlagPre | (excl + cnt));
        }
        S.gstart[d] = pass_base[d] + excl;
    }
    // tile-local starts: exclusive scan of cnt over the 256 digits (warps 0..7)
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31 && wid < kBins / 32) S.wsum[wid] = x;
    __syncthreads();
    if (has_digit) {
        uint32_t wpre = 0;
#pragma unroll
        for (int w = 0; w < kBins / 32; ++w)
            if (w < wid) wpre += S.wsum[w];
        S.tstart[d] = wpre + x - cnt;
    }
    __syncthreads();
    // ---- exchange through shared memory in tile order
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t i = base + r * 32 + lane;
        if (i < n) {
            const uint32_t dg = (uint32_t)((k[r] >> shift) & 0xFF);
            const uint32_t pos = S.tstart[dg] + S.woff[wid][dg] + rk[r];
            S.key[pos] = k[r];
            if (kVals) S.val[pos] = v[r];
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < tile_n; q += kThreads) {
        const uint64_t kk = S.key[q];
        const uint32_t dg = (uint32_t)((kk >> shift) & 0xFF);
        const unsigned long long dst = S.gstart[dg] + (uint32_t)(q - S.tstart[dg]);
        keys_out[dst] = kk;
        if (kVals) vals_out[dst] = S.val[q];
    }
}

}  // namespace

template <bool kVals>
bool radix_sort_impl(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt, int64_t n,
                     uint64_t varying, cudaStream_t s, uint64_t bias, bool* biased) {
    if (biased) *biased = false;
    if (n <= 1 || varying == 0) return false;
    if (biased) *biased = true;
    uint32_t digit_mask = 0;
    for (int d = 0; d < 8; ++d)
        if ((varying >> (8 * d)) & 0xFFull) digit_mask |= 1u << d;
    const int64_t ntiles = ceil_div(n, (int64_t)tile_items<kVals>());
    DBuf<unsigned long long> hist(8 * kBins, s);
    VRB_CUDA(cudaMemsetAsync(hist.get(), 0, hist.bytes(), s));
    const unsigned hg = (unsigned)std::min<int64_t>(ceil_div(n, kThreads), (int64_t)device_sm_count() * 8);
    k_histograms<<<hg, kThreads, 0, s>>>(keys, n, digit_mask, hist.get(), bias);
    VRB_LAUNCH_CHECK();
    k_scan_bins<<<8, 32, 0, s>>>(hist.get());
    VRB_LAUNCH_CHECK();
    const int npass = __builtin_popcount(digit_mask);
    DBuf<unsigned long long> status((size_t)ntiles * kBins * npass, s);
    DBuf<unsigned> counters(npass, s);
    VRB_CUDA(cudaMemsetAsync(status.get(), 0, status.bytes(), s));
    VRB_CUDA(cudaMemsetAsync(counters.get(), 0, counters.bytes(), s));
    const size_t smem = sizeof(SweepSmem<kVals>);
    VRB_CUDA(cudaFuncSetAttribute(k_onesweep<kVals>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bool alt = false;
    int pass = 0;
    for (int d = 0; d < 8; ++d) {
        if (!((digit_mask >> d) & 1u)) continue;
        uint64_t* kin = alt ? keys_alt : keys;
        uint64_t* kout = alt ? keys : keys_alt;
        uint32_t* vin = alt ? vals_alt : vals;
        uint32_t* vout = alt ? vals : vals_alt;
        k_onesweep<kVals><<<(unsigned)ntiles, kThreads, smem, s>>>(kin, vin, kout, vout, n, 8 * d, hist.get() + d * kBins,
                                                            status.get() + (size_t)pass * ntiles * kBins,
                                                            counters.get() + pass, pass == 0 ? bias : 0ull);
        VRB_LAUNCH_CHECK();
        alt = !alt;
        ++pass;
    }
    return alt;
}

bool radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt, int64_t n,
                      uint64_t varying, cudaStream_t s, uint64_t bias, bool* biased) {
    return radix_sort_impl<true>(keys, keys_alt, vals, vals_alt, n, varying, s, bias, biased);
}

bool radix_sort_keys(uint64_t* keys, uint64_t* keys_alt, int64_t n, uint64_t varying, cudaStream_t s) {
    return radix_sort_impl<false>(keys, keys_alt, nullptr, nullptr, n, varying, s, 0, nullptr);
}

}  // namespace vrb
