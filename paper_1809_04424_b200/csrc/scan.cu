// scan.cu -- device-wide prefix sums and small helpers (reduce-then-scan).
#include "vrb_internal.cuh"

namespace vrb {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;                      // per thread per tile
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T warp_inclusive(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide inclusive scan of one value per thread; returns (inclusive, total).
template <class T>
__device__ __forceinline__ T block_inclusive(T v, T* smem_warp, T& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_inclusive(v);
    if (lane == 31) smem_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = lane < (kScanThreads / 32) ? smem_warp[lane] : T(0);
        w = warp_inclusive(w);
        if (lane < (kScanThreads / 32)) smem_warp[lane] = w;
    }
    __syncthreads();
    T prefix = wid ? smem_warp[wid - 1] : T(0);
    total = smem_warp[kScanThreads / 32 - 1];
    __syncthreads();
    return inc + prefix;
}

// In: a pointer, or an index view such as HeadFlags
template <class In, class Tacc>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(In in, int64_t n, Tacc* __restrict__ sums) {
    __shared__ Tacc red[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    Tacc acc = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        int64_t i = base + it * kScanThreads + threadIdx.x;
        if (i < n) acc += (Tacc)in[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        Tacc t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += red[w];
        sums[blockIdx.x] = t;
    }
}

// Scan one tile with a per-tile offset.  Exclusive: out has n + 1 entries.
template <class In, class Tout, bool kInclusive>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(In in, int64_t n, const Tout* __restrict__ tile_off,
                                                            Tout* __restrict__ out) {
    __shared__ Tout warp_tot[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    Tout carry = tile_off ? tile_off[blockIdx.x] : Tout(0);
    for (int it = 0; it < kScanItems; ++it) {
        int64_t i = base + it * kScanThreads + threadIdx.x;
        Tout v = i < n ? (Tout)in[i] : Tout(0);
        Tout total;
        Tout inc = block_inclusive<Tout>(v, warp_tot, total);
        if (i < n) out[i] = carry + (kInclusive ? inc : inc - v);
        if (!kInclusive && i == n) out[n] = carry + inc - v;   // grand total slot
        carry += total;
    }
    if (!kInclusive && n % kScanTile == 0 && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
        out[n] = carry;
}

template <class In, class Tout, bool kInclusive>
void scan_impl(In in, Tout* out, int64_t n, cudaStream_t s) {
    if (n == 0) {
        if (!kInclusive) VRB_CUDA(cudaMemsetAsync(out, 0, sizeof(Tout), s));
        return;
    }
    const int64_t tiles = ceil_div(n, kScanTile);
    if (tiles == 1) {
        k_tile_scan<In, Tout, kInclusive><<<1, kScanThreads, 0, s>>>(in, n, nullptr, out);
        VRB_LAUNCH_CHECK();
        return;
    }
    DBuf<Tout> sums(tiles, s), offs(tiles + 1, s);
    k_tile_sums<In, Tout><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, sums.get());
    VRB_LAUNCH_CHECK();
    scan_impl<const Tout*, Tout, false>(sums.get(), offs.get(), tiles, s);
    k_tile_scan<In, Tout, kInclusive><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, offs.get(), out);
    VRB_LAUNCH_CHECK();
}

// head flags of a sorted key array as a scan input: 1 where a run of equal
// keys starts (dense ranks = their inclusive scan, reading A3)
struct HeadFlags {
    const uint64_t* key;
    __device__ __forceinline__ uint32_t operator[](int64_t i) const {
        return (i == 0 || __ldg(key + i) != __ldg(key + i - 1)) ? 1u : 0u;
    }
};

__global__ void k_varying(const uint64_t* __restrict__ k, int64_t n, unsigned long long* out) {
    const uint64_t k0 = k[0];
    uint64_t acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc |= k[i] ^ k0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc |= __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicOr(out, (unsigned long long)acc);
}

__global__ void k_minmax(const uint64_t* __restrict__ k, int64_t n, unsigned long long* out) {
    uint64_t mn = ~0ull, mx = 0, any = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = k[i];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
        any |= v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t a = __shfl_down_sync(0xffffffffu, mn, o), b = __shfl_down_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
        any |= __shfl_down_sync(0xffffffffu, any, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], (unsigned long long)mn);
        atomicMax(&out[1], (unsigned long long)mx);
        atomicOr(&out[2], (unsigned long long)any);
    }
}

__global__ void k_fill_u32(uint32_t* p, uint32_t v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_iota_u32(uint32_t* p, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

unsigned grid_for(int64_t n, int threads) {
    int64_t g = ceil_div(n, threads);
    int64_t cap = (int64_t)device_sm_count() * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void exclusive_scan(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s) {
    scan_impl<const uint32_t*, uint64_t, false>(in, out, n, s);
}
void dense_ranks(const uint64_t* sorted_keys, uint32_t* out, int64_t n, cudaStream_t s) {
    scan_impl<HeadFlags, uint32_t, true>(HeadFlags{sorted_keys}, out, n, s);
}
void exclusive_scan(const uint64_t* in, uint64_t* out, int64_t n, cudaStream_t s) {
    scan_impl<const uint64_t*, uint64_t, false>(in, out, n, s);
}
void inclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s) {
    scan_impl<const uint32_t*, uint32_t, true>(in, out, n, s);
}

uint64_t varying_bits(const uint64_t* keys, int64_t n, cudaStream_t s) {
    if (n <= 1) return 0;
    DBuf<unsigned long long> acc(1, s);
    VRB_CUDA(cudaMemsetAsync(acc.get(), 0, sizeof(unsigned long long), s));
    k_varying<<<grid_for(n, 256), 256, 0, s>>>(keys, n, acc.get());
    VRB_LAUNCH_CHECK();
    unsigned long long h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, acc.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return (uint64_t)h;
}

uint64_t key_range(const uint64_t* keys, int64_t n, cudaStream_t s, uint64_t* kmin,
                   const unsigned long long* reduced) {
    *kmin = 0;
    if (n <= 0) return 0;
    DBuf<unsigned long long> acc;
    if (!reduced) {
        acc.alloc(3, s);
        const unsigned long long init[3] = {~0ull, 0ull, 0ull};
        VRB_CUDA(cudaMemcpyAsync(acc.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_minmax<<<grid_for(n, 256), 256, 0, s>>>(keys, n, acc.get());
        VRB_LAUNCH_CHECK();
    }
    unsigned long long h[3] = {0, 0, 0};
    VRB_CUDA(cudaMemcpyAsync(h, reduced ? reduced : acc.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    *kmin = h[0];
    uint64_t d = h[1] - h[0], mask = 0;
    while (d) { mask = (mask << 1) | 1ull; d >>= 1; }
    // bits below the lowest set bit of any key are zero in every key, and so
    // in every (key - min): those digits never vary (e.g. integer-valued
    // lengths, HIV's Hamming distances)
    if (h[2]) {
        const int tz = __builtin_ctzll(h[2]);
        mask &= tz >= 64 ? 0ull : ~((1ull << tz) - 1ull);
    }
    return mask;
}

void fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_fill_u32<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
    VRB_LAUNCH_CHECK();
}

void iota_u32(uint32_t* p, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_iota_u32<<<grid_for(n, 256), 256, 0, s>>>(p, n);
    VRB_LAUNCH_CHECK();
}

}  // namespace vrb
