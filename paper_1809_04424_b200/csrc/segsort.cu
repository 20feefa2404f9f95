// segsort.cu -- S7 for tie groups: lex re-sort of the simplices whose owner
// edges share a filtration level.
//
// The owner-edge enumeration emits each level's simplices grouped by owner
// edge.  When a level holds a single edge this is already the (filt, lex)
// order; when several edges share the level (length ties, reading A3: equal
// lengths share a level; reading A4: ties broken lexicographically
// "does not determine a total ordering") the level's range must be sorted by
// the lex code of its vertex tuple.  Levels are contiguous output ranges
// [off[g0], off[g1]), so this is a segmented sort over the (few, usually tiny)
// tie ranges: one CTA bitonic sort per segment up to kSmall entries, the
// global radix sort beyond.  Lex codes pack the sorted vertex tuple into 64
// bits: 3 x 21 bits for triangles, 4 x 16 bits for tetrahedra.
#include <algorithm>
#include <vector>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kSortThreads = 512;
template <int K>
__host__ __device__ constexpr int small_cap() { return K == 2 ? 2048 : 1024; }   // static shared memory < 48 KB

struct Seg {
    uint64_t start;
    uint64_t len;
};

// One thread per level start; appends (start, len) segments of tie levels.
__global__ void k_find_ties(const uint32_t* __restrict__ efilt, const uint64_t* __restrict__ off, int64_t E,
                            int64_t p_lo, int64_t p_hi, uint64_t slot0, Seg* __restrict__ segs,
                            unsigned long long* __restrict__ nseg) {
    for (int64_t p = p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p_hi;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = efilt[p];
        if (p > 0 && efilt[p - 1] == f) continue;          // not a level start
        if (p + 1 >= E || efilt[p + 1] != f) continue;     // single-edge level: already lex
        int64_t q = p + 1;
        while (q < E && efilt[q] == f) ++q;
        const uint64_t len = off[q] - off[p];
        if (len < 2) continue;
        const unsigned long long at = atomicAdd(nseg, 1ull);
        segs[at] = Seg{off[p] - slot0, len};
    }
}

template <int K>
struct Code {
    static constexpr int kBitsPer = K == 2 ? 21 : 16;
    static constexpr uint64_t kMask = (1ull << kBitsPer) - 1;
    __device__ static uint64_t pack(const uint32_t* v) {
        uint64_t c = 0;
#pragma unroll
        for (int i = 0; i <= K; ++i) c = (c << kBitsPer) | v[i];
        return c;
    }
    __device__ static void unpack(uint64_t c, uint32_t* v) {
#pragma unroll
        for (int i = K; i >= 0; --i) { v[i] = (uint32_t)(c & kMask); c >>= kBitsPer; }
    }
};

template <int K>
__global__ void __launch_bounds__(kSortThreads) k_sort_small(const Seg* __restrict__ segs, int64_t nseg,
                                                             uint32_t* __restrict__ verts, uint32_t* __restrict__ rows) {
    constexpr int kSmall = small_cap<K>();
    __shared__ uint64_t key[kSmall];
    __shared__ uint16_t idx[kSmall];
    __shared__ uint32_t rbuf[kSmall * (K + 1)];
    for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const Seg S = segs[sg];
        if (S.len > (uint64_t)kSmall) continue;
        const int len = (int)S.len;
        int N = 1;
        while (N < len) N <<= 1;
        for (int q = threadIdx.x; q < N; q += kSortThreads) {
            if (q < len) {
                key[q] = Code<K>::pack(verts + (K + 1) * (S.start + q));
                if (rows)
                    for (int c = 0; c <= K; ++c) rbuf[(K + 1) * q + c] = rows[(K + 1) * (S.start + q) + c];
            } else {
                key[q] = ~0ull;
            }
            idx[q] = (uint16_t)q;
        }
        __syncthreads();
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < N; i += kSortThreads) {
                    const int l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        const uint64_t a = key[i], b = key[l];
                        if ((a > b) == up) {
                            key[i] = b; key[l] = a;
                            const uint16_t t = idx[i]; idx[i] = idx[l]; idx[l] = t;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int q = threadIdx.x; q < len; q += kSortThreads) {
            uint32_t v[K + 1];
            Code<K>::unpack(key[q], v);
            uint32_t* o = verts + (K + 1) * (S.start + q);
            for (int c = 0; c <= K; ++c) o[c] = v[c];
            if (rows) {
                const int src = idx[q];
                for (int c = 0; c <= K; ++c) rows[(K + 1) * (S.start + q) + c] = rbuf[(K + 1) * src + c];
            }
        }
        __syncthreads();
    }
}

template <int K>
__global__ void k_seg_keys(const uint32_t* __restrict__ verts, uint64_t start, int64_t len, uint64_t* __restrict__ key) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < len; q += (int64_t)gridDim.x * blockDim.x)
        key[q] = Code<K>::pack(verts + (K + 1) * (start + q));
}

template <int K>
__global__ void k_seg_apply(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ rows_copy, uint64_t start, int64_t len,
                            uint32_t* __restrict__ verts, uint32_t* __restrict__ rows) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < len; q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v[K + 1];
        Code<K>::unpack(key[q], v);
        uint32_t* o = verts + (K + 1) * (start + q);
        for (int c = 0; c <= K; ++c) o[c] = v[c];
        if (rows) {
            const uint32_t src = perm[q];
            for (int c = 0; c <= K; ++c) rows[(K + 1) * (start + q) + c] = rows_copy[(K + 1) * (int64_t)src + c];
        }
    }
}

template <int K>
void sort_ties(const uint32_t* efilt, const uint64_t* off, int64_t E, int64_t p_lo, int64_t p_hi, uint32_t* verts,
               uint32_t* rows, cudaStream_t s) {
    uint64_t slot0 = 0;
    VRB_CUDA(cudaMemcpyAsync(&slot0, off + p_lo, sizeof(slot0), cudaMemcpyDeviceToHost, s));
    const int64_t span = p_hi - p_lo;
    DBuf<Seg> segs((size_t)span, s);
    DBuf<unsigned long long> nseg(1, s);
    VRB_CUDA(cudaMemsetAsync(nseg.get(), 0, sizeof(unsigned long long), s));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(span, 256), (int64_t)device_sm_count() * 16);
    k_find_ties<<<g, 256, 0, s>>>(efilt, off, E, p_lo, p_hi, slot0, segs.get(), nseg.get());
    VRB_LAUNCH_CHECK();
    unsigned long long h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, nseg.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h == 0) return;
    const unsigned gs = (unsigned)std::min<unsigned long long>(h, (unsigned long long)device_sm_count() * 4);
    k_sort_small<K><<<gs, kSortThreads, 0, s>>>(segs.get(), (int64_t)h, verts, rows);
    VRB_LAUNCH_CHECK();
    std::vector<Seg> hs(h);
    VRB_CUDA(cudaMemcpyAsync(hs.data(), segs.get(), h * sizeof(Seg), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    for (const Seg& S : hs) {
        if (S.len <= (uint64_t)small_cap<K>()) continue;
        const int64_t len = (int64_t)S.len;
        DBuf<uint64_t> k0(len, s), k1(len, s);
        DBuf<uint32_t> v0(len, s), v1(len, s);
        const unsigned gg = (unsigned)std::min<int64_t>(ceil_div(len, 256), 4096);
        k_seg_keys<K><<<gg, 256, 0, s>>>(verts, S.start, len, k0.get());
        VRB_LAUNCH_CHECK();
        iota_u32(v0.get(), len, s);
        const uint64_t vary = varying_bits(k0.get(), len, s);
        const bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), len, vary, s);
        DBuf<uint32_t> rcopy;
        if (rows) {
            rcopy.alloc((size_t)((K + 1) * len), s);
            VRB_CUDA(cudaMemcpyAsync(rcopy.get(), rows + (K + 1) * S.start, (K + 1) * len * sizeof(uint32_t),
                                     cudaMemcpyDeviceToDevice, s));
        }
        k_seg_apply<K><<<gg, 256, 0, s>>>(alt ? k1.get() : k0.get(), alt ? v1.get() : v0.get(), rcopy.get(),
                                          S.start, len, verts, rows);
        VRB_LAUNCH_CHECK();
    }
}

}  // namespace

void sort_tie_groups(int k, const uint32_t* efilt, const uint64_t* off, int64_t E, int64_t p_lo, int64_t p_hi,
                     int64_t n, uint32_t* verts, uint32_t* rows, cudaStream_t s) {
    if (p_lo >= p_hi) return;
    if (k == 2) {
        sort_ties<2>(efilt, off, E, p_lo, p_hi, verts, rows, s);
    } else {
        if (n > 65536) fail(VRB_ENOTSUP, "tetrahedra tie sort needs n <= 65536 (16-bit lex codes)");
        sort_ties<3>(efilt, off, E, p_lo, p_hi, verts, rows, s);
    }
}

}  // namespace vrb
