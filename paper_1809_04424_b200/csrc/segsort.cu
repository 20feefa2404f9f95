// segsort.cu -- S7 for tie groups: lex re-sort of the simplices whose owner
// edges share a filtration level.
//
// The owner-edge enumeration emits each level's simplices grouped by owner
// edge.  When a level holds a single edge this is already the (filt, lex)
// order; when several edges share the level (length ties, reading A3: equal
// lengths share a level; reading A4: ties broken lexicographically
// "does not determine a total ordering") the level's range must be sorted by
// the lex code of its vertex tuple.  Levels are contiguous ranges
// [toff[g0], toff[g1]) of the output, so this is a segmented sort over the
// (few, usually tiny) tie ranges: one CTA bitonic sort per segment up to
// kSmall entries, the global radix sort beyond.
#include <algorithm>
#include <vector>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kSmall = 2048;
constexpr int kSortThreads = 512;

struct Seg {
    uint64_t start;
    uint64_t len;
};

// One thread per tie-group start; appends (start, len) segments.
__global__ void k_find_ties(const uint32_t* __restrict__ efilt, const uint64_t* __restrict__ toff, int64_t E,
                            int64_t p_lo, int64_t p_hi, uint64_t slot0, Seg* __restrict__ segs,
                            unsigned long long* __restrict__ nseg) {
    for (int64_t p = p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p_hi;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = efilt[p];
        if (p > 0 && efilt[p - 1] == f) continue;          // not a level start
        if (p + 1 >= E || efilt[p + 1] != f) continue;     // single-edge level: already lex
        int64_t q = p + 1;
        while (q < E && efilt[q] == f) ++q;
        const uint64_t len = toff[q] - toff[p];
        if (len < 2) continue;
        const unsigned long long at = atomicAdd(nseg, 1ull);
        segs[at] = Seg{toff[p] - slot0, len};
    }
}

__device__ __forceinline__ uint64_t lex_code(const uint32_t* v) {
    return ((uint64_t)v[0] << 42) | ((uint64_t)v[1] << 21) | (uint64_t)v[2];
}

__global__ void __launch_bounds__(kSortThreads) k_sort_small(const Seg* __restrict__ segs, int64_t nseg,
                                                             uint32_t* __restrict__ tv, uint32_t* __restrict__ rows) {
    __shared__ uint64_t key[kSmall];
    __shared__ uint16_t idx[kSmall];
    __shared__ uint32_t rbuf[kSmall * 3];
    for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const Seg S = segs[sg];
        if (S.len > (uint64_t)kSmall) continue;
        const int len = (int)S.len;
        int N = 1;
        while (N < len) N <<= 1;
        for (int q = threadIdx.x; q < N; q += kSortThreads) {
            if (q < len) {
                key[q] = lex_code(tv + 3 * (S.start + q));
                if (rows) {
                    rbuf[3 * q] = rows[3 * (S.start + q)];
                    rbuf[3 * q + 1] = rows[3 * (S.start + q) + 1];
                    rbuf[3 * q + 2] = rows[3 * (S.start + q) + 2];
                }
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
            const uint64_t c = key[q];
            uint32_t* v = tv + 3 * (S.start + q);
            v[0] = (uint32_t)(c >> 42);
            v[1] = (uint32_t)((c >> 21) & 0x1FFFFF);
            v[2] = (uint32_t)(c & 0x1FFFFF);
            if (rows) {
                const int src = idx[q];
                uint32_t* r = rows + 3 * (S.start + q);
                r[0] = rbuf[3 * src]; r[1] = rbuf[3 * src + 1]; r[2] = rbuf[3 * src + 2];
            }
        }
        __syncthreads();
    }
}

__global__ void k_seg_keys(const uint32_t* __restrict__ tv, uint64_t start, int64_t len, uint64_t* __restrict__ key) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < len; q += (int64_t)gridDim.x * blockDim.x)
        key[q] = lex_code(tv + 3 * (start + q));
}

__global__ void k_seg_apply(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ rows_copy, uint64_t start, int64_t len,
                            uint32_t* __restrict__ tv, uint32_t* __restrict__ rows) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < len; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t c = key[q];
        uint32_t* v = tv + 3 * (start + q);
        v[0] = (uint32_t)(c >> 42);
        v[1] = (uint32_t)((c >> 21) & 0x1FFFFF);
        v[2] = (uint32_t)(c & 0x1FFFFF);
        if (rows) {
            const uint32_t src = perm[q];
            rows[3 * (start + q)] = rows_copy[3 * (int64_t)src];
            rows[3 * (start + q) + 1] = rows_copy[3 * (int64_t)src + 1];
            rows[3 * (start + q) + 2] = rows_copy[3 * (int64_t)src + 2];
        }
    }
}

}  // namespace

void sort_tie_groups(const uint32_t* efilt, const uint64_t* toff, int64_t E, int64_t p_lo, int64_t p_hi,
                     int64_t n, uint32_t* tv, uint32_t* rows, cudaStream_t s) {
    (void)n;
    if (p_lo >= p_hi) return;
    uint64_t slot0 = 0;
    VRB_CUDA(cudaMemcpyAsync(&slot0, toff + p_lo, sizeof(slot0), cudaMemcpyDeviceToHost, s));
    const int64_t span = p_hi - p_lo;
    DBuf<Seg> segs((size_t)span, s);
    DBuf<unsigned long long> nseg(1, s);
    VRB_CUDA(cudaMemsetAsync(nseg.get(), 0, sizeof(unsigned long long), s));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(span, 256), (int64_t)device_sm_count() * 16);
    k_find_ties<<<g, 256, 0, s>>>(efilt, toff, E, p_lo, p_hi, slot0, segs.get(), nseg.get());
    VRB_LAUNCH_CHECK();
    unsigned long long h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, nseg.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h == 0) return;
    const unsigned gs = (unsigned)std::min<unsigned long long>(h, (unsigned long long)device_sm_count() * 4);
    k_sort_small<<<gs, kSortThreads, 0, s>>>(segs.get(), (int64_t)h, tv, rows);
    VRB_LAUNCH_CHECK();
    // large segments: global radix sort each
    std::vector<Seg> hs(h);
    VRB_CUDA(cudaMemcpyAsync(hs.data(), segs.get(), h * sizeof(Seg), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    for (const Seg& S : hs) {
        if (S.len <= (uint64_t)kSmall) continue;
        const int64_t len = (int64_t)S.len;
        DBuf<uint64_t> k0(len, s), k1(len, s);
        DBuf<uint32_t> v0(len, s), v1(len, s);
        const unsigned gg = (unsigned)std::min<int64_t>(ceil_div(len, 256), 4096);
        k_seg_keys<<<gg, 256, 0, s>>>(tv, S.start, len, k0.get());
        VRB_LAUNCH_CHECK();
        iota_u32(v0.get(), len, s);
        const uint64_t vary = varying_bits(k0.get(), len, s);
        const bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), len, vary, s);
        DBuf<uint32_t> rcopy;
        if (rows) {
            rcopy.alloc((size_t)(3 * len), s);
            VRB_CUDA(cudaMemcpyAsync(rcopy.get(), rows + 3 * S.start, 3 * len * sizeof(uint32_t),
                                     cudaMemcpyDeviceToDevice, s));
        }
        k_seg_apply<<<gg, 256, 0, s>>>(alt ? k1.get() : k0.get(), alt ? v1.get() : v0.get(), rcopy.get(),
                                       S.start, len, tv, rows);
        VRB_LAUNCH_CHECK();
    }
}

}  // namespace vrb
