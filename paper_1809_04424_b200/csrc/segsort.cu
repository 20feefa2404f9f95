// segsort.cu -- S7 for tie groups: lex re-sort of the simplices whose owner
// edges share a filtration level.
//
// The owner-edge enumeration emits each level's simplices grouped by owner
// edge.  When a level holds a single edge this is already the (filt, lex)
// order; when several edges share the level (length ties, reading A3: equal
// lengths share a level; reading A4: ties broken lexicographically
// "does not determine a total ordering") the level's range must be sorted by
// the lex code of its vertex tuple.  Levels are contiguous output ranges
// [off[g0], off[g1]), so this is a segmented sort over the tie ranges:
//   levels : head flags over the owner edges + a scan list every level start
//            (no thread walks a level);
//   small  : one CTA bitonic sort per segment of <= kSmall entries;
//   large  : ALL larger segments in ONE radix sort of (segment, lex code)
//            keys -- packed into 64 bits when they fit (n <= 2^16 for
//            triangles with up to 2^16 segments, ...), else two stable LSD
//            sorts (code, then segment) -- and one scatter back, so a tie-heavy
//            input (HIV's Hamming distances) costs a few device-wide
//            passes, not a host loop of per-level sorts.
// Lex codes pack the sorted vertex tuple: 3 x 21 bits for triangles, 4 x 16
// bits for tetrahedra.
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

// level heads over the owner edges [p_lo, p_hi)
__global__ void k_level_heads(const uint32_t* __restrict__ efilt, int64_t p_lo, int64_t p_hi,
                              uint32_t* __restrict__ head) {
    for (int64_t p = p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p_hi;
         p += (int64_t)gridDim.x * blockDim.x)
        head[p - p_lo] = (p == p_lo || efilt[p - 1] != efilt[p]) ? 1u : 0u;
}

// level starts, compacted in order (starts[nlev] = p_hi)
__global__ void k_level_starts(const uint32_t* __restrict__ head, const uint64_t* __restrict__ pos, int64_t p_lo,
                               int64_t span, uint32_t* __restrict__ starts) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < span; q += (int64_t)gridDim.x * blockDim.x)
        if (head[q]) starts[pos[q]] = (uint32_t)(p_lo + q);
}

// one thread per level: levels of >= 2 edges and >= 2 simplices are tie segments
__global__ void k_tie_segs(const uint32_t* __restrict__ starts, int64_t nlev, int64_t p_hi,
                           const uint64_t* __restrict__ off, uint64_t slot0, Seg* __restrict__ segs,
                           unsigned long long* __restrict__ nseg) {
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nlev; l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = starts[l], b = l + 1 < nlev ? (int64_t)starts[l + 1] : p_hi;
        if (b - a < 2) continue;
        const uint64_t len = off[b] - off[a];
        if (len < 2) continue;
        segs[atomicAdd(nseg, 1ull)] = Seg{off[a] - slot0, len};
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

// segment of element q of the concatenated large segments (segoff: nseg + 1
// ascending offsets): binary search, element-parallel kernels below
__device__ __forceinline__ int64_t seg_of(const uint64_t* __restrict__ segoff, int64_t nseg, uint64_t q) {
    int64_t lo = 0, hi = nseg;   // last g with segoff[g] <= q
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(segoff + mid) <= q) lo = mid; else hi = mid;
    }
    return lo;
}

// the same with a per-thread cached segment: grid-stride steps mostly land in
// the same or the next segment (segments are long), so the binary search
// (a chain of dependent loads) is the exception
__device__ __forceinline__ int64_t seg_cached(const uint64_t* __restrict__ segoff, int64_t nseg, uint64_t q,
                                              int64_t& g) {
    if (g >= 0 && g < nseg) {
        const uint64_t a = __ldg(segoff + g), b = __ldg(segoff + g + 1);
        if (q >= a && q < b) return g;
        if (q >= b && g + 1 < nseg && q < __ldg(segoff + g + 2)) return ++g;
    }
    g = seg_of(segoff, nseg, q);
    return g;
}

#define ELEM_STRIDE(q, M) \
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (uint64_t)(M); \
         q += (uint64_t)gridDim.x * blockDim.x)

// Keys of the large segments: element q (0..M) of the concatenated segments
// (segment g at [segoff[g], segoff[g+1])) -> (g << cbits | code) when packed,
// else the code alone; vals = the element's slot.
template <int K>
__global__ void k_big_keys(const Seg* __restrict__ segs, const uint64_t* __restrict__ segoff, int64_t nseg,
                           int64_t M, const uint32_t* __restrict__ verts, int cbits, int packed,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
    int64_t gc = -1;
    ELEM_STRIDE(q, M) {
        const int64_t g = seg_cached(segoff, nseg, q, gc);
        const uint64_t slot = segs[g].start + (q - segoff[g]);
        const uint64_t code = Code<K>::pack(verts + (K + 1) * slot);
        key[q] = packed ? (((uint64_t)g << cbits) | code) : code;
        val[q] = (uint32_t)slot;
    }
}

// segment index of each sorted element's slot (two-pass path): binary search
// in the segment starts (segments sorted by start)
__global__ void k_seg_of(const uint32_t* __restrict__ val, int64_t M, const Seg* __restrict__ segs, int64_t nseg,
                         uint64_t* __restrict__ key) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < M; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t slot = val[q];
        int64_t lo = 0, hi = nseg;   // last segment with start <= slot
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (segs[mid].start <= slot) lo = mid; else hi = mid;
        }
        key[q] = (uint64_t)lo;
    }
}

// gather the rows of the sorted elements (before any is overwritten)
template <int K>
__global__ void k_big_rows(const uint32_t* __restrict__ val, int64_t M, const uint32_t* __restrict__ rows,
                           uint32_t* __restrict__ rcopy) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < M; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t src = val[q];
#pragma unroll
        for (int c = 0; c <= K; ++c) rcopy[(K + 1) * q + c] = rows[(K + 1) * src + c];
    }
}

// scatter: the q-th sorted element goes to slot segs[g].start + (q - segoff[g])
// of its segment g; its vertices are decoded from its code
template <int K>
__global__ void k_big_apply(const Seg* __restrict__ segs, const uint64_t* __restrict__ segoff, int64_t nseg,
                            int64_t M, const uint64_t* __restrict__ codes, const uint32_t* __restrict__ rcopy,
                            uint32_t* __restrict__ verts, uint32_t* __restrict__ rows) {
    int64_t gc = -1;
    ELEM_STRIDE(q, M) {
        const int64_t g = seg_cached(segoff, nseg, q, gc);
        const uint64_t slot = segs[g].start + (q - segoff[g]);
        uint32_t v[K + 1];
        Code<K>::unpack(codes[q], v);
        uint32_t* out = verts + (K + 1) * slot;
        for (int c = 0; c <= K; ++c) out[c] = v[c];
        if (rows)
            for (int c = 0; c <= K; ++c) rows[(K + 1) * slot + c] = rcopy[(K + 1) * q + c];
    }
}

__global__ void k_codes_of(const uint32_t* __restrict__ val, int64_t M, const uint32_t* __restrict__ verts, int k,
                           uint64_t* __restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < M; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* v = verts + (uint64_t)(k + 1) * val[q];
        uint64_t c = 0;
        const int bits = k == 2 ? 21 : 16;
        for (int i = 0; i <= k; ++i) c = (c << bits) | v[i];
        out[q] = c;
    }
}

// ---- keys-only path (triangles, n <= kTableMaxN): the key packs (segment,
// v0, v1, v2) with vbits per vertex; after the sort the vertices are decoded
// from the key and the D_2 rows recomputed from an n x n table of edge
// positions (L2-resident for the tie-heavy inputs: HIV's 1088 vertices take
// 4.7 MB), so no row or value moves through the sort.
constexpr int64_t kTableMaxN = 8192;

__global__ void k_tab_positions(const uint32_t* __restrict__ ev, int64_t E, int64_t n, uint32_t* __restrict__ tab) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = ev[2 * p], b = ev[2 * p + 1];
        tab[a * (uint64_t)n + b] = (uint32_t)p;
        tab[b * (uint64_t)n + a] = (uint32_t)p;
    }
}

__global__ void k_tri_keys(const Seg* __restrict__ segs, const uint64_t* __restrict__ segoff, int64_t nseg,
                           int64_t M, const uint32_t* __restrict__ verts, int vb, uint64_t* __restrict__ key) {
    int64_t gc = -1;
    ELEM_STRIDE(q, M) {
        const int64_t g = seg_cached(segoff, nseg, q, gc);
        const uint32_t* v = verts + 3 * (segs[g].start + (q - segoff[g]));
        key[q] = ((uint64_t)g << (3 * vb)) | ((uint64_t)v[0] << (2 * vb)) | ((uint64_t)v[1] << vb) | v[2];
    }
}

__global__ void k_tri_apply(const Seg* __restrict__ segs, const uint64_t* __restrict__ segoff, int64_t nseg,
                            int64_t M, const uint64_t* __restrict__ key, int vb, const uint32_t* __restrict__ tab,
                            int64_t n, uint32_t* __restrict__ verts, uint32_t* __restrict__ rows) {
    const uint64_t m = (1ull << vb) - 1ull;
    int64_t gc = -1;
    ELEM_STRIDE(q, M) {
        const int64_t g = seg_cached(segoff, nseg, q, gc);
        const uint64_t slot = segs[g].start + (q - segoff[g]);
        const uint64_t kk = key[q];
        const uint32_t a = (uint32_t)((kk >> (2 * vb)) & m), b = (uint32_t)((kk >> vb) & m), c = (uint32_t)(kk & m);
        uint32_t* out = verts + 3 * slot;
        out[0] = a;
        out[1] = b;
        out[2] = c;
        if (rows) {
            uint32_t r0 = __ldg(tab + (uint64_t)a * n + b), r1 = __ldg(tab + (uint64_t)a * n + c),
                     r2 = __ldg(tab + (uint64_t)b * n + c);
            uint32_t t;
            if (r0 > r1) { t = r0; r0 = r1; r1 = t; }
            if (r1 > r2) { t = r1; r1 = r2; r2 = t; }
            if (r0 > r1) { t = r0; r0 = r1; r1 = t; }
            uint32_t* rw = rows + 3 * slot;
            rw[0] = r0;
            rw[1] = r1;
            rw[2] = r2;
        }
    }
}

int bits_for(uint64_t v) {   // bits to hold 0..v
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

template <int K>
void sort_ties(const uint32_t* efilt, const uint64_t* off, int64_t E, int64_t p_lo, int64_t p_hi, int64_t n,
               uint32_t* verts, uint32_t* rows, const uint32_t* ev, cudaStream_t s) {
    uint64_t slot0 = 0;
    VRB_CUDA(cudaMemcpyAsync(&slot0, off + p_lo, sizeof(slot0), cudaMemcpyDeviceToHost, s));
    const int64_t span = p_hi - p_lo;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(span, 256), (int64_t)device_sm_count() * 16);
    // ---- levels (heads + scan), then tie segments
    DBuf<uint32_t> head(span, s), starts(span, s);
    DBuf<uint64_t> hpos(span + 1, s);
    k_level_heads<<<g, 256, 0, s>>>(efilt, p_lo, p_hi, head.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(head.get(), hpos.get(), span, s);
    uint64_t nlev = 0;
    VRB_CUDA(cudaMemcpyAsync(&nlev, hpos.get() + span, sizeof(nlev), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (nlev == (uint64_t)span) return;   // every level holds one edge: nothing to re-sort
    k_level_starts<<<g, 256, 0, s>>>(head.get(), hpos.get(), p_lo, span, starts.get());
    VRB_LAUNCH_CHECK();
    DBuf<Seg> segs((size_t)nlev, s);
    DBuf<unsigned long long> nseg(1, s);
    VRB_CUDA(cudaMemsetAsync(nseg.get(), 0, sizeof(unsigned long long), s));
    const unsigned gl = (unsigned)std::min<int64_t>(ceil_div((int64_t)nlev, 256), (int64_t)device_sm_count() * 16);
    k_tie_segs<<<gl, 256, 0, s>>>(starts.get(), (int64_t)nlev, p_hi, off, slot0, segs.get(), nseg.get());
    VRB_LAUNCH_CHECK();
    unsigned long long h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, nseg.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    head.reset();
    starts.reset();
    hpos.reset();
    if (h == 0) return;
    // ---- small segments: one CTA each
    const unsigned gs = (unsigned)std::min<unsigned long long>(h, (unsigned long long)device_sm_count() * 4);
    k_sort_small<K><<<gs, kSortThreads, 0, s>>>(segs.get(), (int64_t)h, verts, rows);
    VRB_LAUNCH_CHECK();
    // ---- large segments: one batched sort
    std::vector<Seg> hs(h);
    VRB_CUDA(cudaMemcpyAsync(hs.data(), segs.get(), h * sizeof(Seg), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    std::vector<Seg> big;
    for (const Seg& S : hs)
        if (S.len > (uint64_t)small_cap<K>()) big.push_back(S);
    if (big.empty()) return;
    std::sort(big.begin(), big.end(), [](const Seg& a, const Seg& b) { return a.start < b.start; });
    const int64_t nb = (int64_t)big.size();
    std::vector<uint64_t> hoff(nb + 1, 0);
    for (int64_t q = 0; q < nb; ++q) hoff[q + 1] = hoff[q] + big[q].len;
    const int64_t M = (int64_t)hoff[nb];
    DBuf<Seg> dseg(nb, s);
    DBuf<uint64_t> dsegoff(nb + 1, s);
    VRB_CUDA(cudaMemcpyAsync(dseg.get(), big.data(), nb * sizeof(Seg), cudaMemcpyHostToDevice, s));
    VRB_CUDA(cudaMemcpyAsync(dsegoff.get(), hoff.data(), (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    const int vbits = bits_for((uint64_t)std::max<int64_t>(n - 1, 1));
    const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(M, 256), (int64_t)device_sm_count() * 16);
    if (K == 2 && (!rows || (ev && n <= kTableMaxN)) && 3 * vbits + bits_for((uint64_t)std::max<int64_t>(nb - 1, 1)) <= 64) {
        DBuf<uint32_t> tab;
        if (rows) {
            tab.alloc((size_t)(n * n), s);
            VRB_CUDA(cudaMemsetAsync(tab.get(), 0xFF, tab.bytes(), s));
            k_tab_positions<<<(unsigned)std::min<int64_t>(ceil_div(E, 256), (int64_t)device_sm_count() * 16), 256, 0,
                              s>>>(ev, E, n, tab.get());
            VRB_LAUNCH_CHECK();
        }
        DBuf<uint64_t> k0(M, s), k1(M, s);
        k_tri_keys<<<gb, 256, 0, s>>>(dseg.get(), dsegoff.get(), nb, M, verts, vbits, k0.get());
        VRB_LAUNCH_CHECK();
        const uint64_t vary = varying_bits(k0.get(), M, s);
        const bool alt = radix_sort_keys(k0.get(), k1.get(), M, vary, s);
        k_tri_apply<<<gb, 256, 0, s>>>(dseg.get(), dsegoff.get(), nb, M, alt ? k1.get() : k0.get(), vbits, tab.get(), n,
                                       verts, rows);
        VRB_LAUNCH_CHECK();
        return;
    }
    const int cbits = (K + 1) * Code<K>::kBitsPer;   // as packed by Code<K>
    // the code's top (K + 1) * kBitsPer bits hold K + 1 ids of vbits each:
    // only its low (K + 1 - 1) * kBitsPer + vbits bits can be nonzero
    const int code_bits = K * Code<K>::kBitsPer + vbits;
    const bool packed = code_bits + bits_for((uint64_t)std::max<int64_t>(nb - 1, 1)) <= 64;
    (void)cbits;
    DBuf<uint64_t> k0(M, s), k1(M, s);
    DBuf<uint32_t> v0(M, s), v1(M, s);
    k_big_keys<K><<<gb, 256, 0, s>>>(dseg.get(), dsegoff.get(), nb, M, verts, code_bits, packed ? 1 : 0, k0.get(),
                                    v0.get());
    VRB_LAUNCH_CHECK();
    const uint64_t vary = varying_bits(k0.get(), M, s);
    bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), M, vary, s);
    uint64_t* sk = alt ? k1.get() : k0.get();
    uint32_t* sv = alt ? v1.get() : v0.get();
    const unsigned gm = (unsigned)std::min<int64_t>(ceil_div(M, 256), (int64_t)device_sm_count() * 16);
    if (!packed) {
        // stable second pass on the segment index (LSD: code, then segment)
        uint64_t* ok = alt ? k0.get() : k1.get();
        uint32_t* ov = alt ? v0.get() : v1.get();
        k_seg_of<<<gm, 256, 0, s>>>(sv, M, dseg.get(), nb, sk);
        VRB_LAUNCH_CHECK();
        const uint64_t vary2 = varying_bits(sk, M, s);
        const bool alt2 = radix_sort_pairs(sk, ok, sv, ov, M, vary2, s);
        if (alt2) { sk = ok; sv = ov; }
        k_codes_of<<<gm, 256, 0, s>>>(sv, M, verts, K, sk);   // the sorted elements' codes
        VRB_LAUNCH_CHECK();
    } else {
        // strip the segment bits: keys are then the codes
        k_codes_of<<<gm, 256, 0, s>>>(sv, M, verts, K, sk);
        VRB_LAUNCH_CHECK();
    }
    DBuf<uint32_t> rcopy;
    if (rows) {
        rcopy.alloc((size_t)(K + 1) * M, s);
        k_big_rows<K><<<gm, 256, 0, s>>>(sv, M, rows, rcopy.get());
        VRB_LAUNCH_CHECK();
    }
    k_big_apply<K><<<gb, 256, 0, s>>>(dseg.get(), dsegoff.get(), nb, M, sk, rcopy.get(), verts, rows);
    VRB_LAUNCH_CHECK();
}

}  // namespace

void sort_tie_groups(int k, const uint32_t* efilt, const uint64_t* off, int64_t E, int64_t p_lo, int64_t p_hi,
                     int64_t n, uint32_t* verts, uint32_t* rows, cudaStream_t s, const uint32_t* ev) {
    if (p_lo >= p_hi) return;
    if (k == 2) {
        sort_ties<2>(efilt, off, E, p_lo, p_hi, n, verts, rows, ev, s);
    } else {
        if (n > 65536) fail(VRB_ENOTSUP, "tetrahedra tie sort needs n <= 65536 (16-bit lex codes)");
        sort_ties<3>(efilt, off, E, p_lo, p_hi, n, verts, rows, ev, s);
    }
}

}  // namespace vrb
