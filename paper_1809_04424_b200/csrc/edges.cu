// edges.cu -- S3 (edge ranking) and S4 (neighbourhood lists + owner-edge plan).
//
// S3 follows the paper's GPU sortperm (sec. 4.5: order the
// distance entries, then read ranks off the permutation) with the readings of
// order by (len, i, j) (A4), filt = dense rank of len (A3, A14).
// The kept edges arrive in lex order, so a STABLE radix sort on the length
// bits alone yields (len, i, j) order.  Head flags + an inclusive scan give
// the dense rank; heads also write value_of_rank.
//
// S4 builds, per vertex v, (a) its neighbours in edge-position order (the
// "older-neighbour prefix" of an edge is a prefix of this list) and (b) its
// neighbours in id order with their edge positions.  Each edge p = (a, b) is
// then assigned to the endpoint x with the SHORTER prefix of neighbours older
// than p (to be scanned) and the other endpoint y (the "host", whose full
// neighbourhood is held as a dense map in shared memory during enumeration).
#include <algorithm>
#include <cstdlib>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

unsigned grid_for(int64_t n, int threads) {
    int64_t g = ceil_div(n, threads);
    int64_t cap = (int64_t)device_sm_count() * 32;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

#define GRID_STRIDE(i, n)                                                          \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n);       \
         i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_edge_outputs(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                               const uint32_t* __restrict__ ei, const uint32_t* __restrict__ ej,
                               const uint32_t* __restrict__ efilt, int64_t E, uint32_t* __restrict__ ev,
                               double* __restrict__ vor, uint64_t bias) {
    GRID_STRIDE(p, E) {
        const uint32_t lex = perm[p];
        ev[2 * p] = ei[lex];
        ev[2 * p + 1] = ej[lex];
        if (p == 0 || key[p] != key[p - 1]) vor[efilt[p] - 1] = __longlong_as_double((long long)(key[p] + bias));
    }
}

// packed ids (n <= 65536): the sorted values are (i << 16 | j) themselves
__global__ void k_edge_outputs_packed(const uint64_t* __restrict__ key, const uint32_t* __restrict__ pij,
                                      const uint32_t* __restrict__ efilt, int64_t E, uint2* __restrict__ ev,
                                      double* __restrict__ vor, uint64_t bias) {
    GRID_STRIDE(p, E) {
        const uint32_t v = pij[p];
        ev[p] = make_uint2(v >> 16, v & 0xFFFFu);
        const uint64_t k = key[p];
        if (p == 0 || k != key[p - 1]) vor[efilt[p] - 1] = __longlong_as_double((long long)(k + bias));
    }
}

// (vertex << 32 | entry): a keys-only sort on the vertex bits, stable, keeps
// each vertex's entries in position order
__global__ void k_keys_vertex(const uint32_t* __restrict__ ev, int64_t n2, uint64_t* __restrict__ key) {
    GRID_STRIDE(q, n2) key[q] = ((uint64_t)ev[q] << 32) | (uint64_t)q;
}

__global__ void k_keys_vertex_nbr(const uint32_t* __restrict__ ev, int64_t n2, uint64_t* __restrict__ key) {
    GRID_STRIDE(q, n2) key[q] = ((uint64_t)ev[q] << 21) | ev[q ^ 1];
}

// list offsets from the vertex-sorted entries: off[u] = first slot with
// key >= u (binary search per vertex; off[n] = 2E)
__global__ void k_offsets_from_sorted(const uint64_t* __restrict__ skey, int64_t n2, int64_t n,
                                      uint64_t* __restrict__ off) {
    GRID_STRIDE(u, n + 1) {
        int64_t lo = 0, hi = n2;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((skey[mid] >> 32) < (uint64_t)u) lo = mid + 1; else hi = mid;
        }
        off[u] = (uint64_t)lo;
    }
}

// position-ordered lists: slot s holds entry q = sorted[s] of vertex skey[s]
// listidx (entry -> its index in the vertex's list) is written only when the
// large-n rank path needs it; the scanned-endpoint choice instead takes, per
// edge, the minimum of (index << 1 | side) over its two entries (a shared-
// nothing atomicMin into an L2-resident word per edge, where the scatter of
// listidx made partial-sector DRAM writes)
__global__ void k_pos_lists(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ ev,
                            const uint64_t* __restrict__ off, int64_t n2, uint32_t* __restrict__ nkr,
                            uint32_t* __restrict__ np, uint32_t* __restrict__ listidx,
                            unsigned* __restrict__ scanpack) {
    GRID_STRIDE(s, n2) {
        const uint64_t kk = skey[s];
        const uint32_t q = (uint32_t)kk;
        const uint32_t v = (uint32_t)(kk >> 32);
        nkr[s] = ev[q ^ 1];
        np[s] = q >> 1;
        const uint32_t t = (uint32_t)(s - (int64_t)off[v]);
        if (listidx) listidx[q] = t;
        atomicMin(scanpack + (q >> 1), (t << 1) | (q & 1u));
    }
}

// id-ordered lists: slot s holds entry q = sorted[s]; its rank s - off[v] is
// recorded at the entry's slot of the position-ordered list
__global__ void k_id_ranks(const uint32_t* __restrict__ sorted, const uint32_t* __restrict__ ev,
                           const uint64_t* __restrict__ off, const uint32_t* __restrict__ listidx,
                           int64_t n2, int packed, uint32_t* __restrict__ nkr, uint32_t* __restrict__ nr) {
    GRID_STRIDE(s, n2) {
        const uint32_t q = sorted[s];
        const uint64_t o = off[ev[q]];
        const uint32_t r = (uint32_t)(s - (int64_t)o);
        const uint64_t slot = o + listidx[q];
        if (packed)
            nkr[slot] |= r << 16;
        else
            nr[slot] = r;
    }
}

// krank by counting (n <= kRankBitmapMax): one CTA per vertex v marks its
// neighbours in an n-bit shared bitmap; krank(k) = #neighbours with smaller id
// = prefix popcount of the bitmap below bit k.
constexpr int64_t kRankBitmapMax = 262144;

__global__ void __launch_bounds__(256) k_ranks_bitmap(const uint64_t* __restrict__ off, int64_t n, int packed,
                                                      uint32_t* __restrict__ nkr, uint32_t* __restrict__ nr,
                                                      const uint32_t* __restrict__ np, uint2* __restrict__ idl) {
    extern __shared__ uint32_t sm[];
    const int64_t nw = (n + 31) >> 5;
    uint32_t* bm = sm;
    uint32_t* wp = sm + nw;
    __shared__ uint32_t warp_tot[8];
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const uint64_t o0 = off[v], o1 = off[v + 1];
        if (o1 == o0) continue;
        for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) bm[w] = 0u;
        __syncthreads();
        for (uint64_t t = o0 + threadIdx.x; t < o1; t += blockDim.x) {
            const uint32_t k = nkr[t];
            atomicOr(&bm[k >> 5], 1u << (k & 31));
        }
        __syncthreads();
        // exclusive prefix popcount over the words: thread owns a contiguous run
        const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
        const int64_t w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
        uint32_t tot = 0;
        for (int64_t w = w0; w < w1; ++w) tot += __popc(bm[w]);
        uint32_t x = tot;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
        for (int q = 1; q < 32; q <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, q);
            if (lane >= q) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        uint32_t run = x - tot;
        for (int w = 0; w < wid; ++w) run += warp_tot[w];
        for (int64_t w = w0; w < w1; ++w) { wp[w] = run; run += __popc(bm[w]); }
        __syncthreads();
        for (uint64_t t = o0 + threadIdx.x; t < o1; t += blockDim.x) {
            const uint32_t k = nkr[t];
            const uint32_t r = wp[k >> 5] + __popc(bm[k >> 5] & ((1u << (k & 31)) - 1u));
            if (packed) {
                nkr[t] = k | (r << 16);
                if (idl) idl[o0 + r] = make_uint2(k, np[t]);   // the id-ordered list, fused
            } else {
                nr[t] = r;
            }
        }
        __syncthreads();
    }
}

// the endpoint with the shorter prefix (ties: the first endpoint)
__global__ void k_assign(const uint32_t* __restrict__ ev, const unsigned* __restrict__ scanpack, int64_t E,
                         uint32_t* __restrict__ scan_v, uint32_t* __restrict__ scan_len) {
    GRID_STRIDE(p, E) {
        const unsigned w = scanpack[p];
        scan_v[p] = ev[2 * p + (w & 1u)];
        scan_len[p] = w >> 1;
    }
}

// plan sort key of the owner edges p_lo + [0, m): host, then longest prefix
// first (LPT order inside a host, by prefix length in buckets of 2^lsh so
// that host and length fit 24 bits: three radix passes)
__global__ void k_host_keys(const uint32_t* __restrict__ ev, const uint32_t* __restrict__ scan_v,
                            const uint32_t* __restrict__ scan_len, int64_t p_lo, int64_t m, int lbits, int lsh,
                            uint64_t* __restrict__ host_key) {
    const uint32_t lmax = (1u << lbits) - 1u;
    GRID_STRIDE(q, m) {
        const int64_t p = p_lo + q;
        const uint32_t a = ev[2 * p], b = ev[2 * p + 1], x = scan_v[p];
        const uint32_t lb = min(scan_len[p] >> lsh, lmax);
        host_key[q] = ((uint64_t)(x == a ? b : a) << lbits) | (lmax - lb);
    }
}

__global__ void k_hosted_work(const uint32_t* __restrict__ hosted, const uint64_t* __restrict__ host_key,
                              const uint32_t* __restrict__ scan_v, const uint32_t* __restrict__ scan_len,
                              const uint64_t* __restrict__ off, int64_t E, int64_t p_lo, int lbits,
                              uint32_t* __restrict__ hosted_v, uint4* __restrict__ plan, uint32_t* __restrict__ work) {
    GRID_STRIDE(i, E) {
        const uint32_t p = (uint32_t)(p_lo + hosted[i]);
        const uint32_t x = scan_v[p], len = scan_len[p];
        hosted_v[i] = (uint32_t)(host_key[i] >> lbits);
        plan[i] = make_uint4(p, x, len, (uint32_t)(off[x + 1] - off[x]));
        work[i] = len;
    }
}

// (k, pos) of every neighbour in neighbour-ID order (packed lists): one warp
// per vertex scatters its position-ordered entries by their id rank
__global__ void k_id_lists(const uint64_t* __restrict__ off, int64_t n, const uint32_t* __restrict__ nkr,
                           const uint32_t* __restrict__ np, uint2* __restrict__ idl) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = w0; v < n; v += nw) {
        const uint64_t o0 = off[v], o1 = off[v + 1];
        for (uint64_t t = o0 + lane; t < o1; t += 32) {
            const uint32_t w = nkr[t];
            idl[o0 + (w >> 16)] = make_uint2(w & 0xFFFFu, np[t]);
        }
    }
}

__global__ void k_max_deg(const uint64_t* __restrict__ off, int64_t n, unsigned* __restrict__ out) {
    unsigned m = 0;
    GRID_STRIDE(v, n) m = max(m, (unsigned)(off[v + 1] - off[v]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Sort (keys, vals) where vals start as 0..m-1; returns the buffer with the
// sorted values (the other buffers are scratch).
uint32_t* sort_ids(DBuf<uint64_t>& k0, DBuf<uint64_t>& k1, DBuf<uint32_t>& v0, DBuf<uint32_t>& v1,
                   int64_t m, cudaStream_t s, uint64_t** sorted_keys = nullptr) {
    iota_u32(v0.get(), m, s);
    const uint64_t vary = varying_bits(k0.get(), m, s);
    const bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), m, vary, s);
    if (sorted_keys) *sorted_keys = alt ? k1.get() : k0.get();
    return alt ? v1.get() : v0.get();
}

}  // namespace

#ifndef VRB_EDGE_TOP_DIGITS
#define VRB_EDGE_TOP_DIGITS 4
#endif
#ifndef VRB_EDGE_RUN_MAX
#define VRB_EDGE_RUN_MAX 64
#endif
// After a sort on the high digits only (bits >= shift): runs of equal high
// bits are tiny for continuous data; sort each by the full key in place
// (insertion sort, stable, so equal keys keep their lex order).  A run longer
// than 64 whose keys are not all equal sets *fallback (full sort needed).
__global__ void k_fixup_runs(uint64_t* __restrict__ key, uint32_t* __restrict__ val, int64_t n, int shift,
                             int* __restrict__ fallback) {
    // lanes hold consecutive keys: the neighbours come by shuffles, so the
    // common case (a run of one) costs one coalesced load per key; only the
    // starts of real runs walk them
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
        const int64_t p = base + lane;
        const uint64_t k = p < n ? key[p] : ~0ull;
        uint64_t kprev = __shfl_up_sync(0xffffffffu, k, 1);
        uint64_t knext = __shfl_down_sync(0xffffffffu, k, 1);
        if (lane == 0) kprev = p > 0 && p < n ? key[p - 1] : ~0ull;
        if (lane == 31) knext = p + 1 < n ? key[p + 1] : ~0ull;
        if (p >= n) continue;
        const uint64_t hp = k >> shift;
        if (p > 0 && (kprev >> shift) == hp) continue;        // not the start of a run
        if (p + 1 >= n || (knext >> shift) != hp) continue;   // a run of one
        int64_t q = p + 1;
        while (q < n && q - p <= VRB_EDGE_RUN_MAX && (key[q] >> shift) == hp) ++q;
        if (q - p < 2) continue;
        if (q - p > VRB_EDGE_RUN_MAX) {
            const uint64_t k0 = key[p];
            for (int64_t r = p + 1; r < n && (key[r] >> shift) == hp; ++r)
                if (key[r] != k0) { atomicOr(fallback, 1); break; }
            continue;
        }
        for (int64_t a = p + 1; a < q; ++a) {
            const uint64_t k = key[a];
            const uint32_t v = val[a];
            int64_t b = a - 1;
            while (b >= p && key[b] > k) {
                key[b + 1] = key[b];
                val[b + 1] = val[b];
                --b;
            }
            key[b + 1] = k;
            val[b + 1] = v;
        }
    }
}

// Sort the kept edges by (len, i, j): a stable radix sort of the length bits
// (the input is in lex order), on the 4 highest varying digits only.  Results:
// so.key[q] + so.bias = length bits of the q-th edge, so.val[q] = its packed
// (i, j) (ke.packed) or lex index.  *shift_out > 0: the keys are ordered by
// (key >> shift) only -- runs of equal high bits still need their full-key
// order (k_fixup_runs, or the fused ranking pass).
static void sort_edges_top(KeptEdges& ke, cudaStream_t s, SortedEdges& so, int* shift_out, bool* alt_out) {
    const int64_t E = ke.E;
    so.E = E;
    so.packed = ke.packed;
    *shift_out = 0;
    *alt_out = false;
    if (E == 0) return;
    DBuf<uint64_t>& key_alt = so.key_alt;
    key_alt.alloc(E, s);
    // values: the packed (i, j) ids, or the lex index (permutation) for large n
    DBuf<uint32_t>& perm = so.perm;
    DBuf<uint32_t>& perm_alt = so.perm_alt;
    perm_alt.alloc(E, s);
    uint32_t* vals = ke.pij.get();
    if (!ke.packed) {
        perm.alloc(E, s);
        iota_u32(perm.get(), E, s);
        vals = perm.get();
    }
    // sort (len bits - min): only the digits of (max - min) vary
    uint64_t kmin = 0;
    const uint64_t vary = key_range(ke.key.get(), E, s, &kmin, ke.range.get());
    // radix passes on the 4 highest varying digits only (~31+ significant
    // bits); the runs left with equal high bits are finished afterwards
    int hi_digit = -1;
    for (int dg = 7; dg >= 0; --dg)
        if ((vary >> (8 * dg)) & 0xFFull) { hi_digit = dg; break; }
    const int shift = hi_digit >= VRB_EDGE_TOP_DIGITS ? 8 * (hi_digit - (VRB_EDGE_TOP_DIGITS - 1)) : 0;
    const uint64_t vary_top = shift ? (vary & ~((1ull << shift) - 1ull)) : vary;
    bool biased = false;
    const bool alt = radix_sort_pairs(ke.key.get(), key_alt.get(), vals, perm_alt.get(), E, vary_top, s, kmin, &biased);
    so.key = alt ? key_alt.get() : ke.key.get();
    so.val = alt ? perm_alt.get() : vals;
    so.bias = biased ? kmin : 0ull;
    *shift_out = (shift && (vary & ((1ull << shift) - 1ull))) ? shift : 0;   // varying bits below the sorted digits
    *alt_out = alt;
}

// Complete the order by a full-key radix sort (the fallback when a run of
// equal high bits is too long for the in-place fix-up).
static void sort_edges_full(KeptEdges& ke, cudaStream_t s, SortedEdges& so, bool alt) {
    const int64_t E = ke.E;
    uint64_t* k1 = const_cast<uint64_t*>(so.key);
    uint32_t* v1 = const_cast<uint32_t*>(so.val);
    uint32_t* vals0 = ke.packed ? ke.pij.get() : so.perm.get();
    uint64_t* k2 = alt ? ke.key.get() : so.key_alt.get();
    uint32_t* v2 = alt ? vals0 : so.perm_alt.get();
    const uint64_t vary = varying_bits(k1, E, s);
    const bool alt2 = radix_sort_pairs(k1, k2, v1, v2, E, vary, s);
    if (alt2) {
        so.key = k2;
        so.val = v2;
    }
}

void sort_edges(KeptEdges& ke, cudaStream_t s, SortedEdges& so) {
    int shift = 0;
    bool alt = false;
    sort_edges_top(ke, s, so, &shift, &alt);
    if (!shift) return;
    const int64_t E = ke.E;
    DBuf<int> fb(1, s);
    VRB_CUDA(cudaMemsetAsync(fb.get(), 0, sizeof(int), s));
    k_fixup_runs<<<grid_for(E, 256), 256, 0, s>>>(const_cast<uint64_t*>(so.key), const_cast<uint32_t*>(so.val), E,
                                                  shift, fb.get());
    VRB_LAUNCH_CHECK();
    int h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, fb.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h) sort_edges_full(ke, s, so, alt);   // heavy clustering of the high bits: every digit
}

namespace {
// Fused S3 epilogue (one pass over the high-bit-sorted keys, in place of the
// run fix-up, the two-pass head-flag scan and the output kernel).  A tile
// of 2048 positions is staged in shared memory with halos; every run of
// equal high bits (C5A: 47% of the edges sit in runs of 2..10) is put in
// full-key order by ranking each item within its run (stable: equal keys
// keep their lex order) -- a run belongs to the tile it starts in, a run
// longer than kRkRunMax must hold equal keys (its order stands; otherwise
// the caller re-sorts).  Heads of equal-length runs are counted by warp
// ballots, turned into dense ranks by a chained scan over tiles (decoupled
// look-back, tiles taken in order), and each warp writes its positions'
// (i, j), filt and value_of_rank in lane-consecutive (coalesced) rounds.
constexpr int kRkThreads = 256;
constexpr int kRkWarps = kRkThreads / 32;
constexpr int kRkTile = 2048;
constexpr int kRkRunMax = 64;
constexpr int kRkHalo = kRkRunMax + 1;
constexpr int kRkStage = kRkTile + 2 * kRkHalo;
constexpr unsigned long long kRkAgg = 1ull << 62, kRkPre = 2ull << 62, kRkVal = (1ull << 62) - 1;

struct RankArgs {
    const uint64_t* key;   // + bias = length bits
    const uint32_t* val;   // packed (i << 16 | j), or the lex index into ei / ej
    int64_t E;
    int shift;             // > 0: ordered only by key >> shift so far
    uint64_t bias;
    const uint32_t* ei;
    const uint32_t* ej;    // null when packed
    uint32_t* ev;
    uint32_t* efilt;
    double* vor;
    unsigned long long* status;
    unsigned* tile_counter;
    int* fallback;
};

__device__ __forceinline__ uint2 edge_of(const RankArgs& A, uint32_t v) {
    return A.ej ? make_uint2(__ldg(A.ei + v), __ldg(A.ej + v)) : make_uint2(v >> 16, v & 0xFFFFu);
}

__global__ void __launch_bounds__(kRkThreads) k_rank_edges(RankArgs A) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wtot[kRkWarps];
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned s_own_lo, s_own_hi;         // owned positions, relative to t0
    __shared__ uint64_t s_key[kRkStage];            // window [t0 - halo, t1 + halo), as sorted so far
    __shared__ uint32_t s_val[kRkStage];
    __shared__ uint16_t s_perm[kRkTile + kRkHalo];  // owned positions (from t0) -> window index
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(A.tile_counter, 1u);
        s_own_lo = 0xFFFFFFFFu;
        s_own_hi = 0u;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t E = A.E;
    const int sh = A.shift;
    const int64_t t0 = (int64_t)tile * kRkTile;
    const int64_t wb = t0 - kRkHalo;                 // window base (may be negative)
    const int t1r = (int)(min(t0 + kRkTile, E) - t0);   // tile length
    const int h0r = (int)(max(t0 - kRkHalo, (int64_t)0) - wb), h1r = (int)(min(t0 + kRkTile + kRkHalo, E) - wb);
    for (int w = h0r + threadIdx.x; w < h1r; w += kRkThreads) {
        s_key[w] = __ldcs(A.key + wb + w);
        s_val[w] = __ldcs(A.val + wb + w);
    }
    __syncthreads();
    const int T0 = kRkHalo, T1 = kRkHalo + t1r;      // the tile in window coordinates
    // ---- final places (s_perm) of the owned items
    unsigned my_lo = 0xFFFFFFFFu, my_hi = 0u;
    for (int w = T0 + threadIdx.x; w < h1r; w += kRkThreads) {
        const uint64_t kq = s_key[w];
        if (!sh) {   // fully sorted: every item in place
            if (w < T1) {
                s_perm[w - T0] = (uint16_t)w;
                my_lo = min(my_lo, (unsigned)(w - T0));
                my_hi = max(my_hi, (unsigned)(w - T0 + 1));
            }
            continue;
        }
        const uint64_t top = kq >> sh;
        const int64_t q = wb + w;
        const bool starts = q == 0 || (s_key[w - 1] >> sh) != top;
        const bool ends = q + 1 >= E || (w + 1 < h1r ? (s_key[w + 1] >> sh) : (A.key[q + 1] >> sh)) != top;
        if (starts && ends) {   // a run of one (the common case)
            if (w < T1) {
                s_perm[w - T0] = (uint16_t)w;
                my_lo = min(my_lo, (unsigned)(w - T0));
                my_hi = max(my_hi, (unsigned)(w - T0 + 1));
            }
            continue;
        }
        int rs = w, re = w + 1;
        bool lng = false;
        while (rs > h0r && (s_key[rs - 1] >> sh) == top) {
            --rs;
            if (w - rs >= kRkRunMax) { lng = true; break; }
        }
        if (!lng && rs >= T1) continue;   // a run of a later tile (long or short: not ours)
        if (!lng) {
            while (re < h1r && (s_key[re] >> sh) == top) {
                ++re;
                if (re - rs > kRkRunMax) { lng = true; break; }
            }
            if (!lng && re == h1r && wb + h1r < E && (A.key[wb + h1r] >> sh) == top) lng = true;
        }
        if (lng) {
            // a long run: every key must be equal (then the lex order of the
            // stable radix passes stands); otherwise the caller re-sorts
            if ((w > h0r && (s_key[w - 1] >> sh) == top && s_key[w - 1] != kq) ||
                (w + 1 < h1r && (s_key[w + 1] >> sh) == top && s_key[w + 1] != kq))
                atomicOr(A.fallback, 1);
            if (w < T1) {
                s_perm[w - T0] = (uint16_t)w;
                my_lo = min(my_lo, (unsigned)(w - T0));
                my_hi = max(my_hi, (unsigned)(w - T0 + 1));
            }
            continue;
        }
        if (rs < T0) continue;   // a short run of an earlier tile
        int pos = rs;
        for (int a = rs; a < re; ++a) {
            const uint64_t ka = s_key[a];
            pos += (ka < kq || (ka == kq && a < w)) ? 1 : 0;
        }
        s_perm[pos - T0] = (uint16_t)w;
        my_lo = min(my_lo, (unsigned)(w - T0));
        my_hi = max(my_hi, (unsigned)(w - T0 + 1));
    }
    my_lo = __reduce_min_sync(0xffffffffu, my_lo);
    my_hi = __reduce_max_sync(0xffffffffu, my_hi);
    if (lane == 0) {
        atomicMin(&s_own_lo, my_lo);
        atomicMax(&s_own_hi, my_hi);
    }
    __syncthreads();
    const int olo = s_own_lo == 0xFFFFFFFFu ? 0 : (int)s_own_lo;   // owned [olo, ohi), relative to t0
    const int ohi = s_own_lo == 0xFFFFFFFFu ? 0 : (int)s_own_hi;
    // ---- heads in the final order, per warp over a contiguous chunk of the
    // owned positions (32 per round).  The position before olo holds the
    // previous run's item: it differs in its high bits, or is equal within a
    // long run, so the staged key (any order) decides.
    const int nown = ohi - olo;
    const int chunk = ((nown + kRkWarps - 1) / kRkWarps + 31) & ~31;
    const int c0 = min(olo + wid * chunk, ohi), c1 = min(c0 + chunk, ohi);
    auto key_final = [&](int r) -> uint64_t { return s_key[s_perm[r]]; };
    auto head_at = [&](int r, uint64_t kq) -> bool {
        const int64_t q = t0 + r;
        if (q == 0) return true;
        const uint64_t kp = r == olo ? (T0 + r - 1 >= h0r ? s_key[T0 + r - 1] : A.key[q - 1]) : key_final(r - 1);
        return kq != kp;
    };
    uint32_t wheads = 0;
    for (int r0 = c0; r0 < c1; r0 += 32) {
        const int r = r0 + lane;
        const bool h = r < c1 && head_at(r, key_final(r));
        wheads += __popc(__ballot_sync(0xffffffffu, h));
    }
    if (lane == 0) s_wtot[wid] = wheads;
    __syncthreads();
    if (wid == 0) {
        const uint32_t v = lane < kRkWarps ? s_wtot[lane] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < kRkWarps; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, kRkWarps - 1);
        volatile unsigned long long* st = A.status;
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st[0] = kRkPre | (unsigned long long)total;
        } else {
            if (lane == 0) st[tile] = kRkAgg | (unsigned long long)total;
            // look-back: the warp reads 32 predecessors' status words at a time
            int64_t j = (int64_t)tile - 1;
            for (;;) {
                const int64_t jj = j - lane;
                unsigned long long sv = kRkPre;   // below tile 0: an inclusive prefix of 0
                if (jj >= 0) {
                    sv = st[jj];
                    while ((sv & (kRkAgg | kRkPre)) == 0) sv = st[jj];
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (sv & kRkPre) != 0);
                const int first = pre ? __ffs(pre) - 1 : 32;   // nearest predecessor with a prefix
                unsigned long long part = lane <= first ? (sv & kRkVal) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (pre) break;
                j -= 32;
            }
            if (lane == 0) {
                __threadfence();
                st[tile] = kRkPre | (excl + total);
            }
        }
        if (lane < kRkWarps) s_wtot[lane] = incl - v;   // exclusive per warp
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    // ---- outputs: lane-consecutive rounds, ranks by ballot prefix counts
    uint32_t run = (uint32_t)(s_prefix + s_wtot[wid]);
    const unsigned lle = (2u << lane) - 1u;   // lanes <= this one
    for (int r0 = c0; r0 < c1; r0 += 32) {
        const int r = r0 + lane;
        const bool in = r < c1;
        const int w = in ? s_perm[r] : 0;
        const uint64_t kq = in ? s_key[w] : 0ull;
        const bool h = in && head_at(r, kq);
        const unsigned b = __ballot_sync(0xffffffffu, h);
        if (in) {
            const uint32_t filt = run + __popc(b & lle);
            if (h) A.vor[filt - 1] = __longlong_as_double((long long)(kq + A.bias));
            const int64_t q = t0 + r;
            __stcs(reinterpret_cast<uint2*>(A.ev) + q, edge_of(A, s_val[w]));
            __stcs(A.efilt + q, filt);
        }
        run += __popc(b);
    }
}
}  // namespace

static thread_local int t_edge_path = -1;
int last_edge_path() { return t_edge_path; }

int64_t rank_edges(KeptEdges& ke, uint32_t* ev, uint32_t* efilt, double* vor, cudaStream_t s) {
    const int64_t E = ke.E;
    t_edge_path = -1;
    if (E == 0) return 0;
    // the bucket path (edge_buckets.cu) unless the distribution does not
    // allow it; VRB_EDGE_PATH=radix forces the radix path (tests, experiments)
    // (measured: for E of a few million the radix passes are as fast or
    // faster -- C3 0.28 vs 0.32 ms, C5B 0.79 vs 0.80 ms -- C5A 12.4 vs 10.1 ms)
    const char* ep = std::getenv("VRB_EDGE_PATH");   // "radix" | "bucket" (any E) | unset: bucket from 2^24 edges
    const bool bucket = ep ? ep[0] == 'b' : E >= ((int64_t)1 << 24);
    if (bucket) {
        int64_t nv = 0;
        if (rank_edges_buckets(ke, ke.n, ev, efilt, vor, s, &nv)) {
            t_edge_path = 1;
            return nv;
        }
    }
    t_edge_path = 0;
    SortedEdges so;
    const char* un = std::getenv("VRB_EDGE_UNFUSED");   // experiment knob: the three-kernel epilogue
    if (un && un[0] == '1') {
        sort_edges(ke, s, so);
        dense_ranks(so.key, efilt, E, s);
        if (ke.packed)
            k_edge_outputs_packed<<<grid_for(E, 256), 256, 0, s>>>(so.key, so.val, efilt, E,
                                                                   reinterpret_cast<uint2*>(ev), vor, so.bias);
        else
            k_edge_outputs<<<grid_for(E, 256), 256, 0, s>>>(so.key, so.val, ke.ei.get(), ke.ej.get(), efilt, E, ev,
                                                            vor, so.bias);
        VRB_LAUNCH_CHECK();
    } else {
        int shift = 0;
        bool alt = false;
        sort_edges_top(ke, s, so, &shift, &alt);
        const int64_t tiles = ceil_div(E, kRkTile);
        DBuf<unsigned long long> status(tiles, s);
        DBuf<unsigned> counter(1, s);
        DBuf<int> fb(1, s);
        VRB_CUDA(cudaMemsetAsync(status.get(), 0, tiles * sizeof(unsigned long long), s));
        VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned), s));
        VRB_CUDA(cudaMemsetAsync(fb.get(), 0, sizeof(int), s));
        RankArgs A{};
        A.key = so.key;
        A.val = so.val;
        A.E = E;
        A.shift = shift;
        A.bias = so.bias;
        A.ei = ke.packed ? nullptr : ke.ei.get();
        A.ej = ke.packed ? nullptr : ke.ej.get();
        A.ev = ev;
        A.efilt = efilt;
        A.vor = vor;
        A.status = status.get();
        A.tile_counter = counter.get();
        A.fallback = fb.get();
        k_rank_edges<<<(unsigned)tiles, kRkThreads, 0, s>>>(A);
        VRB_LAUNCH_CHECK();
        int h = 0;
        VRB_CUDA(cudaMemcpyAsync(&h, fb.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        if (h) {
            // a run of equal high bits too long for the in-place sort: complete
            // the order on every digit, then the three-kernel epilogue
            sort_edges_full(ke, s, so, alt);
            dense_ranks(so.key, efilt, E, s);
            if (ke.packed)
                k_edge_outputs_packed<<<grid_for(E, 256), 256, 0, s>>>(so.key, so.val, efilt, E,
                                                                       reinterpret_cast<uint2*>(ev), vor, so.bias);
            else
                k_edge_outputs<<<grid_for(E, 256), 256, 0, s>>>(so.key, so.val, ke.ei.get(), ke.ej.get(), efilt, E,
                                                                ev, vor, so.bias);
            VRB_LAUNCH_CHECK();
        }
    }
    uint32_t nvals = 0;
    VRB_CUDA(cudaMemcpyAsync(&nvals, efilt + E - 1, sizeof(nvals), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return nvals;
}

void build_graph(const uint32_t* ev, int64_t n, int64_t E, cudaStream_t s, Graph& g) {
    build_lists(ev, n, E, s, g);
    build_plan(ev, 0, E, s, g);
}

void build_lists(const uint32_t* ev, int64_t n, int64_t E, cudaStream_t s, Graph& g) {
    g.n = n;
    g.E = E;
    const int64_t n2 = 2 * E;
    g.off.alloc(n + 1, s);
    // (a) lists in edge-position order: stable sort of the 2E entries by
    // vertex; the list offsets are the run starts of the sorted keys
    if (n2 >= (int64_t)1 << 32) fail(VRB_EOVERFLOW, "%lld list entries exceed u32 entry ids", (long long)n2);
    DBuf<uint64_t> lk0, lk1;
    DBuf<uint32_t> lv0, lv1;
    const uint64_t* lskeys = nullptr;
    if (n2) {
        lk0.alloc(n2, s);
        lk1.alloc(n2, s);
        k_keys_vertex<<<grid_for(n2, 256), 256, 0, s>>>(ev, n2, lk0.get());
        VRB_LAUNCH_CHECK();
        int vb = 1;
        while (vb < 32 && ((uint64_t)(n - 1) >> vb)) ++vb;
        const bool alt = radix_sort_keys(lk0.get(), lk1.get(), n2, ((1ull << vb) - 1ull) << 32, s);
        lskeys = alt ? lk1.get() : lk0.get();
        k_offsets_from_sorted<<<grid_for(n + 1, 256), 256, 0, s>>>(lskeys, n2, n, g.off.get());
        VRB_LAUNCH_CHECK();
    } else {
        VRB_CUDA(cudaMemsetAsync(g.off.get(), 0, g.off.bytes(), s));
    }
    {
        DBuf<unsigned> mx(1, s);
        VRB_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned), s));
        if (n) k_max_deg<<<grid_for(n, 256), 256, 0, s>>>(g.off.get(), n, mx.get());
        VRB_LAUNCH_CHECK();
        unsigned h = 0;
        VRB_CUDA(cudaMemcpyAsync(&h, mx.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        g.max_deg = h;
    }
    // packed (krank << 16 | k) lists when ids and ranks fit 16 bits; the wide
    // layout can be forced for testing with VRB_FORCE_WIDE_LISTS=1
    const char* force_wide = std::getenv("VRB_FORCE_WIDE_LISTS");
    g.packed = n <= 65536 && g.max_deg <= 65536 && !(force_wide && force_wide[0] == '1');
    // +4 entries: the enumeration kernels read lists in aligned 16-byte groups
    g.nkr.alloc(n2 + 4, s);
    // the padding is read by the last list's 16-byte groups: vertex 0, rank 0
    // (the triangle count looks every word of a group up before masking)
    VRB_CUDA(cudaMemsetAsync(g.nkr.get() + n2, 0, 4 * sizeof(uint32_t), s));
    if (!g.packed) g.nr.alloc(n2 + 4, s);
    g.np.alloc(n2 + 4, s);
    const char* force_sort = std::getenv("VRB_FORCE_SORT_RANKS");   // testing knob
    const bool bitmap_ranks = n <= kRankBitmapMax && !(force_sort && force_sort[0] == '1');
    if (!bitmap_ranks) g.listidx.alloc(n2, s);
    g.scan_v.alloc(E, s);
    g.scan_len.alloc(E, s);
    if (E == 0) return;
    DBuf<unsigned> scanpack(E, s);
    VRB_CUDA(cudaMemsetAsync(scanpack.get(), 0xFF, E * sizeof(unsigned), s));
    {
        DBuf<uint64_t>& k0 = lk0;
        DBuf<uint64_t>& k1 = lk1;
        DBuf<uint32_t>& v0 = lv0;
        DBuf<uint32_t>& v1 = lv1;
        k_pos_lists<<<grid_for(n2, 256), 256, 0, s>>>(lskeys, ev, g.off.get(), n2, g.nkr.get(), g.np.get(),
                                                       g.listidx.get(), scanpack.get());
        VRB_LAUNCH_CHECK();
        const uint32_t* sorted = nullptr;
        // (b) ranks in neighbour-id order
        if (bitmap_ranks) {
            const size_t smem = (size_t)2 * ((n + 31) >> 5) * sizeof(uint32_t);
            VRB_CUDA(cudaFuncSetAttribute(k_ranks_bitmap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)device_sm_count() * 8);
            if (g.packed) g.idl.alloc(n2, s);
            k_ranks_bitmap<<<grid, 256, smem, s>>>(g.off.get(), n, g.packed ? 1 : 0, g.nkr.get(), g.nr.get(),
                                                   g.np.get(), g.packed ? g.idl.get() : nullptr);
            VRB_LAUNCH_CHECK();
        } else {
            // large n: sort entries by (vertex, neighbour)
            v0.alloc(n2, s);
            v1.alloc(n2, s);
            k_keys_vertex_nbr<<<grid_for(n2, 256), 256, 0, s>>>(ev, n2, k0.get());
            VRB_LAUNCH_CHECK();
            sorted = sort_ids(k0, k1, v0, v1, n2, s);
            k_id_ranks<<<grid_for(n2, 256), 256, 0, s>>>(sorted, ev, g.off.get(), g.listidx.get(), n2,
                                                          g.packed ? 1 : 0, g.nkr.get(), g.nr.get());
            VRB_LAUNCH_CHECK();
        }
    }
    if (g.packed && !g.idl.get()) {   // (the bitmap rank path wrote it already)
        g.idl.alloc(n2, s);
        const unsigned gw = (unsigned)std::min<int64_t>(ceil_div(n * 32, 256), (int64_t)device_sm_count() * 16);
        k_id_lists<<<gw, 256, 0, s>>>(g.off.get(), n, g.nkr.get(), g.np.get(), g.idl.get());
        VRB_LAUNCH_CHECK();
    }
    // (c) scanned endpoint of every edge: the one with the shorter prefix of
    // neighbours older than the edge
    k_assign<<<grid_for(E, 256), 256, 0, s>>>(ev, scanpack.get(), E, g.scan_v.get(), g.scan_len.get());
    VRB_LAUNCH_CHECK();
}

// fill plan of the x-major triangle fill: owner edges [p_lo, p_hi) grouped
// by their SCANNED endpoint x, longest prefix first: (p, host y, prefix
// length, deg x); work = prefix length
__global__ void k_scan_keys(const uint32_t* __restrict__ scan_v, const uint32_t* __restrict__ scan_len, int64_t p_lo,
                            int64_t m, uint64_t* __restrict__ key) {
    GRID_STRIDE(q, m) {
        const int64_t p = p_lo + q;
        key[q] = ((uint64_t)scan_v[p] << 32) | (uint32_t)~scan_len[p];
    }
}

__global__ void k_fill_plan(const uint32_t* __restrict__ sorted, const uint32_t* __restrict__ ev,
                            const uint32_t* __restrict__ scan_v, const uint32_t* __restrict__ scan_len,
                            const uint64_t* __restrict__ off, int64_t m, int64_t p_lo, uint32_t* __restrict__ group_v,
                            uint4* __restrict__ plan, uint32_t* __restrict__ work) {
    GRID_STRIDE(i, m) {
        const uint32_t p = (uint32_t)(p_lo + sorted[i]);
        const uint32_t x = scan_v[p], a = ev[2 * (uint64_t)p], b = ev[2 * (uint64_t)p + 1];
        const uint32_t len = scan_len[p];
        group_v[i] = x;
        plan[i] = make_uint4(p, x == a ? b : a, len, (uint32_t)(off[x + 1] - off[x]));
        work[i] = len + 32;   // + a per-edge constant: the edge's fixed costs
    }
}

void build_fill_plan(const uint32_t* ev, int64_t p_lo, int64_t p_hi, cudaStream_t s, const Graph& g,
                     DBuf<uint4>& plan, DBuf<uint32_t>& group_v, DBuf<uint64_t>& work_pre, int64_t& m_out,
                     uint64_t& work) {
    const int64_t m = p_hi > p_lo ? p_hi - p_lo : 0;
    m_out = m;
    plan.alloc(m, s);
    group_v.alloc(m, s);
    work_pre.alloc(m + 1, s);
    work = 0;
    if (m == 0) {
        VRB_CUDA(cudaMemsetAsync(work_pre.get(), 0, sizeof(uint64_t), s));
        return;
    }
    DBuf<uint64_t> k0(m, s), k1(m, s);
    DBuf<uint32_t> v0(m, s), v1(m, s);
    k_scan_keys<<<grid_for(m, 256), 256, 0, s>>>(g.scan_v.get(), g.scan_len.get(), p_lo, m, k0.get());
    VRB_LAUNCH_CHECK();
    const uint32_t* sorted = sort_ids(k0, k1, v0, v1, m, s);
    DBuf<uint32_t> w(m, s);
    k_fill_plan<<<grid_for(m, 256), 256, 0, s>>>(sorted, ev, g.scan_v.get(), g.scan_len.get(), g.off.get(), m, p_lo,
                                                 group_v.get(), plan.get(), w.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(w.get(), work_pre.get(), m, s);
    VRB_CUDA(cudaMemcpyAsync(&work, work_pre.get() + m, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
}

void build_plan(const uint32_t* ev, int64_t p_lo, int64_t p_hi, cudaStream_t s, Graph& g) {
    // owner-edge plan of the owner edges [p_lo, p_hi): scanned endpoint,
    // prefix length, host; hosted slots grouped by host
    const int64_t m = p_hi > p_lo ? p_hi - p_lo : 0;
    g.nplan = m;
    g.plan.alloc(m, s);
    g.hosted_v.alloc(m, s);
    g.work_pre.alloc(m + 1, s);
    if (m == 0) {
        VRB_CUDA(cudaMemsetAsync(g.work_pre.get(), 0, sizeof(uint64_t), s));
        g.work = 0;
        return;
    }
    DBuf<uint64_t> k0(m, s), k1(m, s);
    DBuf<uint32_t> v0(m, s), v1(m, s);
    auto bits_of = [](uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return b; };
    const int hbits = std::max(1, bits_of((uint64_t)std::max<int64_t>(g.n - 1, 1)));
    const int lbits = std::max(1, 24 - hbits);
    const int lsh = std::max(0, bits_of(g.max_deg) - lbits);
    k_host_keys<<<grid_for(m, 256), 256, 0, s>>>(ev, g.scan_v.get(), g.scan_len.get(), p_lo, m, lbits, lsh, k0.get());
    VRB_LAUNCH_CHECK();
    uint64_t* skeys = nullptr;
    const uint32_t* sorted = sort_ids(k0, k1, v0, v1, m, s, &skeys);
    DBuf<uint32_t> work(m, s);
    k_hosted_work<<<grid_for(m, 256), 256, 0, s>>>(sorted, skeys, g.scan_v.get(), g.scan_len.get(), g.off.get(), m,
                                                   p_lo, lbits, g.hosted_v.get(), g.plan.get(), work.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(work.get(), g.work_pre.get(), m, s);
    VRB_CUDA(cudaMemcpyAsync(&g.work, g.work_pre.get() + m, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vrb
