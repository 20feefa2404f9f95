// edge_buckets.cu -- S3 edge ranking by ONE bucket scatter and an on-chip
// finish (SURVEY 8(d) "Edges work the same way"; the paper's row D, GPU
// sortperm, sec. 4.5).  Replaces the LSD radix passes of
// radix_sort.cu on the edge keys whenever the length distribution allows it.
//
// The order is (len, i, j) (readings A3/A4) and lengths are non-negative
// doubles, so the order of their bit patterns is the order of the lengths.
// With kmin = the smallest key, d = key - kmin:
//   bucket   b = d >> shift                   (monotone in the key)
//   record   r = ((d mod 2^shift) >> tz) << vb | id
// where id is (i << bn | j) when the packed ids fit beside the residual (or E
// is too large to gather ids later), else the edge's lex index q (its slot
// in the lex-ordered kept-edge arrays) -- both order as (i, j) -- and tz the
// trailing zero bits common to every d.  Inside a bucket, r orders exactly as
// (len, i, j): one u64 per edge.
//   k_bk_hist    : bucket counts (global atomics on an L2-resident array)
//   scan         : bucket offsets
//   k_bk_scatter : r to slot atomicAdd(cur[b]) (the order inside a bucket is
//                  arbitrary: the record restores it), in slices of the bucket
//                  range so the partially written sector of each bucket stays
//                  in L2 until it fills
//   k_bk_rank    : per chunk of whole buckets (< 2 kBkC items; records by one
//                  TMA bulk copy on an mbarrier), in shared memory: the bucket
//                  of each position by a warp fill over the staged offsets,
//                  each bucket of m_b items split into 2^(ceil(log2 m_b) + 1)
//                  sub-buckets by its residual's high bits (a counting sort
//                  with packed u16 counters), each item ranked inside its
//                  sub-bucket by comparing records (equal lengths found there
//                  too: the chunk's level count is published before the
//                  outputs); dense ranks by a chained scan over chunks
//                  (decoupled look-back, chunks taken in order); (i, j), filt
//                  and value_of_rank written in lane-consecutive rounds.
// HBM: 8 B read (hist) + (12 B read per slice) + 8 B written (scatter) + 8 B
// read + 12 B written + <= 8 B value_of_rank (rank) per edge, against 4 radix
// passes of 24 B and a 32 B epilogue.  A bucket larger than kBkC items after
// two refinements of the bucket width (ties, or a very spiky distribution),
// or a record that would not fit 64 bits: the caller runs the radix path.
#include <algorithm>
#include <cstdlib>
#include <functional>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

#ifndef VRB_BK_ITEMS
#define VRB_BK_ITEMS 4   // keys per thread in flight in the scatter (8: slower, more partial-sector traffic)
#endif
#ifndef VRB_BK_KEEP
#define VRB_BK_KEEP 1    // scatter stores with an L2 evict_last policy
#endif
#ifndef VRB_BK_C
#define VRB_BK_C 2048
#endif
#ifndef VRB_BK_THREADS
#define VRB_BK_THREADS 512
#endif
// -DVRB_BK_CHECKS: device asserts on every shared-memory index and scatter
// slot (an experiment build, tests/test_edge_buckets_gpu.py under it; the
// pool has no compute-sanitizer)
#ifdef VRB_BK_CHECKS
#include <cassert>
#define BK_ASSERT(c) assert(c)
#else
#define BK_ASSERT(c) ((void)0)
#endif
constexpr int kBkC = VRB_BK_C;          // chunk k = the buckets whose first item lies in [k C, (k+1) C)
constexpr int kBkMax = 2 * kBkC;        // items of a chunk: < C + largest bucket <= 2 C
constexpr int kBkThreads = VRB_BK_THREADS;
constexpr int kBkMinBlocks = (2048 / kBkThreads) < 2 ? 1 : (2048 / kBkThreads) / 2;
constexpr int kBkWarps = kBkThreads / 32;
#ifndef VRB_BK_OFFSTAGE
#define VRB_BK_OFFSTAGE 1024
#endif
constexpr int kBkOffStage = VRB_BK_OFFSTAGE;       // a chunk's bucket offsets staged in shared memory up to this many buckets
constexpr int kBkMaxLogNB = 23;
constexpr unsigned long long kBkAgg = 1ull << 62, kBkPre = 2ull << 62, kBkVal = (1ull << 62) - 1;

#ifndef VRB_BK_FILLBL
#define VRB_BK_FILLBL 1   // staged chunks: the bucket of each position by a warp fill, not a search
#endif
#ifndef VRB_BK_TMA
#define VRB_BK_TMA 1   // the chunk's records come in by one cp.async.bulk (TMA) copy on an mbarrier
#endif
constexpr size_t kBkSmem = (kBkMax + 2) * sizeof(uint64_t)    // s_rec (+ 16-byte alignment slack)
                           + 4 * kBkMax * sizeof(uint16_t)    // s_c16 (sub-bucket counts, then ends; packed u16)
                           + kBkMax * sizeof(uint32_t)        // s_bl (bucket of an item, chunk-relative)
                           + 3 * kBkMax * sizeof(uint16_t)    // s_sb, s_tmp, s_perm
                           + (kBkOffStage + 8) * sizeof(uint16_t);

unsigned grid_cap(int64_t work, int threads) {
    int64_t g = ceil_div(work, threads);
    const int64_t cap = (int64_t)device_sm_count() * 16;
    return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

template <int kItems>
__global__ void __launch_bounds__(256) k_bk_hist(const uint64_t* __restrict__ key, int64_t E, uint64_t kmin, int shift,
                                                 uint32_t* __restrict__ cnt) {
    const int64_t step = (int64_t)gridDim.x * 256 * kItems;
    for (int64_t b0 = (int64_t)blockIdx.x * 256 * kItems + threadIdx.x; b0 < E; b0 += step) {
        uint64_t k[kItems];
#pragma unroll
        for (int u = 0; u < kItems; ++u) {
            const int64_t q = b0 + (int64_t)u * 256;
            k[u] = q < E ? __ldcs(reinterpret_cast<const unsigned long long*>(key) + q) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kItems; ++u)
            if (b0 + (int64_t)u * 256 < E) atomicAdd(&cnt[(k[u] - kmin) >> shift], 1u);
    }
}

__global__ void k_bk_max(const uint32_t* __restrict__ cnt, int64_t nb, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        m = max(m, cnt[b]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void k_bk_cursor(const uint64_t* __restrict__ off, int64_t nb, uint32_t* __restrict__ cur) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        cur[b] = (uint32_t)off[b];
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_keep(uint64_t* p, uint64_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// kIds: the record's low field is (i << bn | j), from the packed ids
// (i << 16 | j) of the kept edges; otherwise it is the lex index q (vb bits).
template <int kItems, bool kIds>
__global__ void __launch_bounds__(256) k_bk_scatter(const uint64_t* __restrict__ key, int64_t E, uint64_t kmin,
                                                    int shift, int tz, int lowbits, const uint32_t* __restrict__ pij,
                                                    int bn, uint32_t* __restrict__ cur, uint64_t* __restrict__ rec,
                                                    const uint32_t* __restrict__ slices, int slice) {
    // this pass scatters the buckets [b_lo, b_hi) only (a slice of about
    // E / passes items): its partially written sectors stay in L2
    const uint64_t b_lo = slices[slice], b_hi = slices[slice + 1];
    const uint64_t low = shift >= 64 ? ~0ull : ((1ull << shift) - 1ull);
    const uint64_t pol = l2_evict_last_policy();
    const int64_t step = (int64_t)gridDim.x * 256 * kItems;
    for (int64_t b0 = (int64_t)blockIdx.x * 256 * kItems + threadIdx.x; b0 < E; b0 += step) {
        uint64_t k[kItems];
#pragma unroll
        for (int u = 0; u < kItems; ++u) {
            const int64_t q = b0 + (int64_t)u * 256;
            k[u] = q < E ? __ldcs(reinterpret_cast<const unsigned long long*>(key) + q) : 0ull;
        }
        uint32_t slot[kItems];
        bool inr[kItems];
#pragma unroll
        for (int u = 0; u < kItems; ++u) {
            const uint64_t b = (k[u] - kmin) >> shift;
            inr[u] = b0 + (int64_t)u * 256 < E && b >= b_lo && b < b_hi;
        }
#pragma unroll
        for (int u = 0; u < kItems; ++u)
            if (inr[u]) {
#if defined(VRB_BK_TIMING_NOATOM)   // timing experiment only (wrong output): random slots, no atomics
                slot[u] = (uint32_t)(((uint64_t)(b0 + u * 256) * 2654435761ull) % (uint64_t)E);
#elif defined(VRB_BK_TIMING_SEQ)    // timing experiment only (wrong output): atomics, sequential stores
                slot[u] = atomicAdd(&cur[(k[u] - kmin) >> shift], 1u) * 0u + (uint32_t)(b0 + u * 256);
#else
                slot[u] = atomicAdd(&cur[(k[u] - kmin) >> shift], 1u);
#endif
            }
        uint64_t idv[kItems];
#pragma unroll
        for (int u = 0; u < kItems; ++u) {
            const int64_t q = b0 + (int64_t)u * 256;
            if (kIds) {
                const uint32_t v = inr[u] ? __ldcs(pij + q) : 0u;
                idv[u] = ((uint64_t)(v >> 16) << bn) | (uint64_t)(v & 0xFFFFu);
            } else {
                idv[u] = (uint64_t)q;
            }
        }
#pragma unroll
        for (int u = 0; u < kItems; ++u) {
            if (inr[u]) {
                const uint64_t d = k[u] - kmin;
                const uint64_t r = (((d & low) >> tz) << lowbits) | idv[u];
                BK_ASSERT(slot[u] < (uint64_t)E);
                if (VRB_BK_KEEP)
                    st_keep(rec + slot[u], r, pol);
                else
                    rec[slot[u]] = r;
            }
        }
    }
}

// entry k -> first bucket with offset >= k * step (the last entry: nb);
// chunks (step kBkC) and scatter slices
__global__ void k_bk_chunks(const uint64_t* __restrict__ off, int64_t nb, int64_t nchunks, uint64_t step,
                            uint32_t* __restrict__ cb) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nchunks;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = (uint64_t)k * step;
        int64_t lo = 0, hi = nb;   // off[nb] = E
        if (off[nb] < x) {
            cb[k] = (uint32_t)nb;
            continue;
        }
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid] >= x) hi = mid; else lo = mid + 1;
        }
        cb[k] = (uint32_t)lo;
    }
}

struct BkArgs {
    const uint64_t* rec;
    const uint64_t* off;   // nb + 1 bucket offsets
    const uint32_t* cb;    // nchunks + 1 first buckets
    int64_t n;
    uint64_t kmin;
    int shift, tz, vb;     // vb: bits of the record's low field
    int bn;                // > 0: the low field is (i << bn | j); else the lex index, with
    const uint32_t* pij;   // packed (i << 16 | j) per lex index, or
    const uint32_t* ei;    // i, j per lex index
    const uint32_t* ej;
    uint32_t* ev;
    uint32_t* efilt;
    double* vor;
    unsigned long long* status;
    unsigned* counter;
};

__global__ void __launch_bounds__(kBkThreads, kBkMinBlocks) k_bk_rank(BkArgs A) {
    extern __shared__ __align__(16) unsigned char bk_smem[];
    uint64_t* s_raw = reinterpret_cast<uint64_t*>(bk_smem);
    uint32_t* s_cw = reinterpret_cast<uint32_t*>(s_raw + kBkMax + 2);   // 4 kBkMax u16 counters, two per word
    uint16_t* s_c16 = reinterpret_cast<uint16_t*>(s_cw);
    uint32_t* s_bl = s_cw + 2 * kBkMax;
    uint16_t* s_sb = reinterpret_cast<uint16_t*>(s_bl + kBkMax);
    uint16_t* s_tmp = s_sb + kBkMax;
    uint16_t* s_perm = s_tmp + kBkMax;
    uint16_t* s_off = s_perm + kBkMax;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wtot[kBkWarps];
    __shared__ unsigned long long s_prefix;
    __shared__ uint32_t s_hm[kBkMax / 32];   // head flags of the final order, one ballot per 32 positions
    __shared__ __align__(8) uint64_t s_bar;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(A.counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t ba = A.cb[tile], bb = A.cb[tile + 1];
    const int64_t p0 = (int64_t)A.off[ba];
    const int m = (int)((int64_t)A.off[bb] - p0);
    const uint32_t nbk = bb - ba;
#if VRB_BK_TMA
    // records [p0, p0 + m) by one bulk copy from the 16-byte aligned address
    // at or below (rec is padded by two records), while the threads stage the
    // offsets and clear the counters
    const uint64_t* src = A.rec + p0;
    const int lead = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
    uint64_t* s_rec = s_raw + lead;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    if (tid == 0 && m > 0) {
        const uint32_t bytes = (uint32_t)(((m + lead) * 8 + 15) & ~15);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(s_raw)), "l"(src - lead), "r"(bytes), "r"(bar)
                     : "memory");
    }
#else
    uint64_t* s_rec = s_raw;
#endif
    BK_ASSERT(m >= 0 && m <= kBkMax);
    const bool staged = nbk <= (uint32_t)kBkOffStage;
    if (staged)
        for (int t = tid; t <= (int)nbk; t += kBkThreads) s_off[t] = (uint16_t)(A.off[ba + t] - p0);
#if !VRB_BK_TMA
    for (int t = tid; t < m; t += kBkThreads)
        s_rec[t] = __ldcs(reinterpret_cast<const unsigned long long*>(A.rec) + p0 + t);
#endif
    for (int t = tid; t < 2 * m; t += kBkThreads) s_cw[t] = 0u;   // 4m u16 counters
    __syncthreads();   // (the barrier is initialised before any thread waits on it)
#if VRB_BK_TMA
    if (m > 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar) : "memory");
    }
#endif
    auto off_of = [&](uint32_t bl) -> int { return staged ? (int)s_off[bl] : (int)((int64_t)A.off[ba + bl] - p0); };
    const int vb = A.vb;
    const int rbits = A.shift - A.tz;   // residual bits
    // ---- sub-bucket of every item: bucket bl (chunk-relative) of m_b items
    // owns sub-buckets [4 off(bl), 4 off(bl) + 2^L), 2 m_b <= 2^L < 4 m_b, by
    // the residual's L high bits (about 1 item per 2 to 4 sub-buckets)
    // staged chunks: each warp writes the bucket index over its buckets'
    // positions (lane-strided); others: a binary search in off[] per item
#if VRB_BK_FILLBL
    if (staged) {
        __syncthreads();   // the TMA copy's barrier wait and s_off are complete for all
        for (int bl = wid; bl < (int)nbk; bl += kBkWarps) {
            const int st = s_off[bl], en = s_off[bl + 1];
            for (int t = st + lane; t < en; t += 32) s_bl[t] = (uint32_t)bl;
        }
        __syncthreads();
    }
#endif
    for (int t = tid; t < m; t += kBkThreads) {
        uint32_t lo = 0, hi = nbk;   // off(lo) <= t < off(hi)
#if VRB_BK_FILLBL
        if (staged) {
            lo = s_bl[t];
        } else
#endif
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (off_of(mid) <= t) lo = mid; else hi = mid;
        }
        const int st = off_of(lo), mb = off_of(lo + 1) - st;
        const int L = (mb > 1 ? 32 - __clz(mb - 1) : 0) + 1;
        const uint64_t res = s_rec[t] >> vb;
        const uint32_t sub = L >= rbits ? (uint32_t)(res << (L - rbits)) : (uint32_t)(res >> (rbits - L));
        const uint32_t sb = 4u * (uint32_t)st + sub;
        BK_ASSERT(st <= t && t < st + mb && sub < (1u << L) && sb < 4u * (uint32_t)(st + mb));
        s_sb[t] = (uint16_t)sb;
        s_bl[t] = lo;
        atomicAdd(&s_cw[sb >> 1], 1u << (16 * (sb & 1)));
    }
    __syncthreads();
    // ---- exclusive scan of the 2m sub-bucket counts
    {
        const int ns = 2 * m;   // words of two u16 counters
        const int per = (ns + kBkThreads - 1) / kBkThreads;
        const int a0 = min(tid * per, ns), a1 = min(a0 + per, ns);
        uint32_t sum = 0;
        for (int a = a0; a < a1; ++a) {
            const uint32_t c = s_cw[a];
            sum += (c & 0xFFFFu) + (c >> 16);
        }
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_wtot[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const uint32_t v = lane < kBkWarps ? s_wtot[lane] : 0u;
            uint32_t iw = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, iw, o);
                if (lane >= o) iw += y;
            }
            if (lane < kBkWarps) s_wtot[lane] = iw - v;
        }
        __syncthreads();
        uint32_t run = s_wtot[wid] + inc - sum;
        for (int a = a0; a < a1; ++a) {
            const uint32_t c = s_cw[a];
            const uint32_t lo16 = c & 0xFFFFu;
            s_cw[a] = run | ((run + lo16) << 16);
            run += lo16 + (c >> 16);
        }
    }
    __syncthreads();
    // ---- counting-sort scatter by sub-bucket; afterwards s_c16[x] = end of x
    for (int t = tid; t < m; t += kBkThreads) {
        const uint32_t sb = s_sb[t], sh = 16 * (sb & 1);
        const uint32_t slot = (atomicAdd(&s_cw[sb >> 1], 1u << sh) >> sh) & 0xFFFFu;
        BK_ASSERT(slot < (uint32_t)m);
        s_tmp[slot] = (uint16_t)t;
    }
    __syncthreads();
    // ---- final place: rank inside the sub-bucket (records are distinct);
    // an item with an equal residual (an equal length: same bucket, same
    // sub-bucket) and a smaller record is not a head of its level
    uint32_t dups = 0;
    for (int t = tid; t < m; t += kBkThreads) {
        const uint32_t sb = s_sb[t];
        const int lo = sb ? (int)s_c16[sb - 1] : 0, hi = (int)s_c16[sb];
        const uint64_t r = s_rec[t];
        int pos = lo;
        bool dup = false;
        for (int u = lo; u < hi; ++u) {
            const uint64_t ru = s_rec[s_tmp[u]];
            pos += ru < r ? 1 : 0;
            dup |= ru < r && (ru >> vb) == (r >> vb);
        }
        BK_ASSERT(lo <= pos && pos < hi && hi <= m);
        s_perm[pos] = (uint16_t)t;
        dups += dup ? 1u : 0u;
    }
    dups = __reduce_add_sync(0xffffffffu, dups);
    if (lane == 0) s_hm[wid] = dups;   // (s_hm reused below for head ballots)
    __syncthreads();
    // the chunk's distinct-length count goes out first (successors look back
    // on it); then every warp records its head ballots and writes its (i, j)
    // -- they need no rank offset -- and warp 0 looks back for the prefix
    volatile unsigned long long* st = A.status;
    uint32_t total = 0;
    if (wid == 0) {
        uint32_t dsum = lane < kBkWarps ? s_hm[lane] : 0u;
        dsum = __reduce_add_sync(0xffffffffu, dsum);
        total = (uint32_t)m - dsum;
        if (lane == 0) st[tile] = (tile == 0 ? kBkPre : kBkAgg) | (unsigned long long)total;
    }
    __syncthreads();   // s_hm free again
    // ---- heads in the final order: a bucket start (the chunk's first item
    // too: the previous chunk ends with another bucket) or a new residual
    const int chunk = ((m + kBkWarps - 1) / kBkWarps + 31) & ~31;
    const int c0 = min(wid * chunk, m), c1 = min(c0 + chunk, m);
    auto head_at = [&](int t, int w) -> bool {
        if (t == 0) return true;
        const int wp = s_perm[t - 1];
        return s_bl[w] != s_bl[wp] || (s_rec[w] >> vb) != (s_rec[wp] >> vb);
    };
    uint32_t wheads = 0;
    {
        const uint64_t qmask = (1ull << vb) - 1ull;
        const uint64_t jmask = (1ull << A.bn) - 1ull;
        for (int r0 = c0; r0 < c1; r0 += 32) {   // r0: a multiple of 32
            const int t = r0 + lane;
            const int w = t < c1 ? s_perm[t] : 0;
            const bool h = t < c1 && head_at(t, w);
            const unsigned bal = __ballot_sync(0xffffffffu, h);
            if (lane == 0) s_hm[r0 >> 5] = bal;
            wheads += __popc(bal);
            if (t < c1) {
                const uint64_t q = s_rec[w] & qmask;
                uint2 e;
                if (A.bn) {
                    e = make_uint2((uint32_t)(q >> A.bn), (uint32_t)(q & jmask));
                } else if (A.pij) {
                    const uint32_t v = __ldg(A.pij + q);
                    e = make_uint2(v >> 16, v & 0xFFFFu);
                } else {
                    e = make_uint2(__ldg(A.ei + q), __ldg(A.ej + q));
                }
                __stcs(reinterpret_cast<uint2*>(A.ev) + p0 + t, e);
            }
        }
    }
    if (lane == 0) s_wtot[wid] = wheads;
    __syncthreads();
    if (wid == 0) {
        const uint32_t v = lane < kBkWarps ? s_wtot[lane] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        BK_ASSERT(__shfl_sync(0xffffffffu, incl, 31) == total);
        if (lane < kBkWarps) s_wtot[lane] = incl - v;   // exclusive per warp
    }
    if (wid == 0) {
        unsigned long long excl = 0;
        if (tile > 0) {
            int64_t j = (int64_t)tile - 1;
            for (;;) {
                const int64_t jj = j - lane;
                unsigned long long sv = kBkPre;   // below chunk 0: an inclusive prefix of 0
                if (jj >= 0) {
                    sv = st[jj];
                    while ((sv & (kBkAgg | kBkPre)) == 0) sv = st[jj];
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (sv & kBkPre) != 0);
                const int first = pre ? __ffs(pre) - 1 : 32;
                unsigned long long part = lane <= first ? (sv & kBkVal) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (pre) break;
                j -= 32;
            }
            if (lane == 0) {
                __threadfence();
                st[tile] = kBkPre | (excl + total);
            }
        }
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    // ---- filt and value_of_rank
    uint32_t run = (uint32_t)(s_prefix + s_wtot[wid]);
    const unsigned lle = (2u << lane) - 1u;
    for (int r0 = c0; r0 < c1; r0 += 32) {
        const int t = r0 + lane;
        const bool in = t < c1;
        const int w = in ? s_perm[t] : 0;
        const unsigned b = s_hm[r0 >> 5];
        const bool h = (b >> lane) & 1u;
        if (in) {
            const uint32_t filt = run + __popc(b & lle);
            if (h) {
                const uint64_t r = s_rec[w];
                const uint64_t bits = A.kmin + ((uint64_t)(ba + s_bl[w]) << A.shift) + ((r >> vb) << A.tz);
                A.vor[filt - 1] = __longlong_as_double((long long)bits);
            }
            __stcs(A.efilt + p0 + t, filt);
        }
        run += __popc(b);
    }
}

}  // namespace

namespace {
// The bucket parameters and the common finish (scan, scatter passes, chunk
// ranking) of both front ends: hist(shift, cnt) counts the buckets of
// (key - kmin) >> shift; scatter(P, cur, rec, slices, slice) writes the
// records of the buckets in the slice.
struct BkPlan {
    int64_t E = 0, n = 0;
    uint64_t kmin = 0, vary = 0;
    int bn_avail = 0;      // > 0: packed ids of bn bits available for the record
};
using HistFn = std::function<void(const FoldBk&)>;
using ScatterFn = std::function<void(const FoldBk&)>;

bool bucket_rank(const BkPlan& P, const HistFn& hist, const ScatterFn& scatter, const KeptEdges* ke, uint32_t* ev,
                 uint32_t* efilt, double* vor, cudaStream_t s, int64_t* nvals) {
    const int64_t E = P.E;
    const uint64_t vary = P.vary, kmin = P.kmin;
    if (E < 2 || !vary) return false;   // one length: the radix path is trivial
    const int blen = 64 - __builtin_clzll(vary);
    const int tz = __builtin_ctzll(vary);
    int lgE = 0;
    while (((int64_t)1 << lgE) < E) ++lgE;
    const int logNB = std::max(10, std::min(21, lgE - 5));
    int shift = std::max(tz, blen - logNB);
    // record low field: the lex index (vb bits; the rank pass gathers the
    // ids), or for packed ids (i << bn | j) when that fits the bucket width
    // or E is too large for random id gathers
    int vb = 1;
    while (vb < 64 && ((uint64_t)(E - 1) >> vb)) ++vb;
    int bn = 0;
    if (P.bn_avail && ((shift - tz) + 2 * P.bn_avail <= 64 || E > ((int64_t)1 << 26)))
        bn = P.bn_avail;
    if (bn) vb = 2 * bn;
    if ((shift - tz) + vb > 64) shift = (64 - vb) + tz;   // more buckets so the record fits
    if (blen - shift > kBkMaxLogNB) return false;
    FoldBk F;
    F.kmin = kmin;
    F.tz = tz;
    F.vb = vb;
    F.bn = bn;
    DBuf<uint32_t> cnt;
    DBuf<unsigned> mx(1, s);
    int64_t nb = 0;
    for (int attempt = 0;; ++attempt) {
        nb = (int64_t)(vary >> shift) + 1;
        cnt.alloc(nb, s);
        VRB_CUDA(cudaMemsetAsync(cnt.get(), 0, nb * sizeof(uint32_t), s));
        VRB_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned), s));
        F.shift = shift;
        F.nb = nb;
        F.cnt = cnt.get();
        hist(F);
        k_bk_max<<<grid_cap(nb, 256), 256, 0, s>>>(cnt.get(), nb, mx.get());
        VRB_LAUNCH_CHECK();
        unsigned h = 0;
        VRB_CUDA(cudaMemcpyAsync(&h, mx.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        if (h <= (unsigned)kBkC) break;
        // finer buckets: by the factor the largest one is over
        int more = 0;
        while (((uint64_t)kBkC << more) < h) ++more;
        if (attempt >= 2 || shift - more < tz || blen - (shift - more) > kBkMaxLogNB) return false;
        shift -= more;
    }
    DBuf<uint64_t> off(nb + 1, s);
    exclusive_scan(cnt.get(), off.get(), nb, s);
    k_bk_cursor<<<grid_cap(nb, 256), 256, 0, s>>>(off.get(), nb, cnt.get());   // cnt becomes the cursors
    VRB_LAUNCH_CHECK();
    DBuf<uint64_t> rec(E + 2, s);   // + 2: the chunk copies round to 16 bytes
    // the scatter in slices of the bucket range, so that the sectors it
    // writes partially (one per bucket) stay L2-resident until complete
    const int64_t frontier = nb * 32;   // bytes of partial sectors if all buckets were active
    int passes = (int)std::min<int64_t>(16, std::max<int64_t>(1, ceil_div(frontier, (int64_t)16 << 20)));
    if (const char* ep = std::getenv("VRB_BK_PASSES")) passes = std::max(1, std::atoi(ep));
    DBuf<uint32_t> slices(passes + 1, s);
    k_bk_chunks<<<1, 32, 0, s>>>(off.get(), nb, passes, (uint64_t)ceil_div(E, passes), slices.get());
    VRB_LAUNCH_CHECK();
    F.cnt = cnt.get();
    F.rec = rec.get();
    F.slices = slices.get();
    for (int sl = 0; sl < passes; ++sl) {
        F.slice = sl;
        scatter(F);
    }
    cnt.reset();
    const int64_t nchunks = ceil_div(E, kBkC);
    DBuf<uint32_t> cb(nchunks + 1, s);
    k_bk_chunks<<<grid_cap(nchunks + 1, 256), 256, 0, s>>>(off.get(), nb, nchunks, (uint64_t)kBkC, cb.get());
    VRB_LAUNCH_CHECK();
    DBuf<unsigned long long> status(nchunks, s);
    DBuf<unsigned> counter(1, s);
    VRB_CUDA(cudaMemsetAsync(status.get(), 0, nchunks * sizeof(unsigned long long), s));
    VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned), s));
    VRB_CUDA(cudaFuncSetAttribute(k_bk_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBkSmem));
    BkArgs A{};
    A.rec = rec.get();
    A.off = off.get();
    A.cb = cb.get();
    A.n = P.n;
    A.kmin = kmin;
    A.shift = shift;
    A.tz = tz;
    A.vb = vb;
    A.bn = bn;
    if (!bn) {   // lex-index records: the ids are gathered
        A.pij = ke->packed ? ke->pij.get() : nullptr;
        A.ei = ke->packed ? nullptr : ke->ei.get();
        A.ej = ke->packed ? nullptr : ke->ej.get();
    }
    A.ev = ev;
    A.efilt = efilt;
    A.vor = vor;
    A.status = status.get();
    A.counter = counter.get();
    k_bk_rank<<<(unsigned)nchunks, kBkThreads, kBkSmem, s>>>(A);
    VRB_LAUNCH_CHECK();
    uint32_t nv = 0;
    VRB_CUDA(cudaMemcpyAsync(&nv, efilt + E - 1, sizeof(nv), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    *nvals = nv;
    return true;
}

int bits_of(int64_t n) {
    int b = 1;
    while (((uint64_t)(n - 1) >> b)) ++b;
    return b;
}
}  // namespace

bool rank_edges_buckets(KeptEdges& ke, int64_t n, uint32_t* ev, uint32_t* efilt, double* vor, cudaStream_t s,
                        int64_t* nvals) {
    const int64_t E = ke.E;
    if (E < 2) return false;
    BkPlan P;
    P.E = E;
    P.n = n;
    P.vary = key_range(ke.key.get(), E, s, &P.kmin, ke.range.get());
    P.bn_avail = ke.packed ? bits_of(n) : 0;
    const uint64_t* key = ke.key.get();
    const uint32_t* pij = ke.pij.get();
    auto hist = [&](const FoldBk& F) {
        k_bk_hist<4><<<grid_cap(E, 256 * 4), 256, 0, s>>>(key, E, F.kmin, F.shift, F.cnt);
        VRB_LAUNCH_CHECK();
    };
    auto scatter = [&](const FoldBk& F) {
        if (F.bn)
            k_bk_scatter<VRB_BK_ITEMS, true><<<grid_cap(E, 256 * VRB_BK_ITEMS), 256, 0, s>>>(
                key, E, F.kmin, F.shift, F.tz, F.vb, pij, F.bn, F.cnt, F.rec, F.slices, F.slice);
        else
            k_bk_scatter<VRB_BK_ITEMS, false><<<grid_cap(E, 256 * VRB_BK_ITEMS), 256, 0, s>>>(
                key, E, F.kmin, F.shift, F.tz, F.vb, nullptr, 0, F.cnt, F.rec, F.slices, F.slice);
        VRB_LAUNCH_CHECK();
    };
    return bucket_rank(P, hist, scatter, &ke, ev, efilt, vor, s, nvals);
}

}  // namespace vrb
