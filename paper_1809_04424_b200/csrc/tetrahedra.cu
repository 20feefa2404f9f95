// tetrahedra.cu -- S6 (tetrahedron enumeration), S7 and S8 for dimension 3.
//
// Definition ("a solid tetrahedra is constructed if all its face
// triangles have been created"; readings A3/A4/A7): {a,b,c,d} is a
// tetrahedron iff its six edges are kept; filt = max edge filt; dimension 3
// is ordered by (filt, lex); its D_3 column holds the positions of its four
// face triangles in the dimension-2 order, ascending.
//
// Owner-edge order, as for triangles (triangles.cu): the owner of a
// tetrahedron is its edge of largest position p = (y, x).  Its other two
// vertices k < l are both in S(p) = {k : pos(x,k) < p, pos(y,k) < p} (the
// apex set of p's triangles) and are adjacent with pos(k,l) < p.  For a fixed
// owner, (k, l) lex order is the lex order of the sorted 4-tuple, so a count
// pass, an exclusive scan and a fill pass place every tetrahedron directly;
// tie levels are re-sorted afterwards (segsort.cu).
//
// Per owner edge (one warp, the host y's position map in shared memory):
//   S     : x's older-neighbour prefix -> bitmap by rank in x's id list ->
//           S sorted by id, with pos(x,k), in shared memory; S's vertices
//           also flagged in an n-bit vertex bitmap
//   pairs : for each k in S (ascending), stream k's neighbours older than p
//           (a prefix of k's position-ordered list, found by binary search);
//           l in S with l > k (vertex bitmap, then binary search in S for its
//           index) marks bit idx(l) of a small bitmap; its popcount ranks give
//           the (k, l) emission order
//   D_3   : faces (y,x,k), (y,x,l) are p's own triangles (direct index when
//           p's level is a single edge); faces (y,k,l), (x,k,l) are found by
//           binary search in the triangle range of their owner edge.
#include <algorithm>
#include <cstdlib>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kBits = 4096;     // ranks of x's id list per round
constexpr int kWords = kBits / 32;
constexpr int kS = 512;         // max |S(p)| in warp scratch (larger: k_tets_big)
constexpr int64_t kDenseMaxN = 16384;   // n x n u32 edge-position table (<= 1 GiB)

struct TetArgs {
    int64_t n, E;
    const uint64_t* off;
    const uint32_t* nkr;
    const uint32_t* nr;
    const uint32_t* np;
    int packed;
    const uint4* plan;
    const uint32_t* hosted_v;
    const uint64_t* work_pre;
    uint64_t chunk;
    int64_t ntasks, task_lo, task_hi;
    unsigned long long* task_counter;
    unsigned* ovf_n;          // owner edges with |S(p)| > kS: their hosted slots are
    uint32_t* ovf_list;       // listed here and handled by k_tets_big
    const uint2* idl;         // (k, pos) in neighbour-id order (packed lists), for k_tets_big
    uint32_t* big;            // k_tets_big scratch, big_stride u32 per CTA
    uint64_t big_stride;
    uint32_t max_deg;
    // triangles (dimension 2, global arrays)
    const uint64_t* toff;     // E + 1
    const uint64_t* tlo;      // E: start of the triangle range of p's level
    const uint64_t* thi;      // E: end of it
    const uint4* frec;        // 2E: 32-byte face record per owner edge (k_level_ranges)
    const uint32_t* tv;       // 3T (dimension-2 vertices, global order)
    const ulonglong2* hslots;   // triangle lex code -> position: slot = (code, position), open addressing
    uint64_t hmask;
    const uint16_t* apex;       // per triangle: its vertex off the owner edge (null: use the hash)
    const uint32_t* dense;      // n x n edge positions (NONE32 = no edge), or null
    // count
    uint32_t* cnt;
    // fill
    const uint32_t* efilt;
    const uint64_t* qoff;
    int64_t p_lo, p_hi;
    uint64_t slot0;
    uint32_t* qv;
    uint32_t* qf;
    uint32_t* rows;
};

struct TetScratch {
    uint32_t bits[kWords];
    uint32_t wpre[kWords];
    uint32_t Sk[kS];          // S sorted by id
    uint32_t Spx[kS];         // pos(x, k)
    uint32_t lbits[kS / 32];  // l in S (by index) adjacent to the current k through an older edge
    uint32_t lpre[kS / 32];
    uint32_t lpos[kS];        // pos(k, l) for the marked l
    uint32_t plen[kS];        // #neighbours of Sk[i] older than p (prefix of its position list)
};

__device__ __forceinline__ int64_t lb_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t v) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t ub_u32(const uint32_t* a, int64_t lo, int64_t hi, uint32_t v) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// first index in [lo, hi) of the ascending u32 array a with a[i] >= v
__device__ __forceinline__ uint32_t lb_u32(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t v) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Warp-cooperative lower bound in an ascending u32 array: 32 probes per
// round, so ~log32(n) dependent loads instead of log2(n).
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t v) {
    const int lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = n;
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t idx = min(hi - 1, lo + (uint32_t)(lane + 1) * step - 1);
        const bool less = __ldg(a + idx) < v;
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, less));
        const uint32_t nlo = lo + c * step;
        hi = min(hi, nlo + step);
        lo = min(nlo, hi);
    }
    const bool less = lo + lane < hi && __ldg(a + lo + lane) < v;
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

__device__ __forceinline__ void sort3v(uint32_t& a, uint32_t& b, uint32_t& c) {
    uint32_t t;
    if (a > b) { t = a; a = b; b = t; }
    if (b > c) { t = b; b = c; c = t; }
    if (a > b) { t = a; a = b; b = t; }
}

__device__ __forceinline__ void sort4v(uint32_t* v) {
#pragma unroll
    for (int i = 1; i < 4; ++i)
#pragma unroll
        for (int j = i; j > 0; --j)
            if (v[j - 1] > v[j]) { const uint32_t t = v[j]; v[j] = v[j - 1]; v[j - 1] = t; }
}

// Position of triangle {a, b, c} (a < b < c) whose owner edge is f: binary
// search by lex triple inside the (lex-sorted) triangle range of f's level.
__device__ __forceinline__ uint32_t tri_pos(const TetArgs& A, uint32_t f, uint32_t a, uint32_t b, uint32_t c) {
    uint64_t lo = A.tlo[f], hi = A.thi[f];
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint32_t* t = A.tv + 3 * mid;
        const uint32_t t0 = t[0], t1 = t[1], t2 = t[2];
        const bool less = t0 < a || (t0 == a && (t1 < b || (t1 == b && t2 < c)));
        if (less) lo = mid + 1; else hi = mid;
    }
    return (uint32_t)lo;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 33; z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

__device__ __forceinline__ uint64_t tri_code(uint32_t a, uint32_t b, uint32_t c) {
    return ((uint64_t)a << 42) | ((uint64_t)b << 21) | (uint64_t)c;
}

// Position of triangle {a < b < c}: hash lookup (the key is always present).
__device__ __forceinline__ uint32_t tri_lookup(const TetArgs& A, uint32_t a, uint32_t b, uint32_t c) {
    const uint64_t code = tri_code(a, b, c);
    uint64_t h = mix64(code) & A.hmask;
    for (;;) {
        const ulonglong2 sl = __ldg(A.hslots + h);   // key and position in one 16-byte slot
        if (sl.x == code) return (uint32_t)sl.y;
        h = (h + 1) & A.hmask;
    }
}

// Positions of two triangles at once: both first probes are issued before
// either is resolved (two independent DRAM round trips in flight per lane).
__device__ __forceinline__ void tri_lookup2(const TetArgs& A, uint64_t c1, uint64_t c2, uint32_t& p1, uint32_t& p2) {
    uint64_t h1 = mix64(c1) & A.hmask, h2 = mix64(c2) & A.hmask;
    ulonglong2 s1 = __ldg(A.hslots + h1), s2 = __ldg(A.hslots + h2);
    while (s1.x != c1) { h1 = (h1 + 1) & A.hmask; s1 = __ldg(A.hslots + h1); }
    while (s2.x != c2) { h2 = (h2 + 1) & A.hmask; s2 = __ldg(A.hslots + h2); }
    p1 = (uint32_t)s1.y;
    p2 = (uint32_t)s2.y;
}

__device__ __forceinline__ uint64_t tri_code_sorted(uint32_t a, uint32_t b, uint32_t c) {
    sort3v(a, b, c);
    return tri_code(a, b, c);
}

// Faces of a tetrahedron by owner-edge search.  The triangle with owner edge
// f (its largest edge position) and apex a (its vertex off f): when f is alone
// at its filtration level, f's triangles sit at [toff[f], toff[f+1]) in apex
// order, so its position is toff[f] + #apexes of f below a -- an 8-ary search
// in the (L2-resident) apex array.  One 32-byte record per owner edge (one
// sector) holds toff[f], the count and 12 separators (every b-th apex,
// b = ceil(count / 13)); it selects the block of <= b entries that holds a,
// which two 16-byte reads finish for counts <= 104: two dependent L2 round
// trips per face.
// A tie level is lex-sorted as a whole: binary search by triple in tv.
struct FaceQuery {
    uint32_t f, a, a0, a1, a2;
};

__device__ __forceinline__ FaceQuery face_query(uint32_t u, uint32_t v, uint32_t w, uint32_t puv, uint32_t puw,
                                                uint32_t pvw) {
    FaceQuery q{puv, w, u, v, w};
    if (puw > q.f) { q.f = puw; q.a = v; }
    if (pvw > q.f) { q.f = pvw; q.a = u; }
    sort3v(q.a0, q.a1, q.a2);
    return q;
}

// 8-ary rounds of 7 independent probes over apex[lo, hi) (ascending) until
// <= 8 entries are left that hold the first entry >= a.
__device__ __forceinline__ void apex_narrow(const uint16_t* __restrict__ apex, uint32_t& lo, uint32_t& hi,
                                            uint32_t a) {
    while (hi - lo > 8) {
        const uint32_t step = (hi - lo + 7) >> 3;
        uint32_t c = 0;
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            const uint32_t q = lo + (uint32_t)i * step;
            if (q < hi) c += __ldg(apex + q) < a ? 1u : 0u;
        }
        const uint32_t nlo = lo + c * step;
        hi = min(hi, nlo + step);
        lo = nlo;
    }
}

// The <= 8 entries [lo, hi) lie in two aligned 16-byte chunks of the apex
// array (padded by 16 entries): load them ...
__device__ __forceinline__ void apex_chunks(const uint16_t* __restrict__ apex, uint32_t lo, uint32_t hi, uint4& c0,
                                            uint4& c1) {
    const uint32_t base = lo & ~7u;
    const uint4* pv = reinterpret_cast<const uint4*>(apex + base);
    c0 = __ldg(pv);
    c1 = hi - base > 8 ? __ldg(pv + 1) : make_uint4(~0u, ~0u, ~0u, ~0u);
}

// ... and return lo + #entries of [lo, hi) below a, compared 2 entries per
// 32-bit add when ids < 0x7FFF (bit 15 of each half of w + 0x8000 - a is set
// iff that entry >= a).
__device__ __forceinline__ uint32_t apex_count(const uint4& c0, const uint4& c1, uint32_t lo, uint32_t hi, uint32_t a,
                                               bool small_ids) {
    const uint32_t base = lo & ~7u;
    const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    uint32_t ltm = 0;
    if (small_ids) {
        const uint32_t K = 0x80008000u - a * 0x10001u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t lt = ~(w[i] + K);   // bit 15 / 31: low / high entry < a
            ltm |= ((lt >> 15) & 1u) << (2 * i) | (lt >> 31) << (2 * i + 1);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t lt = __vcmpltu2(w[i], a * 0x10001u);   // 0xFFFF per 16-bit lane below a
            ltm |= ((lt & 1u) | ((lt >> 15) & 2u)) << (2 * i);
        }
    }
    const uint32_t valid = ((1u << (hi - base)) - 1u) & ~((1u << (lo - base)) - 1u);
    return lo + (uint32_t)__popc(ltm & valid);
}

// Block of the triangle with owner edge f and apex a from f's face record:
// returns false when f shares its filtration level (tie: search by triple).
__device__ __forceinline__ bool face_block(const uint4& r0, const uint4& r1, uint32_t a, bool small_ids, uint32_t& lo,
                                           uint32_t& hi) {
    if (r0.y >> 31) return false;
    const uint32_t start = r0.x, len = r0.y;
    const uint32_t b = max(1u, (len + 12) / 13);
    const uint32_t sw[6] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    uint32_t c = 0;
    if (small_ids) {   // separators past the end are 0x7FFF > a
        const uint32_t K = 0x80008000u - (a + 1) * 0x10001u;
#pragma unroll
        for (int i = 0; i < 6; ++i) c += __popc(~(sw[i] + K) & 0x80008000u);
    } else {
#pragma unroll
        for (int i = 0; i < 12; ++i)
            c += ((uint32_t)(i + 1) * b < len && ((sw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu) <= a) ? 1u : 0u;
    }
    lo = start + c * b;
    hi = min(lo + b, start + len);
    return true;
}

// Positions of the two faces: both records read together, both blocks
// narrowed (no-op for counts <= 104), all four 16-byte chunks read together.
__device__ __forceinline__ void face_pos2(const TetArgs& A, const FaceQuery& q1, const FaceQuery& q2, uint32_t& r1,
                                          uint32_t& r2) {
    const bool small_ids = A.n < 0x7FFF;
    const uint4 a0 = __ldg(A.frec + 2 * (uint64_t)q1.f), a1 = __ldg(A.frec + 2 * (uint64_t)q1.f + 1);
    const uint4 b0 = __ldg(A.frec + 2 * (uint64_t)q2.f), b1 = __ldg(A.frec + 2 * (uint64_t)q2.f + 1);
    uint32_t lo1 = 0, hi1 = 0, lo2 = 0, hi2 = 0;
    const bool d1 = face_block(a0, a1, q1.a, small_ids, lo1, hi1);
    const bool d2 = face_block(b0, b1, q2.a, small_ids, lo2, hi2);
    if (d1) apex_narrow(A.apex, lo1, hi1, q1.a);
    if (d2) apex_narrow(A.apex, lo2, hi2, q2.a);
    // a block of one entry is the face itself (the apex is in the list): no
    // second round trip (every owner edge of <= 13 triangles: the record's
    // separators are its apexes)
    const bool x1 = d1 && hi1 - lo1 > 1, x2 = d2 && hi2 - lo2 > 1;
    uint4 c10, c11, c20, c21;
    if (x1) apex_chunks(A.apex, lo1, hi1, c10, c11);
    if (x2) apex_chunks(A.apex, lo2, hi2, c20, c21);
    r1 = d1 ? (x1 ? apex_count(c10, c11, lo1, hi1, q1.a, small_ids) : lo1) : tri_pos(A, q1.f, q1.a0, q1.a1, q1.a2);
    r2 = d2 ? (x2 ? apex_count(c20, c21, lo2, hi2, q2.a, small_ids) : lo2) : tri_pos(A, q2.f, q2.a0, q2.a1, q2.a2);
}

__global__ void k_tri_hash(const uint32_t* __restrict__ tv, int64_t T, ulonglong2* __restrict__ slots,
                           uint64_t mask) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < T; q += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t code = tri_code(tv[3 * q], tv[3 * q + 1], tv[3 * q + 2]);
        uint64_t h = mix64(code) & mask;
        for (;;) {
            const unsigned long long prev = atomicCAS(&slots[h].x, ~0ull, (unsigned long long)code);
            if (prev == ~0ull || prev == code) { slots[h].y = (unsigned long long)q; break; }
            h = (h + 1) & mask;
        }
    }
}

// Warp: S(p) sorted by id into W->Sk / W->Spx, flags S in the vertex bitmap.
// Returns |S| (may exceed kS: caller checks).
template <int kB, class Scratch>
__device__ uint32_t build_S(const TetArgs& A, const uint32_t* __restrict__ map, Scratch* __restrict__ W,
                           uint32_t* __restrict__ vbits, uint32_t p, uint32_t x, uint32_t len, uint64_t offx,
                           uint32_t degx) {
    constexpr int kBits = kB, kWords = kB / 32;
    const int lane = threadIdx.x & 31;
    const uint32_t* lk = A.nkr + offx;
    const uint32_t* lr = A.nr + offx;
    const uint32_t* lp = A.np + offx;
    const uint32_t kmask = A.packed ? 0xFFFFu : 0xFFFFFFFFu;
    uint32_t total = 0;
    for (uint32_t R = 0; R < degx; R += kBits) {
        const uint32_t lim = min((uint32_t)kBits, degx - R);
        const uint32_t nwords = (lim + 31) >> 5;
        for (uint32_t w = lane; w < nwords; w += 32) W->bits[w] = 0u;
        __syncwarp();
        for (uint32_t t = lane; t < len; t += 32) {
            const uint32_t w = __ldg(lk + t);
            const uint32_t k = w & kmask;
            const uint32_t r = (A.packed ? (w >> 16) : __ldg(lr + t)) - R;
            if (r < (uint32_t)kBits && map[k] < p) atomicOr(&W->bits[r >> 5], 1u << (r & 31));
        }
        __syncwarp();
        // prefix popcount, 4 words per lane
        uint32_t c[kWords / 32], tot = 0;
#pragma unroll
        for (int j = 0; j < kWords / 32; ++j) {
            const uint32_t wd = (kWords / 32) * lane + j;
            c[j] = wd < nwords ? __popc(W->bits[wd]) : 0u;
            tot += c[j];
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t run = incl - tot;
#pragma unroll
        for (int j = 0; j < kWords / 32; ++j) { W->wpre[(kWords / 32) * lane + j] = run; run += c[j]; }
        const uint32_t count = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        for (uint32_t t = lane; t < len; t += 32) {
            const uint32_t w = __ldg(lk + t);
            const uint32_t r = (A.packed ? (w >> 16) : __ldg(lr + t)) - R;
            if (r >= (uint32_t)kBits) continue;
            const uint32_t wd = W->bits[r >> 5];
            if (!((wd >> (r & 31)) & 1u)) continue;
            const uint32_t idx = total + W->wpre[r >> 5] + __popc(wd & ((1u << (r & 31)) - 1u));
            if (idx < (uint32_t)kS) {
                const uint32_t k = w & kmask;
                W->Sk[idx] = k;
                W->Spx[idx] = __ldg(lp + t);
                if (vbits) atomicOr(&vbits[k >> 5], 1u << (k & 31));
            }
        }
        __syncwarp();
        total += count;
    }
    return total;
}

__device__ void clear_S(TetScratch* __restrict__ W, uint32_t* __restrict__ vbits, uint32_t m) {
    const int lane = threadIdx.x & 31;
    for (uint32_t i = lane; i < m; i += 32) {
        const uint32_t k = W->Sk[i];
        atomicAnd(&vbits[k >> 5], ~(1u << (k & 31)));
    }
    __syncwarp();
}

// For k = Sk[ki]: mark l in S, l > k, pos(k,l) < p; returns #marked and
// fills lpre.
__device__ uint32_t mark_l(const TetArgs& A, TetScratch* __restrict__ W, const uint32_t* __restrict__ vbits,
                           const uint32_t* __restrict__ vpre, uint32_t p, uint32_t ki, uint32_t m) {
    const int lane = threadIdx.x & 31;
    const uint32_t k = W->Sk[ki];
    const uint64_t ok0 = A.off[k], ok1 = A.off[k + 1];
    const uint32_t* npk = A.np + ok0;
    // k's neighbours older than p: a prefix of its position-ordered list
    const uint32_t plen = W->plen[ki];
    (void)ok1;
    const uint32_t nw = (m + 31) >> 5;
    for (uint32_t w = lane; w < nw; w += 32) W->lbits[w] = 0u;
    __syncwarp();
    const uint32_t kmask = A.packed ? 0xFFFFu : 0xFFFFFFFFu;
    const uint32_t* lk = A.nkr + ok0;
    for (uint32_t t = lane; t < plen; t += 32) {
        const uint32_t l = __ldg(lk + t) & kmask;
        const uint32_t vw = vbits[l >> 5];
        if (l <= k || !((vw >> (l & 31)) & 1u)) continue;
        const uint32_t j = vpre[l >> 5] + __popc(vw & ((1u << (l & 31)) - 1u));   // index of l in S
        atomicOr(&W->lbits[j >> 5], 1u << (j & 31));
        W->lpos[j] = __ldg(npk + t);
    }
    __syncwarp();
    uint32_t tot = 0;
    for (uint32_t w = lane; w < nw; w += 32) tot += __popc(W->lbits[w]);
    // words in order: lane w holds word w (nw <= 32)
    const uint32_t c = lane < (int)nw ? __popc(W->lbits[lane]) : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane < (int)nw) W->lpre[lane] = incl - c;
    __syncwarp();
    (void)tot;
    return __shfl_sync(0xffffffffu, incl, 31);
}

template <bool kFill>
__global__ void __launch_bounds__(kThreads, 1) k_tets(TetArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* map = reinterpret_cast<uint32_t*>(smem);
    const int64_t nvw = (A.n + 31) >> 5;
    const size_t map_b = (size_t)((A.n * 4 + 15) / 16) * 16;
    const size_t vb_b = (size_t)((nvw * 4 + 15) / 16) * 16;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nthreads = blockDim.x;
    uint32_t* vbits = reinterpret_cast<uint32_t*>(smem + map_b + (size_t)wid * 2 * vb_b);
    uint32_t* vpre = vbits + vb_b / 4;
    TetScratch* W = reinterpret_cast<TetScratch*>(smem + map_b + (size_t)(nthreads / 32) * 2 * vb_b) + wid;
    __shared__ int64_t s_lo, s_hi, s_end;
    __shared__ uint32_t s_y;
    __shared__ unsigned s_next;
    for (int64_t q = threadIdx.x; q < A.n; q += nthreads) map[q] = NONE32;
    for (int64_t q = lane; q < nvw; q += 32) vbits[q] = 0u;
    __syncthreads();
    const uint32_t kmask = A.packed ? 0xFFFFu : 0xFFFFFFFFu;
    for (;;) {
        if (threadIdx.x == 0) {
            const int64_t task = A.task_lo + (int64_t)atomicAdd(A.task_counter, 1ull);
            if (task >= A.task_hi) {
                s_lo = s_hi = -1;
            } else {
                s_lo = lb_u64(A.work_pre, 0, A.E + 1, (uint64_t)task * A.chunk);
                s_hi = task == A.ntasks - 1 ? A.E : lb_u64(A.work_pre, 0, A.E + 1, (uint64_t)(task + 1) * A.chunk);
                if (s_lo > A.E) s_lo = A.E;
                if (s_hi > A.E) s_hi = A.E;
            }
        }
        __syncthreads();
        const int64_t lo = s_lo, hi = s_hi;
        __syncthreads();
        if (lo < 0) break;
        for (int64_t seg = lo; seg < hi;) {
            if (threadIdx.x == 0) {
                const uint32_t y = A.hosted_v[seg];
                s_y = y;
                s_end = ub_u32(A.hosted_v, seg, hi, y);
                s_next = 0;
            }
            __syncthreads();
            const uint32_t y = s_y;
            const int64_t end = s_end;
            const uint64_t oy = A.off[y], oy1 = A.off[y + 1];
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = A.np[t];
            __syncthreads();
            for (;;) {
                unsigned my = 0;
                if (lane == 0) my = atomicAdd(&s_next, 1u);
                const int64_t e = seg + (int64_t)__shfl_sync(0xffffffffu, my, 0);
                if (e >= end) break;
                const uint4 pl = A.plan[e];
                const uint32_t p = pl.x, x = pl.y, len = pl.z;
                if (len < 2) continue;
                if (kFill && ((int64_t)p < A.p_lo || (int64_t)p >= A.p_hi)) continue;
                const uint64_t offx = A.off[x];
                const uint32_t m = build_S<kBits>(A, map, W, vbits, p, x, len, offx, pl.w);
                if (m > (uint32_t)kS) {   // too large for warp scratch: k_tets_big
                    if (lane == 0) A.ovf_list[atomicAdd(A.ovf_n, 1u)] = (uint32_t)e;
                    clear_S(W, vbits, kS);
                    continue;
                }
                // older-neighbour prefix length of every k in S, one lane per k
                for (uint32_t i = lane; i < m; i += 32) {
                    const uint32_t k = W->Sk[i];
                    const uint64_t o0 = A.off[k], o1 = A.off[k + 1];
                    W->plen[i] = lb_u32(A.np + o0, 0, (uint32_t)(o1 - o0), p);
                }
                {   // vpre[w] = #S members in words < w (index of a member = its rank by id)
                    const uint32_t per = (uint32_t)((nvw + 31) >> 5);
                    const uint32_t w0 = lane * per, w1 = min((uint32_t)nvw, w0 + per);
                    uint32_t tot = 0;
                    for (uint32_t w = w0; w < w1; ++w) tot += __popc(vbits[w]);
                    uint32_t incl = tot;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += v;
                    }
                    uint32_t run = incl - tot;
                    for (uint32_t w = w0; w < w1; ++w) { vpre[w] = run; run += __popc(vbits[w]); }
                    __syncwarp();
                }
                uint64_t slot = 0;
                uint32_t filt = 0;
                bool direct = false;
                uint64_t tbase = 0;
                if (kFill) {
                    slot = A.qoff[p] - A.slot0;
                    filt = A.efilt[p];
                    tbase = A.toff[p];
                    direct = !(A.frec[2 * (uint64_t)p].y >> 31);   // p alone at its level
                }
                uint32_t total = 0;
                for (uint32_t ki = 0; ki + 1 < m; ++ki) {
                    const uint32_t c = mark_l(A, W, vbits, vpre, p, ki, m);
                    if (kFill && c) {
                    const uint32_t k = W->Sk[ki];
                    const uint32_t f_yxk = direct ? (uint32_t)(tbase + ki) : 0u;
                    const uint32_t nw = (m + 31) >> 5;
                    // dense lanes: lane takes the i-th marked l (i = lane, lane + 32, ...)
                    for (uint32_t i = lane; i < c; i += 32) {
                        uint32_t w = 0;
                        while (w + 1 < nw && W->lpre[w + 1] <= i) ++w;
                        const uint32_t j = 32 * w + (uint32_t)__fns(W->lbits[w], 0, (int)(i - W->lpre[w] + 1));
                        const uint32_t l = W->Sk[j];
                        const uint64_t s = slot + total + i;
                        uint32_t v[4] = {y, x, k, l};
                        sort4v(v);
                        uint4* qv = reinterpret_cast<uint4*>(A.qv + 4 * s);
                        *qv = make_uint4(v[0], v[1], v[2], v[3]);
                        A.qf[s] = filt;
                        if (A.rows) {
                            uint32_t r[4];
                            if (direct) {
                                r[0] = f_yxk;
                                r[1] = (uint32_t)(tbase + j);
                            } else if (A.apex) {
                                uint32_t a0 = y, a1 = x, a2 = k;
                                sort3v(a0, a1, a2);
                                r[0] = tri_pos(A, p, a0, a1, a2);
                                a0 = y; a1 = x; a2 = l;
                                sort3v(a0, a1, a2);
                                r[1] = tri_pos(A, p, a0, a1, a2);
                            } else {
                                tri_lookup2(A, tri_code_sorted(y, x, k), tri_code_sorted(y, x, l), r[0], r[1]);
                            }
                            if (A.apex) {
                                const uint32_t pkl = W->lpos[j];
                                face_pos2(A, face_query(y, k, l, map[k], map[l], pkl),
                                          face_query(x, k, l, W->Spx[ki], W->Spx[j], pkl), r[2], r[3]);
                            } else {
                                tri_lookup2(A, tri_code_sorted(y, k, l), tri_code_sorted(x, k, l), r[2], r[3]);
                            }
                            sort4v(r);
                            *reinterpret_cast<uint4*>(A.rows + 4 * s) = make_uint4(r[0], r[1], r[2], r[3]);
                        }
                    }
                }
                    total += c;
                    __syncwarp();
                }
                if (!kFill && lane == 0) A.cnt[p] = total;
                clear_S(W, vbits, m);
            }
            __syncthreads();
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = NONE32;
            __syncthreads();
            seg = end;
        }
    }
}

// ---------------------------------------------------------------------------
// Dense-table variant (n <= kDenseMaxN; needs the apex array).  The pairs
// (k, l), k < l, of S(p) are tested directly -- pos(k, l) < p in an n x n
// table of edge positions (L2-resident for the configs of interest) --
// instead of streaming every k's older-neighbour prefix.  The pairs are
// walked in row-major (k, l) order, 32 per warp step: a ballot and a
// prefix popcount place each tetrahedron, so emission is in lex order and
// the stores of a step are contiguous.
// ---------------------------------------------------------------------------
constexpr int kBitsD = 1024;   // ranks of x's id list per build_S round (dense path)
struct TetScratchD {
    uint32_t bits[kBitsD / 32];
    uint32_t wpre[kBitsD / 32];
    uint32_t Sk[kS];          // S sorted by id
    uint32_t Spx[kS];         // pos(x, k)
};

// row i of the upper-triangular pair index q (rows of m - 1 - i pairs)
__device__ __forceinline__ void pair_of(uint32_t q, uint32_t m, uint32_t& i, uint32_t& j) {
    const float b = (float)(2 * m - 1);
    int ii = (int)((b - sqrtf(b * b - 8.0f * (float)q)) * 0.5f);
    ii = max(0, min(ii, (int)m - 2));
    auto start = [&](int r) { return (uint32_t)(r * (2 * (int)m - r - 1) / 2); };
    while (ii > 0 && start(ii) > q) --ii;
    while (ii + 1 < (int)m - 1 && start(ii + 1) <= q) ++ii;
    i = (uint32_t)ii;
    j = q - start(ii) + (uint32_t)ii + 1u;
}

template <bool kFill>
__global__ void __launch_bounds__(1024, 1) k_tets_dense(TetArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* map = reinterpret_cast<uint32_t*>(smem);
    const size_t map_b = (size_t)((A.n * 4 + 15) / 16) * 16;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int nthreads = blockDim.x;
    TetScratchD* W = reinterpret_cast<TetScratchD*>(smem + map_b) + wid;
    __shared__ int64_t s_lo, s_hi, s_end;
    __shared__ uint32_t s_y;
    __shared__ unsigned s_next;
    for (int64_t q = threadIdx.x; q < A.n; q += nthreads) map[q] = NONE32;
    __syncthreads();
    const uint32_t kmask = A.packed ? 0xFFFFu : 0xFFFFFFFFu;
    const uint64_t n = (uint64_t)A.n;
    for (;;) {
        if (threadIdx.x == 0) {
            const int64_t task = A.task_lo + (int64_t)atomicAdd(A.task_counter, 1ull);
            if (task >= A.task_hi) {
                s_lo = s_hi = -1;
            } else {
                s_lo = lb_u64(A.work_pre, 0, A.E + 1, (uint64_t)task * A.chunk);
                s_hi = task == A.ntasks - 1 ? A.E : lb_u64(A.work_pre, 0, A.E + 1, (uint64_t)(task + 1) * A.chunk);
                if (s_lo > A.E) s_lo = A.E;
                if (s_hi > A.E) s_hi = A.E;
            }
        }
        __syncthreads();
        const int64_t lo = s_lo, hi = s_hi;
        __syncthreads();
        if (lo < 0) break;
        for (int64_t seg = lo; seg < hi;) {
            if (threadIdx.x == 0) {
                const uint32_t y = A.hosted_v[seg];
                s_y = y;
                s_end = ub_u32(A.hosted_v, seg, hi, y);
                s_next = 0;
            }
            __syncthreads();
            const uint32_t y = s_y;
            const int64_t end = s_end;
            const uint64_t oy = A.off[y], oy1 = A.off[y + 1];
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = A.np[t];
            __syncthreads();
            for (;;) {
                unsigned my = 0;
                if (lane == 0) my = atomicAdd(&s_next, 1u);
                const int64_t e = seg + (int64_t)__shfl_sync(0xffffffffu, my, 0);
                if (e >= end) break;
                const uint4 pl = A.plan[e];
                const uint32_t p = pl.x, x = pl.y, len = pl.z;
                if (len < 2) continue;
                if (kFill && ((int64_t)p < A.p_lo || (int64_t)p >= A.p_hi)) continue;
                const uint32_t m = build_S<kBitsD>(A, map, W, nullptr, p, x, len, A.off[x], pl.w);
                if (m > (uint32_t)kS) {   // too large for warp scratch: k_tets_big
                    if (lane == 0) A.ovf_list[atomicAdd(A.ovf_n, 1u)] = (uint32_t)e;
                    continue;
                }
                uint64_t slot = 0, tbase = 0;
                uint32_t filt = 0;
                bool direct = false;
                if (kFill) {
                    slot = A.qoff[p] - A.slot0;
                    filt = A.efilt[p];
                    tbase = A.toff[p];
                    direct = !(A.frec[2 * (uint64_t)p].y >> 31);
                }
                const uint32_t npairs = m * (m - 1) / 2;
                uint32_t total = 0;
                // the table read of the next warp step is issued before this
                // step's faces are searched (two L2 round trips overlap)
                uint32_t i_n = 0, j_n = 0, pkl_n = NONE32;
                if ((uint32_t)lane < npairs) {
                    pair_of(lane, m, i_n, j_n);
                    pkl_n = __ldg(A.dense + (uint64_t)W->Sk[i_n] * n + W->Sk[j_n]);
                }
                for (uint32_t q0 = 0; q0 < npairs; q0 += 32) {
                    const uint32_t i = i_n, j = j_n, pkl = pkl_n;
                    {
                        const uint32_t qn = q0 + 32 + lane;
                        pkl_n = NONE32;
                        if (qn < npairs) {   // advance 32 pairs in row-major order
                            j_n += 32;
                            while (j_n >= m) { ++i_n; j_n = j_n - m + i_n + 1; }
                            pkl_n = __ldg(A.dense + (uint64_t)W->Sk[i_n] * n + W->Sk[j_n]);
                        }
                    }
                    const bool valid = pkl < p;
                    const uint32_t bal = __ballot_sync(0xffffffffu, valid);
                    if (kFill && valid) {
                        const uint32_t k = W->Sk[i], l = W->Sk[j];
                        const uint64_t s = slot + total + __popc(bal & lt);
                        uint32_t v[4] = {y, x, k, l};
                        sort4v(v);
                        __stcs(reinterpret_cast<uint4*>(A.qv + 4 * s), make_uint4(v[0], v[1], v[2], v[3]));
                        __stcs(A.qf + s, filt);
                        if (A.rows) {
                            uint32_t r[4];
                            if (direct) {
                                r[0] = (uint32_t)(tbase + i);
                                r[1] = (uint32_t)(tbase + j);
                            } else {
                                uint32_t a0 = y, a1 = x, a2 = k;
                                sort3v(a0, a1, a2);
                                r[0] = tri_pos(A, p, a0, a1, a2);
                                a0 = y; a1 = x; a2 = l;
                                sort3v(a0, a1, a2);
                                r[1] = tri_pos(A, p, a0, a1, a2);
                            }
                            face_pos2(A, face_query(y, k, l, map[k], map[l], pkl),
                                      face_query(x, k, l, W->Spx[i], W->Spx[j], pkl), r[2], r[3]);
                            sort4v(r);
                            __stcs(reinterpret_cast<uint4*>(A.rows + 4 * s), make_uint4(r[0], r[1], r[2], r[3]));
                        }
                    }
                    total += __popc(bal);
                }
                if (!kFill && lane == 0) A.cnt[p] = total;
                __syncwarp();
            }
            __syncthreads();
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = NONE32;
            __syncthreads();
            seg = end;
        }
    }
}


// ---------------------------------------------------------------------------
// Owner edges whose apex set S(p) exceeds the warp scratch (|S| > kS = 512):
// one CTA per such edge, S and the per-row counts in global scratch.  The
// definition is the same: S(p) = the common neighbours k of the
// owner's endpoints with both edges older than p, sorted by id (an
// intersection of x's and y's id-ordered lists); the tetrahedra of p are the
// pairs k < l of S adjacent through an edge older than p (k's id-ordered list
// merged with S), emitted row by row in (k, l) order -- the lex order of the
// sorted 4-tuples -- at slots from an exclusive scan of the row counts.
// ---------------------------------------------------------------------------
constexpr int kBigThreads = 512;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh, uint32_t& total) {
    // sh: >= 32 words of shared scratch
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) sh[wid] = incl;
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
        const uint32_t c = sh[w];
        if (w < wid) before += c;
        tot += c;
    }
    __syncthreads();
    total = tot;
    return before + incl - v;
}

template <bool kFill>
__global__ void __launch_bounds__(kBigThreads) k_tets_big(TetArgs A) {
    __shared__ uint32_t sh[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t* Sk = A.big + (uint64_t)blockIdx.x * A.big_stride;
    uint32_t* Spx = Sk + A.max_deg;
    uint32_t* Spy = Spx + A.max_deg;
    uint32_t* crow = Spy + A.max_deg;   // row counts, then row offsets
    const unsigned nbig = *A.ovf_n;
    for (unsigned q = blockIdx.x; q < nbig; q += gridDim.x) {
        const uint32_t e = A.ovf_list[q];
        const uint4 pl = A.plan[e];
        const uint32_t p = pl.x, x = pl.y, y = A.hosted_v[e];
        const uint64_t ox = A.off[x], oy = A.off[y];
        const uint32_t dx = (uint32_t)(A.off[x + 1] - ox), dy = (uint32_t)(A.off[y + 1] - oy);
        // ---- S(p), sorted by id, with pos(x, k) and pos(y, k)
        uint32_t m = 0;
        for (uint32_t b0 = 0; b0 < dx; b0 += blockDim.x) {
            const uint32_t t = b0 + threadIdx.x;
            bool v = false;
            uint32_t k = 0, px = 0, py = 0;
            if (t < dx) {
                const uint2 ek = __ldg(A.idl + ox + t);
                k = ek.x;
                px = ek.y;
                if (px < p) {
                    uint32_t lo = 0, hi = dy;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (__ldg(&A.idl[oy + mid].x) < k) lo = mid + 1; else hi = mid;
                    }
                    if (lo < dy) {
                        const uint2 fy = __ldg(A.idl + oy + lo);
                        if (fy.x == k && fy.y < p) { v = true; py = fy.y; }
                    }
                }
            }
            uint32_t tot = 0;
            const uint32_t at = m + block_excl_scan(v ? 1u : 0u, sh, tot);
            if (v) { Sk[at] = k; Spx[at] = px; Spy[at] = py; }
            m += tot;
        }
        __syncthreads();
        // ---- row i (k = Sk[i]): the l in S, l > k, with pos(k, l) < p
        auto row_pass = [&](uint32_t i, bool emit, uint32_t base, uint64_t slot, uint32_t filt, bool direct,
                            uint64_t tbase) -> uint32_t {
            const uint32_t k = Sk[i];
            const uint64_t ok = A.off[k];
            const uint32_t dk = (uint32_t)(A.off[k + 1] - ok);
            // first entry of k's id list above k
            uint32_t lo = 0, hi = dk;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(&A.idl[ok + mid].x) <= k) lo = mid + 1; else hi = mid;
            }
            uint32_t c = 0;
            for (uint32_t t0 = lo; t0 < dk; t0 += 32) {
                const uint32_t t = t0 + lane;
                bool v = false;
                uint32_t j = 0, pkl = 0, l = 0;
                if (t < dk) {
                    const uint2 el = __ldg(A.idl + ok + t);
                    l = el.x;
                    pkl = el.y;
                    if (pkl < p) {
                        uint32_t a = i + 1, b = m;
                        while (a < b) {
                            const uint32_t mid = (a + b) >> 1;
                            if (Sk[mid] < l) a = mid + 1; else b = mid;
                        }
                        if (a < m && Sk[a] == l) { v = true; j = a; }
                    }
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, v);
                if (emit && v) {
                    const uint64_t s = slot + base + c + __popc(bal & lt);
                    uint32_t vv[4] = {y, x, k, l};
                    sort4v(vv);
                    __stcs(reinterpret_cast<uint4*>(A.qv + 4 * s), make_uint4(vv[0], vv[1], vv[2], vv[3]));
                    __stcs(A.qf + s, filt);
                    if (A.rows) {
                        uint32_t r[4];
                        if (direct) {
                            r[0] = (uint32_t)(tbase + i);
                            r[1] = (uint32_t)(tbase + j);
                        } else {
                            uint32_t a0 = y, a1 = x, a2 = k;
                            sort3v(a0, a1, a2);
                            r[0] = tri_pos(A, p, a0, a1, a2);
                            a0 = y; a1 = x; a2 = l;
                            sort3v(a0, a1, a2);
                            r[1] = tri_pos(A, p, a0, a1, a2);
                        }
                        if (A.apex)
                            face_pos2(A, face_query(y, k, l, Spy[i], Spy[j], pkl),
                                      face_query(x, k, l, Spx[i], Spx[j], pkl), r[2], r[3]);
                        else
                            tri_lookup2(A, tri_code_sorted(y, k, l), tri_code_sorted(x, k, l), r[2], r[3]);
                        sort4v(r);
                        __stcs(reinterpret_cast<uint4*>(A.rows + 4 * s), make_uint4(r[0], r[1], r[2], r[3]));
                    }
                }
                c += __popc(bal);
            }
            return c;
        };
        for (uint32_t i = wid; i < m; i += nwarps) {
            const uint32_t c = row_pass(i, false, 0, 0, 0, false, 0);
            if (lane == 0) crow[i] = c;
        }
        __syncthreads();
        if (!kFill) {
            uint32_t part = 0;
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) part += crow[i];
            uint32_t tot = 0;
            block_excl_scan(part, sh, tot);
            if (threadIdx.x == 0) A.cnt[p] = tot;
        } else {
            // exclusive offsets of the rows, in chunks of blockDim
            uint32_t run = 0;
            for (uint32_t b0 = 0; b0 < m; b0 += blockDim.x) {
                const uint32_t i = b0 + threadIdx.x;
                const uint32_t c = i < m ? crow[i] : 0u;
                uint32_t tot = 0;
                const uint32_t ex = block_excl_scan(c, sh, tot);
                if (i < m) crow[i] = run + ex;
                run += tot;
            }
            __syncthreads();
            const uint64_t slot = A.qoff[p] - A.slot0;
            const uint32_t filt = A.efilt[p];
            const uint64_t tbase = A.toff[p];
            const bool direct = !(A.frec[2 * (uint64_t)p].y >> 31);
            for (uint32_t i = wid; i < m; i += nwarps) row_pass(i, true, crow[i], slot, filt, direct, tbase);
        }
        __syncthreads();
    }
}

__global__ void k_dense_positions(const uint32_t* __restrict__ ev, int64_t E, int64_t n, uint32_t* __restrict__ tab) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = ev[2 * p], b = ev[2 * p + 1];
        tab[a * (uint64_t)n + b] = (uint32_t)p;
        tab[b * (uint64_t)n + a] = (uint32_t)p;
    }
}

// tlo / thi: the triangle range of each edge's filtration level; frec: the
// face record of each owner edge (see face_pos)
__global__ void k_level_ranges(const uint32_t* __restrict__ efilt, const uint64_t* __restrict__ toff, int64_t E,
                               const uint16_t* __restrict__ apex, uint32_t sentinel, uint64_t* __restrict__ tlo,
                               uint64_t* __restrict__ thi, uint4* __restrict__ frec) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        if (p > 0 && efilt[p - 1] == efilt[p]) continue;   // not a level start
        int64_t q = p + 1;
        while (q < E && efilt[q] == efilt[p]) ++q;
        const uint32_t shared = q - p > 1 ? 0x80000000u : 0u;
        for (int64_t r = p; r < q; ++r) {
            tlo[r] = toff[p];
            thi[r] = toff[q];
            const uint32_t start = (uint32_t)toff[r], len = (uint32_t)(toff[r + 1] - toff[r]);
            const uint32_t b = max(1u, (len + 12) / 13);
            uint32_t sep[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) {
                const uint32_t o = (uint32_t)(i + 1) * b;
                sep[i] = (apex && o < len) ? (uint32_t)apex[start + o] : sentinel;
            }
            frec[2 * r] = make_uint4(start, len | shared, sep[0] | sep[1] << 16, sep[2] | sep[3] << 16);
            frec[2 * r + 1] = make_uint4(sep[4] | sep[5] << 16, sep[6] | sep[7] << 16, sep[8] | sep[9] << 16,
                                         sep[10] | sep[11] << 16);
        }
    }
}

size_t tet_smem(int64_t n, int warps) {
    const int64_t nvw = (n + 31) >> 5;
    return (size_t)((n * 4 + 15) / 16) * 16 + (size_t)warps * 2 * ((size_t)((nvw * 4 + 15) / 16) * 16) +
           (size_t)warps * sizeof(TetScratch);
}

int tet_warps(int64_t n) {
    const int64_t avail = (int64_t)device_max_smem_optin() - 1024;
    for (int w = kWarps; w >= 4; w /= 2)
        if ((int64_t)tet_smem(n, w) <= avail) return w;
    return 0;
}

#ifndef VRB_TET_CTA_WARPS
#define VRB_TET_CTA_WARPS 10
#endif
#ifndef VRB_TET_DENSE_CTAS
#define VRB_TET_DENSE_CTAS 3
#endif
// dense path: CTAs of up to VRB_TET_CTA_WARPS warps, 3 per SM when the map
// is small (C4 fill: 8 warps 10.7 ms, 10 warps 10.0 ms; 16-warp CTAs two per
// SM are slower: longer per-host barrier tails, hosts own ~E/n edges each)
int tet_dense_warps(int64_t n) {
    const int64_t avail = (int64_t)device_max_smem_optin() - 1024 - (int64_t)((n * 4 + 15) / 16) * 16;
    return (int)std::min<int64_t>(VRB_TET_CTA_WARPS, avail / (int64_t)sizeof(TetScratchD));
}

// The owner edges the main kernel listed (|S(p)| > kS): one CTA each.
void launch_big(TetArgs A, bool fill, cudaStream_t s) {
    unsigned h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, A.ovf_n, sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h == 0) return;
    if (!A.idl) fail(VRB_ENOTSUP, "an edge owns more than %d triangles and the lists are not packed", kS);
    const unsigned grid = std::min<unsigned>(h, (unsigned)device_sm_count() * 2);
    A.big_stride = 4 * (uint64_t)A.max_deg + 4;
    DBuf<uint32_t> scratch((size_t)grid * A.big_stride, s);
    A.big = scratch.get();
    if (fill)
        k_tets_big<true><<<grid, kBigThreads, 0, s>>>(A);
    else
        k_tets_big<false><<<grid, kBigThreads, 0, s>>>(A);
    VRB_LAUNCH_CHECK();
}

void launch_tets(TetArgs A, bool fill, uint64_t work, int part, int nparts, cudaStream_t s) {
    if (A.dense && tet_dense_warps(A.n) >= 8) {
        const int warps = tet_dense_warps(A.n);
        const size_t smem = (size_t)((A.n * 4 + 15) / 16) * 16 + (size_t)warps * sizeof(TetScratchD);
        if (fill)
            VRB_CUDA(cudaFuncSetAttribute(k_tets_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else
            VRB_CUDA(cudaFuncSetAttribute(k_tets_dense<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        uint64_t chunk = work / 8192 + 1;
        if (chunk < 16384) chunk = 16384;
        A.chunk = chunk;
        A.ntasks = (int64_t)((work + chunk - 1) / chunk);
        if (A.ntasks < 1) A.ntasks = 1;
        A.task_lo = A.ntasks * part / nparts;
        A.task_hi = A.ntasks * (part + 1) / nparts;
        if (A.task_lo >= A.task_hi) return;
        DBuf<unsigned long long> counter(1, s);
        DBuf<unsigned> ovf_n(1, s);
        DBuf<uint32_t> ovf_list(A.E, s);
        VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned long long), s));
        VRB_CUDA(cudaMemsetAsync(ovf_n.get(), 0, sizeof(unsigned), s));
        A.task_counter = counter.get();
        A.ovf_n = ovf_n.get();
        A.ovf_list = ovf_list.get();
        // fill: at most VRB_TET_DENSE_CTAS CTAs per SM, the rest of the
        // unified on-chip memory left to L1 (the face searches live on L1
        // hits; 4 CTAs: 14.4 ms, 3: 11.1 ms on C4); the count takes 4
        const int cap = fill ? VRB_TET_DENSE_CTAS : 4;
        const int carve = (int)std::min<int64_t>(
            100, (int64_t)ceil_div((int64_t)cap * (int64_t)(smem + 1024) * 100, (int64_t)228 * 1024));
        int per_sm = 1;
        if (fill) {
            VRB_CUDA(cudaFuncSetAttribute(k_tets_dense<true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tets_dense<true>, warps * 32, smem));
        } else {
            VRB_CUDA(cudaFuncSetAttribute(k_tets_dense<false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tets_dense<false>, warps * 32, smem));
        }
        per_sm = std::min(per_sm, cap);
        const unsigned grid =
            (unsigned)std::min<int64_t>((int64_t)device_sm_count() * std::max(1, per_sm), A.task_hi - A.task_lo);
        if (fill)
            k_tets_dense<true><<<grid, warps * 32, smem, s>>>(A);
        else
            k_tets_dense<false><<<grid, warps * 32, smem, s>>>(A);
        VRB_LAUNCH_CHECK();
        launch_big(A, fill, s);
        return;
    }
    const int warps = tet_warps(A.n);
    if (warps < 4) fail(VRB_ENOTSUP, "tetrahedron kernel: n = %lld leaves no shared memory", (long long)A.n);
    const int threads = warps * 32;
    const size_t smem = tet_smem(A.n, warps);
    if (fill)
        VRB_CUDA(cudaFuncSetAttribute(k_tets<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    else
        VRB_CUDA(cudaFuncSetAttribute(k_tets<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    uint64_t chunk = work / 8192 + 1;
    if (chunk < 16384) chunk = 16384;
    A.chunk = chunk;
    A.ntasks = (int64_t)((work + chunk - 1) / chunk);
    if (A.ntasks < 1) A.ntasks = 1;
    A.task_lo = A.ntasks * part / nparts;
    A.task_hi = A.ntasks * (part + 1) / nparts;
    if (A.task_lo >= A.task_hi) return;
    DBuf<unsigned long long> counter(1, s);
    DBuf<unsigned> ovf_n(1, s);
    DBuf<uint32_t> ovf_list(A.E, s);
    VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned long long), s));
    VRB_CUDA(cudaMemsetAsync(ovf_n.get(), 0, sizeof(unsigned), s));
    A.task_counter = counter.get();
    A.ovf_n = ovf_n.get();
    A.ovf_list = ovf_list.get();
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)device_sm_count(), A.task_hi - A.task_lo);
    if (fill)
        k_tets<true><<<grid, threads, smem, s>>>(A);
    else
        k_tets<false><<<grid, threads, smem, s>>>(A);
    VRB_LAUNCH_CHECK();
    launch_big(A, fill, s);
}

}  // namespace

// Largest vertex count the tetrahedron stage supports on this device: the
// tie-group sort packs lex codes in 16-bit ids (n <= 65536), and the sparse
// kernel keeps an n-entry host map plus per-warp vertex bitmaps in shared
// memory (>= 4 warps; ~38k vertices with 227 KB of shared memory).
int64_t tets_max_n() {
    int64_t lo = 0, hi = 65536;
    while (lo < hi) {   // largest n with tet_warps(n) >= 4
        const int64_t mid = (lo + hi + 1) / 2;
        if (tet_warps(mid) >= 4) lo = mid; else hi = mid - 1;
    }
    return lo;
}

namespace {

TetArgs tet_args(const Graph& g, const TriLevels& L) {
    TetArgs A{};
    A.n = g.n;
    A.E = g.nplan;   // hosted slots of the plan (A.E bounds the plan and work_pre)
    A.off = g.off.get();
    A.nkr = g.nkr.get();
    A.nr = g.nr.get();
    A.np = g.np.get();
    A.packed = g.packed ? 1 : 0;
    A.plan = g.plan.get();
    A.hosted_v = g.hosted_v.get();
    A.work_pre = g.work_pre.get();
    A.idl = g.idl.get();
    A.max_deg = g.max_deg;
    A.toff = L.toff;
    A.tlo = L.tlo.get();
    A.thi = L.thi.get();
    A.frec = L.frec.get();
    A.tv = L.tv;
    A.hslots = L.hslots.get();
    A.apex = L.apex;
    A.dense = L.dense.get();
    A.hmask = L.hmask;
    return A;
}

}  // namespace

void triangle_levels(const uint32_t* efilt, const uint64_t* toff, int64_t E, const uint32_t* tv, cudaStream_t s,
                     TriLevels& L) {
    L.toff = toff;
    L.tv = tv;
    L.tlo.alloc(E, s);
    L.thi.alloc(E, s);
    L.frec.alloc(2 * E, s);
    if (E == 0) return;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(E, 256), (int64_t)device_sm_count() * 16);
    k_level_ranges<<<g, 256, 0, s>>>(efilt, toff, E, L.apex, L.n < 0x7FFF ? 0x7FFFu : 0xFFFFu, L.tlo.get(),
                                     L.thi.get(), L.frec.get());
    VRB_LAUNCH_CHECK();
    if (L.apex) {   // face positions by owner-edge search (face_pos2)
        const char* fs = std::getenv("VRB_FORCE_SPARSE_TETS");   // testing knob: the k_tets path
        if (L.n <= kDenseMaxN && !(fs && fs[0] == '1')) {   // pair tests through an n x n table of edge positions
            L.dense.alloc((size_t)(L.n * L.n), s);
            VRB_CUDA(cudaMemsetAsync(L.dense.get(), 0xFF, L.dense.bytes(), s));
            const unsigned gd = (unsigned)std::min<int64_t>(ceil_div(E, 256), (int64_t)device_sm_count() * 16);
            k_dense_positions<<<gd, 256, 0, s>>>(L.ev, E, L.n, L.dense.get());
            VRB_LAUNCH_CHECK();
        }
        return;
    }
    // triangle position hash (load factor <= 1/2)
    uint64_t T = 0;
    VRB_CUDA(cudaMemcpyAsync(&T, toff + E, sizeof(T), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    uint64_t cap = 1024;
    while (cap < T + T / 2) cap <<= 1;   // load factor in (1/3, 2/3]
    L.hmask = cap - 1;
    L.hslots.alloc(cap, s);
    VRB_CUDA(cudaMemsetAsync(L.hslots.get(), 0xFF, L.hslots.bytes(), s));
    if (T) {
        const unsigned gh = (unsigned)std::min<int64_t>(ceil_div((int64_t)T, 256), (int64_t)device_sm_count() * 16);
        k_tri_hash<<<gh, 256, 0, s>>>(tv, (int64_t)T, L.hslots.get(), L.hmask);
        VRB_LAUNCH_CHECK();
    }
}

void count_tets(const Graph& g, const TriLevels& L, uint32_t* cnt, int part, int nparts, cudaStream_t s) {
    if (g.E == 0) return;
    VRB_CUDA(cudaMemsetAsync(cnt, 0, g.E * sizeof(uint32_t), s));
    if (g.work == 0) return;
    TetArgs A = tet_args(g, L);
    A.cnt = cnt;
    launch_tets(A, false, g.work, part, nparts, s);
}

void fill_tets(const Graph& g, const TriLevels& L, const uint32_t* efilt, const uint64_t* qoff, int64_t p_lo,
               int64_t p_hi, uint64_t slot0, uint32_t* qv, uint32_t* qf, uint32_t* rows, cudaStream_t s) {
    if (g.E == 0 || g.work == 0 || p_lo >= p_hi) return;
    TetArgs A = tet_args(g, L);
    A.efilt = efilt;
    A.qoff = qoff;
    A.p_lo = p_lo;
    A.p_hi = p_hi;
    A.slot0 = slot0;
    A.qv = qv;
    A.qf = qf;
    A.rows = rows;
    launch_tets(A, true, g.work, 0, 1, s);
}

}  // namespace vrb
