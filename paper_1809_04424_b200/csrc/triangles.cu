// triangles.cu -- S5 (triangle enumeration), S7 (filtration order) and S8
// (boundary rows) fused into one owner-edge enumeration.
//
// Definition ("a solid triangle is created if all its three edges have
// been generated"; readings A3/A4/A7): triangle {u,v,w} exists iff its three
// edges are kept; filt = max edge filt; dimension 2 is ordered by (filt, lex);
// its D_2 column holds the positions of its three edges, ascending.
//
// Owner-edge order (B200 design).  Every triangle has a unique
// OWNER: its edge of largest position p in the (len, i, j) edge order.  Its
// filt is filt(p), and for a fixed owner (y, x) the triangles (y, x, k) with
// both other edges older than p are exactly the apexes
//     k in N(x) with pos(x,k) < p   and   pos(y,k) < p,
// and for a fixed owner, increasing k is increasing lex order of the sorted
// vertex triple.  So, when no two edges share a level, the global (filt, lex)
// order is (owner position, apex id): a count pass per owner edge, an
// exclusive scan, and a fill pass that writes each triangle straight to its
// final slot -- no sort of the 2e9 triangles of C5B.  Owner edges sharing a
// level (ties) get their small ranges re-sorted by lex afterwards (segsort.cu).
//
// Kernel shape.  Edges are grouped by a "host" endpoint y; a CTA holds the
// whole neighbourhood of y as a dense map pos_y[k] (n u32; shared memory, or
// a per-CTA slice of global memory when n is too large) and its warps take
// the host's owner edges one at a time (longest first, grabbed dynamically).
// For edge p = (y, x) a warp streams the older-neighbour PREFIX of x (x's
// neighbours in position order, cut at p; the endpoint with the shorter
// prefix is scanned) and tests pos_y[k] < p.  Two kernels:
//   count: per owner edge, the valid apexes' ranks in x's ID-ordered list are
//          OR-ed into a shared bitmap, which is stored (the "apex bitmap",
//          ceil(deg x / 32) words) and popcounted -> cnt[p].
//   fill : (single rank, packed lists, degrees <= 8192: the default) the
//          bitmap is reloaded in 32-word register chunks; a warp scan of the
//          popcounts gives each valid apex its slot (#valid apexes of smaller
//          id) -- a counting sort by apex id with no data movement; the set
//          bits of a window of slots are walked, (k, pos(x, k)) is gathered
//          from x's id-ordered list in rank order, pos(y, k) read from the
//          map, and 32 triangles at a time are staged in shared memory and
//          written as whole 16-byte chunks.
//          (Several ranks, or larger degrees: the fill re-enumerates -- mark
//          as the count does, rank, re-stream the prefix with its positions
//          staging (k, pos(x, k)) by slot, flush.)
//          Streams run 4/2/1 groups per lane so short prefixes waste few lanes.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kWarps = 32;               // max warps per CTA (fewer when the map is large)
constexpr int kThreads = kWarps * 32;
constexpr int kBits = 4096;              // apex ranks per round (bitmap bits per warp)
constexpr int kWords = kBits / 32;
static_assert(kWords % 32 == 0, "bitmap words must split evenly over the lanes");
#ifndef VRB_TRI_WIN
#define VRB_TRI_WIN 512
#endif
// VRB_TRI_MODE selects the packed-list fill (experiment knob, tools/variants.py):
//   3 (default) warp_fill_kp: the emit streams the prefix with its edge
//     positions and stages (k, pos(x, k)), so the flush needs no gathers
//   0 warp_fill (the wide-list algorithm): staged (k, t), pos(x, k) gathered
#ifndef VRB_TRI_MODE
#define VRB_TRI_MODE 3
#endif
#ifndef VRB_TRI_WIN3
#define VRB_TRI_WIN3 512
#endif
constexpr int kWin = VRB_TRI_WIN;        // triangles staged per output window (packed records)
constexpr int kRegGroups = 4;            // uint4 groups per lane in flight when streaming

struct TriArgs {
    int64_t n, E;
    const uint64_t* off;
    const uint32_t* nkr;     // packed ? (krank << 16 | k) : k, position-ordered lists
    const uint32_t* nr;      // krank when !packed
    const uint32_t* np;      // edge position of each list entry
    int packed;
    const uint4* plan;       // per hosted slot: (p, x, prefix length, deg x)
    const uint32_t* hosted_v;
    const uint64_t* work_pre;
    uint64_t chunk;
    int64_t ntasks;             // tasks of the whole work
    int64_t task_lo, task_hi;   // this launch's task range
    unsigned long long* task_counter;
    // count
    uint32_t* cnt;
    // fill
    const uint32_t* efilt;
    const uint64_t* toff;
    int64_t p_lo, p_hi;
    uint64_t slot0;
    uint32_t* tv;
    uint32_t* tf;
    uint32_t* rows;
    uint16_t* apex;   // K >= 3, n <= 65536: apex id of each triangle (its vertex off the owner edge)
    uint32_t* gmap;            // global-memory host maps (n u32 per CTA) when n is too large for
                               // shared memory, else null (the map lives in shared memory)
    uint32_t* bm;              // apex bitmaps (count writes, fill reads), or null
    int bm_mode;               // 1: by id rank in x's list (deg x bits); 2: by prefix entry (len bits)
    const uint64_t* bmoff;     // per hosted slot: word offset of its bitmap
    const uint2* idl;          // (k, pos) in neighbour-ID order
    int debug;   // ablation (experiment builds with -DVRB_ABLATION only): 1 = stop after mark, 2 = skip the flush
    // x-major path (records): per owner edge p (by position), its scanned
    // prefix's validity bits (tb + tb_off[p], ceil(len/32) words) and the host
    // positions pos(y, k) of its valid apexes in prefix order (rec + rec_off[p])
    uint32_t* rec;
    const uint64_t* rec_off;
    uint32_t* tb;
    const uint64_t* tb_off;
    const uint4* fplan;        // fill plan: slots grouped by scanned vertex x: (p, host y, len, deg x)
    const uint32_t* fgroup_v;  // x of each fill-plan slot
    int lists_cap;             // shared-memory list capacity (entries) of the x-major fill
};

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t upper_bound_u32(const uint32_t* a, int64_t lo, int64_t hi, uint32_t v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void sort3(uint32_t& a, uint32_t& b, uint32_t& c) {
    uint32_t t;
    if (a > b) { t = a; a = b; b = t; }
    if (b > c) { t = b; b = c; c = t; }
    if (a > b) { t = a; a = b; b = t; }
}

// Prefix streaming: lane-owned 16-byte aligned groups of 4 consecutive list
// entries.  `mis` = entries before the list start inside the first group.
// Entry e of group i is list index t = 4 i + e - mis (valid iff 0 <= t < len).
__device__ __forceinline__ const uint4* aligned_groups(const uint32_t* lst, int& mis) {
    mis = (int)((reinterpret_cast<uintptr_t>(lst) >> 2) & 3);
    return reinterpret_cast<const uint4*>(lst - mis);
}

__device__ __forceinline__ uint32_t pick(const uint4& q, int e) {
    return e == 0 ? q.x : (e == 1 ? q.y : (e == 2 ? q.z : q.w));
}

// Neighbour-list loads (read-only path).  L2 evict-last cache hints on these
// loads were measured and did not help.
__device__ __forceinline__ uint4 ld_list(const uint4* a) { return __ldg(a); }
__device__ __forceinline__ uint32_t ld_list(const uint32_t* a) { return __ldg(a); }
__device__ __forceinline__ uint2 ld_idl(const uint2* a) { return __ldg(a); }

__device__ __forceinline__ uint4 no_group() { return make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu); }

// Stream the groups of a list prefix: G uint4 groups per lane in flight;
// f(word, t) for every entry t in [0, len).
template <int G, class F>
__device__ __forceinline__ void stream_range(const uint4* __restrict__ g, int start, int stop, int ngroups, int mis,
                                             uint32_t len, F&& f) {
    const int lane = threadIdx.x & 31;
    for (int i0 = start; i0 < stop; i0 += 32 * G) {
        uint4 q[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
            q[u] = i < ngroups ? ld_list(g + i) : no_group();
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t t = (uint32_t)(4 * i + e - mis);
                if (t < len) f(pick(q[u], e), t);
            }
        }
    }
}
#ifndef VRB_TRI_TAIL
#define VRB_TRI_TAIL 1
#endif
// The whole prefix: 4-group iterations while >= 128 groups remain, then
// 2- and 1-group iterations (VRB_TRI_TAIL), so at most 127 entry slots per
// lane-sweep are idle; without VRB_TRI_TAIL one 1- or G-group stride.
template <int G, class F>
__device__ __forceinline__ void stream_prefix(const uint4* __restrict__ g, int ngroups, int mis, uint32_t len,
                                              F&& f) {
#if VRB_TRI_TAIL
    const int f4 = (ngroups / 128) * 128;
    const int f2 = f4 + ((ngroups - f4) / 64) * 64;
    stream_range<4>(g, 0, f4, ngroups, mis, len, f);
    stream_range<2>(g, f4, f2, ngroups, mis, len, f);
    stream_range<1>(g, f2, ngroups, ngroups, mis, len, f);
#else
    stream_range<G>(g, 0, ngroups, ngroups, mis, len, f);
#endif
}

// Per-warp shared scratch of the fill kernel (3 KB: 32 warps + the vertex
// map fit one SM).
struct WarpScratch {
    uint32_t bits[kWords];   // valid apexes of this round, bitmap by rank in x's id-ordered list
    uint32_t wpre[kWords];   // exclusive prefix popcount per bitmap word
    uint32_t rec[kWin];      // staged window: packed: apex k | prefix index t << 16;
                             //                wide:   (k, t) word pairs, kWin / 2 slots
};

// Per-warp shared scratch of the (k, pos) fill (VRB_TRI_MODE 3).
constexpr int kWin3 = VRB_TRI_WIN3;      // slots per window
struct WarpScratch3 {
    uint32_t bits[kWords];   // valid apexes of this round, bitmap by rank in x's id-ordered list
    uint32_t wpre[kWords];   // exclusive prefix popcount per bitmap word
    uint2 rec[kWin3];        // staged window: (apex k, pos(x, k)) per slot
};

// Stream two parallel list prefixes (same layout): f(word_a, word_b, t).
template <int G, class F>
__device__ __forceinline__ void stream_range2(const uint4* __restrict__ ga, const uint4* __restrict__ gb, int start,
                                              int stop, int ngroups, int mis, uint32_t len, F&& f) {
    const int lane = threadIdx.x & 31;
    for (int i0 = start; i0 < stop; i0 += 32 * G) {
        uint4 qa[G], qb[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
            qa[u] = i < ngroups ? ld_list(ga + i) : no_group();
            qb[u] = i < ngroups ? ld_list(gb + i) : no_group();
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t t = (uint32_t)(4 * i + e - mis);
                if (t < len) f(pick(qa[u], e), pick(qb[u], e), t);
            }
        }
    }
}
template <int G, class F>
__device__ __forceinline__ void stream_prefix2(const uint4* __restrict__ ga, const uint4* __restrict__ gb, int ngroups,
                                               int mis, uint32_t len, F&& f) {
#if VRB_TRI_TAIL
    const int f2 = (ngroups / 64) * 64;
    stream_range2<2>(ga, gb, 0, f2, ngroups, mis, len, f);
    stream_range2<1>(ga, gb, f2, ngroups, ngroups, mis, len, f);
#else
    stream_range2<G>(ga, gb, 0, ngroups, ngroups, mis, len, f);
#endif
}

// Clear the bitmap words of a round of lim ranks (before marking).
template <class WS>
__device__ __forceinline__ void clear_bits(WS* __restrict__ W, uint32_t lim) {
    const int lane = threadIdx.x & 31;
    const uint32_t nwords = (lim + 31) >> 5;
    for (uint32_t w = lane; w < nwords; w += 32) W->bits[w] = 0u;
    __syncwarp();
}

// Exclusive per-word prefix popcounts of the round's bitmap (lim ranks);
// returns the number of valid apexes of the round.
template <int kNW, class WS>
__device__ __forceinline__ uint32_t rank_bits(WS* __restrict__ W, uint32_t lim) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    constexpr int kWpl = kNW / 32;         // bitmap words per lane (lane owns kWpl consecutive words)
    const uint32_t nwords = (lim + 31) >> 5;
    uint32_t c[kWpl], tot = 0;
#pragma unroll
    for (int j = 0; j < kWpl; ++j) {
        const uint32_t wd = kWpl * lane + j;
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
    for (int j = 0; j < kWpl; ++j) { W->wpre[kWpl * lane + j] = run; run += c[j]; }
    __syncwarp();
    return __shfl_sync(0xffffffffu, incl, 31);
}

// Exclusive per-word prefix popcounts of nw bitmap words (any nw), warp-wide.
__device__ __forceinline__ void rank_bits_n(const uint32_t* __restrict__ bits, uint32_t* __restrict__ wpre,
                                            uint32_t nw) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    uint32_t carry = 0;
    for (uint32_t w0 = 0; w0 < nw; w0 += 32) {
        const uint32_t wd = w0 + lane;
        const uint32_t c = wd < nw ? __popc(bits[wd]) : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (wd < nw) wpre[wd] = carry + incl - c;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
}

// Write the staged window [s0, s0 + m), one lane per triangle, kU position
// gathers in flight per lane: record -> (k, t); pos(x, k) = np[offx + t] (the
// prefix just streamed: L1/L2), pos(y, k) = map[k].
template <bool kPacked>
__device__ __forceinline__ void flush_window(const TriArgs& A, const uint32_t* __restrict__ map,
                                             const WarpScratch* __restrict__ W, uint32_t m, uint64_t s0,
                                             uint32_t p, uint32_t y, uint32_t x, uint32_t filt,
                                             const uint32_t* __restrict__ npx) {
    const int lane = threadIdx.x & 31;
    constexpr int kU = 4;
    for (uint32_t j0 = 0; j0 < m; j0 += 32 * kU) {
        uint32_t kk[kU], px[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint32_t j = j0 + 32 * q + lane;
            kk[q] = 0;
            px[q] = 0;
            if (j < m) {
                uint32_t t;
                if (kPacked) {
                    const uint32_t rc = W->rec[j];
                    kk[q] = rc & 0xFFFFu;
                    t = rc >> 16;
                } else {
                    kk[q] = W->rec[2 * j];
                    t = W->rec[2 * j + 1];
                }
                px[q] = ld_list(npx + t);
            }
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint32_t j = j0 + 32 * q + lane;
            if (j >= m) continue;
            const uint32_t k = kk[q];
            const uint32_t py = map[k];
            uint32_t a0 = y, a1 = x, a2 = k;
            sort3(a0, a1, a2);
            uint32_t* tv = A.tv + 3 * (s0 + j);
            __stcs(tv, a0);
            __stcs(tv + 1, a1);
            __stcs(tv + 2, a2);
            if (A.rows) {
                uint32_t* rw = A.rows + 3 * (s0 + j);
                __stcs(rw, min(px[q], py));
                __stcs(rw + 1, max(px[q], py));
                __stcs(rw + 2, p);
            }
            __stcs(A.tf + s0 + j, filt);
            if (A.apex) A.apex[s0 + j] = (uint16_t)k;
        }
    }
}

// Warp: emit the triangles of owner edge p = (y, x) in apex-id order.
//  mark : stream x's older-neighbour prefix (kRegGroups 16-byte groups per
//         lane in flight); every apex k with pos_y[k] < p sets bit krank(k)
//         of the warp's bitmap (shared atomic OR: as cheap as a byte store on
//         B200, measured by tools/micro/smem_atomics.cu)
//  rank : exclusive per-word prefix popcounts
//  emit : stream the prefix again (L1/L2-hot); a valid apex's slot is
//         prefix(word) + popc(word below its bit); stage (k, t) in the window
//  flush: one lane per triangle (flush_window)
// kBits ranks per round (rounds only when deg x > kBits), kWin slots per window.
template <bool kPacked, bool kOneRound>
__device__ __forceinline__ void warp_fill_impl(const TriArgs& A, const uint32_t* __restrict__ map,
                                               WarpScratch* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                               uint32_t len, uint64_t offx, uint32_t degx, uint64_t slot,
                                               uint32_t filt) {
    const int lane = threadIdx.x & 31;
    int mis;
    const uint4* gk = aligned_groups(A.nkr + offx, mis);
    const uint4* gr = kPacked ? nullptr : reinterpret_cast<const uint4*>(A.nr + offx - mis);
    const uint32_t* __restrict__ npx = A.np + offx;
    const int ngroups = (int)((len + mis + 3) >> 2);
    const uint32_t win = kPacked ? (uint32_t)kWin : (uint32_t)kWin / 2;
    for (uint32_t R = 0; R < degx; R += kBits) {
        const uint32_t lim = kOneRound ? degx : min((uint32_t)kBits, degx - R);
        clear_bits(W, lim);
        // ---- mark
        if constexpr (kPacked) {
            auto mark = [&](uint32_t w, uint32_t) {
                const uint32_t r = (w >> 16) - R;
                if ((kOneRound || r < (uint32_t)kBits) && map[w & 0xFFFFu] < p)
                    atomicOr(&W->bits[r >> 5], 1u << (r & 31));
            };
            if (ngroups <= 32) stream_prefix<1>(gk, ngroups, mis, len, mark);
            else stream_prefix<kRegGroups>(gk, ngroups, mis, len, mark);
        } else
        for (int i0 = 0; i0 < ngroups; i0 += 32 * kRegGroups) {
            uint4 qk[kRegGroups], qr[kRegGroups];
#pragma unroll
            for (int u = 0; u < kRegGroups; ++u) {
                const int i = i0 + u * 32 + lane;
                qk[u] = i < ngroups ? ld_list(gk + i) : no_group();
                if (!kPacked) qr[u] = i < ngroups ? __ldg(gr + i) : no_group();
            }
#pragma unroll
            for (int u = 0; u < kRegGroups; ++u) {
                const int i = i0 + u * 32 + lane;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t t = (uint32_t)(4 * i + e - mis);
                    const uint32_t w = pick(qk[u], e);
                    const uint32_t k = kPacked ? (w & 0xFFFFu) : w;
                    const uint32_t r = (kPacked ? (w >> 16) : pick(qr[u], e)) - R;
                    if (t < len && (kOneRound || r < (uint32_t)kBits) && map[k] < p)
                        atomicOr(&W->bits[r >> 5], 1u << (r & 31));
                }
            }
        }
        const uint32_t count = rank_bits<kWords>(W, lim);
        if (A.debug == 1) { slot += count; continue; }
        // ---- emit + flush, one window per pass over the prefix
        for (uint32_t w0 = 0; w0 < count; w0 += win) {
            if constexpr (kPacked) {
                auto emit = [&](uint32_t w, uint32_t t) {
                    const uint32_t r = (w >> 16) - R;
                    if (!kOneRound && r >= (uint32_t)kBits) return;
                    const uint32_t wd = W->bits[r >> 5];
                    if (!((wd >> (r & 31)) & 1u)) return;
                    const uint32_t pos = W->wpre[r >> 5] + __popc(wd & ((2u << (r & 31)) - 1u)) - 1u - w0;
                    if (pos < win) W->rec[pos] = (w & 0xFFFFu) | (t << 16);
                };
                if (ngroups <= 32) stream_prefix<1>(gk, ngroups, mis, len, emit);
                else stream_prefix<kRegGroups>(gk, ngroups, mis, len, emit);
            } else
            for (int i0 = 0; i0 < ngroups; i0 += 32 * kRegGroups) {
                uint4 qk[kRegGroups], qr[kRegGroups];
#pragma unroll
                for (int u = 0; u < kRegGroups; ++u) {
                    const int i = i0 + u * 32 + lane;
                    qk[u] = i < ngroups ? ld_list(gk + i) : no_group();
                    if (!kPacked) qr[u] = i < ngroups ? __ldg(gr + i) : no_group();
                }
#pragma unroll
                for (int u = 0; u < kRegGroups; ++u) {
                    const int i = i0 + u * 32 + lane;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t t = (uint32_t)(4 * i + e - mis);
                        const uint32_t w = pick(qk[u], e);
                        const uint32_t r = (kPacked ? (w >> 16) : pick(qr[u], e)) - R;
                        if (t >= len || (!kOneRound && r >= (uint32_t)kBits)) continue;
                        const uint32_t wd = W->bits[r >> 5];
                        const uint32_t below = wd & ((2u << (r & 31)) - 1u);   // bits <= r
                        if (!((wd >> (r & 31)) & 1u)) continue;
                        const uint32_t pos = W->wpre[r >> 5] + __popc(below) - 1u - w0;
                        if (pos >= win) continue;
                        if (kPacked) {
                            W->rec[pos] = (w & 0xFFFFu) | (t << 16);
                        } else {
                            W->rec[2 * pos] = w;
                            W->rec[2 * pos + 1] = t;
                        }
                    }
                }
            }
            __syncwarp();
            if (A.debug != 2) {
                flush_window<kPacked>(A, map, W, min(win, count - w0), slot + w0, p, y, x, filt, npx);
            }
            __syncwarp();
        }
        slot += count;
        if (kOneRound) break;
    }
}

template <bool kPacked>
__device__ __forceinline__ void warp_fill(const TriArgs& A, const uint32_t* __restrict__ map,
                                          WarpScratch* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                          uint32_t len, uint64_t offx, uint32_t degx, uint64_t slot,
                                          uint32_t filt) {
    if (degx <= (uint32_t)kBits)
        warp_fill_impl<kPacked, true>(A, map, W, p, y, x, len, offx, degx, slot, filt);
    else
        warp_fill_impl<kPacked, false>(A, map, W, p, y, x, len, offx, degx, slot, filt);
}

// Warp: count the apexes of owner edge p (host y's map in smem).
template <bool kPacked>
__device__ __forceinline__ uint32_t warp_count_apexes(const TriArgs& A, const uint32_t* __restrict__ map, uint32_t p,
                                                      uint64_t offx, uint32_t len) {
    int mis;
    const uint4* g = aligned_groups(A.nkr + offx, mis);
    const int ngroups = (int)((len + mis + 3) >> 2);
    uint32_t c = 0;
    auto test = [&](uint32_t w, uint32_t) { c += map[kPacked ? (w & 0xFFFFu) : w] < p; };
    if (ngroups <= 32)
        stream_prefix<1>(g, ngroups, mis, len, test);
    else
        stream_prefix<kRegGroups>(g, ngroups, mis, len, test);
    return __reduce_add_sync(0xffffffffu, c);
}

// (k, pos) fill of owner edge p = (y, x) (packed lists).
//  mark : as warp_fill_impl (bitmap by rank of the valid apexes)
//  emit : re-stream the prefix together with its edge positions (both
//         coalesced 16-byte groups) and stage (k, pos(x, k)) at the apex's slot
//  flush: one lane per triangle, no global gathers: pos(y, k) = map[k]
template <bool kOneRound>
__device__ __forceinline__ void warp_fill_kp(const TriArgs& A, const uint32_t* __restrict__ map,
                                             WarpScratch3* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                             uint32_t len, uint64_t offx, uint32_t degx, uint64_t slot,
                                             uint32_t filt) {
    const int lane = threadIdx.x & 31;
    int mis;
    const uint4* gk = aligned_groups(A.nkr + offx, mis);
    const uint4* gp = reinterpret_cast<const uint4*>(A.np + offx - mis);
    const int ngroups = (int)((len + mis + 3) >> 2);
    for (uint32_t R = 0; R < degx; R += kBits) {
        const uint32_t lim = kOneRound ? degx : min((uint32_t)kBits, degx - R);
        clear_bits(W, lim);
        auto mark = [&](uint32_t w, uint32_t) {
            const uint32_t r = (w >> 16) - R;
            if ((kOneRound || r < (uint32_t)kBits) && map[w & 0xFFFFu] < p)
                atomicOr(&W->bits[r >> 5], 1u << (r & 31));
        };
        if (ngroups <= 32) stream_prefix<1>(gk, ngroups, mis, len, mark);
        else stream_prefix<kRegGroups>(gk, ngroups, mis, len, mark);
        const uint32_t count = rank_bits<kWords>(W, lim);
        if (A.debug == 1) { slot += count; if (kOneRound) break; continue; }
        for (uint32_t w0 = 0; w0 < count; w0 += kWin3) {
            auto emit = [&](uint32_t w, uint32_t px, uint32_t) {
                const uint32_t r = (w >> 16) - R;
                if (!kOneRound && r >= (uint32_t)kBits) return;
                const uint32_t wd = W->bits[r >> 5];
                if (!((wd >> (r & 31)) & 1u)) return;
                const uint32_t pos = W->wpre[r >> 5] + __popc(wd & ((2u << (r & 31)) - 1u)) - 1u - w0;
                if (pos < (uint32_t)kWin3) W->rec[pos] = make_uint2(w & 0xFFFFu, px);
            };
            if (ngroups <= 32) stream_prefix2<1>(gk, gp, ngroups, mis, len, emit);
            else stream_prefix2<2>(gk, gp, ngroups, mis, len, emit);
            __syncwarp();
            const uint32_t m = min((uint32_t)kWin3, count - w0);
            if (A.debug != 2) {
                const uint64_t s0 = slot + w0;
                for (uint32_t j = lane; j < m; j += 32) {
                    const uint2 rc = W->rec[j];
                    const uint32_t k = rc.x, px = rc.y;
                    const uint32_t py = map[k];
                    uint32_t a0 = y, a1 = x, a2 = k;
                    sort3(a0, a1, a2);
                    uint32_t* tv = A.tv + 3 * (s0 + j);
                    __stcs(tv, a0);
                    __stcs(tv + 1, a1);
                    __stcs(tv + 2, a2);
                    if (A.rows) {
                        uint32_t* rw = A.rows + 3 * (s0 + j);
                        __stcs(rw, min(px, py));
                        __stcs(rw + 1, max(px, py));
                        __stcs(rw + 2, p);
                    }
                    __stcs(A.tf + s0 + j, filt);
                    if (A.apex) A.apex[s0 + j] = (uint16_t)k;
                }
            }
            __syncwarp();
        }
        slot += count;
        if (kOneRound) break;
    }
}

// ---------------------------------------------------------------------------
// Apex-bitmap path (single rank, packed lists, degrees <= kApexBitmapMaxDeg).
// The count pass keeps what it computes: per owner edge, the bitmap of its
// valid apexes by rank r in x's id-ordered list (ceil(deg x / 32) words,
// written coalesced).  The fill then never touches the candidates again:
// it loads the bitmap, prefix-popcounts its words, walks the set bits of a
// window of slots (lane owns words lane, lane + 32, ...) staging r, and
// flushes one lane per triangle with (k, pos(x, k)) = idl[off x + r] -- a
// gather in rank order, so a warp's 32 loads fall in a few sectors.
// ---------------------------------------------------------------------------
#ifndef VRB_BATCH_DIV
#define VRB_BATCH_DIV 2
#endif
#ifndef VRB_BATCH_MAX
#define VRB_BATCH_MAX 32
#endif
#ifndef VRB_COUNT_OR0
#define VRB_COUNT_OR0 0
#endif
#ifndef VRB_COUNT_PRED
#define VRB_COUNT_PRED 1
#endif
#ifndef VRB_COUNT_BATCH
#define VRB_COUNT_BATCH 1
#endif
#ifndef VRB_FILL_BATCH
#define VRB_FILL_BATCH 1
#endif
#ifndef VRB_TRI_COUNT_WARPS
#define VRB_TRI_COUNT_WARPS 16
#endif
constexpr int kBmWords = (int)(kApexBitmapMaxDeg / 32);
#ifndef VRB_WINB
#define VRB_WINB 512
#endif
constexpr int kWinB = VRB_WINB;   // slots per window of the bitmap fill
struct WarpScratchC {              // count
    uint32_t bits[kBmWords];
};
#ifndef VRB_FILL_BULK
#define VRB_FILL_BULK 0
#endif
struct WarpScratchB {              // fill: the staged window (apex ranks by slot)
    uint16_t rec[kWinB];
#if VRB_FILL_BULK
    alignas(16) uint32_t st[2][96];   // double-buffered: one bulk copy in flight per buffer
    alignas(16) uint32_t sr[2][96];
#else
    alignas(16) uint32_t st[96];   // 32 triangles' vertices, then D_2 rows: re-cut into
    alignas(16) uint32_t sr[96];   // 16-byte chunks for full-sector vector stores
#endif
};

#if VRB_FILL_BULK
// TMA bulk store (cp.async.bulk shared::cta -> global, one issuing lane):
// the staged 384-byte group leaves shared memory without passing through
// registers; bulk groups are per thread, so lane 0 issues, commits and waits.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
#endif

__device__ __forceinline__ uint32_t warp_count_bm(const TriArgs& A, const uint32_t* __restrict__ map,
                                                  WarpScratchC* __restrict__ W, uint32_t p, uint64_t offx,
                                                  uint32_t len, uint32_t degx, int64_t e) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (degx + 31) >> 5;
    // the bitmap words start at zero (cleared at kernel start, and re-zeroed
    // as they are stored below); the output offset is loaded before the
    // stream so its latency hides behind it
    uint32_t* out = A.bm + __ldg(A.bmoff + e);
    int mis;
    const uint4* g = aligned_groups(A.nkr + offx, mis);
    const int ngroups = (int)((len + mis + 3) >> 2);
#if VRB_COUNT_PRED
    const uint32_t bits_s = (uint32_t)__cvta_generic_to_shared(W->bits);
    // branch-free marking: every lane looks its entry up (entries past the
    // prefix, or of a missing group (word 0, vertex 0), are looked up too and
    // masked out), so the loop carries no divergent branches
    auto run = [&](auto G_) {
        constexpr int G = decltype(G_)::value;
        return [&](int start, int stop) {
            for (int i0 = start; i0 < stop; i0 += 32 * G) {
                uint4 q[G];
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int i = i0 + u * 32 + lane;
                    q[u] = i < ngroups ? ld_list(g + i) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int i = i0 + u * 32 + lane;
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const uint32_t t = (uint32_t)(4 * i + e2 - mis);
                        const uint32_t w = pick(q[u], e2);
                        const uint32_t py = map[w & 0xFFFFu];
                        const uint32_t ok = (uint32_t)(t < len) & (uint32_t)(py < p);
                        const uint32_t addr = bits_s + ((w >> 19) & ~3u);   // word r >> 5 of the bitmap
#if VRB_COUNT_OR0
                        // every lane ORs (a zero when not an apex): no branch at all
                        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"((0u - ok) & (1u << ((w >> 16) & 31u)))
                                     : "memory");
#else
                        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}"
                                     ::"r"(addr), "r"(1u << ((w >> 16) & 31u)), "r"(ok) : "memory");
#endif
                    }
                }
            }
        };
    };
    {
        const int f4 = (ngroups / 128) * 128;
        const int f2 = f4 + ((ngroups - f4) / 64) * 64;
        run(std::integral_constant<int, 4>())(0, f4);
        run(std::integral_constant<int, 2>())(f4, f2);
        run(std::integral_constant<int, 1>())(f2, ngroups);
    }
#else
    auto mark = [&](uint32_t w, uint32_t) {
        if (map[w & 0xFFFFu] < p) {
            const uint32_t r = w >> 16;
            atomicOr(&W->bits[r >> 5], 1u << (r & 31));
        }
    };
    stream_prefix<kRegGroups>(g, ngroups, mis, len, mark);
#endif
    __syncwarp();
    uint32_t c = 0;
    for (uint32_t w = lane; w < nw; w += 32) {
        const uint32_t b = W->bits[w];
        W->bits[w] = 0u;
#ifndef VRB_ABL_NOSTORE
        __stcg(out + w, b);
#endif
        c += __popc(b);
    }
    __syncwarp();
    return __reduce_add_sync(0xffffffffu, c);
}

// known_count: the edge's triangle count when the caller has it (toff), else
// ~0u; a count within one window takes a walk with no window tests
template <bool kSmemBits = false, bool kApex = true>
__device__ __forceinline__ void warp_fill_bm(const TriArgs& A, const uint32_t* __restrict__ map,
                                             WarpScratchB* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                             uint64_t offx, uint32_t degx, uint64_t bmo, uint64_t slot,
                                             uint32_t filt, const uint32_t* smem_bits = nullptr,
                                             uint32_t known_count = ~0u) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (degx + 31) >> 5;
    const uint32_t nchunks = (nw + 31) >> 5;
    const uint32_t* __restrict__ in = kSmemBits ? smem_bits : A.bm + bmo;
    const uint2* __restrict__ idx = A.idl + (A.debug == 3 ? 0 : offx);   // debug 3: ablation, one hot list
    if (known_count == 0) return;
    // Windows of kWinB slots.  Each pass walks the bitmap in chunks of 32
    // words held in registers (lane = word): a warp scan of the popcounts
    // gives every word's first slot, and each lane stages the ranks of its
    // set bits that fall in the window.  The first pass also yields count.
    uint32_t count = 0;
    for (uint32_t w0 = 0; w0 == 0 || w0 < count; w0 += kWinB) {
        const uint32_t w1 = w0 + kWinB;
        const bool one_window = known_count <= (uint32_t)kWinB;
        uint32_t carry = 0;
        for (uint32_t ch = 0; ch < nchunks; ++ch) {
            if (w0 > 0 && carry >= w1) break;
            const uint32_t wd = 32 * ch + lane;
            uint32_t b = wd < nw ? (kSmemBits ? in[wd] : __ldg(in + wd)) : 0u;
            const uint32_t c = __popc(b);
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            uint32_t s = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
            if (one_window) {   // every slot is in the window
                const uint32_t base = 32 * wd;
                while (b) {
                    W->rec[s++] = (uint16_t)(base + (uint32_t)(__ffs(b) - 1));
                    b &= b - 1;
                }
            } else if (s < w1 && s + c > w0) {
                while (b) {
                    const int bit = __ffs(b) - 1;
                    b &= b - 1;
                    if (s >= w0 && s < w1) W->rec[s - w0] = (uint16_t)(32 * wd + bit);
                    ++s;
                }
            }
        }
        if (w0 == 0) count = carry;
        __syncwarp();
        if (count == 0) break;
        const uint32_t m = min((uint32_t)kWinB, count - w0);
        if (A.debug != 2) {
            const uint64_t s0 = slot + w0;
            // the window's output pointers (32-bit offsets from here on)
            uint32_t* __restrict__ const tfw = A.tf + s0;
            uint32_t* __restrict__ const tvw = A.tv + 3 * s0;
            uint32_t* __restrict__ const rww = A.rows ? A.rows + 3 * s0 : nullptr;
            // one triangle: slot j of the window, (k, pos(x, k)) gathered
            const uint32_t vlo = min(x, y), vhi = max(x, y);
            auto tri = [&](uint32_t j, uint2 kp, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& r0,
                           uint32_t& r1) {
                const uint32_t k = kp.x, px = kp.y, py = map[k];
#ifdef VRB_SORT3
                a0 = y; a1 = x; a2 = k;
                sort3(a0, a1, a2);
#else
                // the owner edge's ends are fixed: place the apex among them
                a0 = k < vlo ? k : vlo;
                a1 = k < vlo ? vlo : (k < vhi ? k : vhi);
                a2 = k < vhi ? vhi : k;
#endif
                r0 = min(px, py);
                r1 = max(px, py);
                __stcs(tfw + j, filt);
                if (kApex && A.apex) A.apex[s0 + j] = (uint16_t)k;
            };
            auto scalar = [&](uint32_t j, uint2 kp) {
                uint32_t a0, a1, a2, r0, r1;
                tri(j, kp, a0, a1, a2, r0, r1);
                uint32_t* tv = tvw + 3 * j;
                __stcs(tv, a0);
                __stcs(tv + 1, a1);
                __stcs(tv + 2, a2);
                if (rww) {
                    uint32_t* rw = rww + 3 * j;
                    __stcs(rw, r0);
                    __stcs(rw + 1, r1);
                    __stcs(rw + 2, p);
                }
            };
            // head: slots before the first multiple of 4 (16-byte aligned triples)
            const uint32_t h = min(m, (uint32_t)((4u - (uint32_t)(s0 & 3u)) & 3u));
#if VRB_FILL_BULK
            uint32_t nbulk = 0;
#endif
            if ((uint32_t)lane < h) scalar(lane, ld_idl(idx + W->rec[lane]));
#ifndef VRB_TRI_BM_UNROLL
#define VRB_TRI_BM_UNROLL 8
#endif
            // groups of 32 triangles (384 bytes of vertices, 384 of rows): staged in
            // shared memory and stored as 24 16-byte chunks each -- every L2 sector
            // is written whole by one instruction; kU groups of gathers in flight
            constexpr int kU = VRB_TRI_BM_UNROLL;
            for (uint32_t g0 = h; g0 < m; g0 += 32 * kU) {
                uint2 kq[kU];
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const uint32_t j = g0 + 32 * q + lane;
                    kq[q] = j < m ? ld_idl(idx + W->rec[j]) : make_uint2(0u, 0u);
                }
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const uint32_t g = g0 + 32 * q;
                    if (g >= m) break;
                    const uint32_t j = g + lane;
                    if (g + 32 <= m) {
                        uint32_t a0, a1, a2, r0, r1;
                        tri(j, kq[q], a0, a1, a2, r0, r1);
#if VRB_FILL_BULK
                        // buffer nb was last read by the copy issued two groups ago
                        if (lane == 0 && nbulk >= 2) bulk_wait_read<1>();
                        __syncwarp();
                        uint32_t* st = W->st[nbulk & 1];
                        uint32_t* sr = W->sr[nbulk & 1];
                        st[3 * lane] = a0;
                        st[3 * lane + 1] = a1;
                        st[3 * lane + 2] = a2;
                        sr[3 * lane] = r0;
                        sr[3 * lane + 1] = r1;
                        sr[3 * lane + 2] = p;
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            bulk_s2g(tvw + 3 * g, st, 384u);
                            if (rww) bulk_s2g(rww + 3 * g, sr, 384u);
                            bulk_commit();
                        }
                        ++nbulk;
#else
                        W->st[3 * lane] = a0;
                        W->st[3 * lane + 1] = a1;
                        W->st[3 * lane + 2] = a2;
                        W->sr[3 * lane] = r0;
                        W->sr[3 * lane + 1] = r1;
                        W->sr[3 * lane + 2] = p;
                        __syncwarp();
                        if (lane < 24) {
                            __stcs(reinterpret_cast<uint4*>(tvw + 3 * g) + lane,
                                   reinterpret_cast<const uint4*>(W->st)[lane]);
                            if (rww)
                                __stcs(reinterpret_cast<uint4*>(rww + 3 * g) + lane,
                                       reinterpret_cast<const uint4*>(W->sr)[lane]);
                        }
                        __syncwarp();
#endif
                    } else if (j < m) {
                        scalar(j, kq[q]);
                    }
                }
            }
#if VRB_FILL_BULK
            // the staging buffers are reused by the next window / owner edge
            if (lane == 0 && nbulk) bulk_wait_read<0>();
#endif
        }
        __syncwarp();
    }
}

// Mark-in-fill (mode 4, VRB_TRI_PATH=markfill): the count stores nothing
// but the counts; the fill marks the apex bitmap itself (as the bitmap count
// does) in shared memory, then walks it as warp_fill_bm.
struct WarpScratchM {
    uint32_t bits[kBmWords];
    WarpScratchB b;
};

__device__ __forceinline__ void warp_markfill(const TriArgs& A, const uint32_t* __restrict__ map,
                                              WarpScratchM* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                              uint64_t offx, uint32_t len, uint32_t degx, uint64_t slot,
                                              uint32_t filt) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (degx + 31) >> 5;
    for (uint32_t w = lane; w < nw; w += 32) W->bits[w] = 0u;
    __syncwarp();
    int mis;
    const uint4* g = aligned_groups(A.nkr + offx, mis);
    const int ngroups = (int)((len + mis + 3) >> 2);
    auto mark = [&](uint32_t w, uint32_t) {
        if (map[w & 0xFFFFu] < p) {
            const uint32_t r = w >> 16;
            atomicOr(&W->bits[r >> 5], 1u << (r & 31));
        }
    };
    stream_prefix<kRegGroups>(g, ngroups, mis, len, mark);
    __syncwarp();
    warp_fill_bm<true>(A, map, &W->b, p, y, x, offx, degx, 0, slot, filt, W->bits);
}


// ---------------------------------------------------------------------------
// Position-bitmap path (the default for single-rank-range builds with packed
// lists and degrees <= kApexBitmapMaxDeg).  The count stores, per owner edge,
// one bit per entry t of the scanned prefix (bit t of word t / 32: entry t is
// a valid apex), built by ballots -- 32 candidates per map lookup + vote, no
// shared-memory atomics.  The fill then reads those words, marks the valid
// entries' id ranks (krank, in the packed list word) in a shared bitmap,
// prefix-popcounts it -- the slot of an apex is the number of valid apexes of
// smaller id -- and places (k, pos(x, k)) read from the prefix itself (nkr,
// np: contiguous, coalesced) into a window of slots, flushed as 16-byte
// chunks.  No per-apex gathers from another list.
// ---------------------------------------------------------------------------
constexpr int kWinT = 512;
struct WarpScratchT {              // fill (position bitmaps)
    uint32_t bits[kBmWords];       // valid apexes by id rank in x's list
    uint32_t wpre[kBmWords];       // exclusive prefix popcounts
    uint16_t reck[kWinT];          // staged window: apex ids ...
    uint32_t recp[kWinT];          // ... and pos(x, k)
    alignas(16) uint32_t st[96];
    alignas(16) uint32_t sr[96];
};
struct WarpScratchNone {
    uint32_t unused;
};

__device__ __forceinline__ uint32_t warp_count_tbm(const TriArgs& A, const uint32_t* __restrict__ map, uint32_t p,
                                                   uint64_t offx, uint32_t len, int64_t e) {
    const int lane = threadIdx.x & 31;
    const uint32_t* __restrict__ lst = A.nkr + offx;
    uint32_t* __restrict__ out = A.bm + A.bmoff[e];
    const uint32_t nch = (len + 31) >> 5;
    uint32_t c = 0;
    constexpr int U = 8;
    for (uint32_t c0 = 0; c0 < nch; c0 += U) {
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = 32 * (c0 + u) + lane;
            w[u] = t < len ? ld_list(lst + t) : 0u;
        }
        uint32_t mine = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = 32 * (c0 + u) + lane;
            const bool v = t < len && map[w[u] & 0xFFFFu] < p;
            const uint32_t b = __ballot_sync(0xffffffffu, v);
            if (lane == u) mine = b;
            c += __popc(b);
        }
        if (lane < U && c0 + lane < nch) __stcg(out + c0 + lane, mine);
    }
    return c;
}

// Store slots [0, m) of a window at output slot s0: kp_of(j) = (k, pos(x, k))
// of slot j; pos(y, k) = map[k].  Groups of 32 triangles are staged in shared
// memory and stored as 16-byte chunks (every L2 sector written whole).
template <int kU, class KP>
__device__ __forceinline__ void store_window(const TriArgs& A, const uint32_t* __restrict__ map,
                                             uint32_t* __restrict__ st, uint32_t* __restrict__ sr, uint64_t s0,
                                             uint32_t m, uint32_t p, uint32_t y, uint32_t x, uint32_t filt,
                                             KP&& kp_of) {
    const int lane = threadIdx.x & 31;
    auto tri = [&](uint32_t j, uint2 kp, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& r0, uint32_t& r1) {
        const uint32_t k = kp.x, px = kp.y, py = map[k];
        a0 = y; a1 = x; a2 = k;
        sort3(a0, a1, a2);
        r0 = min(px, py);
        r1 = max(px, py);
        __stcs(A.tf + s0 + j, filt);
        if (A.apex) A.apex[s0 + j] = (uint16_t)k;
    };
    auto scalar = [&](uint32_t j, uint2 kp) {
        uint32_t a0, a1, a2, r0, r1;
        tri(j, kp, a0, a1, a2, r0, r1);
        uint32_t* tv = A.tv + 3 * (s0 + j);
        __stcs(tv, a0);
        __stcs(tv + 1, a1);
        __stcs(tv + 2, a2);
        if (A.rows) {
            uint32_t* rw = A.rows + 3 * (s0 + j);
            __stcs(rw, r0);
            __stcs(rw + 1, r1);
            __stcs(rw + 2, p);
        }
    };
    const uint32_t h = min(m, (uint32_t)((4u - (uint32_t)(s0 & 3u)) & 3u));
    if ((uint32_t)lane < h) scalar(lane, kp_of(lane));
    for (uint32_t g0 = h; g0 < m; g0 += 32 * kU) {
        uint2 kq[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint32_t j = g0 + 32 * q + lane;
            kq[q] = j < m ? kp_of(j) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint32_t g = g0 + 32 * q;
            if (g >= m) break;
            const uint32_t j = g + lane;
            if (g + 32 <= m) {
                uint32_t a0, a1, a2, r0, r1;
                tri(j, kq[q], a0, a1, a2, r0, r1);
                st[3 * lane] = a0;
                st[3 * lane + 1] = a1;
                st[3 * lane + 2] = a2;
                sr[3 * lane] = r0;
                sr[3 * lane + 1] = r1;
                sr[3 * lane + 2] = p;
                __syncwarp();
                if (lane < 24) {
                    __stcs(reinterpret_cast<uint4*>(A.tv + 3 * (s0 + g)) + lane, reinterpret_cast<const uint4*>(st)[lane]);
                    if (A.rows)
                        __stcs(reinterpret_cast<uint4*>(A.rows + 3 * (s0 + g)) + lane,
                               reinterpret_cast<const uint4*>(sr)[lane]);
                }
                __syncwarp();
            } else if (j < m) {
                scalar(j, kq[q]);
            }
        }
    }
}

__device__ __forceinline__ void warp_fill_tbm(const TriArgs& A, const uint32_t* __restrict__ map,
                                              WarpScratchT* __restrict__ W, uint32_t p, uint32_t y, uint32_t x,
                                              uint32_t len, uint64_t offx, uint32_t degx, uint64_t tbo, uint64_t slot,
                                              uint32_t filt) {
    const int lane = threadIdx.x & 31;
    const uint32_t* __restrict__ lk = A.nkr + offx;
    const uint32_t* __restrict__ lp = A.np + offx;
    const uint32_t* __restrict__ tb = A.bm + tbo;
    const uint32_t nch = (len + 31) >> 5;
    const uint32_t nw = (degx + 31) >> 5;
    for (uint32_t w = lane; w < nw; w += 32) W->bits[w] = 0u;
    __syncwarp();
    constexpr int U = 8;
    // ---- mark the id ranks of the valid entries
    for (uint32_t c0 = 0; c0 < nch; c0 += U) {
        const uint32_t wl = (lane < U && c0 + lane < nch) ? __ldg(tb + c0 + lane) : 0u;
        uint32_t ent[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t word = __shfl_sync(0xffffffffu, wl, u);
            ent[u] = ((word >> lane) & 1u) ? ld_list(lk + 32 * (c0 + u) + lane) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (ent[u] != 0xFFFFFFFFu) {
                const uint32_t r = ent[u] >> 16;
                atomicOr(&W->bits[r >> 5], 1u << (r & 31));
            }
    }
    const uint32_t count = rank_bits<kBmWords>(W, degx);
    // ---- windows of kWinT slots: place (k, pos(x, k)) by slot, then store
    for (uint32_t w0 = 0; w0 < count; w0 += kWinT) {
        for (uint32_t c0 = 0; c0 < nch; c0 += U) {
            const uint32_t wl = (lane < U && c0 + lane < nch) ? __ldg(tb + c0 + lane) : 0u;
            uint32_t ent[U], pos[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t word = __shfl_sync(0xffffffffu, wl, u);
                const bool v = (word >> lane) & 1u;
                const uint32_t t = 32 * (c0 + u) + lane;
                ent[u] = v ? ld_list(lk + t) : 0xFFFFFFFFu;
                pos[u] = v ? ld_list(lp + t) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (ent[u] != 0xFFFFFFFFu) {
                    const uint32_t r = ent[u] >> 16;
                    const uint32_t wd = W->bits[r >> 5];
                    const uint32_t sl = W->wpre[r >> 5] + __popc(wd & ((2u << (r & 31)) - 1u)) - 1u - w0;
                    if (sl < (uint32_t)kWinT) {
                        W->reck[sl] = (uint16_t)(ent[u] & 0xFFFFu);
                        W->recp[sl] = pos[u];
                    }
                }
        }
        __syncwarp();
        const uint32_t m = min((uint32_t)kWinT, count - w0);
        store_window<4>(A, map, W->st, W->sr, slot + w0, m, p, y, x, filt,
                        [&](uint32_t j) { return make_uint2(W->reck[j], W->recp[j]); });
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// x-major path ("records"; packed lists, degrees <= kApexBitmapMaxDeg).
//   count (hosted by y, the host map on chip): per owner edge p, x's
//          older-neighbour prefix is streamed as in the bitmap count; each
//          step (32 lanes x one entry of their 16-byte groups) takes one map
//          lookup and one ballot: the ballot word is the step's validity
//          word (stored, 32 per coalesced store) and the valid lanes append
//          the host positions pos(y, k) in step order (a coalesced run per
//          step).  No shared atomics, no per-edge bitmap.
//   fill  (x-major): a CTA holds the scanned vertex x's position-ordered
//          list (krank << 16 | k, pos(x, k)) in shared memory and its warps
//          take x's owner edges.  Per edge: the validity words give the
//          valid prefix entries t in step order (= the records' order); a
//          compaction puts them in a shared arrival list; their id ranks
//          (in the list word) are marked in a shared bitmap and prefix-
//          popcounted -- the slot of an apex is the number of valid apexes
//          of smaller id (the lex order); each arrival is staged at its slot
//          with pos(y, k) read from its record (coalesced), and the staged
//          window is written as whole 16-byte chunks.  No neighbourhood is
//          re-read from DRAM per owner edge: the fill reads 4 B per triangle
//          and a bit per candidate besides writing its 28 B per triangle.
// Step order: chunk c of 32 groups, entry e of the group, lane: step s =
// 4 c + e covers the prefix entries t = 4 (32 c + lane) + e - mis.
// ---------------------------------------------------------------------------
template <int G, class F>
__device__ __forceinline__ void stream_range_s(const uint4* __restrict__ g, int start, int stop, int ngroups, int mis,
                                               uint32_t len, F&& f) {
    const int lane = threadIdx.x & 31;
    for (int i0 = start; i0 < stop; i0 += 32 * G) {
        uint4 q[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
            q[u] = i < ngroups ? ld_list(g + i) : no_group();
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const int i = i0 + u * 32 + lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t t = (uint32_t)(4 * i + e - mis);
                f(pick(q[u], e), t < len);   // every lane calls (ballots inside)
            }
        }
    }
}
template <class F>
__device__ __forceinline__ void stream_prefix_s(const uint4* __restrict__ g, int ngroups, int mis, uint32_t len,
                                                F&& f) {
    const int f4 = (ngroups / 128) * 128;
    const int f2 = f4 + ((ngroups - f4) / 64) * 64;
    stream_range_s<4>(g, 0, f4, ngroups, mis, len, f);
    stream_range_s<2>(g, f4, f2, ngroups, mis, len, f);
    stream_range_s<1>(g, f2, ngroups, ngroups, mis, len, f);
}

__host__ __device__ __forceinline__ uint32_t rec_steps(uint32_t len, uint32_t mis) {
    const uint32_t ngroups = (len + mis + 3) >> 2;
    return 4u * ((ngroups + 31u) >> 5);
}

__device__ __forceinline__ uint32_t warp_count_rec(const TriArgs& A, const uint32_t* __restrict__ map, uint32_t p,
                                                   uint64_t offx, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t* __restrict__ rec = A.rec + __ldg(A.rec_off + p);
    uint32_t* __restrict__ tb = A.tb + __ldg(A.tb_off + p);
    int mis;
    const uint4* g = aligned_groups(A.nkr + offx, mis);
    const int ngroups = (int)((len + mis + 3) >> 2);
    uint32_t na = 0, step = 0, mine = 0;
    stream_prefix_s(g, ngroups, mis, len, [&](uint32_t w, bool in) {
        const uint32_t py = in ? map[w & 0xFFFFu] : NONE32;
        const bool v = py < p;
        const uint32_t b = __ballot_sync(0xffffffffu, v);
        if (v) __stcg(rec + na + __popc(b & lt), py);
        na += __popc(b);
        if ((step & 31u) == (uint32_t)lane) mine = b;
        ++step;
        if ((step & 31u) == 0) __stcg(tb + step - 32 + lane, mine);
    });
    if (step & 31u) {
        if ((uint32_t)lane < (step & 31u)) __stcg(tb + (step & ~31u) + lane, mine);
    }
    return na;
}

#ifndef VRB_XM_WIN
#define VRB_XM_WIN 1024
#endif
constexpr int kWinX = VRB_XM_WIN;   // slots per window of the x-major fill
struct WarpScratchX {
    uint32_t rbits[kBmWords];   // valid apexes by id rank in x's list
    uint32_t wpre[kBmWords];    // exclusive prefix popcount per word
    uint32_t py[kWinX];         // staged: pos(y, k) by slot
    uint16_t cand[kWinX];       // arrival list: prefix index t of the valid entries (record order)
    uint16_t st[kWinX];         // staged: prefix index t by slot
    alignas(16) uint32_t ov[96];   // 32 triangles' vertices, then D_2 rows: 16-byte chunks
    alignas(16) uint32_t orw[96];
};

// every valid entry of the edge in record order: f(t, j) (lane-serial over
// the set bits of lane-owned validity words; j = record index)
template <class F>
__device__ __forceinline__ void walk_valid(const uint32_t* __restrict__ tb, uint32_t nsteps, uint32_t mis, F&& f) {
    const int lane = threadIdx.x & 31;
    uint32_t run = 0;
    for (uint32_t s0 = 0; s0 < nsteps; s0 += 32) {
        const uint32_t s = s0 + lane;
        uint32_t word = s < nsteps ? __ldg(tb + s) : 0u;
        const uint32_t c = __popc(word);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t j = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t tb0 = 4u * 32u * (s >> 2) + (s & 3u) - mis;   // t of bit 0
        while (word) {
            const int b = __ffs(word) - 1;
            word &= word - 1;
            f(tb0 + 4u * (uint32_t)b, j);
            ++j;
        }
    }
}

__device__ __forceinline__ uint32_t xm_slot(const WarpScratchX* __restrict__ W, uint32_t r) {
    return W->wpre[r >> 5] + __popc(W->rbits[r >> 5] & ((1u << (r & 31)) - 1u));
}

// emit the staged window [0, m) at output slots s0 + [0, m)
__device__ __forceinline__ void flush_x(const TriArgs& A, const uint32_t* __restrict__ lk,
                                        const uint32_t* __restrict__ lp, WarpScratchX* __restrict__ W, uint64_t s0,
                                        uint32_t m, uint32_t p, uint32_t y, uint32_t x, uint32_t filt) {
    const int lane = threadIdx.x & 31;
    auto tri = [&](uint32_t j, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& r0, uint32_t& r1) {
        const uint32_t t = W->st[j];
        const uint32_t k = lk[t] & 0xFFFFu, px = lp[t], py = W->py[j];
        a0 = y; a1 = x; a2 = k;
        sort3(a0, a1, a2);
        r0 = min(px, py);
        r1 = max(px, py);
        __stcs(A.tf + s0 + j, filt);
        if (A.apex) A.apex[s0 + j] = (uint16_t)k;
    };
    auto scalar = [&](uint32_t j) {
        uint32_t a0, a1, a2, r0, r1;
        tri(j, a0, a1, a2, r0, r1);
        uint32_t* tv = A.tv + 3 * (s0 + j);
        __stcs(tv, a0);
        __stcs(tv + 1, a1);
        __stcs(tv + 2, a2);
        if (A.rows) {
            uint32_t* rw = A.rows + 3 * (s0 + j);
            __stcs(rw, r0);
            __stcs(rw + 1, r1);
            __stcs(rw + 2, p);
        }
    };
    const uint32_t h = min(m, (uint32_t)((4u - (uint32_t)(s0 & 3u)) & 3u));
    if ((uint32_t)lane < h) scalar(lane);
    for (uint32_t g = h; g < m; g += 32) {
        const uint32_t j = g + lane;
        if (g + 32 <= m) {
            uint32_t a0, a1, a2, r0, r1;
            tri(j, a0, a1, a2, r0, r1);
            W->ov[3 * lane] = a0;
            W->ov[3 * lane + 1] = a1;
            W->ov[3 * lane + 2] = a2;
            W->orw[3 * lane] = r0;
            W->orw[3 * lane + 1] = r1;
            W->orw[3 * lane + 2] = p;
            __syncwarp();
            if (lane < 24) {
                __stcs(reinterpret_cast<uint4*>(A.tv + 3 * (s0 + g)) + lane, reinterpret_cast<const uint4*>(W->ov)[lane]);
                if (A.rows)
                    __stcs(reinterpret_cast<uint4*>(A.rows + 3 * (s0 + g)) + lane,
                           reinterpret_cast<const uint4*>(W->orw)[lane]);
            }
            __syncwarp();
        } else if (j < m) {
            scalar(j);
        }
    }
}

__device__ __forceinline__ void warp_fill_x(const TriArgs& A, const uint32_t* __restrict__ lk,
                                            const uint32_t* __restrict__ lp, WarpScratchX* __restrict__ W, uint32_t p,
                                            uint32_t y, uint32_t x, uint32_t len, uint32_t degx, uint32_t mis,
                                            uint64_t slot, uint32_t count, uint32_t filt) {
    const int lane = threadIdx.x & 31;
    const uint32_t* __restrict__ tb = A.tb + __ldg(A.tb_off + p);
    const uint32_t* __restrict__ rec = A.rec + __ldg(A.rec_off + p);
    const uint32_t nsteps = rec_steps(len, mis);
    const uint32_t nw = (degx + 31) >> 5;
    if (count <= (uint32_t)kWinX) {
        // arrivals -> shared list, then mark, rank, place, flush
        walk_valid(tb, nsteps, mis, [&](uint32_t t, uint32_t j) { W->cand[j] = (uint16_t)t; });
        __syncwarp();
        for (uint32_t j = lane; j < count; j += 32) {
            const uint32_t r = lk[W->cand[j]] >> 16;
            atomicOr(&W->rbits[r >> 5], 1u << (r & 31));
        }
        rank_bits_n(W->rbits, W->wpre, nw);
        for (uint32_t j = lane; j < count; j += 32) {
            const uint32_t t = W->cand[j];
            const uint32_t s = xm_slot(W, lk[t] >> 16);
            W->st[s] = (uint16_t)t;
            W->py[s] = __ldcs(rec + j);
        }
        __syncwarp();
        flush_x(A, lk, lp, W, slot, count, p, y, x, filt);
    } else {
        // more apexes than a window: mark from the validity words, then per
        // window of slots place the arrivals that fall in it
        walk_valid(tb, nsteps, mis, [&](uint32_t t, uint32_t) {
            const uint32_t r = lk[t] >> 16;
            atomicOr(&W->rbits[r >> 5], 1u << (r & 31));
        });
        rank_bits_n(W->rbits, W->wpre, nw);
        for (uint32_t w0 = 0; w0 < count; w0 += kWinX) {
            walk_valid(tb, nsteps, mis, [&](uint32_t t, uint32_t j) {
                const uint32_t s = xm_slot(W, lk[t] >> 16) - w0;
                if (s < (uint32_t)kWinX) {
                    W->st[s] = (uint16_t)t;
                    W->py[s] = __ldg(rec + j);
                }
            });
            __syncwarp();
            flush_x(A, lk, lp, W, slot + w0, min((uint32_t)kWinX, count - w0), p, y, x, filt);
            __syncwarp();
        }
    }
    __syncwarp();
    for (uint32_t w = lane; w < nw; w += 32) W->rbits[w] = 0u;
    __syncwarp();
}

// The x-major fill: CTAs take tasks (work-balanced ranges of fill-plan slots),
// each slot range grouped by scanned vertex x; per x the CTA loads x's
// position-ordered list into shared memory once and its warps take x's owner
// edges (the next edge's validity words and records are prefetched to L2).
__global__ void __launch_bounds__(512, 1) k_tri_fill_x(TriArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* lk = reinterpret_cast<uint32_t*>(smem);
    uint32_t* lp = lk + A.lists_cap;
    WarpScratchX* scratch = reinterpret_cast<WarpScratchX*>(smem + (size_t)8 * A.lists_cap);
    __shared__ int64_t s_lo, s_hi, s_end;
    __shared__ uint32_t s_x;
    __shared__ unsigned s_next;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nthreads = blockDim.x;
    for (int q = lane; q < kBmWords; q += 32) scratch[wid].rbits[q] = 0u;
    for (;;) {
        if (threadIdx.x == 0) {
            const int64_t task = A.task_lo + (int64_t)atomicAdd(A.task_counter, 1ull);
            if (task >= A.task_hi) {
                s_lo = s_hi = -1;
            } else {
                s_lo = lower_bound_u64(A.work_pre, 0, A.E + 1, (uint64_t)task * A.chunk);
                s_hi = task == A.ntasks - 1 ? A.E
                                            : lower_bound_u64(A.work_pre, 0, A.E + 1, (uint64_t)(task + 1) * A.chunk);
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
                const uint32_t x = A.fgroup_v[seg];
                s_x = x;
                s_end = upper_bound_u32(A.fgroup_v, seg, hi, x);
                s_next = 0;
            }
            __syncthreads();
            const uint32_t x = s_x;
            const int64_t end = s_end;
            const uint64_t ox = A.off[x];
            const uint32_t degx = (uint32_t)(A.off[x + 1] - ox);
            const uint32_t mis = (uint32_t)(ox & 3u);   // the lists are 16-byte aligned
            for (uint32_t t = threadIdx.x; t < degx; t += nthreads) {
                lk[t] = A.nkr[ox + t];
                lp[t] = A.np[ox + t];
            }
            __syncthreads();
            auto grab = [&]() -> int64_t {
                unsigned my = 0;
                if (lane == 0) my = atomicAdd(&s_next, 1u);
                return seg + (int64_t)__shfl_sync(0xffffffffu, my, 0);
            };
            // software pipeline over x's owner edges: plans three ahead, the
            // per-edge offsets two ahead, the L2 prefetch of the validity
            // words and records one ahead of the edge being filled
            struct Meta {
                uint64_t t0, tbo, reco;
                uint32_t count, filt;
            };
            auto plan_of = [&](int64_t e) -> uint4 {
                uint4 pl = e < end ? A.fplan[e] : make_uint4(0, 0, 0, 0);
                if ((int64_t)pl.x < A.p_lo || (int64_t)pl.x >= A.p_hi) pl.z = 0;
                return pl;
            };
            auto meta_of = [&](const uint4& pl) -> Meta {
                Meta m{0, 0, 0, 0, 0};
                if (pl.z) {
                    m.t0 = A.toff[pl.x];
                    m.count = (uint32_t)(A.toff[pl.x + 1] - m.t0);
                    m.filt = A.efilt[pl.x];
                    m.tbo = A.tb_off[pl.x];
                    m.reco = A.rec_off[pl.x];
                }
                return m;
            };
            auto prefetch = [&](const uint4& pl, const Meta& m) {
                if (!pl.z || !m.count) return;
                const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.tb + m.tbo) & ~(uintptr_t)127;
                const uintptr_t a1 = reinterpret_cast<uintptr_t>(A.tb + m.tbo + rec_steps(pl.z, mis));
                for (uintptr_t a = a0 + 128 * (uintptr_t)lane; a < a1; a += 128 * 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                const uintptr_t b0 = reinterpret_cast<uintptr_t>(A.rec + m.reco) & ~(uintptr_t)127;
                const uintptr_t b1 = reinterpret_cast<uintptr_t>(A.rec + m.reco + m.count);
                for (uintptr_t a = b0 + 128 * (uintptr_t)lane; a < b1; a += 128 * 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
            };
            int64_t e0 = grab();
            uint4 pl0 = plan_of(e0);
            int64_t e1 = grab();
            uint4 pl1 = plan_of(e1);
            int64_t e2 = grab();
            uint4 pl2 = plan_of(e2);
            Meta m0 = meta_of(pl0), m1 = meta_of(pl1);
            prefetch(pl0, m0);
            while (e0 < end) {
                const int64_t e3 = grab();
                const uint4 pl3 = plan_of(e3);
                const Meta m2 = meta_of(pl2);
                prefetch(pl1, m1);
                if (pl0.z && m0.count)
                    warp_fill_x(A, lk, lp, scratch + wid, pl0.x, pl0.y, x, pl0.z, degx, mis, m0.t0 - A.slot0,
                                m0.count, m0.filt);
                e0 = e1; pl0 = pl1; m0 = m1;
                e1 = e2; pl1 = pl2; m1 = m2;
                e2 = e3; pl2 = pl3;
            }
            __syncthreads();
            seg = end;
        }
    }
}

// kGmap: the host map is a per-CTA slice of global memory (large n); else it
// is in shared memory, and the compile-time choice lets every map lookup be
// an LDS with a 32-bit address instead of a generic 64-bit load
template <bool kFill, bool kPacked, int kBm, bool kGmap>
__global__ void __launch_bounds__(kFill ? kThreads : (kBm ? VRB_TRI_COUNT_WARPS * 32 : kThreads / 2),
                                   (!kFill && kBm == 3) ? 2 : 1) k_triangles(TriArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* map = kGmap ? A.gmap + (size_t)blockIdx.x * (size_t)A.n : reinterpret_cast<uint32_t*>(smem);
    using WS = typename std::conditional<
        kBm == 4, WarpScratchM,
        typename std::conditional<
        kBm >= 2, typename std::conditional<kFill, WarpScratchT, WarpScratchNone>::type,
        typename std::conditional<
            kBm == 1, typename std::conditional<kFill, WarpScratchB, WarpScratchC>::type,
            typename std::conditional<kPacked && VRB_TRI_MODE == 3, WarpScratch3, WarpScratch>::type>::type>::type>::type;
    WS* scratch = reinterpret_cast<WS*>(smem + (kGmap ? 0 : ((A.n * 4 + 15) / 16) * 16));
    __shared__ int64_t s_lo, s_hi, s_end;
    __shared__ uint32_t s_y;
    __shared__ unsigned s_next;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nthreads = blockDim.x;
    for (int64_t q = threadIdx.x; q < A.n; q += nthreads) map[q] = NONE32;
    if ((kFill && !kBm) || (!kFill && kBm == 1))   // cleared after every use, so they must start at 0
        for (int q = threadIdx.x; q < (int)((nthreads / 32) * sizeof(WS) / 4); q += nthreads)
            reinterpret_cast<uint32_t*>(scratch)[q] = 0u;
    __syncthreads();
    const uint32_t kmask = kPacked ? 0xFFFFu : 0xFFFFFFFFu;
    for (;;) {
        if (threadIdx.x == 0) {
            const int64_t task = A.task_lo + (int64_t)atomicAdd(A.task_counter, 1ull);
            if (task >= A.task_hi) {
                s_lo = s_hi = -1;
            } else {
                s_lo = lower_bound_u64(A.work_pre, 0, A.E + 1, (uint64_t)task * A.chunk);
                s_hi = task == A.ntasks - 1 ? A.E
                                            : lower_bound_u64(A.work_pre, 0, A.E + 1, (uint64_t)(task + 1) * A.chunk);
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
                s_end = upper_bound_u32(A.hosted_v, seg, hi, y);
                s_next = 0;
            }
            __syncthreads();
            const uint32_t y = s_y;
            const int64_t end = s_end;
            const uint64_t oy = A.off[y], oy1 = A.off[y + 1];
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = A.np[t];
            __syncthreads();
#if VRB_COUNT_BATCH
            if constexpr (kBm == 1 && !kFill) {
                // the bitmap count in batches (as the bitmap fill below)
                const int nwarps = nthreads >> 5;
                for (;;) {
                    unsigned my = 0, bb = 0;
                    if (lane == 0) {
                        const int64_t rem = end - seg - (int64_t)*(volatile unsigned*)&s_next;
                        const int64_t want = rem / (VRB_BATCH_DIV * nwarps);
                        bb = want < 1 ? 1u : (want > VRB_BATCH_MAX ? (unsigned)VRB_BATCH_MAX : (unsigned)want);
                        my = atomicAdd(&s_next, bb);
                    }
                    my = __shfl_sync(0xffffffffu, my, 0);
                    bb = __shfl_sync(0xffffffffu, bb, 0);
                    const int64_t eb = seg + (int64_t)my;
                    if (eb >= end) break;
                    const int nb = (int)(end - eb < (int64_t)bb ? end - eb : (int64_t)bb);
                    uint4 pl = make_uint4(0, 0, 0, 0);
                    uint64_t offx = 0;
                    if (lane < nb) {
                        pl = A.plan[eb + lane];
                        if (pl.z) offx = A.off[pl.y];
                    }
                    for (int i = 0; i < nb; ++i) {
                        const uint32_t len = __shfl_sync(0xffffffffu, pl.z, i);
                        if (!len) continue;
                        const uint32_t p = __shfl_sync(0xffffffffu, pl.x, i), degx = __shfl_sync(0xffffffffu, pl.w, i);
                        const uint64_t oi = __shfl_sync(0xffffffffu, offx, i);
                        const uint32_t c = warp_count_bm(A, map, scratch + wid, p, oi, len, degx, eb + i);
                        if (lane == 0) A.cnt[p] = c;
                    }
                }
                __syncthreads();
                for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = NONE32;
                __syncthreads();
                seg = end;
                continue;
            }
#endif
#if VRB_FILL_BATCH
            if constexpr (kBm == 1 && kFill) {
                // The bitmap fill takes the host's edges in batches (up to 32,
                // shrinking with what is left so the warps stay balanced): one
                // shared atomic per batch, the batch's plans, offsets, counts
                // and bitmap offsets loaded lane-parallel, the batch's bitmaps
                // prefetched to L2 together; the edges then run one by one
                // with their parameters broadcast from the lanes.
                const int nwarps = nthreads >> 5;
                for (;;) {
                    unsigned my = 0, bb = 0;
                    if (lane == 0) {
                        const int64_t rem = end - seg - (int64_t)*(volatile unsigned*)&s_next;
                        const int64_t want = rem / (VRB_BATCH_DIV * nwarps);
                        bb = want < 1 ? 1u : (want > VRB_BATCH_MAX ? (unsigned)VRB_BATCH_MAX : (unsigned)want);
                        my = atomicAdd(&s_next, bb);
                    }
                    my = __shfl_sync(0xffffffffu, my, 0);
                    bb = __shfl_sync(0xffffffffu, bb, 0);
                    const int64_t eb = seg + (int64_t)my;
                    if (eb >= end) break;
                    const int nb = (int)(end - eb < (int64_t)bb ? end - eb : (int64_t)bb);
                    uint4 pl = make_uint4(0, 0, 0, 0);
                    uint64_t offx = 0, slot = 0, bmo = 0;
                    uint32_t filt = 0, tc = 0;
                    if (lane < nb) {
                        pl = A.plan[eb + lane];
                        if ((int64_t)pl.x < A.p_lo || (int64_t)pl.x >= A.p_hi) pl.z = 0;
                        if (pl.z) {
                            offx = A.off[pl.y];
                            const uint64_t t0 = A.toff[pl.x];
                            slot = t0 - A.slot0;
                            tc = (uint32_t)(A.toff[pl.x + 1] - t0);
                            filt = A.efilt[pl.x];
                            bmo = A.bmoff[eb + lane];
                        }
                        if (pl.z && tc) {
                            const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.bm + bmo) & ~(uintptr_t)127;
                            const uintptr_t a1 = reinterpret_cast<uintptr_t>(A.bm + bmo + ((pl.w + 31) >> 5));
                            for (uintptr_t a = a0; a < a1; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                        }
                    }
                    for (int i = 0; i < nb; ++i) {
                        const uint32_t len = __shfl_sync(0xffffffffu, pl.z, i);
                        const uint32_t tci = __shfl_sync(0xffffffffu, tc, i);
                        if (!len || !tci) continue;
                        const uint32_t p = __shfl_sync(0xffffffffu, pl.x, i), x = __shfl_sync(0xffffffffu, pl.y, i),
                                       degx = __shfl_sync(0xffffffffu, pl.w, i),
                                       fi = __shfl_sync(0xffffffffu, filt, i);
                        const uint64_t oi = __shfl_sync(0xffffffffu, offx, i), si = __shfl_sync(0xffffffffu, slot, i),
                                       bi = __shfl_sync(0xffffffffu, bmo, i);
                        if (A.apex)
                            warp_fill_bm<false, true>(A, map, scratch + wid, p, y, x, oi, degx, bi, si, fi, nullptr,
                                                      tci);
                        else
                            warp_fill_bm<false, false>(A, map, scratch + wid, p, y, x, oi, degx, bi, si, fi, nullptr,
                                                       tci);
                    }
                }
                __syncthreads();
                for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = NONE32;
                __syncthreads();
                seg = end;
                continue;
            }
#endif
            // Edges of this host, longest prefix first, grabbed dynamically and
            // software-pipelined two deep: while edge e0 is processed, the
            // plan of e2 and the offsets of e1 are in flight.
            auto grab = [&]() -> int64_t {
                unsigned my = 0;
                if (lane == 0) my = atomicAdd(&s_next, 1u);
                return seg + (int64_t)__shfl_sync(0xffffffffu, my, 0);
            };
            auto plan_of = [&](int64_t e) -> uint4 {
                uint4 pl = e < end ? A.plan[e] : make_uint4(0, 0, 0, 0);
                if (kFill && ((int64_t)pl.x < A.p_lo || (int64_t)pl.x >= A.p_hi)) pl.z = 0;
                return pl;
            };
            int64_t e0 = grab();
            uint4 pl0 = plan_of(e0);
            int64_t e1 = grab();
            uint4 pl1 = plan_of(e1);
            uint64_t off0 = pl0.z ? A.off[pl0.y] : 0, off1 = pl1.z ? A.off[pl1.y] : 0;
            uint64_t slot0 = 0, slot1 = 0;
            uint32_t filt0 = 0, filt1 = 0;
            uint32_t tc0 = 0, tc1 = 0;     // the pipelined edges' triangle counts
            uint64_t bmo0 = 0, bmo1 = 0;   // bitmap fill: word offsets of the pipelined edges' bitmaps
            if (kFill) {
                if (pl0.z) {
                    slot0 = A.toff[pl0.x] - A.slot0;
                    tc0 = (uint32_t)(A.toff[pl0.x + 1] - A.toff[pl0.x]);
                    filt0 = A.efilt[pl0.x];
                }
                if (pl1.z) {
                    slot1 = A.toff[pl1.x] - A.slot0;
                    tc1 = (uint32_t)(A.toff[pl1.x + 1] - A.toff[pl1.x]);
                    filt1 = A.efilt[pl1.x];
                }
                if (kBm && kBm != 4) {
                    if (pl0.z) bmo0 = A.bmoff[e0];
                    if (pl1.z) bmo1 = A.bmoff[e1];
                }
            }
            while (e0 < end) {
                const int64_t e2 = grab();
                const uint4 pl2 = plan_of(e2);
                if (kBm && kBm != 4 && kFill && pl1.z && (kBm != 1 || tc1)) {
                    // pull the next edge's bitmap into L2 while this edge runs
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.bm + bmo1) & ~(uintptr_t)127;
                    const uintptr_t a1 =
                        reinterpret_cast<uintptr_t>(A.bm + bmo1 + (((kBm == 2 ? pl1.z : pl1.w) + 31) >> 5));
                    for (uintptr_t a = a0 + 128 * (uintptr_t)lane; a < a1; a += 128 * 32)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                }
                if (pl0.z) {
                    const uint32_t p = pl0.x, x = pl0.y, len = pl0.z;
                    if constexpr (kBm == 4 && kFill) {
                        warp_markfill(A, map, scratch + wid, p, y, x, off0, len, pl0.w, slot0, filt0);
                    } else if constexpr (kBm == 3 && !kFill) {
                        const uint32_t c = warp_count_rec(A, map, p, off0, len);
                        if (lane == 0) A.cnt[p] = c;
                    } else if constexpr (kBm == 2 && kFill) {
                        warp_fill_tbm(A, map, scratch + wid, p, y, x, len, off0, pl0.w, bmo0, slot0, filt0);
                    } else if constexpr (kBm == 2) {
                        const uint32_t c = warp_count_tbm(A, map, p, off0, len, e0);
                        if (lane == 0) A.cnt[p] = c;
                    } else if constexpr (kBm && kFill) {
                        if (A.apex)
                            warp_fill_bm<false, true>(A, map, scratch + wid, p, y, x, off0, pl0.w, bmo0, slot0,
                                                      filt0, nullptr, tc0);
                        else
                            warp_fill_bm<false, false>(A, map, scratch + wid, p, y, x, off0, pl0.w, bmo0, slot0,
                                                       filt0, nullptr, tc0);
                    } else if constexpr (kBm) {
                        const uint32_t c = warp_count_bm(A, map, scratch + wid, p, off0, len, pl0.w, e0);
                        if (lane == 0) A.cnt[p] = c;
                    } else if constexpr (kFill && kPacked && VRB_TRI_MODE == 3) {
                        if (pl0.w <= (uint32_t)kBits)
                            warp_fill_kp<true>(A, map, scratch + wid, p, y, x, len, off0, pl0.w, slot0, filt0);
                        else
                            warp_fill_kp<false>(A, map, scratch + wid, p, y, x, len, off0, pl0.w, slot0, filt0);
                    } else if constexpr (kFill && kPacked) {
                        warp_fill<true>(A, map, scratch + wid, p, y, x, len, off0, pl0.w, slot0, filt0);
                    } else if constexpr (kFill) {
                        warp_fill<false>(A, map, scratch + wid, p, y, x, len, off0, pl0.w, slot0, filt0);
                    } else {
                        const uint32_t c = warp_count_apexes<kPacked>(A, map, p, off0, len);
                        if (lane == 0) A.cnt[p] = c;
                    }
                }
                uint64_t off2 = pl2.z ? A.off[pl2.y] : 0, slot2 = 0, bmo2 = 0;
                uint32_t filt2 = 0, tc2 = 0;
                if (kFill && pl2.z) {
                    slot2 = A.toff[pl2.x] - A.slot0;
                    tc2 = (uint32_t)(A.toff[pl2.x + 1] - A.toff[pl2.x]);
                    filt2 = A.efilt[pl2.x];
                    if (kBm && kBm != 4) bmo2 = A.bmoff[e2];
                }
                e0 = e1; pl0 = pl1; off0 = off1; slot0 = slot1; filt0 = filt1; bmo0 = bmo1; tc0 = tc1;
                e1 = e2; pl1 = pl2; off1 = off2; slot1 = slot2; filt1 = filt2; bmo1 = bmo2; tc1 = tc2;
            }
            __syncthreads();
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += nthreads) map[A.nkr[t] & kmask] = NONE32;
            __syncthreads();
            seg = end;
        }
    }
}

size_t map_bytes(int64_t n) { return (size_t)((n * 4 + 15) / 16) * 16; }

size_t scratch_bytes(bool packed) {
    return packed && VRB_TRI_MODE == 3 ? sizeof(WarpScratch3) : sizeof(WarpScratch);
}

template <bool kFill, bool kPacked, int kBm, bool kGmap>
void launch_kg(TriArgs A, int threads, size_t smem, int64_t nctas_cap, cudaStream_t s) {
    VRB_CUDA(cudaFuncSetAttribute(k_triangles<kFill, kPacked, kBm, kGmap>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_triangles<kFill, kPacked, kBm, kGmap>, threads,
                                                           smem));
    if (per_sm < 1) fail(VRB_ENOTSUP, "triangle kernel does not fit (n = %lld)", (long long)A.n);
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)device_sm_count() * per_sm, nctas_cap);
    DBuf<uint32_t> maps;
    if (kGmap) {   // one n-entry host map per CTA in global memory (L2-resident for moderate n)
        maps.alloc((size_t)grid * (size_t)A.n, s);
        A.gmap = maps.get();
    } else {
        A.gmap = nullptr;
    }
    k_triangles<kFill, kPacked, kBm, kGmap><<<grid, threads, smem, s>>>(A);
    VRB_LAUNCH_CHECK();
}

template <bool kFill, bool kPacked, int kBm>
void launch_k(TriArgs A, int threads, size_t smem, int64_t nctas_cap, bool gmap, cudaStream_t s) {
    if (gmap)
        launch_kg<kFill, kPacked, kBm, true>(A, threads, smem, nctas_cap, s);
    else
        launch_kg<kFill, kPacked, kBm, false>(A, threads, smem, nctas_cap, s);
}

void launch(const TriArgs& base, bool fill, uint64_t work, int part, int nparts, cudaStream_t s) {
    TriArgs A = base;
    const bool packed = A.packed != 0;
    const bool markfill = fill && A.bm_mode == 4;   // mark-in-fill (no stored bitmaps)
    const bool recm = A.rec != nullptr;   // x-major path: the count stores records
    const bool bm = A.bm != nullptr || recm;
    const bool tbm = (A.bm != nullptr && A.bm_mode == 2) || recm;
    // fill: one CTA per SM (the vertex map + per-warp scratch); count:
    // 16-warp CTAs, two per SM (shorter per-host barrier tails)
    // the host map goes to global memory when it would leave shared memory for
    // fewer than 8 warps of scratch (n above ~40-50k), or when forced (tests)
    size_t per_warp = markfill ? sizeof(WarpScratchM)
                    : tbm ? (fill ? sizeof(WarpScratchT) : sizeof(WarpScratchNone))
                          : bm ? (fill ? sizeof(WarpScratchB) : sizeof(WarpScratchC)) : (fill ? scratch_bytes(packed) : 0);
    const char* fg = std::getenv("VRB_FORCE_GLOBAL_MAP");   // testing knob
    const bool gmap = (fg && fg[0] == '1') ||
                      (int64_t)map_bytes(A.n) + 8 * (int64_t)std::max<size_t>(per_warp, 64) + 1024 >
                          (int64_t)device_max_smem_optin();
    const size_t mapb = gmap ? 0 : map_bytes(A.n);
    const int64_t avail = (int64_t)device_max_smem_optin() - (int64_t)mapb - 1024;
    int warps;
    if (bm || markfill) {
        // count: 16-warp CTAs, 8 when the vertex map is small (more CTAs per SM)
        const int cw = mapb <= 32768 ? VRB_TRI_COUNT_WARPS / 2 : VRB_TRI_COUNT_WARPS;
        // fill: 32-warp CTAs (one per SM) when the host map is large (C5B:
        // 16 / 8 warps 27.4 / 28.2 ms against 22.5), 8-warp CTAs when it is
        // small (C3, 8 KB map: 8.9 ms against 9.9); VRB_TRI_FILL_WARPS overrides
        const char* fw = std::getenv("VRB_TRI_FILL_WARPS");
        const int fill_warps = fw ? std::max(4, std::min(kWarps, std::atoi(fw))) : ((!gmap && mapb <= 32768) ? 8 : kWarps);
        warps = (int)std::min<int64_t>(fill ? fill_warps : cw, avail / (int64_t)per_warp);
    } else if (fill) {
        warps = (int)std::min<int64_t>(kWarps, avail / (int64_t)per_warp);
    } else {
        warps = kWarps / 2;
    }
    if (warps < 4) fail(VRB_ENOTSUP, "triangle kernel: n = %lld leaves no shared memory", (long long)A.n);
    const int threads = warps * 32;
    const size_t smem = mapb + (size_t)warps * per_warp;
    // Task size depends on the work only (identical on every rank, so a
    // partition of the task range is a partition of the owner edges):
    // ~8k tasks, but not below ~64k candidate tests each.
    uint64_t chunk = work / 8192 + 1;
    if (chunk < 65536) chunk = 65536;
    A.chunk = chunk;
    A.ntasks = (int64_t)((work + chunk - 1) / chunk);
    if (A.ntasks < 1) A.ntasks = 1;
    A.task_lo = A.ntasks * part / nparts;
    A.task_hi = A.ntasks * (part + 1) / nparts;
    if (A.task_lo >= A.task_hi) return;
    DBuf<unsigned long long> counter(1, s);
    VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned long long), s));
    A.task_counter = counter.get();
    const int64_t cap = A.task_hi - A.task_lo;
    if (markfill) {
        launch_k<true, true, 4>(A, threads, smem, cap, gmap, s);
    } else if (recm) {
        launch_k<false, true, 3>(A, threads, smem, cap, gmap, s);
    } else if (tbm) {
        if (fill) launch_k<true, true, 2>(A, threads, smem, cap, gmap, s);
        else launch_k<false, true, 2>(A, threads, smem, cap, gmap, s);
    } else if (bm) {
        if (fill) launch_k<true, true, 1>(A, threads, smem, cap, gmap, s);
        else launch_k<false, true, 1>(A, threads, smem, cap, gmap, s);
    } else if (fill) {
        if (packed) launch_k<true, true, 0>(A, threads, smem, cap, gmap, s);
        else launch_k<true, false, 0>(A, threads, smem, cap, gmap, s);
    } else {
        if (packed) launch_k<false, true, 0>(A, threads, smem, cap, gmap, s);
        else launch_k<false, false, 0>(A, threads, smem, cap, gmap, s);
    }
}

__global__ void k_bm_words(const uint4* __restrict__ plan, int64_t E, int mode, uint32_t* __restrict__ words) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        words[e] = ((mode == 2 ? plan[e].z : plan[e].w) + 31u) >> 5;
}

// 1 = id-rank bitmaps (default), 2 = position bitmaps (VRB_TRI_BITMAPS=pos:
// an experiment, measured slower on C5B -- count 8.4 ms instead of 9.3, fill
// 34.0 ms instead of 22.6 -- DESIGN.md section 10)
int bitmap_mode() {
    const char* m = std::getenv("VRB_TRI_BITMAPS");
    return (m && m[0] == 'p') ? 2 : 1;
}

TriArgs graph_args(const Graph& g) {
    TriArgs A{};
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
    return A;
}

}  // namespace


void count_triangles(const Graph& g, uint32_t* cnt, int part, int nparts, cudaStream_t s) {
    if (g.E == 0) return;
    VRB_CUDA(cudaMemsetAsync(cnt, 0, g.E * sizeof(uint32_t), s));
    if (g.work == 0) return;
    TriArgs A = graph_args(g);
    A.cnt = cnt;
    launch(A, false, g.work, part, nparts, s);
}

// mark-in-fill (VRB_TRI_PATH=markfill): packed lists, degrees <= 8192, no
// stored bitmaps (build_impl then runs the plain count)
bool markfill_apply(const Graph& g) {
    const char* m = std::getenv("VRB_TRI_PATH");
    return g.packed && g.idl.get() && g.max_deg <= kApexBitmapMaxDeg && m && m[0] == 'm';
}

bool apex_bitmaps_apply(const Graph& g) {
    const char* off = std::getenv("VRB_NO_APEX_BITMAPS");   // testing knob: force the re-enumerating fill
    return g.packed && g.idl.get() && g.max_deg <= kApexBitmapMaxDeg && !(off && off[0] == '1') &&
           !markfill_apply(g);
}

void apex_bitmap_offsets(const Graph& g, DBuf<uint64_t>& bmoff, uint64_t& words, cudaStream_t s) {
    const int64_t m = g.nplan;
    bmoff.alloc(m + 1, s);
    words = 0;
    if (m == 0) {
        VRB_CUDA(cudaMemsetAsync(bmoff.get(), 0, sizeof(uint64_t), s));
        return;
    }
    DBuf<uint32_t> w(m, s);
    k_bm_words<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), (int64_t)device_sm_count() * 16), 256, 0, s>>>(
        g.plan.get(), m, bitmap_mode(), w.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(w.get(), bmoff.get(), m, s);
    VRB_CUDA(cudaMemcpyAsync(&words, bmoff.get() + m, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
}

void count_triangles_bm(const Graph& g, uint32_t* cnt, uint32_t* bm, const uint64_t* bmoff, cudaStream_t s) {
    if (g.E == 0) return;
    VRB_CUDA(cudaMemsetAsync(cnt, 0, g.E * sizeof(uint32_t), s));
    if (g.work == 0) return;
    TriArgs A = graph_args(g);
    A.cnt = cnt;
    A.bm = bm;
    A.bm_mode = bitmap_mode();
    A.bmoff = bmoff;
    launch(A, false, g.work, 0, 1, s);
}

namespace {
__global__ void k_rec_words(const uint32_t* __restrict__ scan_len, const uint32_t* __restrict__ scan_v,
                            const uint64_t* __restrict__ off, int64_t E, int64_t p_lo, int64_t p_hi,
                            uint32_t* __restrict__ nrec, uint32_t* __restrict__ nwords) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t len = (p >= p_lo && p < p_hi) ? scan_len[p] : 0u;
        nrec[p] = len;   // capacity: a record per candidate at most
        nwords[p] = len ? rec_steps(len, (uint32_t)(off[scan_v[p]] & 3u)) : 0u;
    }
}
}  // namespace

// The x-major path is an experiment (VRB_TRI_PATH=xmajor): correct, but
// measured slower than the apex-bitmap path on C5B (round 2, second version:
// ballot-compacted records, arrival lists, a 3-deep software pipeline and L2
// prefetch in the fill -- count 12.6 ms against 9.0, fill 30.0 against 22.5;
// C3 fill 30.6 against 8.9, most of its edges exceeding a 1024-slot window).
// Both fills are bound by per-owner-edge work (ncu: 14.0e9 instructions for
// 9.7e6 edges and 2.0e9 triangles), not by the gathers the x-major layout
// removes.
bool records_apply(const Graph& g) {
    const char* m = std::getenv("VRB_TRI_PATH");
    return g.packed && g.idl.get() && g.max_deg <= kApexBitmapMaxDeg && m && m[0] == 'x';
}

void count_triangles_rec(const Graph& g, const uint32_t* ev, int64_t p_lo, int64_t p_hi, uint32_t* cnt,
                         TriRecords& R, cudaStream_t s) {
    const int64_t E = g.E;
    if (E == 0) return;
    VRB_CUDA(cudaMemsetAsync(cnt, 0, E * sizeof(uint32_t), s));
    R.rec_off.alloc(E + 1, s);
    R.tb_off.alloc(E + 1, s);
    {
        DBuf<uint32_t> a(E, s), b(E, s);
        k_rec_words<<<(unsigned)std::min<int64_t>(ceil_div(E, 256), (int64_t)device_sm_count() * 16), 256, 0, s>>>(
            g.scan_len.get(), g.scan_v.get(), g.off.get(), E, p_lo, p_hi, a.get(), b.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(a.get(), R.rec_off.get(), E, s);
        exclusive_scan(b.get(), R.tb_off.get(), E, s);
    }
    uint64_t nrec = 0, nw = 0;
    VRB_CUDA(cudaMemcpyAsync(&nrec, R.rec_off.get() + E, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaMemcpyAsync(&nw, R.tb_off.get() + E, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    R.rec.alloc(std::max<uint64_t>(nrec, 1), s);   // a slot per candidate (only the valid ones are written)
    R.tb.alloc(std::max<uint64_t>(nw, 1), s);
    build_fill_plan(ev, p_lo, p_hi, s, g, R.fplan, R.fgroup_v, R.fwork_pre, R.nfplan, R.fwork);
    if (g.work == 0) return;
    TriArgs A = graph_args(g);
    A.cnt = cnt;
    A.rec = R.rec.get();
    A.rec_off = R.rec_off.get();
    A.tb = R.tb.get();
    A.tb_off = R.tb_off.get();
    launch(A, false, g.work, 0, 1, s);
}

void fill_triangles_x(const Graph& g, const TriRecords& R, const uint32_t* efilt, const uint64_t* toff, int64_t p_lo,
                      int64_t p_hi, uint64_t slot0, uint32_t* tv, uint32_t* tf, uint32_t* rows, uint16_t* apex,
                      cudaStream_t s) {
    if (g.E == 0 || R.nfplan == 0 || R.fwork == 0 || p_lo >= p_hi) return;
    TriArgs A = graph_args(g);
    A.E = R.nfplan;
    A.work_pre = R.fwork_pre.get();
    A.fplan = R.fplan.get();
    A.fgroup_v = R.fgroup_v.get();
    A.rec = const_cast<uint32_t*>(R.rec.get());
    A.rec_off = R.rec_off.get();
    A.tb = const_cast<uint32_t*>(R.tb.get());
    A.tb_off = R.tb_off.get();
    A.efilt = efilt;
    A.toff = toff;
    A.p_lo = p_lo;
    A.p_hi = p_hi;
    A.slot0 = slot0;
    A.tv = tv;
    A.tf = tf;
    A.rows = rows;
    A.apex = g.n <= 65536 ? apex : nullptr;
    A.lists_cap = (int)((g.max_deg + 3) & ~3u);
    const size_t lists = (size_t)8 * A.lists_cap;
    const int64_t avail = (int64_t)device_max_smem_optin() - (int64_t)lists - 1024;
    const char* fw = std::getenv("VRB_TRI_FILL_WARPS");
    int warps = (int)std::min<int64_t>(fw ? std::max(4, std::min(16, std::atoi(fw))) : 16,
                                       avail / (int64_t)sizeof(WarpScratchX));
    if (warps < 4) fail(VRB_ENOTSUP, "x-major triangle fill: degree %u leaves no shared memory", g.max_deg);
    const int threads = warps * 32;
    const size_t smem = lists + (size_t)warps * sizeof(WarpScratchX);
    VRB_CUDA(cudaFuncSetAttribute(k_tri_fill_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tri_fill_x, threads, smem));
    if (per_sm < 1) fail(VRB_ENOTSUP, "x-major triangle fill does not fit");
    uint64_t chunk = R.fwork / 8192 + 1;
    if (chunk < 65536) chunk = 65536;
    A.chunk = chunk;
    A.ntasks = (int64_t)((R.fwork + chunk - 1) / chunk);
    if (A.ntasks < 1) A.ntasks = 1;
    A.task_lo = 0;
    A.task_hi = A.ntasks;
    DBuf<unsigned long long> counter(1, s);
    VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned long long), s));
    A.task_counter = counter.get();
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)device_sm_count() * per_sm, A.ntasks);
    k_tri_fill_x<<<grid, threads, smem, s>>>(A);
    VRB_LAUNCH_CHECK();
}

void fill_triangles(const Graph& g, const uint32_t* efilt, const uint64_t* toff, int64_t p_lo, int64_t p_hi,
                    uint64_t slot0, uint32_t* tv, uint32_t* tf, uint32_t* rows, uint16_t* apex, cudaStream_t s,
                    const uint32_t* bm, const uint64_t* bmoff) {
    if (g.E == 0 || g.work == 0 || p_lo >= p_hi) return;
    TriArgs A = graph_args(g);
    A.efilt = efilt;
    A.toff = toff;
    A.p_lo = p_lo;
    A.p_hi = p_hi;
    A.slot0 = slot0;
    A.tv = tv;
    A.tf = tf;
    A.rows = rows;
    A.apex = g.n <= 65536 ? apex : nullptr;
    A.bm = const_cast<uint32_t*>(bm);
    A.bm_mode = bm ? bitmap_mode() : (markfill_apply(g) ? 4 : 0);
    A.bmoff = bmoff;
#ifdef VRB_ABLATION
    // ablation timing of experiment builds only (tools/variants.py
    // -DVRB_ABLATION=<mode>); it breaks the outputs, so the shipped library
    // (built without the macro) has no such knob
    A.debug = VRB_ABLATION;
#else
    A.debug = 0;
#endif
    launch(A, true, g.work, 0, 1, s);
}

}  // namespace vrb
