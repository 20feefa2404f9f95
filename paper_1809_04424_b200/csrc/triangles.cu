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
// Kernel shape.  Edges are grouped by a "host" endpoint y; a CTA loads the
// whole neighbourhood of y as a dense shared-memory map pos_y[k] (n u32) and
// its warps take the host's owner edges one at a time.  For edge p = (y, x)
// a warp streams the older-neighbour PREFIX of x (x's neighbours in position
// order, cut at p; the endpoint with the shorter prefix is scanned) and tests
// pos_y[k] < p.  Count: popc of ballots.  Fill: valid apexes are marked in a
// per-warp byte map indexed by the apex's rank in x's id-ordered list, which is
// then read back in id order (the lex order) and written coalesced.
#include <algorithm>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kBM = 4096;        // byte-map entries per warp (apex ranks per round)
constexpr int kU = 4;            // loads in flight per lane in the prefix scan

struct TriArgs {
    int64_t n, E;
    const uint64_t* off;
    const uint32_t* nbr_pos;
    const uint32_t* krank_pos;
    const uint64_t* kord;
    const uint32_t* scan_v;
    const uint32_t* scan_len;
    const uint32_t* hosted;
    const uint32_t* hosted_v;
    const uint64_t* work_pre;
    uint64_t chunk;
    int64_t ntasks;          // tasks of the whole work
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

// Warp: count apexes of owner edge p (host y's map in smem).
__device__ __forceinline__ uint32_t warp_count(const TriArgs& A, const uint32_t* __restrict__ map,
                                               uint32_t p, uint32_t x, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uint32_t* __restrict__ lst = A.nbr_pos + A.off[x];
    uint32_t c = 0;
    for (uint32_t t0 = 0; t0 < len; t0 += 32 * kU) {
        uint32_t k[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + u * 32 + lane;
            k[u] = t < len ? __ldg(lst + t) : NONE32;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) c += (k[u] != NONE32 && map[k[u]] < p) ? 1u : 0u;
    }
    return __reduce_add_sync(0xffffffffu, c);
}

// Warp: emit the triangles of owner edge p in apex-id order.
__device__ __forceinline__ void warp_fill(const TriArgs& A, const uint32_t* __restrict__ map,
                                          uint8_t* __restrict__ bm, uint32_t& stamp, uint32_t p,
                                          uint32_t y, uint32_t x, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uint64_t offx = A.off[x];
    const uint32_t degx = (uint32_t)(A.off[x + 1] - offx);
    const uint32_t* __restrict__ lst = A.nbr_pos + offx;
    const uint32_t* __restrict__ krk = A.krank_pos + offx;
    const uint64_t* __restrict__ kord = A.kord + offx;
    const uint32_t filt = A.efilt[p];
    uint64_t slot = A.toff[p] - A.slot0;
    for (uint32_t R = 0; R < degx; R += kBM) {
        if (++stamp == 256) {     // wrap: clear this warp's byte map
            for (int q = lane; q < kBM / 4; q += 32) reinterpret_cast<uint32_t*>(bm)[q] = 0u;
            stamp = 1;
            __syncwarp();
        }
        const uint8_t st = (uint8_t)stamp;
        // mark valid apexes by their rank in x's id-ordered list
        for (uint32_t t0 = 0; t0 < len; t0 += 32 * kU) {
            uint32_t k[kU], r[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t t = t0 + u * 32 + lane;
                k[u] = t < len ? __ldg(lst + t) : NONE32;
                r[u] = t < len ? __ldg(krk + t) : NONE32;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t rr = r[u] - R;
                if (k[u] != NONE32 && rr < (uint32_t)kBM && map[k[u]] < p) bm[rr] = st;
            }
        }
        __syncwarp();
        // read back in id order and write
        const uint32_t lim = min((uint32_t)kBM, degx - R);
        for (uint32_t w0 = 0; w0 < lim; w0 += 128) {
            const uint32_t idx = w0 + 4 * lane;
            uint32_t m4 = 0;
            if (idx < lim) {
                const uint32_t word = reinterpret_cast<const uint32_t*>(bm)[idx >> 2];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (((word >> (8 * b)) & 0xFF) == st && idx + b < lim) m4 |= 1u << b;
            }
            const uint32_t c = __popc(m4);
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            uint64_t s = slot + (incl - c);
            while (m4) {
                const int b = __ffs(m4) - 1;
                m4 &= m4 - 1;
                const uint64_t kp = __ldg(reinterpret_cast<const unsigned long long*>(kord) + R + idx + b);
                const uint32_t k = (uint32_t)kp;
                const uint32_t px = (uint32_t)(kp >> 32);
                const uint32_t py = map[k];
                uint32_t a0 = y, a1 = x, a2 = k;
                sort3(a0, a1, a2);
                uint32_t* tv = A.tv + 3 * s;
                tv[0] = a0; tv[1] = a1; tv[2] = a2;
                A.tf[s] = filt;
                if (A.rows) {
                    uint32_t* rw = A.rows + 3 * s;
                    rw[0] = min(px, py); rw[1] = max(px, py); rw[2] = p;
                }
                ++s;
            }
            slot += total;
        }
        __syncwarp();
    }
}

template <bool kFill>
__global__ void __launch_bounds__(kThreads) k_triangles(TriArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* map = reinterpret_cast<uint32_t*>(smem);
    uint8_t* bm_all = smem + ((A.n * 4 + 15) / 16) * 16;
    __shared__ int64_t s_lo, s_hi, s_end;
    __shared__ uint32_t s_y;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t* bm = bm_all + (size_t)wid * kBM;
    uint32_t stamp = 0;
    for (int64_t q = threadIdx.x; q < A.n; q += kThreads) map[q] = NONE32;
    if (kFill)
        for (int q = threadIdx.x; q < kWarps * kBM / 4; q += kThreads) reinterpret_cast<uint32_t*>(bm_all)[q] = 0u;
    __syncthreads();
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
            }
            __syncthreads();
            const uint32_t y = s_y;
            const int64_t end = s_end;
            const uint64_t oy = A.off[y], oy1 = A.off[y + 1];
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += kThreads) {
                const uint64_t kp = A.kord[t];
                map[(uint32_t)kp] = (uint32_t)(kp >> 32);
            }
            __syncthreads();
            for (int64_t e = seg + wid; e < end; e += kWarps) {
                const uint32_t p = A.hosted[e];
                if (kFill && ((int64_t)p < A.p_lo || (int64_t)p >= A.p_hi)) continue;
                const uint32_t len = A.scan_len[p];
                if (len == 0) {
                    if (!kFill && lane == 0) A.cnt[p] = 0;
                    continue;
                }
                const uint32_t x = A.scan_v[p];
                if (kFill) {
                    warp_fill(A, map, bm, stamp, p, y, x, len);
                } else {
                    const uint32_t c = warp_count(A, map, p, x, len);
                    if (lane == 0) A.cnt[p] = c;
                }
            }
            __syncthreads();
            for (uint64_t t = oy + threadIdx.x; t < oy1; t += kThreads) map[(uint32_t)A.kord[t]] = NONE32;
            __syncthreads();
            seg = end;
        }
    }
}

size_t smem_bytes(int64_t n, bool fill) {
    return (size_t)((n * 4 + 15) / 16) * 16 + (fill ? (size_t)kWarps * kBM : 0);
}

void launch(const TriArgs& base, bool fill, uint64_t work, int part, int nparts, cudaStream_t s) {
    TriArgs A = base;
    const size_t smem = smem_bytes(A.n, fill);
    const int nsm = device_sm_count();
    int per_sm = 1;
    if (fill) {
        VRB_CUDA(cudaFuncSetAttribute(k_triangles<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_triangles<true>, kThreads, smem));
    } else {
        VRB_CUDA(cudaFuncSetAttribute(k_triangles<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_triangles<false>, kThreads, smem));
    }
    if (per_sm < 1) fail(VRB_ENOTSUP, "triangle kernel does not fit (n = %lld)", (long long)A.n);
    const int64_t nctas = (int64_t)nsm * per_sm;
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
    const unsigned grid = (unsigned)std::min<int64_t>(nctas, A.task_hi - A.task_lo);
    if (fill)
        k_triangles<true><<<grid, kThreads, smem, s>>>(A);
    else
        k_triangles<false><<<grid, kThreads, smem, s>>>(A);
    VRB_LAUNCH_CHECK();
}

TriArgs graph_args(const Graph& g) {
    TriArgs A{};
    A.n = g.n;
    A.E = g.E;
    A.off = g.off.get();
    A.nbr_pos = g.nbr_pos.get();
    A.krank_pos = g.krank_pos.get();
    A.kord = g.kord.get();
    A.scan_v = g.scan_v.get();
    A.scan_len = g.scan_len.get();
    A.hosted = g.hosted.get();
    A.hosted_v = g.hosted_v.get();
    A.work_pre = g.work_pre.get();
    return A;
}

}  // namespace

int64_t dense_map_limit() {
    const int64_t smem = (int64_t)device_max_smem_optin();
    return (smem - (int64_t)kWarps * kBM - 64) / 4;
}

void count_triangles(const Graph& g, uint32_t* cnt, int part, int nparts, cudaStream_t s) {
    if (g.E == 0) return;
    VRB_CUDA(cudaMemsetAsync(cnt, 0, g.E * sizeof(uint32_t), s));
    if (g.work == 0) return;
    TriArgs A = graph_args(g);
    A.cnt = cnt;
    launch(A, false, g.work, part, nparts, s);
}

void fill_triangles(const Graph& g, const uint32_t* efilt, const uint64_t* toff, int64_t p_lo, int64_t p_hi,
                    uint64_t slot0, uint32_t* tv, uint32_t* tf, uint32_t* rows, cudaStream_t s) {
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
    launch(A, true, g.work, 0, 1, s);
}

}  // namespace vrb
