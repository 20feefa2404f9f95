// h0.cu -- SURVEY 8(f) F1: dimension-0 persistence straight from the ranked
// edges.
//
// Definition.  Every vertex is born at filtration 0 (Fig. 4 caption, P:286:
// the vertices v_s enter first; reading A8).  Reducing D_1 by the column
// algorithm (Algorithm 1) pairs edge column j with a vertex row
// exactly when edge j joins two different components of the complex built
// from the edges before it, in the filtration order (columns in
// filtration order).  Those edges are the minimum spanning forest of the
// 1-skeleton under the total edge order (filt, lex) = edge position -- the
// Kruskal forest.  Each gives the finite bar [0, filt(e)); each component of
// the whole complex gives [0, inf) (Fig. 4: "one additional bar ... death
// time infinity", reading A8).
//
// B200 design.  Positions are unique weights, so the forest is also what
// Boruvka's algorithm returns: every round, each component takes its
// lightest outgoing edge (atomicMin over the edge positions), components
// hook along those edges (the larger root of a mutual pair yields), and
// pointer jumping flattens the forest.  O(log n) rounds, each a streaming
// pass over the edges that still cross components (compacted every round).
// Filter first: the rounds run on the position prefix [0, P) alone (P = 8n):
// that is Kruskal's state after P edges.  Then windows [w, 4w) in turn keep
// only their edges that still join two components, and the rounds continue on
// those; a spanning tree (n - 1 forest edges) ends the search early.  The
// union is the same unique forest (positions are distinct weights).
// The forest's edges, appended as they join and radix-sorted by position,
// are the D_1 pivot columns (the "clearing" set of P:302), and
// filt(e) over them is the sorted list of finite H0 deaths.
#include <algorithm>

#include "vrb_internal.cuh"

namespace vrb {
namespace {

#define GRID_STRIDE(i, n)                                                          \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n);       \
         i += (int64_t)gridDim.x * blockDim.x)

unsigned grid_for(int64_t n) {
    const int64_t g = ceil_div(n, 256), cap = (int64_t)device_sm_count() * 16;
    return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

__global__ void k_iota(uint32_t* __restrict__ a, int64_t n) { GRID_STRIDE(i, n) a[i] = (uint32_t)i; }

// lightest crossing edge per component root; flags[q] = edge still crosses
__global__ void k_best(const uint2* __restrict__ ev, const uint32_t* __restrict__ act, int64_t na,
                       const uint32_t* __restrict__ comp, uint32_t* best) {
    GRID_STRIDE(q, na) {
        const uint32_t e = act ? act[q] : (uint32_t)q;   // act == null: the prefix [0, na)
        const uint2 uv = ev[e];
        const uint32_t cu = comp[uv.x], cv = comp[uv.y];
        if (cu != cv) {
            // the edges come in position order, so a component usually holds a
            // smaller candidate already: test before paying for the atomic
            if (*(volatile const uint32_t*)(best + cu) > e) atomicMin(&best[cu], e);
            if (*(volatile const uint32_t*)(best + cv) > e) atomicMin(&best[cv], e);
        }
    }
}

// root c hooks to the component across its lightest edge; of a mutual pair
// (both roots chose the same edge) the larger root hooks to the smaller
// (root c hooks: its edge joins the forest, appended once -- of a mutual
// pair only the hooking root appends)
__global__ void k_hook(const uint2* __restrict__ ev, int64_t n, const uint32_t* __restrict__ comp,
                       const uint32_t* __restrict__ best, uint32_t* __restrict__ hook, uint32_t* __restrict__ forest,
                       unsigned long long* __restrict__ nforest, int* __restrict__ changed) {
    GRID_STRIDE(c, n) {
        hook[c] = comp[c];
        if (comp[c] != (uint32_t)c) continue;
        const uint32_t e = best[c];
        if (e == NONE32) continue;
        const uint2 uv = ev[e];
        const uint32_t cu = comp[uv.x], cv = comp[uv.y];
        const uint32_t other = cu == (uint32_t)c ? cv : cu;
        *changed = 1;
        if (best[other] == e && other > (uint32_t)c) continue;   // mutual: the smaller root stays
        hook[c] = other;
        forest[atomicAdd(nforest, 1ull)] = e;
    }
}

// comp[v] <- root of v (hook graph is a forest after the mutual-pair rule)
__global__ void k_jump(const uint32_t* __restrict__ hook, int64_t n, uint32_t* __restrict__ comp) {
    GRID_STRIDE(v, n) {
        uint32_t c = hook[comp[v]];
        while (hook[c] != c) c = hook[c];
        comp[v] = c;
    }
}

__global__ void k_cross_flags(const uint2* __restrict__ ev, const uint32_t* __restrict__ act, int64_t na,
                              const uint32_t* __restrict__ comp, uint32_t* __restrict__ flag) {
    GRID_STRIDE(q, na) {
        const uint32_t e = act ? act[q] : (uint32_t)q;
        const uint2 uv = ev[e];
        flag[q] = comp[uv.x] != comp[uv.y] ? 1u : 0u;
    }
}

__global__ void k_compact(const uint32_t* __restrict__ act, int64_t na, const uint32_t* __restrict__ flag,
                          const uint64_t* __restrict__ pre, uint32_t* __restrict__ out) {
    GRID_STRIDE(q, na) if (flag[q]) out[pre[q]] = act ? act[q] : (uint32_t)q;
}

// edges of [e0, E) whose endpoints lie in different components: counted
// (kFill = false) or appended in any order (the rounds do not depend on it)
template <bool kFill>
__global__ void k_tail_cross(const uint2* __restrict__ ev, int64_t e0, int64_t E, const uint32_t* __restrict__ comp,
                             unsigned long long* __restrict__ count, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q - lane < E; q += stride) {
        bool x = false;
        if (q < E) {
            const uint2 uv = ev[q];
            x = comp[uv.x] != comp[uv.y];
        }
        const unsigned b = __ballot_sync(0xffffffffu, x);
        if (!b) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (kFill && x) out[base + __popc(b & ((1u << lane) - 1u))] = (uint32_t)q;
    }
}

__global__ void k_forest_out(const uint64_t* __restrict__ sorted, int64_t nf, const uint32_t* __restrict__ efilt,
                             uint32_t* __restrict__ pos, uint32_t* __restrict__ death) {
    GRID_STRIDE(i, nf) {
        const uint32_t e = (uint32_t)sorted[i];
        pos[i] = e;
        death[i] = efilt[e];
    }
}

__global__ void k_widen(const uint32_t* __restrict__ a, int64_t n, uint64_t* __restrict__ b) {
    GRID_STRIDE(i, n) b[i] = a[i];
}

}  // namespace

int64_t h0_forest(const uint32_t* ev, const uint32_t* efilt, int64_t n, int64_t E, cudaStream_t s,
                  uint32_t* (*alloc_out)(int64_t, void*), void* ctx, uint32_t** pos_out, uint32_t** death_out) {
    *pos_out = *death_out = nullptr;
    if (n == 0 || E == 0) return 0;
    const uint2* ev2 = reinterpret_cast<const uint2*>(ev);
    DBuf<uint32_t> comp(n, s), hook(n, s), best(n, s), forest(n, s);
    DBuf<unsigned long long> nforest(1, s);
    DBuf<int> changed(1, s);
    k_iota<<<grid_for(n), 256, 0, s>>>(comp.get(), n);
    VRB_LAUNCH_CHECK();
    VRB_CUDA(cudaMemsetAsync(nforest.get(), 0, sizeof(unsigned long long), s));
    const int64_t P = std::min<int64_t>(E, 8 * n);   // the prefix the first rounds run on
    DBuf<uint32_t> act, act_next, flag(P, s);
    DBuf<uint64_t> pre(P + 1, s);
    int64_t na = P;   // active (crossing) edges; the first rounds take the prefix positions
    int64_t w1 = P;   // end of the windows processed so far
    for (int round = 0; round < 4096; ++round) {
        while (na == 0) {
            // the windows so far have converged: a spanning tree ends the search;
            // else the next window [w1, 4 w1) keeps its edges that still cross
            unsigned long long nf = 0;
            VRB_CUDA(cudaMemcpyAsync(&nf, nforest.get(), sizeof(nf), cudaMemcpyDeviceToHost, s));
            VRB_CUDA(cudaStreamSynchronize(s));
            if ((int64_t)nf == n - 1 || w1 == E) break;
            const int64_t w0 = w1;
            w1 = std::min<int64_t>(E, 4 * w1);
            DBuf<unsigned long long> cnt(1, s);
            VRB_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
            k_tail_cross<false><<<grid_for(w1 - w0), 256, 0, s>>>(ev2, w0, w1, comp.get(), cnt.get(), nullptr);
            VRB_LAUNCH_CHECK();
            unsigned long long nt = 0;
            VRB_CUDA(cudaMemcpyAsync(&nt, cnt.get(), sizeof(nt), cudaMemcpyDeviceToHost, s));
            VRB_CUDA(cudaStreamSynchronize(s));
            if (nt == 0) continue;
            act.alloc((int64_t)nt, s);
            VRB_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
            k_tail_cross<true><<<grid_for(w1 - w0), 256, 0, s>>>(ev2, w0, w1, comp.get(), cnt.get(), act.get());
            VRB_LAUNCH_CHECK();
            na = (int64_t)nt;
            if ((size_t)na > flag.size()) {
                flag.alloc(na, s);
                pre.alloc(na + 1, s);
            }
        }
        if (na == 0) break;
        VRB_CUDA(cudaMemsetAsync(best.get(), 0xFF, best.bytes(), s));
        VRB_CUDA(cudaMemsetAsync(changed.get(), 0, sizeof(int), s));
        k_best<<<grid_for(na), 256, 0, s>>>(ev2, act.get(), na, comp.get(), best.get());
        VRB_LAUNCH_CHECK();
        k_hook<<<grid_for(n), 256, 0, s>>>(ev2, n, comp.get(), best.get(), hook.get(), forest.get(), nforest.get(),
                                           changed.get());
        VRB_LAUNCH_CHECK();
        k_jump<<<grid_for(n), 256, 0, s>>>(hook.get(), n, comp.get());
        VRB_LAUNCH_CHECK();
        int h = 0;
        VRB_CUDA(cudaMemcpyAsync(&h, changed.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        // drop the edges that no longer cross components
        k_cross_flags<<<grid_for(na), 256, 0, s>>>(ev2, act.get(), na, comp.get(), flag.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(flag.get(), pre.get(), na, s);
        uint64_t nn = 0;
        VRB_CUDA(cudaMemcpyAsync(&nn, pre.get() + na, sizeof(nn), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        if (!h) nn = 0;   // no component has an outgoing edge left in this set
        if ((int64_t)nn > 0) {
            act_next.alloc(nn, s);
            k_compact<<<grid_for(na), 256, 0, s>>>(act.get(), na, flag.get(), pre.get(), act_next.get());
            VRB_LAUNCH_CHECK();
        }
        act = std::move(act_next);
        na = (int64_t)nn;
    }
    // forest edges in position order (<= n - 1 of them)
    unsigned long long nf = 0;
    VRB_CUDA(cudaMemcpyAsync(&nf, nforest.get(), sizeof(nf), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (nf) {
        DBuf<uint64_t> k0(nf, s), k1(nf, s);
        DBuf<uint32_t> v0(nf, s), v1(nf, s);
        k_widen<<<grid_for((int64_t)nf), 256, 0, s>>>(forest.get(), (int64_t)nf, k0.get());
        VRB_LAUNCH_CHECK();
        uint64_t vary = 0;
        for (int64_t b = 1; b <= E; b <<= 1) vary |= (uint64_t)b;   // positions < 2^ceil(log2(E + 1))
        iota_u32(v0.get(), (int64_t)nf, s);
        const bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), (int64_t)nf, vary, s);
        *pos_out = alloc_out((int64_t)nf, ctx);
        *death_out = alloc_out((int64_t)nf, ctx);
        k_forest_out<<<grid_for((int64_t)nf), 256, 0, s>>>(alt ? k1.get() : k0.get(), (int64_t)nf, efilt, *pos_out,
                                                           *death_out);
        VRB_LAUNCH_CHECK();
    }
    return (int64_t)nf;
}

// ---------------------------------------------------------------------------
// "Clear and compress" (Bauer-Kerber-Reininghaus, cited there): the
// pivots of a reduced D_k lie in rows of POSITIVE (k-1)-simplices -- those
// whose own column of D_{k-1} reduces to zero -- so deleting the rows of the
// negative ones leaves every pivot pair of D_k unchanged.  For k = 2 the
// negative edges are exactly the D_1 pivot columns, i.e. the H0 forest, so
// D_2 is compressed by dropping the forest's rows.  Rows are renumbered
// densely in position order (rowmap: new row -> edge position); a column
// keeps 1..3 entries (a forest has no cycle, so never 0), ascending.
// ---------------------------------------------------------------------------
namespace {

__global__ void k_keep_flags(const uint32_t* __restrict__ forest, int64_t nf, uint32_t* __restrict__ keep) {
    GRID_STRIDE(q, nf) keep[forest[q]] = 0u;
}

__global__ void k_rowmap(const uint32_t* __restrict__ keep, const uint64_t* __restrict__ newidx, int64_t E,
                         uint32_t* __restrict__ rowmap) {
    GRID_STRIDE(e, E) if (keep[e]) rowmap[newidx[e]] = (uint32_t)e;
}

// Columns in tiles: a thread takes kCPT consecutive columns (3 kCPT rows,
// read as 16-byte vectors), a CTA of kCTh threads one tile of kCT columns;
// tiles are taken in order (a counter) and chained by a decoupled look-back
// over their kept-row counts, so D_2's rows are read once.  Whether a row
// survives and its new number come from a table of 16-byte entries per 64
// edge positions (the forest's bits there, and the number of forest
// positions below): one L2-resident load per row, all of a thread's issued
// together (C5B: 2.4 MB for 9.7e6 edges).  Each warp stages its output (kept
// rows and colptr) in shared memory and writes both as contiguous runs.
#ifndef VRB_CC_THREADS
#define VRB_CC_THREADS 512
#endif
#ifndef VRB_CC_CPT
#define VRB_CC_CPT 4
#endif
constexpr int kCTh = VRB_CC_THREADS;   // threads per CTA
constexpr int kCPT = VRB_CC_CPT;       // columns per thread (3 kCPT rows, 16-byte loads)
constexpr int kCT = kCTh * kCPT;     // columns per tile
constexpr int kCWarps = kCTh / 32;
constexpr unsigned long long kCAgg = 1ull << 62, kCPre = 2ull << 62, kCVal = (1ull << 62) - 1;

__device__ __forceinline__ bool ftab_kept(const ulonglong2& e, uint32_t r, uint32_t& newr) {
    const int o = (int)(r & 63u);
    newr = r - (uint32_t)(e.y + (uint64_t)__popcll(e.x & ((1ull << o) - 1ull)));
    return !((e.x >> o) & 1ull);
}

__global__ void __launch_bounds__(kCTh) k_col_compress(const uint32_t* __restrict__ rows, int64_t ncols,
                                                       const ulonglong2* __restrict__ ftab,
                                                       unsigned long long* __restrict__ status,
                                                       unsigned* __restrict__ counter, uint64_t* __restrict__ colptr,
                                                       uint32_t* __restrict__ out) {
    __shared__ uint32_t srow_all[kCWarps][32 * 3 * kCPT];
    __shared__ uint64_t scp_all[kCWarps][32 * kCPT];
    __shared__ uint32_t wt[kCWarps];
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_prefix;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* srow = srow_all[wid];
    uint64_t* scp = scp_all[wid];
    const int64_t tiles = (ncols + kCT - 1) / kCT;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
        __syncthreads();
        const int64_t t = s_tile;
        if (t >= tiles) break;
        const int64_t j0 = t * kCT + (int64_t)threadIdx.x * kCPT;
        // rows and their table entries, all loads issued before any use
        uint32_t r[3 * kCPT];
        if (j0 + kCPT <= ncols) {
            const uint4* v = reinterpret_cast<const uint4*>(rows + 3 * j0);
#pragma unroll
            for (int q = 0; q < 3 * kCPT / 4; ++q) {
                const uint4 w = __ldcs(v + q);
                r[4 * q] = w.x; r[4 * q + 1] = w.y; r[4 * q + 2] = w.z; r[4 * q + 3] = w.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3 * kCPT; ++q) r[q] = j0 + q / 3 < ncols ? __ldcs(rows + 3 * j0 + q) : 0u;
        }
        ulonglong2 e[3 * kCPT];
#pragma unroll
        for (int q = 0; q < 3 * kCPT; ++q) e[q] = __ldg(ftab + (r[q] >> 6));
        uint32_t mask = 0, c = 0;
#pragma unroll
        for (int q = 0; q < 3 * kCPT; ++q) {
            uint32_t nr;
            const bool k = j0 + q / 3 < ncols && ftab_kept(e[q], r[q], nr);
            r[q] = nr;
            if (k) { mask |= 1u << q; ++c; }
        }
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t wsum = __shfl_sync(0xffffffffu, x, 31);
        if (lane == 31) wt[wid] = wsum;
        __syncthreads();
        if (wid == 0) {
            const uint32_t v = lane < kCWarps ? wt[lane] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned long long total = __shfl_sync(0xffffffffu, incl, 31);
            volatile unsigned long long* st = status;
            unsigned long long excl = 0;
            if (t == 0) {
                if (lane == 0) st[0] = kCPre | total;
            } else {
                if (lane == 0) st[t] = kCAgg | total;
                int64_t j = t - 1;
                for (;;) {
                    const int64_t jj = j - lane;
                    unsigned long long sv = kCPre;
                    if (jj >= 0) {
                        sv = st[jj];
                        while ((sv & (kCAgg | kCPre)) == 0) sv = st[jj];
                    }
                    const unsigned pre = __ballot_sync(0xffffffffu, (sv & kCPre) != 0);
                    const int first = pre ? __ffs(pre) - 1 : 32;
                    unsigned long long part = lane <= first ? (sv & kCVal) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                    excl += part;
                    if (pre) break;
                    j -= 32;
                }
                if (lane == 0) {
                    __threadfence();
                    st[t] = kCPre | (excl + total);
                }
            }
            if (lane < kCWarps) wt[lane] = incl - v;   // exclusive per warp
            if (lane == 0) s_prefix = excl;
        }
        __syncthreads();
        const uint64_t wbase = s_prefix + wt[wid];   // the warp's first output row
        uint32_t lo = x - c;
#pragma unroll
        for (int q = 0; q < kCPT; ++q) {
            scp[lane * kCPT + q] = wbase + lo;
#pragma unroll
            for (int e2 = 0; e2 < 3; ++e2)
                if ((mask >> (3 * q + e2)) & 1u) srow[lo++] = r[3 * q + e2];
        }
        __syncwarp();
        for (uint32_t i = lane; i < wsum; i += 32) __stcs(out + wbase + i, srow[i]);
        const int64_t c0 = t * kCT + (int64_t)wid * 32 * kCPT;
        for (int i = lane; i < 32 * kCPT; i += 32)
            if (c0 + i < ncols) __stcs(reinterpret_cast<unsigned long long*>(colptr) + c0 + i, scp[i]);
        if (lane == 0 && c0 <= ncols - 1 && ncols - 1 < c0 + 32 * kCPT) colptr[ncols] = wbase + wsum;
        __syncthreads();   // s_tile, wt and the staging are reused
    }
}

// forest table: bits of the forest positions per 64-position block, then
// the count below each block (an exclusive scan of the blocks' popcounts)
__global__ void k_ftab_bits(const uint32_t* __restrict__ forest, int64_t nf, ulonglong2* __restrict__ tab) {
    GRID_STRIDE(q, nf) {
        const uint32_t f = forest[q];
        atomicOr(reinterpret_cast<unsigned long long*>(&tab[f >> 6].x), 1ull << (f & 63u));
    }
}

__global__ void k_ftab_pop(const ulonglong2* __restrict__ tab, int64_t nb, uint32_t* __restrict__ pop) {
    GRID_STRIDE(b, nb) pop[b] = (uint32_t)__popcll(tab[b].x);
}

__global__ void k_ftab_below(ulonglong2* __restrict__ tab, int64_t nb, const uint64_t* __restrict__ below) {
    GRID_STRIDE(b, nb) tab[b].y = below[b];
}


}  // namespace

int64_t compress_d2(const uint32_t* forest, int64_t nf, int64_t E, const uint32_t* rows, int64_t ncols,
                    cudaStream_t s, uint64_t* colptr, uint32_t* (*alloc_out)(int64_t, void*), void* ctx,
                    uint32_t** rowval_out, uint32_t** rowmap_out, int64_t* nrows_out) {
    *rowval_out = nullptr;
    *rowmap_out = nullptr;
    DBuf<uint32_t> keep(std::max<int64_t>(E, 1), s);   // u32 flags for the scan ...
    fill_u32(keep.get(), 1u, E, s);
    if (nf) {
        k_keep_flags<<<grid_for(nf), 256, 0, s>>>(forest, nf, keep.get());
        VRB_LAUNCH_CHECK();
    }
    DBuf<uint64_t> newidx(E + 1, s);
    exclusive_scan(keep.get(), newidx.get(), E, s);
    uint64_t nr = 0;
    VRB_CUDA(cudaMemcpyAsync(&nr, newidx.get() + E, sizeof(nr), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    *nrows_out = (int64_t)nr;
    *rowmap_out = alloc_out((int64_t)nr, ctx);
    if (nr) {
        k_rowmap<<<grid_for(E), 256, 0, s>>>(keep.get(), newidx.get(), E, *rowmap_out);
        VRB_LAUNCH_CHECK();
    }
    keep.reset();
    if (ncols == 0) {
        VRB_CUDA(cudaMemsetAsync(colptr, 0, sizeof(uint64_t), s));
        return 0;
    }
    // the forest table (16 bytes per 64 edge positions)
    const int64_t ntab = (E >> 6) + 1;
    DBuf<ulonglong2> ftab(ntab, s);
    VRB_CUDA(cudaMemsetAsync(ftab.get(), 0, ntab * sizeof(ulonglong2), s));
    if (nf) {
        k_ftab_bits<<<grid_for(nf), 256, 0, s>>>(forest, nf, ftab.get());
        VRB_LAUNCH_CHECK();
    }
    {
        DBuf<uint32_t> pop(ntab, s);
        DBuf<uint64_t> below(ntab + 1, s);
        k_ftab_pop<<<grid_for(ntab), 256, 0, s>>>(ftab.get(), ntab, pop.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(pop.get(), below.get(), ntab, s);
        k_ftab_below<<<grid_for(ntab), 256, 0, s>>>(ftab.get(), ntab, below.get());
        VRB_LAUNCH_CHECK();
    }
    // one pass over D_2: tiles chained by a look-back over their kept counts
    const int64_t tiles = ceil_div(ncols, kCT);
    DBuf<unsigned long long> status(tiles, s);
    DBuf<unsigned> counter(1, s);
    VRB_CUDA(cudaMemsetAsync(status.get(), 0, tiles * sizeof(unsigned long long), s));
    VRB_CUDA(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned), s));
    // nnz: 3 ncols less the forest rows -- known only after the pass, so the
    // output is allocated for 3 ncols and the count read back afterwards
    uint32_t* rv = alloc_out(3 * ncols, ctx);
    *rowval_out = rv;
    int per_sm = 1;
    VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_col_compress, kCTh, 0));
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)device_sm_count() * std::max(1, per_sm));
    k_col_compress<<<grid, kCTh, 0, s>>>(rows, ncols, ftab.get(), status.get(), counter.get(), colptr, rv);
    VRB_LAUNCH_CHECK();
    uint64_t nnz = 0;
    VRB_CUDA(cudaMemcpyAsync(&nnz, colptr + ncols, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return (int64_t)nnz;
}

}  // namespace vrb
