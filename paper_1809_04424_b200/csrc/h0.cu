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
// read as 16-byte vectors), a CTA of kCTh threads one tile of kCT columns.
// Pass 1 sums each tile's kept rows, a scan of the tile sums gives tile
// offsets, pass 2 scans the threads' counts in the block and writes colptr
// and the kept (renumbered) rows -- the D_2 rows are read twice, colptr and
// the output written once.  Whether a row survives and its new number come
// from the (sorted) forest itself, held in shared memory with a coarse
// index: blk[b] = #forest positions below b << shift, so a row r searches
// forest[blk[r >> shift], blk[(r >> shift) + 1]) -- with the shift chosen so
// a block holds about one forest position on average (the forest has n - c
// of E edges, most of them among the shortest) -- instead of two random
// global lookups per row.  Persistent CTAs load the
// index once and stride over the tiles.
constexpr int kCTh = 1024;           // threads per CTA
constexpr int kCPT = 8;              // columns per thread (24 rows = 6 uint4)
constexpr int kCT = kCTh * kCPT;     // columns per tile

struct ForestIndex {
    const uint32_t* f;     // sorted forest positions
    const uint32_t* blk;   // coarse index
    int shift;
    __device__ __forceinline__ bool kept(uint32_t r, uint32_t& newr) const {
        const uint32_t b = r >> shift;
        uint32_t lo = blk[b], hi = blk[b + 1];
        const uint32_t end = hi;
        // lower bound of r in the block's forest positions: the forest's
        // (short) edges crowd the first blocks, so search, not scan
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (f[mid] < r) lo = mid + 1; else hi = mid;
        }
        newr = r - lo;
        return !(lo < end && f[lo] == r);
    }
};

__device__ __forceinline__ ForestIndex load_forest(unsigned char* smem, const uint32_t* __restrict__ forest,
                                                   int64_t nf, const uint32_t* __restrict__ blk, int64_t nblk,
                                                   int shift, bool in_smem) {
    if (!in_smem) return ForestIndex{forest, blk, shift};   // too large for shared memory: read it through L2
    uint32_t* f = reinterpret_cast<uint32_t*>(smem);
    uint32_t* b = f + nf;
    for (int64_t q = threadIdx.x; q < nf; q += blockDim.x) f[q] = forest[q];
    for (int64_t q = threadIdx.x; q <= nblk; q += blockDim.x) b[q] = blk[q];
    __syncthreads();
    return ForestIndex{f, b, shift};
}

// the kCPT columns of thread slot j0 .. j0 + kCPT: kept flags, new rows, and
// the number kept per column (columns >= ncols keep nothing)
struct ColGroup {
    uint32_t r[3 * kCPT];
    uint32_t keepmask;   // bit 3 c + q: row q of column c kept
};

__device__ __forceinline__ uint32_t load_group(const uint32_t* __restrict__ rows, int64_t ncols, int64_t j0,
                                               const ForestIndex& FI, ColGroup& G) {
    if (j0 + kCPT <= ncols) {
        const uint4* v = reinterpret_cast<const uint4*>(rows + 3 * j0);
#pragma unroll
        for (int q = 0; q < 3 * kCPT / 4; ++q) {
            const uint4 w = __ldcs(v + q);
            G.r[4 * q] = w.x; G.r[4 * q + 1] = w.y; G.r[4 * q + 2] = w.z; G.r[4 * q + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 3 * kCPT; ++q) G.r[q] = j0 + q / 3 < ncols ? __ldcs(rows + 3 * j0 + q) : 0u;
    }
    uint32_t mask = 0, cnt = 0;
    uint32_t last = 0xFFFFFFFFu, lastnew = 0;
    bool lastkept = false;
#pragma unroll
    for (int q = 0; q < 3 * kCPT; ++q) {
        if (j0 + q / 3 >= ncols) continue;
        uint32_t nr;
        bool k;
        if (G.r[q] == last) {   // the owner edge's row repeats along its triangles
            nr = lastnew;
            k = lastkept;
        } else {
            k = FI.kept(G.r[q], nr);
            last = G.r[q];
            lastnew = nr;
            lastkept = k;
        }
        G.r[q] = nr;
        if (k) { mask |= 1u << q; ++cnt; }
    }
    G.keepmask = mask;
    return cnt;
}

__global__ void __launch_bounds__(kCTh) k_col_tile_sums(const uint32_t* __restrict__ rows, int64_t ncols,
                                                        const uint32_t* __restrict__ forest, int64_t nf,
                                                        const uint32_t* __restrict__ blk, int64_t nblk, int shift,
                                                        int in_smem, unsigned long long* __restrict__ sums) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long red[kCTh / 32];
    const ForestIndex FI = load_forest(smem, forest, nf, blk, nblk, shift, in_smem != 0);
    const int64_t tiles = (ncols + kCT - 1) / kCT;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        ColGroup G;
        unsigned long long a = load_group(rows, ncols, t * kCT + (int64_t)threadIdx.x * kCPT, FI, G);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long v = red[threadIdx.x];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (threadIdx.x == 0) sums[t] = v;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kCTh) k_col_tile_fill(const uint32_t* __restrict__ rows, int64_t ncols,
                                                        const uint32_t* __restrict__ forest, int64_t nf,
                                                        const uint32_t* __restrict__ blk, int64_t nblk, int shift,
                                                        int in_smem, const uint64_t* __restrict__ tile_off,
                                                        uint64_t* __restrict__ colptr, uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long wt[kCTh / 32];
    const ForestIndex FI = load_forest(smem, forest, nf, blk, nblk, shift, in_smem != 0);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t tiles = (ncols + kCT - 1) / kCT;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t j0 = t * kCT + (int64_t)threadIdx.x * kCPT;
        ColGroup G;
        const uint32_t c = load_group(rows, ncols, j0, FI, G);
        unsigned long long x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wt[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned long long v = wt[lane], s = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wt[lane] = s - v;   // exclusive prefix of the warp totals
        }
        __syncthreads();
        uint64_t o = tile_off[t] + wt[wid] + x - c;
        if (j0 + kCPT <= ncols) {
            uint64_t cp[kCPT];
#pragma unroll
            for (int q = 0; q < kCPT; ++q) {
                cp[q] = o;
#pragma unroll
                for (int e = 0; e < 3; ++e)
                    if ((G.keepmask >> (3 * q + e)) & 1u) out[o++] = G.r[3 * q + e];
            }
            ulonglong2* d = reinterpret_cast<ulonglong2*>(colptr + j0);
#pragma unroll
            for (int q = 0; q < kCPT / 2; ++q) __stcs(d + q, make_ulonglong2(cp[2 * q], cp[2 * q + 1]));
            if (j0 + kCPT == ncols) colptr[ncols] = o;
        } else {
#pragma unroll
            for (int q = 0; q < kCPT; ++q) {
                if (j0 + q >= ncols) break;
                colptr[j0 + q] = o;
#pragma unroll
                for (int e = 0; e < 3; ++e)
                    if ((G.keepmask >> (3 * q + e)) & 1u) out[o++] = G.r[3 * q + e];
                if (j0 + q == ncols - 1) colptr[ncols] = o;
            }
        }
        __syncthreads();
    }
}

__global__ void k_forest_blocks(const uint32_t* __restrict__ forest, int64_t nf, int64_t nblk, int shift,
                                uint32_t* __restrict__ blk) {
    GRID_STRIDE(b, nblk + 1) {
        const uint64_t v = (uint64_t)b << shift;
        int64_t lo = 0, hi = nf;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((uint64_t)forest[mid] < v) lo = mid + 1; else hi = mid;
        }
        blk[b] = (uint32_t)lo;
    }
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
    // coarse index granularity: about one forest position per block, as long
    // as forest + index fit shared memory (else the index goes to L2)
    const int64_t budget = (int64_t)device_max_smem_optin() - 4096;
    int shift = 6;
    while (shift < 31 && (((E >> shift) > 2 * nf + 1024) || 4 * (nf + (E >> shift) + 2) > budget)) ++shift;
    const int64_t nblk = (E >> shift) + 1;
    DBuf<uint32_t> blk(nblk + 1, s);
    k_forest_blocks<<<grid_for(nblk + 1), 256, 0, s>>>(forest, nf, nblk, shift, blk.get());
    VRB_LAUNCH_CHECK();
    size_t smem = (size_t)4 * (nf + nblk + 1);
    int in_smem = 1;
    if ((int64_t)smem > budget) {   // large forests: index in global memory
        smem = 0;
        in_smem = 0;
    }
    VRB_CUDA(cudaFuncSetAttribute(k_col_tile_sums, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VRB_CUDA(cudaFuncSetAttribute(k_col_tile_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    VRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_col_tile_fill, kCTh, smem));
    const int64_t tiles = ceil_div(ncols, kCT);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)device_sm_count() * std::max(1, per_sm));
    DBuf<unsigned long long> sums(tiles, s);
    DBuf<uint64_t> toff(tiles + 1, s);
    k_col_tile_sums<<<grid, kCTh, smem, s>>>(rows, ncols, forest, nf, blk.get(), nblk, shift, in_smem, sums.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(reinterpret_cast<const uint64_t*>(sums.get()), toff.get(), tiles, s);
    uint64_t nnz = 0;
    VRB_CUDA(cudaMemcpyAsync(&nnz, toff.get() + tiles, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    *rowval_out = alloc_out((int64_t)nnz, ctx);
    k_col_tile_fill<<<grid, kCTh, smem, s>>>(rows, ncols, forest, nf, blk.get(), nblk, shift, in_smem, toff.get(),
                                             colptr, *rowval_out);
    VRB_LAUNCH_CHECK();
    VRB_CUDA(cudaStreamSynchronize(s));
    return (int64_t)nnz;
}

}  // namespace vrb
