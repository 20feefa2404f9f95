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
// The forest's edges, flagged per position, are compacted in position order:
// they are the D_1 pivot columns (the "clearing" set of P:302), and
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
        const uint32_t e = act ? act[q] : (uint32_t)q;
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
__global__ void k_hook(const uint2* __restrict__ ev, int64_t n, const uint32_t* __restrict__ comp,
                       const uint32_t* __restrict__ best, uint32_t* __restrict__ hook, uint8_t* __restrict__ in_forest,
                       int* __restrict__ changed) {
    GRID_STRIDE(c, n) {
        hook[c] = comp[c];
        if (comp[c] != (uint32_t)c) continue;
        const uint32_t e = best[c];
        if (e == NONE32) continue;
        const uint2 uv = ev[e];
        const uint32_t cu = comp[uv.x], cv = comp[uv.y];
        const uint32_t other = cu == (uint32_t)c ? cv : cu;
        in_forest[e] = 1;
        *changed = 1;
        if (best[other] == e && other > (uint32_t)c) continue;   // mutual: the smaller root stays
        hook[c] = other;
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

__global__ void k_forest_flags(const uint8_t* __restrict__ in_forest, int64_t E, uint32_t* __restrict__ flag) {
    GRID_STRIDE(e, E) flag[e] = in_forest[e];
}

__global__ void k_forest_out(const uint32_t* __restrict__ flag, const uint64_t* __restrict__ pre, int64_t E,
                             const uint32_t* __restrict__ efilt, uint32_t* __restrict__ pos,
                             uint32_t* __restrict__ death) {
    GRID_STRIDE(e, E) {
        if (flag[e]) {
            pos[pre[e]] = (uint32_t)e;
            death[pre[e]] = efilt[e];
        }
    }
}

}  // namespace

int64_t h0_forest(const uint32_t* ev, const uint32_t* efilt, int64_t n, int64_t E, cudaStream_t s,
                  uint32_t* (*alloc_out)(int64_t, void*), void* ctx, uint32_t** pos_out, uint32_t** death_out) {
    *pos_out = *death_out = nullptr;
    if (n == 0 || E == 0) return 0;
    const uint2* ev2 = reinterpret_cast<const uint2*>(ev);
    DBuf<uint32_t> comp(n, s), hook(n, s), best(n, s);
    DBuf<uint8_t> in_forest(E, s);
    DBuf<int> changed(1, s);
    k_iota<<<grid_for(n), 256, 0, s>>>(comp.get(), n);
    VRB_LAUNCH_CHECK();
    VRB_CUDA(cudaMemsetAsync(in_forest.get(), 0, in_forest.bytes(), s));
    DBuf<uint32_t> act, act_next, flag(E, s);
    DBuf<uint64_t> pre(E + 1, s);
    int64_t na = E;   // active (crossing) edges; the first round takes all positions
    for (int round = 0; round < 64 && na > 0; ++round) {
        VRB_CUDA(cudaMemsetAsync(best.get(), 0xFF, best.bytes(), s));
        VRB_CUDA(cudaMemsetAsync(changed.get(), 0, sizeof(int), s));
        k_best<<<grid_for(na), 256, 0, s>>>(ev2, act.get(), na, comp.get(), best.get());
        VRB_LAUNCH_CHECK();
        k_hook<<<grid_for(n), 256, 0, s>>>(ev2, n, comp.get(), best.get(), hook.get(), in_forest.get(),
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
        if (!h) break;
        if ((int64_t)nn > 0) {
            act_next.alloc(nn, s);
            k_compact<<<grid_for(na), 256, 0, s>>>(act.get(), na, flag.get(), pre.get(), act_next.get());
            VRB_LAUNCH_CHECK();
        }
        act = std::move(act_next);
        na = (int64_t)nn;
    }
    // forest edges in position order
    k_forest_flags<<<grid_for(E), 256, 0, s>>>(in_forest.get(), E, flag.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(flag.get(), pre.get(), E, s);
    uint64_t nf = 0;
    VRB_CUDA(cudaMemcpyAsync(&nf, pre.get() + E, sizeof(nf), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (nf) {
        *pos_out = alloc_out((int64_t)nf, ctx);
        *death_out = alloc_out((int64_t)nf, ctx);
        k_forest_out<<<grid_for(E), 256, 0, s>>>(flag.get(), pre.get(), E, efilt, *pos_out, *death_out);
        VRB_LAUNCH_CHECK();
    }
    return (int64_t)nf;
}

}  // namespace vrb
