// dist.cu -- vrb_build_dist: the multi-GPU build, one process per GPU
// (the paper's own precedent is the column partition of
// blockprodsum, whose master fixes the column pointers "one after the
// other", Fig. BlkProdSum P:1010-1022 -- here that fix-up is an exclusive
// scan of per-rank totals).
//
// Every stage but the neighbour lists is sharded:
//   S1  points: rank 0 places (copy / transpose / finite check) and
//       broadcasts them (n d 8 bytes);
//   S2  distances: rank g computes the pairs of its row block (tile-aligned,
//       balanced by pair count);
//   S3  edge order: each rank sorts its kept edges by (len, i, j); the sorted
//       runs (16 B per edge) are all-gathered and merged (merge path, log2 G
//       rounds), so every rank holds the global edge order, dense ranks and
//       value_of_rank -- the tables D_2's rows and the enumeration need;
//   S4  neighbour lists: rebuilt on every rank from the global edge order
//       (the one replicated stage; it needs no exchange);
//   S5-S8 triangles: rank g owns the owner edges of one position range,
//       level-aligned and balanced by enumeration work; it counts, fills and
//       tie-sorts that range alone (apex bitmaps kept on the rank), and its
//       output slice starts at the exclusive prefix of the per-rank totals
//       (G x 8 bytes all-gathered), so the slices concatenated in rank order
//       are byte-identical to vrb_build (pin P13);
//   S6  tetrahedra (K = 3): the per-edge triangle counts and the triangle
//       vertices / apexes are all-gathered (D_3's faces can be any earlier
//       triangle), then tetrahedra are partitioned like triangles.
// The exchange goes through the caller's vrb_comm callbacks, issued on the
// build stream.
#include <algorithm>
#include <cstring>
#include <vector>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

#define GRID_STRIDE(i, n)                                                          \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n);       \
         i += (int64_t)gridDim.x * blockDim.x)

unsigned grid_of(int64_t n) {
    int64_t g = ceil_div(n, 256), cap = (int64_t)device_sm_count() * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Collective calls through the caller's callbacks (vrb_comm).
struct Comm {
    const vrb_comm* c;
    cudaStream_t s;
    int rank() const { return c->rank; }
    int world() const { return c->world; }
    void allgather(const void* send, void* recv, size_t bytes) const {
        if (c->allgather(send, recv, bytes, (void*)s, c->ctx) != 0) fail(VRB_ECOMM, "allgather of %zu bytes failed", bytes);
    }
    void bcast(void* buf, size_t bytes, int root) const {
        if (c->broadcast(buf, bytes, root, (void*)s, c->ctx) != 0) fail(VRB_ECOMM, "broadcast of %zu bytes failed", bytes);
    }
    // one u64 per rank, in rank order (host)
    std::vector<uint64_t> allgather_u64(uint64_t v) const {
        const int G = world();
        DBuf<uint64_t> d(1, s), all(G, s);
        VRB_CUDA(cudaMemcpyAsync(d.get(), &v, sizeof(v), cudaMemcpyHostToDevice, s));
        allgather(d.get(), all.get(), sizeof(uint64_t));
        std::vector<uint64_t> h(G);
        VRB_CUDA(cudaMemcpyAsync(h.data(), all.get(), G * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        return h;
    }
};

// ---------------------------------------------------------------------------
// S3: runs of (len bits, i << 32 | j), merged
// ---------------------------------------------------------------------------
__global__ void k_make_run(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sval, int64_t m,
                           uint64_t bias, int packed, const uint32_t* __restrict__ ei, const uint32_t* __restrict__ ej,
                           uint64_t* __restrict__ key, uint64_t* __restrict__ ij) {
    GRID_STRIDE(q, m) {
        key[q] = skey[q] + bias;
        const uint32_t v = sval[q];
        ij[q] = packed ? ((uint64_t)(v >> 16) << 32 | (v & 0xFFFFu)) : ((uint64_t)ei[v] << 32 | ej[v]);
    }
}

__device__ __forceinline__ bool item_less(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Merge path: out[d] for d in [0, na + nb) from the sorted runs A and B
// (items are distinct, so the merge is unique).  Each thread finds the split
// of its diagonal by binary search, then merges kPer items sequentially.
constexpr int kPer = 8;
__global__ void k_merge(const uint64_t* __restrict__ ak, const uint64_t* __restrict__ ai, int64_t na,
                        const uint64_t* __restrict__ bk, const uint64_t* __restrict__ bi, int64_t nb,
                        uint64_t* __restrict__ ok, uint64_t* __restrict__ oi) {
    const int64_t total = na + nb;
    for (int64_t d0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPer; d0 < total;
         d0 += (int64_t)gridDim.x * blockDim.x * kPer) {
        // i = number of A items among the first d0 outputs
        int64_t lo = d0 > nb ? d0 - nb : 0, hi = d0 < na ? d0 : na;
        while (lo < hi) {
            const int64_t i = (lo + hi) >> 1, j = d0 - i - 1;   // A[i] vs B[j]
            if (item_less(bk[j], bi[j], ak[i], ai[i])) hi = i; else lo = i + 1;
        }
        int64_t i = lo, j = d0 - lo;
        const int64_t d1 = min(total, d0 + kPer);
        for (int64_t d = d0; d < d1; ++d) {
            const bool take_a = j >= nb || (i < na && item_less(ak[i], ai[i], bk[j], bi[j]));
            if (take_a) { ok[d] = ak[i]; oi[d] = ai[i]; ++i; }
            else { ok[d] = bk[j]; oi[d] = bi[j]; ++j; }
        }
    }
}

__global__ void k_edge_out(const uint64_t* __restrict__ key, const uint64_t* __restrict__ ij,
                           const uint32_t* __restrict__ efilt, int64_t E, uint32_t* __restrict__ ev,
                           double* __restrict__ vor) {
    GRID_STRIDE(p, E) {
        const uint64_t v = ij[p];
        ev[2 * p] = (uint32_t)(v >> 32);
        ev[2 * p + 1] = (uint32_t)v;
        if (p == 0 || key[p] != key[p - 1]) vor[efilt[p] - 1] = __longlong_as_double((long long)key[p]);
    }
}

// ---------------------------------------------------------------------------
// Owner-edge ranges: bounds[g] = the first edge p whose work prefix reaches
// g / G of the total, moved back to the start of its filtration level (a
// level -- and so a tie group -- is never split across ranks).  The same
// function runs on the host (vrb_partition_bounds, CPU tests) and the device.
// ---------------------------------------------------------------------------
__host__ __device__ int64_t partition_bound(const uint64_t* prefix, const uint32_t* efilt, int64_t E, int g, int G) {
    if (g <= 0) return 0;
    if (g >= G) return E;
    const uint64_t W = prefix[E];
    const uint64_t target = (uint64_t)(((unsigned __int128)W * (uint64_t)g) / (uint64_t)G);
    int64_t lo = 0, hi = E;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (prefix[mid] < target) lo = mid + 1; else hi = mid;
    }
    while (lo > 0 && lo < E && efilt[lo - 1] == efilt[lo]) --lo;
    return lo;
}

__global__ void k_bounds(const uint64_t* __restrict__ prefix, const uint32_t* __restrict__ efilt, int64_t E, int G,
                         int64_t* __restrict__ bounds) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= G; g += gridDim.x * blockDim.x)
        bounds[g] = partition_bound(prefix, efilt, E, g, G);
}

// work of owner edge p for the triangle split: its scanned prefix length
__global__ void k_work_tri(const uint32_t* __restrict__ scan_len, int64_t E, uint64_t* __restrict__ w) {
    GRID_STRIDE(p, E) w[p] = scan_len[p];
}

// ... for the tetrahedron split: the pair tests of its apex set (|S| = the
// edge's triangle count) plus its prefix
__global__ void k_work_tet(const uint32_t* __restrict__ tcnt, const uint32_t* __restrict__ scan_len, int64_t E,
                           uint64_t* __restrict__ w) {
    GRID_STRIDE(p, E) {
        const uint64_t c = tcnt[p];
        w[p] = c * (c > 0 ? c - 1 : 0) / 2 + scan_len[p];
    }
}

__global__ void k_sum_slices(const uint32_t* __restrict__ all, int64_t E, int world, uint32_t* __restrict__ out) {
    GRID_STRIDE(p, E) {
        uint32_t s = 0;
        for (int r = 0; r < world; ++r) s += all[(int64_t)r * E + p];
        out[p] = s;
    }
}

// [lo, hi) of this rank for the per-edge work w (E entries)
void owner_range(const uint64_t* w, const uint32_t* efilt, int64_t E, int G, int g, cudaStream_t s, int64_t* b) {
    DBuf<uint64_t> pre(E + 1, s);
    exclusive_scan(w, pre.get(), E, s);
    DBuf<int64_t> bd(G + 1, s);
    k_bounds<<<(unsigned)ceil_div(G + 1, 64), 64, 0, s>>>(pre.get(), efilt, E, G, bd.get());
    VRB_LAUNCH_CHECK();
    VRB_CUDA(cudaMemcpyAsync(b, bd.get() + g, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
}

uint64_t read_u64(const uint64_t* p, cudaStream_t s) {
    uint64_t v = 0;
    VRB_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return v;
}

// Row blocks of the pair matrix: rank g gets rows [r_g, r_{g+1}), multiples
// of the distance tile, with about equal pair counts (row i has n - 1 - i).
std::vector<int64_t> row_blocks(int64_t n, int G) {
    const int64_t T = edge_tile();
    auto pairs_before = [&](int64_t i) { return (double)i * (double)n - (double)i * (double)(i + 1) / 2.0; };
    const double total = pairs_before(n);
    std::vector<int64_t> r(G + 1, 0);
    r[G] = n;
    for (int g = 1; g < G; ++g) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (pairs_before(mid) < total * g / G) lo = mid + 1; else hi = mid;
        }
        int64_t rb = ((lo + T / 2) / T) * T;
        if (rb >= n) rb = n;
        r[g] = std::max(r[g - 1], rb);
    }
    return r;
}

}  // namespace

// Host entry of the partition rule (tests): bounds[0..G] from host arrays.
void partition_bounds_host(const uint64_t* prefix, const uint32_t* efilt, int64_t E, int G, int64_t* bounds) {
    for (int g = 0; g <= G; ++g) bounds[g] = partition_bound(prefix, efilt, E, g, G);
}

void build_dist_impl(const double* X, int64_t n, int32_t d, const vrb_opts* opts, const vrb_comm* comm,
                     cudaStream_t s, DistOut& o) {
    const Comm C{comm, s};
    const int G = C.world(), rk = C.rank();
    const int K = opts->maxdim + 1;
    const bool strict = (opts->flags & VRB_STRICT_RADIUS) != 0;
    StageTimer& timer = *o.timer;
    timer.begin(6);

    // ---- S1: rank 0 places the points, everyone receives them
    DBuf<double> Xd((size_t)(n * d), s);
    {
        DBuf<int64_t> hdr(1, s);
        int64_t bad = 0;
        if (rk == 0) {
            bad = place_points(X, n, d, opts->flags, s, Xd, true) ? 0 : 1;
        }
        VRB_CUDA(cudaMemcpyAsync(hdr.get(), &bad, sizeof(bad), cudaMemcpyHostToDevice, s));
        C.bcast(hdr.get(), sizeof(int64_t), 0);
        VRB_CUDA(cudaMemcpyAsync(&bad, hdr.get(), sizeof(bad), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        if (bad) fail(VRB_EINVAL, "non-finite coordinate in the point cloud (checked on rank 0)");
        if (n * d) C.bcast(Xd.get(), (size_t)(n * d) * sizeof(double), 0);
    }
    timer.mark(6);
    timer.begin(0);
    // ---- S2: this rank's row block
    KeptEdges ke;
    const std::vector<int64_t> rows = row_blocks(n, G);
    build_kept_edges(Xd.get(), n, d, opts->radius, strict, s, ke, rows[rk], rows[rk + 1] == n ? -1 : rows[rk + 1]);
    Xd.reset();
    timer.mark(0);
    timer.begin(1);
    // ---- S3: local sort, all-gather of the runs, merge
    DBuf<uint64_t> rkey, rij;   // this rank's run, padded to the longest
    const std::vector<uint64_t> Es = C.allgather_u64((uint64_t)ke.E);
    uint64_t Eg = 0, maxE = 0;
    for (uint64_t e : Es) { Eg += e; maxE = std::max(maxE, e); }
    if (Eg >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu kept edges exceed u32 positions", (unsigned long long)Eg);
    const int64_t E = (int64_t)Eg;
    rkey.alloc(std::max<uint64_t>(maxE, 1), s);
    rij.alloc(std::max<uint64_t>(maxE, 1), s);
    if (ke.E) {
        SortedEdges so;
        sort_edges(ke, s, so);
        k_make_run<<<grid_of(ke.E), 256, 0, s>>>(so.key, so.val, ke.E, so.bias, so.packed ? 1 : 0, ke.ei.get(),
                                                 ke.ej.get(), rkey.get(), rij.get());
        VRB_LAUNCH_CHECK();
    }
    ke = KeptEdges();
    timer.mark(1);
    timer.begin(6);
    DBuf<uint64_t> ak((size_t)G * std::max<uint64_t>(maxE, 1), s), ai((size_t)G * std::max<uint64_t>(maxE, 1), s);
    if (maxE) {
        C.allgather(rkey.get(), ak.get(), maxE * sizeof(uint64_t));
        C.allgather(rij.get(), ai.get(), maxE * sizeof(uint64_t));
    }
    rkey.reset();
    rij.reset();
    timer.mark(6);
    timer.begin(1);
    // merge rounds: adjacent runs merged pairwise into the other buffer
    // (the first round also compacts the maxE-strided runs), log2 G rounds
    DBuf<uint64_t> bk(std::max<int64_t>(E, 1), s), bi(std::max<int64_t>(E, 1), s);
    struct Run { uint64_t* k; uint64_t* i; int64_t n; };
    std::vector<Run> runs;
    for (int q = 0; q < G; ++q)
        runs.push_back({ak.get() + (size_t)q * maxE, ai.get() + (size_t)q * maxE, (int64_t)Es[q]});
    uint64_t* buf_k[2] = {bk.get(), ak.get()};
    uint64_t* buf_i[2] = {bi.get(), ai.get()};
    int dst = 0;
    do {
        std::vector<Run> next;
        int64_t at = 0;
        for (size_t q = 0; q < runs.size(); q += 2) {
            const Run A = runs[q];
            const Run B = q + 1 < runs.size() ? runs[q + 1] : Run{nullptr, nullptr, 0};
            const int64_t m = A.n + B.n;
            if (m) {
                k_merge<<<grid_of(ceil_div(m, kPer)), 256, 0, s>>>(A.k, A.i, A.n, B.k, B.i, B.n, buf_k[dst] + at,
                                                                  buf_i[dst] + at);
                VRB_LAUNCH_CHECK();
            }
            next.push_back({buf_k[dst] + at, buf_i[dst] + at, m});
            at += m;
        }
        runs.swap(next);
        dst ^= 1;
    } while (runs.size() > 1);
    const uint64_t* gk = runs.empty() ? nullptr : runs[0].k;
    const uint64_t* gi = runs.empty() ? nullptr : runs[0].i;
    o.E = E;
    o.ev = o.alloc_u32(2 * E);
    o.efilt = o.alloc_u32(E);
    o.vor = o.alloc_f64(E);
    o.nvals = 0;
    if (E) {
        dense_ranks(gk, o.efilt, E, s);
        k_edge_out<<<grid_of(E), 256, 0, s>>>(gk, gi, o.efilt, E, o.ev, o.vor);
        VRB_LAUNCH_CHECK();
        uint32_t nv = 0;
        VRB_CUDA(cudaMemcpyAsync(&nv, o.efilt + E - 1, sizeof(nv), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        o.nvals = nv;
    }
    ak.reset(); ai.reset(); bk.reset(); bi.reset();
    timer.mark(1);
    timer.begin(2);
    if (K < 2) return;

    // ---- S4: neighbour lists (every rank), S5: this rank's owner edges
    Graph g;
    build_lists(o.ev, n, E, s, g);
    timer.mark(2);
    timer.begin(3);
    int64_t tb[2] = {0, 0};
    if (E) {
        DBuf<uint64_t> w(E, s);
        k_work_tri<<<grid_of(E), 256, 0, s>>>(g.scan_len.get(), E, w.get());
        VRB_LAUNCH_CHECK();
        owner_range(w.get(), o.efilt, E, G, rk, s, tb);
    }
    build_plan(o.ev, tb[0], tb[1], s, g);
    DBuf<uint32_t> cnt(std::max<int64_t>(E, 1), s);
    DBuf<uint64_t> bmoff;
    DBuf<uint32_t> bm;
    TriRecords R;
    bool xmajor = E && records_apply(g);
    if (xmajor) {
        try {
            count_triangles_rec(g, o.ev, tb[0], tb[1], cnt.get(), R, s);
        } catch (const Error& e) {
            if (e.status != VRB_ENOMEM) throw;
            cudaGetLastError();
            R = TriRecords();
            xmajor = false;
        }
    }
    const bool use_bm = !xmajor && apex_bitmaps_apply(g);
    if (E && !xmajor) {
        if (use_bm) {
            uint64_t words = 0;
            apex_bitmap_offsets(g, bmoff, words, s);
            bm.alloc(words ? words : 1, s);
            count_triangles_bm(g, cnt.get(), bm.get(), bmoff.get(), s);
        } else {
            count_triangles(g, cnt.get(), 0, 1, s);
        }
    }
    DBuf<uint64_t> toff(E + 1, s);   // offsets inside this rank's slice (0 before tb[0])
    if (E) exclusive_scan(cnt.get(), toff.get(), E, s);
    else VRB_CUDA(cudaMemsetAsync(toff.get(), 0, sizeof(uint64_t), s));
    const uint64_t Tl = E ? read_u64(toff.get() + E, s) : 0;
    timer.mark(3);
    timer.begin(6);
    const std::vector<uint64_t> Ts = C.allgather_u64(Tl);
    uint64_t T = 0, t0 = 0, maxT = 0;
    for (int q = 0; q < G; ++q) {
        if (q < rk) t0 += Ts[q];
        T += Ts[q];
        maxT = std::max(maxT, Ts[q]);
    }
    timer.mark(6);
    timer.begin(3);
    if (T >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu triangles exceed u32 positions", (unsigned long long)T);
    o.T = T;
    o.t0 = t0;
    o.Tl = Tl;
    o.tv = o.alloc_u32(3 * Tl);
    o.tf = o.alloc_u32(Tl);
    o.trows = (opts->flags & VRB_SKIP_BOUNDARY) ? nullptr : o.alloc_u32(3 * Tl);
    DBuf<uint16_t> tapex;
    if (K >= 3 && n <= 65536) tapex.alloc((size_t)std::max<uint64_t>(Tl, 1), s);
    timer.mark(3);
    timer.begin(4);
    if (xmajor)
        fill_triangles_x(g, R, o.efilt, toff.get(), tb[0], tb[1], 0, o.tv, o.tf, o.trows, tapex.get(), s);
    else
        fill_triangles(g, o.efilt, toff.get(), tb[0], tb[1], 0, o.tv, o.tf, o.trows, tapex.get(), s, bm.get(),
                       bmoff.get());
    bm.reset();
    R = TriRecords();
    timer.mark(4);
    timer.begin(5);
    sort_tie_groups(2, o.efilt, toff.get(), E, tb[0], tb[1], n, o.tv, o.trows, s, o.ev);
    timer.mark(5);
    timer.begin(6);
    if (K < 3) return;

    // ---- S6: tetrahedra.  Exchange the per-edge triangle counts and the
    // triangles themselves (D_3's faces can be any earlier triangle).
    DBuf<uint32_t> tcnt(std::max<int64_t>(E, 1), s);
    DBuf<uint64_t> gtoff(E + 1, s);
    DBuf<uint32_t> tv_all(std::max<uint64_t>(3 * T, 1), s);
    DBuf<uint16_t> apex_all;
    if (n <= 65536) {
        apex_all.alloc(T + 16, s);   // padded: the face search reads 16-byte chunks past the end
        VRB_CUDA(cudaMemsetAsync(apex_all.get() + T, 0xFF, 16 * sizeof(uint16_t), s));
    }
    if (E) {
        DBuf<uint32_t> all((size_t)E * G, s);
        C.allgather(cnt.get(), all.get(), E * sizeof(uint32_t));
        k_sum_slices<<<grid_of(E), 256, 0, s>>>(all.get(), E, G, tcnt.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(tcnt.get(), gtoff.get(), E, s);
    } else {
        VRB_CUDA(cudaMemsetAsync(gtoff.get(), 0, sizeof(uint64_t), s));
    }
    if (maxT) {
        DBuf<uint32_t> sv(3 * maxT, s), rv((size_t)G * 3 * maxT, s);
        if (Tl) VRB_CUDA(cudaMemcpyAsync(sv.get(), o.tv, 3 * Tl * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        C.allgather(sv.get(), rv.get(), 3 * maxT * sizeof(uint32_t));
        uint64_t at = 0;
        for (int q = 0; q < G; ++q) {
            if (Ts[q])
                VRB_CUDA(cudaMemcpyAsync(tv_all.get() + 3 * at, rv.get() + (size_t)q * 3 * maxT,
                                         3 * Ts[q] * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            at += Ts[q];
        }
        if (apex_all.get()) {
            DBuf<uint16_t> sa(maxT, s), ra((size_t)G * maxT, s);
            if (Tl) VRB_CUDA(cudaMemcpyAsync(sa.get(), tapex.get(), Tl * sizeof(uint16_t), cudaMemcpyDeviceToDevice, s));
            C.allgather(sa.get(), ra.get(), maxT * sizeof(uint16_t));
            at = 0;
            for (int q = 0; q < G; ++q) {
                if (Ts[q])
                    VRB_CUDA(cudaMemcpyAsync(apex_all.get() + at, ra.get() + (size_t)q * maxT, Ts[q] * sizeof(uint16_t),
                                             cudaMemcpyDeviceToDevice, s));
                at += Ts[q];
            }
        }
    }
    tapex.reset();
    timer.mark(6);
    timer.begin(8);
    TriLevels L;
    L.apex = apex_all.get();
    L.ev = o.ev;
    L.n = n;
    triangle_levels(o.efilt, gtoff.get(), E, tv_all.get(), s, L);
    int64_t qb[2] = {0, 0};
    if (E) {
        DBuf<uint64_t> w(E, s);
        k_work_tet<<<grid_of(E), 256, 0, s>>>(tcnt.get(), g.scan_len.get(), E, w.get());
        VRB_LAUNCH_CHECK();
        owner_range(w.get(), o.efilt, E, G, rk, s, qb);
    }
    build_plan(o.ev, qb[0], qb[1], s, g);
    DBuf<uint32_t> qc(std::max<int64_t>(E, 1), s);
    if (E) count_tets(g, L, qc.get(), 0, 1, s);
    DBuf<uint64_t> qoff(E + 1, s);
    if (E) exclusive_scan(qc.get(), qoff.get(), E, s);
    else VRB_CUDA(cudaMemsetAsync(qoff.get(), 0, sizeof(uint64_t), s));
    const uint64_t Ql = E ? read_u64(qoff.get() + E, s) : 0;
    timer.mark(8);
    timer.begin(6);
    const std::vector<uint64_t> Qs = C.allgather_u64(Ql);
    uint64_t Q = 0, q0 = 0;
    for (int q = 0; q < G; ++q) {
        if (q < rk) q0 += Qs[q];
        Q += Qs[q];
    }
    timer.mark(6);
    timer.begin(8);
    if (Q >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu tetrahedra exceed u32 positions", (unsigned long long)Q);
    o.Q = Q;
    o.q0 = q0;
    o.Ql = Ql;
    o.qv = o.alloc_u32(4 * Ql);
    o.qf = o.alloc_u32(Ql);
    o.qrows = (opts->flags & VRB_SKIP_BOUNDARY) ? nullptr : o.alloc_u32(4 * Ql);
    timer.mark(8);
    timer.begin(9);
    fill_tets(g, L, o.efilt, qoff.get(), qb[0], qb[1], 0, o.qv, o.qf, o.qrows, s);
    timer.mark(9);
    timer.begin(5);
    sort_tie_groups(3, o.efilt, qoff.get(), E, qb[0], qb[1], n, o.qv, o.qrows, s);
    timer.mark(5);
}

}  // namespace vrb
