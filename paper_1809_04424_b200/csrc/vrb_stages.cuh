// vrb_stages.cuh -- the stages of the build as host
// launchers over device buffers.  Product path only.
#pragma once

#include <functional>

#include "vrb_internal.cuh"

namespace vrb {

// S1: device copy of the points, row-major n x d, finite-checked (a
// non-finite coordinate: VRB_EINVAL, or with soft a false return).
bool place_points(const double* X, int64_t n, int d, uint32_t flags, cudaStream_t s, DBuf<double>& out,
                  bool soft = false);

// d2 threshold equivalent to the cap on sqrt_rn(d2) (reading A1); < 0: none kept.
double cap_threshold(double r, bool strict);

// S2: kept edges in lexicographic (i, j) order with their length bits.
struct KeptEdges {
    int64_t E = 0;
    DBuf<uint64_t> key;   // bit pattern of len (non-negative doubles order as u64)
    int64_t n = 0;
    bool packed = false;  // n <= 65536: (i << 16 | j) in pij, else i, j in ei, ej
    DBuf<uint32_t> ei, ej, pij;
    DBuf<unsigned long long> range;   // when set: min, max, OR of the key bits (reduced by the distance pass)
};
// Rows [row_lo, row_hi) only (a rank's row block; row_lo and row_hi < n
// multiples of edge_tile(); row_hi = -1: to n): their pairs j > i.
void build_kept_edges(const double* X, int64_t n, int d, double radius, bool strict, cudaStream_t s,
                      KeptEdges& out, int64_t row_lo = 0, int64_t row_hi = -1);
int64_t edge_tile();

// F3: distance-matrix input.  place_matrix copies (if host) and checks D
// (n x n, off-diagonal finite, >= 0, symmetric; VRB_EINVAL otherwise);
// build_kept_edges_dm keeps i < j with D[i][j] <= r (< r strict) in lex order.
void place_matrix(const double* D, int64_t n, uint32_t flags, cudaStream_t s, DBuf<double>& out);
void build_kept_edges_dm(const double* D, int64_t n, double radius, bool strict, cudaStream_t s, KeptEdges& out);
// latlon2euc: latlon n x 2 degrees -> xyz n x 3 (device pointers).
void latlon2euc(const double* latlon, int64_t n, double* xyz, cudaStream_t s);

// S3: edge filtration order (len, i, j), dense ranks, value_of_rank.
//   ev    : 2E u32 (i, j) per edge in position order   (caller-allocated)
//   efilt : E u32 dense rank, 1-based                    (caller-allocated)
//   vor   : >= nvals f64, vor[f-1] = length of level f  (caller-allocated, E entries)
int64_t rank_edges(KeptEdges& ke, uint32_t* ev, uint32_t* efilt, double* vor, cudaStream_t s);
int last_edge_path();   // vrb_last_edge_path (this thread)
void note_edge_path(int path);
bool fused_edges_enabled();   // VRB_EDGE_PATH unset or "fused"
// The bucket path of rank_edges (edge_buckets.cu); false when it does not
// apply (then nothing was written and the radix path runs).
bool rank_edges_buckets(KeptEdges& ke, int64_t n, uint32_t* ev, uint32_t* efilt, double* vor, cudaStream_t s,
                        int64_t* nvals);
// Bucket parameters handed to the count and scatter passes of the bucket
// path (edge_buckets.cu): counts cnt[(bits - kmin) >> shift]; records of the
// buckets in [slices[slice], slices[slice + 1]) at atomicAdd(&cnt[b], 1).
struct FoldBk {
    uint64_t kmin = 0;
    int shift = 0, tz = 0, vb = 0, bn = 0;
    int64_t nb = 0;
    uint32_t* cnt = nullptr;
    uint64_t* rec = nullptr;
    const uint32_t* slices = nullptr;
    int slice = 0;
};
// The sort of rank_edges alone: key[q] + bias = length bits of the q-th edge
// in (len, i, j) order; val[q] = packed (i << 16 | j) when packed, else the
// lex index into ke.ei / ke.ej.  Buffers owned here or by ke (keep both alive).
struct SortedEdges {
    int64_t E = 0;
    bool packed = false;
    const uint64_t* key = nullptr;
    const uint32_t* val = nullptr;
    uint64_t bias = 0;
    DBuf<uint64_t> key_alt;
    DBuf<uint32_t> perm, perm_alt;
};
void sort_edges(KeptEdges& ke, cudaStream_t s, SortedEdges& so);

// S4: neighbourhoods of the edge graph, used by the simplex enumeration.
struct Graph {
    int64_t n = 0, E = 0;
    DBuf<uint64_t> off;        // n + 1: offsets of each vertex's 2E directed entries
    // per vertex, its neighbours in EDGE-POSITION order (the older-neighbour
    // prefix of an edge is a prefix of this list):
    DBuf<uint32_t> nkr;        // 2E: packed ? (krank << 16 | k) : k
    DBuf<uint32_t> nr;         // 2E: krank (only when !packed)
    DBuf<uint32_t> np;         // 2E: position of the entry's edge
    bool packed = false;       // n <= 65536 and every degree <= 65536
    //   krank = index of k in the vertex's neighbour-ID-ordered list
    DBuf<uint32_t> listidx;    // 2E: entry q = 2p + side -> index in the vertex's position list
    DBuf<uint2> idl;           // 2E (packed only): (k, pos of edge (v, k)) in neighbour-ID order
    // owner-edge enumeration plan (triangles and tetrahedra)
    DBuf<uint32_t> scan_v;     // E: endpoint whose older-neighbour prefix is scanned
    DBuf<uint32_t> scan_len;   // E: length of that prefix (older neighbours)
    DBuf<uint4> plan;          // E: per hosted slot (edge position p, scanned x, prefix length, deg x),
                               //    slots sorted by (host endpoint, longest prefix first)
    DBuf<uint32_t> hosted_v;   // E: host endpoint of each hosted slot
    DBuf<uint64_t> work_pre;   // nplan + 1: exclusive prefix of scan_len over hosted order
    int64_t nplan = 0;         // hosted slots in the plan (owner edges of [p_lo, p_hi))
    uint64_t work = 0;
    uint32_t max_deg = 0;
};
// build_graph = build_lists + build_plan over every owner edge
void build_graph(const uint32_t* ev, int64_t n, int64_t E, cudaStream_t s, Graph& g);
// the neighbour lists and the scanned endpoint of every edge (scan_v, scan_len)
void build_lists(const uint32_t* ev, int64_t n, int64_t E, cudaStream_t s, Graph& g);
// the owner-edge plan of the edges [p_lo, p_hi) only (plan, hosted_v, work_pre, nplan, work)
void build_plan(const uint32_t* ev, int64_t p_lo, int64_t p_hi, cudaStream_t s, Graph& g);

// S5 + S7 + S8 for triangles (owner-edge enumeration, see triangles.cu).
// Count per owner edge: cnt[p] (E entries, zero-initialised here).  The
// owner edges are split into work-balanced tasks; this call counts the tasks
// of part `part` of `nparts` (0 of 1 = all) and leaves the others at 0.
void count_triangles(const Graph& g, uint32_t* cnt, int part, int nparts, cudaStream_t s);
// Apex bitmaps (single rank, packed lists, max degree <= kApexBitmapMaxDeg):
// the count pass also stores, per hosted slot e, the bitmap of the valid apexes
// by rank in the scanned endpoint's id-ordered list at bm + bmoff[e]
// (ceil(deg x / 32) words); the fill then emits from the bitmaps.
constexpr uint32_t kApexBitmapMaxDeg = 8192;
bool apex_bitmaps_apply(const Graph& g);
bool markfill_apply(const Graph& g);
void apex_bitmap_offsets(const Graph& g, DBuf<uint64_t>& bmoff, uint64_t& words, cudaStream_t s);
void count_triangles_bm(const Graph& g, uint32_t* cnt, uint32_t* bm, const uint64_t* bmoff, cudaStream_t s);
// Emit triangles of owner edges in [p_lo, p_hi) at slots toff[p] - slot0
// (slot0 = toff[p_lo]).  apex (nullable; n <= 65536): each triangle's vertex
// off its owner edge, for the face-position search of tetrahedra.
void fill_triangles(const Graph& g, const uint32_t* efilt, const uint64_t* toff, int64_t p_lo, int64_t p_hi,
                    uint64_t slot0, uint32_t* tv, uint32_t* tf, uint32_t* rows, uint16_t* apex, cudaStream_t s,
                    const uint32_t* bm = nullptr, const uint64_t* bmoff = nullptr);
// x-major triangle path (triangles.cu, "records"; packed lists, degrees <=
// kApexBitmapMaxDeg): the count (hosted by y) stores per owner edge the
// validity bits of its scanned prefix and the host positions of its valid
// apexes; the fill runs per scanned vertex x with x's list in shared memory.
struct TriRecords {
    DBuf<uint64_t> rec_off, tb_off;   // E + 1 each: per owner edge (0 outside [p_lo, p_hi))
    DBuf<uint32_t> rec, tb;
    DBuf<uint4> fplan;                // fill plan (p, host y, len, deg x), grouped by scanned x
    DBuf<uint32_t> fgroup_v;
    DBuf<uint64_t> fwork_pre;
    int64_t nfplan = 0;
    uint64_t fwork = 0;
};
bool records_apply(const Graph& g);
void count_triangles_rec(const Graph& g, const uint32_t* ev, int64_t p_lo, int64_t p_hi, uint32_t* cnt,
                         TriRecords& R, cudaStream_t s);
void fill_triangles_x(const Graph& g, const TriRecords& R, const uint32_t* efilt, const uint64_t* toff, int64_t p_lo,
                      int64_t p_hi, uint64_t slot0, uint32_t* tv, uint32_t* tf, uint32_t* rows, uint16_t* apex,
                      cudaStream_t s);
void build_fill_plan(const uint32_t* ev, int64_t p_lo, int64_t p_hi, cudaStream_t s, const Graph& g,
                     DBuf<uint4>& plan, DBuf<uint32_t>& group_v, DBuf<uint64_t>& work_pre, int64_t& m_out,
                     uint64_t& work);
// Reorder the k-simplices (k = 2, 3) of every tie group (>= 2 edges sharing a
// level) into lex order (readings A3, A4); only owner edges in [p_lo, p_hi).
// off = per-owner-edge simplex offsets (E + 1); verts/rows: (k+1) u32 each.
// ev (2E edge endpoints, nullable): lets the triangle path recompute D_2 rows
// from an edge-position table instead of carrying them through the sort.
void sort_tie_groups(int k, const uint32_t* efilt, const uint64_t* off, int64_t E, int64_t p_lo, int64_t p_hi,
                     int64_t n, uint32_t* verts, uint32_t* rows, cudaStream_t s, const uint32_t* ev = nullptr);

// S6 + S7 + S8 for tetrahedra (tetrahedra.cu).  Needs the complete triangle
// arrays of dimension 2 (face positions for D_3).
struct TriLevels {
    const uint64_t* toff = nullptr;   // E + 1 triangle offsets per owner edge
    const uint32_t* tv = nullptr;     // 3T vertices (global order)
    const uint16_t* apex = nullptr;   // T: apex of each triangle (owner-edge search); null -> hash
    const uint32_t* ev = nullptr;     // 2E edge endpoints in position order
    int64_t n = 0;
    DBuf<uint32_t> dense;             // n x n edge positions (n <= 16384 with apex), NONE32 = no edge
    DBuf<uint64_t> tlo, thi;          // E: triangle range of each edge's filtration level
    DBuf<uint4> frec;                 // 2E: face record per owner edge (first triangle, count | shared flag,
                                      // 12 apex separators)
    DBuf<ulonglong2> hslots;          // (triangle lex code, position), open addressing
    uint64_t hmask = 0;
};
void triangle_levels(const uint32_t* efilt, const uint64_t* toff, int64_t E, const uint32_t* tv, cudaStream_t s,
                     TriLevels& L);
// largest n for which K = 3 (tetrahedra) is supported (VRB_ENOTSUP above)
int64_t tets_max_n();
void count_tets(const Graph& g, const TriLevels& L, uint32_t* cnt, int part, int nparts, cudaStream_t s);
void fill_tets(const Graph& g, const TriLevels& L, const uint32_t* efilt, const uint64_t* qoff, int64_t p_lo,
               int64_t p_hi, uint64_t slot0, uint32_t* qv, uint32_t* qf, uint32_t* rows, cudaStream_t s);


// F4 (gf2.cu): S = D + C E over GF(2); writes colptr_out (ncols + 1) and
// returns nnz(S) with its rows allocated through alloc_rows.
int64_t gf2_blockprodsum(int64_t nrows, int64_t ncols, int64_t kdim, const uint64_t* dcp, const uint32_t* drv,
                         const uint64_t* ccp, const uint32_t* crv, const uint64_t* ecp, const uint32_t* erv,
                         cudaStream_t s, uint64_t* colptr_out, uint32_t* (*alloc_rows)(int64_t, void*), void* ctx,
                         uint32_t** rowval_out);

// F1 (h0.cu): minimum spanning forest of the edges under the position order
// (Boruvka); returns its size and (through alloc_out) its positions ascending
// and their filt.
int64_t h0_forest(const uint32_t* ev, const uint32_t* efilt, int64_t n, int64_t E, cudaStream_t s,
                  uint32_t* (*alloc_out)(int64_t, void*), void* ctx, uint32_t** pos_out, uint32_t** death_out);   // largest n the shared-memory vertex map supports

// F1 "clear and compress" (h0.cu): D_2 (ncols columns of 3 rows) without
// the rows of the forest edges; colptr (ncols + 1, caller), rows renumbered
// densely, rowmap (new row -> edge position); returns nnz.
int64_t compress_d2(const uint32_t* forest, int64_t nf, int64_t E, const uint32_t* rows, int64_t ncols,
                    cudaStream_t s, uint64_t* colptr, uint32_t* (*alloc_out)(int64_t, void*), void* ctx,
                    uint32_t** rowval_out, uint32_t** rowmap_out, int64_t* nrows_out);

// Multi-GPU build (dist.cu).  Outputs are allocated through the callbacks
// (handle-owned); this rank's slices of dimensions 2 and 3.
struct DistOut {
    StageTimer* timer = nullptr;
    std::function<uint32_t*(size_t)> alloc_u32;
    std::function<double*(size_t)> alloc_f64;
    int64_t E = 0, nvals = 0;
    uint32_t* ev = nullptr;
    uint32_t* efilt = nullptr;
    double* vor = nullptr;
    uint64_t T = 0, t0 = 0, Tl = 0;
    uint32_t *tv = nullptr, *tf = nullptr, *trows = nullptr;
    uint64_t Q = 0, q0 = 0, Ql = 0;
    uint32_t *qv = nullptr, *qf = nullptr, *qrows = nullptr;
};
void build_dist_impl(const double* X, int64_t n, int32_t d, const vrb_opts* opts, const vrb_comm* comm,
                     cudaStream_t s, DistOut& o);
// The owner-edge partition rule (host copy of the device one, for tests):
// bounds[g], g = 0..G, over the work prefix (E + 1 entries).
void partition_bounds_host(const uint64_t* prefix, const uint32_t* efilt, int64_t E, int G, int64_t* bounds);

}  // namespace vrb
