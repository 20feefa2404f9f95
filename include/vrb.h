/*
 * vrb.h -- C ABI of libvrb.so, the B200 (sm_100a) Vietoris-Rips filtration
 * and boundary-matrix build (the data-parallel hot path of Eirene profiled in
 * Hylton, Henselman-Petrusek, Sang, Short, arXiv:1809.04424).
 *
 * Citations: P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md,
 * SURVEY 8(x) = /root/repo/SURVEY.md section 8.  Readings A1..A14 of the
 * paper (inclusive cap, dense ranks, lex tie-break, ...) are listed in
 * DESIGN.md "Readings".
 *
 * Problem statement: C = eirene(x; upperlim, bettimax)
 * -- a point cloud, the maximum homology dimension and an optional radius --
 * gives ranked edges, ranked simplices and the boundary operator whose rows
 * and columns are simplices in filtration order.
 *
 * Conventions (all entry points):
 *  - extern "C", no exceptions cross the ABI; every call returns vrb_status.
 *  - indices are 0-based; vertex ids are u32; positions are u32 (a count that
 *    would not fit u32 returns VRB_EOVERFLOW); colptr offsets are u64.
 *  - "device" pointers are CUDA device memory of the current device; "host"
 *    pointers are ordinary (optionally pinned) host memory.
 *  - work is ordered on the caller's cudaStream_t (0 = legacy default
 *    stream).  A call blocks only at internal count read-backs that size its
 *    allocations, and is complete on the stream when it returns.
 *  - On error no handle is produced, nothing leaks, and vrb_last_error()
 *    holds a one-line description (thread-local, valid until the next vrb_*
 *    call on the same thread).
 *  - Thread safety: distinct handles may be used concurrently; one handle
 *    must not be used by two threads at once.
 */
#ifndef VRB_H
#define VRB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VRB_ABI_VERSION 2

typedef enum {
    VRB_OK = 0,
    VRB_EINVAL = 1,     /* bad argument: n < 0, d < 1, maxdim not in 0..2,
                           radius NaN or < 0, non-finite coordinate,
                           dim / k out of range in an accessor, NaN key */
    VRB_ENOMEM = 2,     /* an allocation (through the allocator hook) failed */
    VRB_EOVERFLOW = 3,  /* a count needs more than 32 bits where the layout
                           stores u32 positions (E, T, Q >= 2^32), or n >= 2^21 */
    VRB_ECUDA = 4,      /* CUDA runtime error; text in vrb_last_error() */
    VRB_ECOMM = 5,      /* the collective callback of vrb_build_dist failed
                           (SURVEY 8(b)'s VRB_ENCCL: the callbacks run NCCL or gloo) */
    VRB_ENOTSUP = 6     /* configuration outside what this build implements:
                           maxdim 2 with n above the tetrahedron kernels'
                           shared-memory map (38 784 on a B200; checked before
                           any work) -- DESIGN.md section 10 "Limits" */
} vrb_status;
/* SURVEY 8(b)'s name for the collective error (the collectives are NCCL when
 * the callbacks use torch.distributed's NCCL backend). */
#define VRB_ENCCL VRB_ECOMM

/* vrb_opts.flags */
#define VRB_STRICT_RADIUS    0x1u  /* keep len < radius instead of len <= radius (reading A1) */
#define VRB_DIM_MAJOR        0x2u  /* X is d x n (rowsare="dimensions") */
#define VRB_POINTS_ON_DEVICE 0x4u  /* X is a device pointer (else host; copied H2D inside) */
#define VRB_SKIP_BOUNDARY    0x8u  /* do not materialise the D_k row arrays (k >= 2) */

typedef struct {
    int32_t maxdim;   /* homology dimension: simplices are built up to
                         K = maxdim + 1 (reading A6); 0, 1 or 2 */
    double radius;    /* upperlim: >= 0 or +INFINITY */
    uint32_t flags;   /* VRB_* flags above */
} vrb_opts;

typedef struct vrb_result* vrb_handle;   /* opaque; owns all device outputs */

/* Allocator hook (e.g. PyTorch's caching allocator; SURVEY 8(b) "library-
 * owned device outputs ... allocated through the hook").  The paper's own
 * native calls take caller-allocated buffers; here the sizes are
 * only known after the count passes, so the library allocates.  Both calls are made on
 * the build's stream and device.  alloc returns NULL on failure.  The default
 * (hook unset or set to NULL) is cudaMallocAsync / cudaFreeAsync.  Process-
 * wide; set it before any build, never while a build runs. */
typedef void* (*vrb_alloc_fn)(size_t bytes, int device, void* stream, void* ctx);
typedef void (*vrb_free_fn)(void* ptr, size_t bytes, int device, void* stream, void* ctx);

int vrb_abi_version(void);
const char* vrb_last_error(void);
vrb_status vrb_set_allocator(vrb_alloc_fn alloc, vrb_free_fn free_fn, void* ctx);

/* Build the filtration for n points of dimension d.
 *   X      : n x d float64, row-major (points are rows) unless VRB_DIM_MAJOR;
 *            host memory unless VRB_POINTS_ON_DEVICE.  Read-only, caller-owned.
 *   opts   : maxdim, radius, flags (above).
 *   stream : cudaStream_t (as void*).
 *   out    : receives the handle; release with vrb_free.
 * Method (P:107-113 VR construction, P:929-941 ranking, P:251 order):
 *   len(i,j) = sqrt_rn(fold_c (x_ic - x_jc)^2) in coordinate order, binary64
 *   round-to-nearest, no contraction (reading A5); an edge is kept iff
 *   len <= radius (len < radius with VRB_STRICT_RADIUS); edge filt = dense
 *   rank of len (1-based, ties share a level, reading A3); a k-simplex's filt
 *   is the max filt of its edges; each dimension is ordered by (filt, lex
 *   vertex tuple) (reading A4).  Errors: VRB_EINVAL, VRB_ENOMEM,
 *   VRB_EOVERFLOW, VRB_ECUDA. */
vrb_status vrb_build(const double* X, int64_t n, int32_t d, const vrb_opts* opts,
                     void* stream, vrb_handle* out);

/* Collective callbacks for vrb_build_dist.  All buffers are DEVICE pointers
 * and every call is ordered on `stream` (the build's stream): the callee
 * must enqueue its collective after the work already on that stream and the
 * library's later work must see its result (e.g. torch.distributed NCCL
 * collectives issued with `stream` as the current stream).  Return 0 on
 * success; anything else makes the build fail with VRB_ECOMM.
 *   allgather: recv (world * bytes) <- every rank's `bytes` bytes of send,
 *              in rank order;
 *   broadcast: buf (bytes) on every rank <- buf of rank `root`. */
typedef int (*vrb_allgather_fn)(const void* send, void* recv, size_t bytes, void* stream, void* ctx);
typedef int (*vrb_bcast_fn)(void* buf, size_t bytes, int root, void* stream, void* ctx);

typedef struct {
    int32_t rank;
    int32_t world;            /* >= 1 */
    vrb_allgather_fn allgather;
    vrb_bcast_fn broadcast;
    void* ctx;                /* passed to the callbacks */
} vrb_comm;

/* Multi-GPU build, one process per GPU (the paper's column
 * partition with its colptr fix-up "one after the other", is
 * here an exclusive scan of per-rank totals).  Every rank calls it with the
 * same n, d and opts; X is read on rank 0 only (other ranks may pass NULL).
 *   S1   rank 0 places and checks the points and broadcasts them;
 *   S2   each rank computes the distances of one row block of the pair
 *        matrix (tile-aligned, balanced by pair count);
 *   S3   each rank sorts its kept edges; the sorted runs are all-gathered
 *        (16 bytes per edge) and merged, so every rank holds the global edge
 *        order, the dense ranks and value_of_rank;
 *   S4   the neighbour lists are rebuilt on every rank (the one replicated
 *        stage);
 *   S5-8 each rank counts, fills and tie-sorts the triangles of one range of
 *        owner edges (level-aligned, balanced by enumeration work); its slice
 *        starts at the exclusive prefix of the per-rank totals (world x 8
 *        bytes all-gathered);
 *   S6   with maxdim 2, the per-edge triangle counts and the triangle
 *        vertices are all-gathered, then tetrahedra are partitioned the same
 *        way.
 * The slices of dimensions 2 and 3, concatenated in rank order, are
 * byte-identical to vrb_build's arrays (pin P13).  Edges (dimension 1) are
 * held whole by every rank; vrb_count reports the slice
 * [E rank / world, E (rank + 1) / world).  Errors as vrb_build (raised on
 * every rank alike, e.g. a non-finite coordinate found on rank 0) plus
 * VRB_ECOMM. */
vrb_status vrb_build_dist(const double* X, int64_t n, int32_t d, const vrb_opts* opts,
                          const vrb_comm* comm, void* stream, vrb_handle* out);

/* The owner-edge partition rule of vrb_build_dist, on HOST arrays (for
 * tests and planning): prefix = E + 1 exclusive work prefix over the edge
 * positions, efilt = E edge levels; bounds (world + 1) receives the first
 * owner edge of each rank: the first p whose prefix reaches g / world of
 * the total, moved back to the start of its level.  VRB_EINVAL on NULL
 * pointers, E < 0 or world < 1. */
vrb_status vrb_partition_bounds(const uint64_t* prefix, const uint32_t* efilt, int64_t E, int32_t world,
                                int64_t* bounds);

/* Counts of dimension dim (0..K) -- the "size of complex" per dimension the
 * paper tabulates (Table OSCmach; C(n, k+1) at full filtration,
 * pin P5): global_n = size of the whole dimension;
 * local_off/local_n = this handle's slice (the whole for vrb_build).  Any
 * output pointer may be NULL.  dim out of range -> VRB_EINVAL. */
vrb_status vrb_count(vrb_handle h, int32_t dim, int64_t* global_n, int64_t* local_off,
                     int64_t* local_n);

/* Simplices of dimension dim in 1..K in filtration order ("ordered
 * according to t"; ties by lex order, reading A4) -- this handle's
 * slice: verts = (dim+1)
 * u32 per simplex, ascending vertex ids, filtration order; filt = u32 level
 * per simplex (vertices, dim 0, are implicit: id order, filt 0).  Device
 * pointers owned by the handle. */
vrb_status vrb_simplices(vrb_handle h, int32_t dim, const uint32_t** verts_dev,
                         const uint32_t** filt_dev);

/* value_of_rank (the paper's ranking of the distance entries into integer
 * filtration levels, with Eirene's "filtration" values P:439-442):
 * nvals float64 lengths, value_of_rank[f-1] = length of level f
 * (strictly increasing; level 0 = vertices = 0.0).  Device, owned. */
vrb_status vrb_rank_values(vrb_handle h, const double** value_of_rank_dev, int64_t* nvals);

/* Boundary matrix D_k, k in 1..K: column j (this handle's
 * slice) has the k+1 rows rowval[(k+1)j .. (k+1)j+k], strictly ascending, each
 * the POSITION of a face in the dimension k-1 filtration order (reading A7).
 * colptr is implicit, (k+1)j.  D_1's rows are the vertex ids, so rowval of
 * D_1 aliases the edge vertex array.  nrows = global size of dim k-1, ncols =
 * local size of dim k.  VRB_SKIP_BOUNDARY builds -> VRB_EINVAL for k >= 2. */
vrb_status vrb_boundary(vrb_handle h, int32_t k, int64_t* nrows, int64_t* ncols,
                        const uint32_t** rowval_dev);

/* Materialise colptr (u64, ncols+1 entries, global offsets (k+1)(local_off+j))
 * into caller device memory on `stream`. */
vrb_status vrb_boundary_colptr(vrb_handle h, int32_t k, uint64_t* colptr_dev, void* stream);

/* Release every device output of the handle (through the allocator hook
 * that allocated it).  NULL is a no-op. */
vrb_status vrb_free(vrb_handle h);

/* Build from a distance matrix ("x is either a
 * point cloud ... or a square symmetric matrix (typically a pairwise distance
 * matrix)"; HIV's Hamming matrix P:520-521).  Same outputs and opts as
 * vrb_build, with S1-S2 replaced by: edge (i, j), i < j, has length
 * D[i*n + j] (+0.0, so -0.0 is 0.0); kept iff length <= radius (< with
 * VRB_STRICT_RADIUS).  D: n x n row-major f64, host (copied H2D) or device
 * (VRB_POINTS_ON_DEVICE), caller-owned, read-only.  VRB_EINVAL if an
 * off-diagonal entry is negative, NaN or infinite, if D[i][j] != D[j][i]
 * (the diagonal is not read), or with VRB_DIM_MAJOR. */
vrb_status vrb_build_dm(const double* D, int64_t n, const vrb_opts* opts, void* stream, vrb_handle* out);

/* latlon2euc (sec. 3): latlon_dev n x 2 f64 (latitude, longitude
 * in degrees, one point per row) -> xyz_dev n x 3 f64 on the unit sphere,
 * (cos lat cos lon, cos lat sin lon, sin lat); device pointers, caller-owned;
 * the result is complete when the call returns.  CUDA's sincos is within
 * 1 ulp (not bit-identical to a host libm). */
vrb_status vrb_latlon2euc(const double* latlon_dev, int64_t n, double* xyz_dev, void* stream);

/* Dimension-0 persistence from the ranked edges (Algorithm 1
 * P:210-227 on D_1, Pers/Barcode P:251-260, Fig. 4 caption P:286, readings
 * A8/A13).  Every vertex is born at filtration 0; edge position e pairs with
 * a vertex row iff e joins two components of the edges before it, i.e. iff e
 * is in the minimum spanning forest under the total (filt, lex) edge order.
 *   forest_pos : device, handle-owned: the n_finite forest edge positions,
 *                ascending (the D_1 pivot columns -- the columns "clear and
 *                compress" removes from the next reduction)
 *   death_filt : device, handle-owned: filt of those edges, so the finite
 *                dim-0 bars are [0, death_filt[i]) (integer levels; real
 *                values via vrb_rank_values; zero-length bars are included)
 *   n_finite   : number of finite bars (= n - n_essential)
 *   n_essential: number of [0, inf) bars = connected components at the cap
 * Computed on the first call (O(log n) Boruvka rounds on `stream`), cached in
 * the handle.  Any pointer may be NULL.  Handles of vrb_build_dist hold every
 * edge on every rank, so each rank gets the whole (identical) result. */
vrb_status vrb_h0(vrb_handle h, void* stream, const uint32_t** forest_pos, const uint32_t** death_filt,
                  int64_t* n_finite, int64_t* n_essential);

/* "Clear and compress" of D_2 ("a preprocessing step
 * motivated by homological algebra, which reduces the size of the boundary
 * operator before it is passed to either Pers or LU", after Bauer, Kerber
 * and Reininghaus).  The pivots of a reduced D_2 lie in the rows of edges
 * whose own D_1 column reduces to zero; the other edges -- the D_1 pivot
 * columns, i.e. the H0 forest of vrb_h0 -- are removed from D_2's rows,
 * which leaves every pivot pair (every dimension-1 bar) unchanged.
 * Output (device, handle-owned, computed on the first call on `stream` and
 * cached; vrb_h0 runs first if it has not):
 *   nrows  : E - (forest size): the edges kept as rows
 *   nnz    : entries of the compressed matrix
 *   colptr : this handle's D_2 columns + 1 u64 offsets (column j of the
 *            slice = rows rowval[colptr[j] .. colptr[j+1]), ascending)
 *   rowval : u32 compressed row indices (nnz of them are meaningful; the
 *            allocation holds 3 x columns, the bound known before the pass)
 *   rowmap : nrows u32, compressed row -> edge position (ascending)
 * A column keeps 1 to 3 rows (a forest holds no triangle's three edges).
 * VRB_EINVAL without dimension 2 or with VRB_SKIP_BOUNDARY. */
vrb_status vrb_compress_d2(vrb_handle h, void* stream, int64_t* nrows, int64_t* nnz, const uint64_t** colptr,
                           const uint32_t** rowval, const uint32_t** rowmap);

/* sortperm (Fig. GPU_sortperm) on device: perm_dev gets
 * the 0-based stable ascending permutation of keys_dev (n doubles; -0.0 ==
 * +0.0; NaN -> VRB_EINVAL), dense_rank_dev (nullable) gets 1-based dense ranks
 * (equal keys share a rank, reading A3).  All pointers device, caller-owned. */
vrb_status vrb_sortperm_f64(const double* keys_dev, int64_t n, int64_t* perm_dev,
                            uint32_t* dense_rank_dev, void* stream);

/* blockprodsum (sec. 4.6, Fig. BlkProdSum): the
 * Schur-complement product-sum of Eirene's reduction, S = D + C E over GF(2)
 * ("using the modulo-2 operation"), all CSC with 0-based rows.
 *   D : nrows x ncols   (d_colptr: ncols+1 u64, d_rowval: u32 < nrows)
 *   C : nrows x k       (c_colptr: k+1 u64,     c_rowval: u32 < nrows)
 *   E : k x ncols       (e_colptr: ncols+1 u64, e_rowval: u32 < k)
 * Rows within an input column need not be sorted; duplicates cancel in
 * pairs.  All pointers device, caller-owned, read-only.  The result is
 * handle-owned: S's rows are ascending within each column; vrb_gf2_csc gives
 * nnz, colptr (ncols+1 u64) and rowval (nnz u32).  VRB_EINVAL if an index is
 * out of range; VRB_EOVERFLOW if the candidate count (nnz(D) + sum over E of
 * the C columns it selects) reaches 2^32. */
typedef struct vrb_gf2* vrb_gf2_handle;
vrb_status vrb_gf2_blockprodsum(int64_t nrows, int64_t ncols, int64_t k, const uint64_t* d_colptr,
                                const uint32_t* d_rowval, const uint64_t* c_colptr, const uint32_t* c_rowval,
                                const uint64_t* e_colptr, const uint32_t* e_rowval, void* stream,
                                vrb_gf2_handle* out);
vrb_status vrb_gf2_csc(vrb_gf2_handle h, int64_t* nnz, const uint64_t** colptr_dev, const uint32_t** rowval_dev);
vrb_status vrb_gf2_free(vrb_gf2_handle h);

/* Stage timings of the last build on this thread (milliseconds, CUDA events
 * on the build stream): [0] points + distances S1-S2, [1] edge sort + ranks
 * S3, [2] neighbourhood lists S4, [3] simplex count + offsets + output
 * allocation, [4] simplex fill kernel S5/S6+S8 alone, [5] tie-group sort S7,
 * [6] exchange (vrb_build_dist), [7] total.  Recorded only while profiling
 * is enabled (events add no synchronisation inside the build).
 * vrb_last_stage_ms_n(ms, n) writes the first n of the extended list, which
 * appends [8] tetrahedron count (levels, count pass, offsets, allocation) and
 * [9] the tetrahedron fill kernel S6/S8 alone; with maxdim >= 2 slot [4]
 * holds the triangle fill only and [5] both tie-group sorts.  Entries past
 * [9] are written as 0.  Errors: VRB_EINVAL for a NULL `ms` or n < 0. */
vrb_status vrb_set_profiling(int32_t enable);
vrb_status vrb_last_stage_ms(double* ms8);
vrb_status vrb_last_stage_ms_n(double* ms, int32_t n);

/* Which S3 edge-ranking path the last vrb_build / vrb_build_dm on this thread
 * took: 1 = bucket scatter + on-chip finish (SURVEY 8(d) "Edges work the
 * same way"; edge_buckets.cu), 0 = LSD radix passes (ties or spiky length
 * distributions: a bucket over 2048 edges), -1 = no build yet or no edges.
 * Both give the same arrays (the (len, i, j) order of P:929-936, A3/A4). */
int32_t vrb_last_edge_path(void);

/* Number of kernels this library has launched in this process (monotonic;
 * the difference across a region is the number of launches inside it). */
unsigned long long vrb_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* VRB_H */
