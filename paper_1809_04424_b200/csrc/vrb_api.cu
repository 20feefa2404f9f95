// vrb_api.cu -- the C ABI of libvrb.so (include/vrb.h): argument checks,
// allocator hook, stage orchestration, result handle and accessors.
#include <cmath>
#include <cstring>
#include <atomic>
#include <mutex>
#include <new>

#include <nvtx3/nvToolsExt.h>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string t_last_error;
static thread_local double t_stage_ms[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
static bool g_profiling = false;

void fail(vrb_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw Error{st, std::string(buf)};
}

bool profiling_enabled() { return g_profiling; }

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// allocator hook
// ---------------------------------------------------------------------------
static vrb_alloc_fn g_alloc = nullptr;
static vrb_free_fn g_free = nullptr;
static void* g_ctx = nullptr;
static std::once_flag g_pool_once[64];

static int current_device() {
    int dev = 0;
    VRB_CUDA(cudaGetDevice(&dev));
    return dev;
}

void* dalloc(size_t bytes, cudaStream_t s) {
    if (bytes == 0) return nullptr;
    const int dev = current_device();
    void* p = nullptr;
    if (g_alloc) {
        p = g_alloc(bytes, dev, (void*)s, g_ctx);
        if (!p) fail(VRB_ENOMEM, "allocator hook failed for %zu bytes", bytes);
        return p;
    }
    std::call_once(g_pool_once[dev & 63], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? VRB_ENOMEM : VRB_ECUDA, "cudaMallocAsync(%zu): %s", bytes,
             cudaGetErrorString(e));
    }
    return p;
}

void dfree(void* p, size_t bytes, cudaStream_t s) {
    if (!p) return;
    if (g_free) {
        g_free(p, bytes, current_device(), (void*)s, g_ctx);
        return;
    }
    cudaFreeAsync(p, s);   // never throws (called from destructors)
}

Alloc dalloc_owned(size_t bytes, cudaStream_t s) {
    Alloc a;
    a.p = dalloc(bytes, s);
    a.bytes = bytes;
    a.fn = g_free;
    a.ctx = g_ctx;
    return a;
}

void dfree_owned(const Alloc& a) {
    if (!a.p) return;
    if (a.fn) {
        a.fn(a.p, a.bytes, current_device(), nullptr, a.ctx);
        return;
    }
    cudaFreeAsync(a.p, 0);
}

int device_sm_count() {
    static int cached[64] = {0};
    const int dev = current_device();
    if (!cached[dev & 63]) {
        int v = 0;
        VRB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        cached[dev & 63] = v;
    }
    return cached[dev & 63];
}

size_t device_max_smem_optin() {
    static int cached[64] = {0};
    const int dev = current_device();
    if (!cached[dev & 63]) {
        int v = 0;
        VRB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        cached[dev & 63] = v;
    }
    return (size_t)cached[dev & 63];
}

// ---------------------------------------------------------------------------
// stage timer
// ---------------------------------------------------------------------------
void StageTimer::start(cudaStream_t st) {
    on = g_profiling;
    s = st;
    if (!on) return;
    cudaEvent_t e;
    VRB_CUDA(cudaEventCreate(&e));
    VRB_CUDA(cudaEventRecord(e, s));
    marks.push_back({-1, e});
}

// NVTX ranges per stage ("vrb/S2 distance", ...; visible to nsys / ncu
// --nvtx): begin(stage) opens one, the next mark() closes it.
static const char* stage_name(int st) {
    switch (st) {
        case 0: return "vrb/S1-S2 points+distance";
        case 1: return "vrb/S3 edge rank";
        case 2: return "vrb/S4 neighbour lists";
        case 3: return "vrb/S5 count+offsets";
        case 4: return "vrb/S5-S8 triangle fill";
        case 5: return "vrb/S7 tie-group sort";
        case 6: return "vrb/exchange";
        case 8: return "vrb/S6 tetrahedron count";
        case 9: return "vrb/S6-S8 tetrahedron fill";
        default: return "vrb/stage";
    }
}

void StageTimer::begin(int stage) {
    if (nvtx_open) nvtxRangePop();
    nvtxRangePushA(stage_name(stage));
    nvtx_open = true;
}

void StageTimer::mark(int stage) {
    if (nvtx_open) {
        nvtxRangePop();
        nvtx_open = false;
    }
    if (!on) return;
    cudaEvent_t e;
    VRB_CUDA(cudaEventCreate(&e));
    VRB_CUDA(cudaEventRecord(e, s));
    marks.push_back({stage, e});
}

void StageTimer::finish() {
    if (!on || marks.empty()) return;
    VRB_CUDA(cudaEventSynchronize(marks.back().second));
    for (int q = 0; q < 10; ++q) t_stage_ms[q] = 0.0;
    for (size_t q = 1; q < marks.size(); ++q) {
        float ms = 0.f;
        VRB_CUDA(cudaEventElapsedTime(&ms, marks[q - 1].second, marks[q].second));
        const int st = marks[q].first;
        if (st >= 0 && st < 10 && st != 7) t_stage_ms[st] += ms;
    }
    float tot = 0.f;
    VRB_CUDA(cudaEventElapsedTime(&tot, marks.front().second, marks.back().second));
    t_stage_ms[7] = tot;
}

StageTimer::~StageTimer() {
    if (nvtx_open) nvtxRangePop();
    for (auto& m : marks) cudaEventDestroy(m.second);
}

}  // namespace vrb

// ---------------------------------------------------------------------------
// result handle
// ---------------------------------------------------------------------------
struct vrb_result {
    int device = 0;
    int64_t n = 0;
    int32_t d = 0, maxdim = 0, K = 0;
    uint32_t flags = 0;
    int64_t count[4] = {0, 0, 0, 0};        // global size per dimension
    int64_t local_off[4] = {0, 0, 0, 0};
    int64_t local_n[4] = {0, 0, 0, 0};
    int64_t nvals = 0;
    uint32_t* verts[4] = {nullptr, nullptr, nullptr, nullptr};   // local slice base, dim 1..3
    uint32_t* filt[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t* rows[4] = {nullptr, nullptr, nullptr, nullptr};    // dim 2..3 (dim 1 aliases verts[1])
    double* vor = nullptr;
    uint32_t* ev_all = nullptr;      // 2E edge vertices of every rank (position order)
    uint32_t* efilt_all = nullptr;   // E edge filt
    bool h0_done = false;            // vrb_h0 cache
    int64_t h0_nf = 0;
    uint32_t* h0_pos = nullptr;
    uint32_t* h0_death = nullptr;
    bool c2_done = false;            // vrb_compress_d2 cache
    int64_t c2_nrows = 0, c2_nnz = 0;
    uint64_t* c2_colptr = nullptr;
    uint32_t* c2_rowval = nullptr;
    uint32_t* c2_rowmap = nullptr;
    std::vector<vrb::Alloc> owned;

    void init(int64_t n_, int32_t d_, const vrb_opts* opts) {
        device = 0;
        VRB_CUDA(cudaGetDevice(&device));
        n = n_;
        d = d_;
        maxdim = opts->maxdim;
        K = opts->maxdim + 1;
        flags = opts->flags;
        count[0] = n;
        local_off[0] = 0;
        local_n[0] = n;
    }
    // edges are held whole; the handle reports the slice of rank / world
    void set_edges(uint32_t* ev, uint32_t* efilt, int rank, int world) {
        ev_all = ev;
        efilt_all = efilt;
        const int64_t E = count[1], lo = E * rank / world, hi = E * (rank + 1) / world;
        local_off[1] = lo;
        local_n[1] = hi - lo;
        verts[1] = ev ? ev + 2 * lo : nullptr;
        filt[1] = efilt ? efilt + lo : nullptr;
    }

    template <class T>
    T* own(size_t n_elems, cudaStream_t s) {
        if (n_elems == 0) return nullptr;
        const vrb::Alloc a = vrb::dalloc_owned(n_elems * sizeof(T), s);
        owned.push_back(a);
        return static_cast<T*>(a.p);
    }
    void release_all() {
        for (auto& a : owned) vrb::dfree_owned(a);
        owned.clear();
    }
};

namespace {

using namespace vrb;

template <class F>
vrb_status guarded(F&& f) {
    try {
        cudaGetLastError();   // an error left by a call outside the library is not this call's

        f();
        t_last_error.clear();
        return VRB_OK;
    } catch (const Error& e) {
        t_last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        t_last_error = "host allocation failed";
        return VRB_ENOMEM;
    } catch (...) {
        t_last_error = "unknown internal error";
        return VRB_ECUDA;
    }
}

void check_opts(const double* X, int64_t n, int32_t d, const vrb_opts* opts, vrb_handle* out, bool x_required) {
    if (!out) fail(VRB_EINVAL, "out handle pointer is NULL");
    *out = nullptr;
    if (!opts) fail(VRB_EINVAL, "opts is NULL");
    if (n < 0) fail(VRB_EINVAL, "n = %lld < 0", (long long)n);
    if (d < 1) fail(VRB_EINVAL, "d = %d < 1", d);
    if (x_required && n > 0 && !X) fail(VRB_EINVAL, "X is NULL");
    if (opts->maxdim < 0 || opts->maxdim > 2) fail(VRB_EINVAL, "maxdim = %d not in 0..2", opts->maxdim);
    if (std::isnan(opts->radius) || opts->radius < 0.0) fail(VRB_EINVAL, "radius must be >= 0 (got %g)", opts->radius);
    if (n >= kMaxN) fail(VRB_EOVERFLOW, "n = %lld exceeds the 21-bit vertex id limit", (long long)n);
    // limits of the layout, checked before any work
    if (opts->maxdim >= 2 && n > tets_max_n())
        fail(VRB_ENOTSUP, "tetrahedra (maxdim 2) need n <= %lld on this device (n = %lld)",
             (long long)tets_max_n(), (long long)n);
}

__global__ void k_colptr(uint64_t* colptr, int64_t ncols, uint64_t k1, uint64_t off) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= ncols; j += (int64_t)gridDim.x * blockDim.x)
        colptr[j] = k1 * (off + (uint64_t)j);
}

__global__ void k_sortable_keys(const double* __restrict__ in, int64_t n, uint64_t* __restrict__ out, int* bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = in[i];
        if (isnan(v)) atomicOr(bad, 1);
        if (v == 0.0) v = 0.0;   // -0.0 == +0.0
        const uint64_t b = (uint64_t)__double_as_longlong(v);
        out[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    }
}

__global__ void k_sortperm_out(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ perm,
                               const uint32_t* __restrict__ rank, int64_t n, int64_t* __restrict__ perm_out,
                               uint32_t* __restrict__ dense) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        perm_out[p] = perm[p];
        if (dense) dense[perm[p]] = rank[p];
    }
}

__global__ void k_heads(const uint64_t* __restrict__ key, int64_t n, uint32_t* __restrict__ head) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        head[p] = (p == 0 || key[p] != key[p - 1]) ? 1u : 0u;
}

unsigned grid_of(int64_t n) {
    int64_t g = ceil_div(n, 256);
    return (unsigned)(g < 1 ? 1 : (g > 4096 ? 4096 : g));
}

// total = off[E]
uint64_t read_total(const uint64_t* off, int64_t E, cudaStream_t s) {
    uint64_t total = 0;
    VRB_CUDA(cudaMemcpyAsync(&total, off + E, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return total;
}

// vrb_build / vrb_build_dm (one GPU).
void build_impl(const double* X, int64_t n, int32_t d, const vrb_opts* opts, cudaStream_t s, vrb_handle* out,
                bool matrix = false) {
    check_opts(X, n, d, opts, out, true);
    vrb_result* h = new vrb_result();
    try {
        h->init(n, d, opts);
        StageTimer timer;
        timer.start(s);
        timer.begin(0);

        DBuf<double> Xd;
        KeptEdges ke;
        if (matrix) {   // F3: X is an n x n distance matrix
            place_matrix(X, n, opts->flags, s, Xd);
            build_kept_edges_dm(Xd.get(), n, opts->radius, (opts->flags & VRB_STRICT_RADIUS) != 0, s, ke);
        } else {
            place_points(X, n, d, opts->flags, s, Xd);
            build_kept_edges(Xd.get(), n, d, opts->radius, (opts->flags & VRB_STRICT_RADIUS) != 0, s, ke);
        }
        Xd.reset();
        timer.mark(0);
        timer.begin(1);
        const int64_t E = ke.E;
        h->count[1] = E;
        uint32_t* ev = h->own<uint32_t>(2 * E, s);
        uint32_t* efilt = h->own<uint32_t>(E, s);
        h->vor = h->own<double>(E, s);
        h->nvals = rank_edges(ke, ev, efilt, h->vor, s);
        h->set_edges(ev, efilt, 0, 1);
        ke = KeptEdges();
        timer.mark(1);
        timer.begin(2);
        if (h->K >= 2) {
            Graph g;
            build_graph(ev, n, E, s, g);
            timer.mark(2);
            timer.begin(3);
            // ---- triangles: count per owner edge, offsets
            DBuf<uint32_t> cnt(E, s);
            // the count pass keeps what the fill needs: validity bits and host
            // positions (x-major path) or the apex bitmaps (round-1 path)
            TriRecords R;
            bool xmajor = records_apply(g);
            if (xmajor) {
                try {
                    count_triangles_rec(g, ev, 0, E, cnt.get(), R, s);
                } catch (const Error& e) {
                    if (e.status != VRB_ENOMEM) throw;
                    cudaGetLastError();
                    R = TriRecords();   // not enough memory for the records: the bitmap path
                    xmajor = false;
                }
            }
            DBuf<uint64_t> bmoff;
            DBuf<uint32_t> bm;
            if (xmajor) {
            } else if (apex_bitmaps_apply(g)) {
                uint64_t words = 0;
                apex_bitmap_offsets(g, bmoff, words, s);
                bm.alloc(words ? words : 1, s);
                count_triangles_bm(g, cnt.get(), bm.get(), bmoff.get(), s);
            } else {
                count_triangles(g, cnt.get(), 0, 1, s);
            }
            DBuf<uint64_t> toff(E + 1, s);
            exclusive_scan(cnt.get(), toff.get(), E, s);
            const uint64_t T = read_total(toff.get(), E, s);
            if (T >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu triangles exceed u32 positions", (unsigned long long)T);
            h->count[2] = (int64_t)T;
            h->local_off[2] = 0;
            h->local_n[2] = (int64_t)T;
            uint32_t* tv = h->own<uint32_t>(3 * T, s);
            uint32_t* tf = h->own<uint32_t>(T, s);
            uint32_t* trows = nullptr;
            if (!(opts->flags & VRB_SKIP_BOUNDARY)) trows = h->own<uint32_t>(3 * T, s);
            // apex of every triangle (tetrahedra: face positions by owner-edge search)
            DBuf<uint16_t> tapex;
            if (h->K >= 3 && n <= 65536) {   // padded: the face search reads 16-byte chunks past the end
                tapex.alloc((size_t)T + 16, s);
                VRB_CUDA(cudaMemsetAsync(tapex.get() + T, 0xFF, 16 * sizeof(uint16_t), s));
            }
            timer.mark(3);
            timer.begin(4);
            if (xmajor)
                fill_triangles_x(g, R, efilt, toff.get(), 0, E, 0, tv, tf, trows, tapex.get(), s);
            else
                fill_triangles(g, efilt, toff.get(), 0, E, 0, tv, tf, trows, tapex.get(), s, bm.get(), bmoff.get());
            bm.reset();
            R = TriRecords();
            timer.mark(4);
            timer.begin(5);
            sort_tie_groups(2, efilt, toff.get(), E, 0, E, n, tv, trows, s, ev);
            timer.mark(5);
            timer.begin(3);
            h->verts[2] = tv;
            h->filt[2] = tf;
            h->rows[2] = trows;
            if (h->K >= 3) {
                // ---- tetrahedra
                TriLevels L;
                L.apex = tapex.get();
                L.ev = ev;
                L.n = n;
                triangle_levels(efilt, toff.get(), E, tv, s, L);
                DBuf<uint32_t> qc(E, s);
                timer.mark(3);
                timer.begin(8);
                count_tets(g, L, qc.get(), 0, 1, s);
                DBuf<uint64_t> qoff(E + 1, s);
                exclusive_scan(qc.get(), qoff.get(), E, s);
                const uint64_t Q = read_total(qoff.get(), E, s);
                if (Q >= 0xFFFFFFFFull)
                    fail(VRB_EOVERFLOW, "%llu tetrahedra exceed u32 positions", (unsigned long long)Q);
                h->count[3] = (int64_t)Q;
                h->local_off[3] = 0;
                h->local_n[3] = (int64_t)Q;
                h->verts[3] = h->own<uint32_t>(4 * Q, s);
                h->filt[3] = h->own<uint32_t>(Q, s);
                if (!(opts->flags & VRB_SKIP_BOUNDARY)) h->rows[3] = h->own<uint32_t>(4 * Q, s);
                timer.mark(8);
                timer.begin(9);
                fill_tets(g, L, efilt, qoff.get(), 0, E, 0, h->verts[3], h->filt[3], h->rows[3], s);
                timer.mark(9);
                timer.begin(5);
                sort_tie_groups(3, efilt, qoff.get(), E, 0, E, n, h->verts[3], h->rows[3], s);
                timer.mark(5);
            }
        }
        VRB_CUDA(cudaStreamSynchronize(s));
        VRB_CUDA(cudaGetLastError());
        timer.finish();
        *out = h;
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaGetLastError();
        h->release_all();
        delete h;
        throw;
    }
}

// vrb_build_dist: this rank's slices (dist.cu) wrapped in a handle.
void build_dist(const double* X, int64_t n, int32_t d, const vrb_opts* opts, const vrb_comm* comm, cudaStream_t s,
                vrb_handle* out) {
    if (!comm) fail(VRB_EINVAL, "comm is NULL");
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world || !comm->allgather || !comm->broadcast)
        fail(VRB_EINVAL, "bad communicator (rank %d, world %d)", comm->rank, comm->world);
    check_opts(X, n, d, opts, out, comm->rank == 0);
    vrb_result* h = new vrb_result();
    try {
        h->init(n, d, opts);
        StageTimer timer;
        timer.start(s);
        DistOut o;
        o.timer = &timer;
        o.alloc_u32 = [&](size_t m) { return h->own<uint32_t>(m, s); };
        o.alloc_f64 = [&](size_t m) { return h->own<double>(m, s); };
        build_dist_impl(X, n, d, opts, comm, s, o);
        h->count[1] = o.E;
        h->vor = o.vor;
        h->nvals = o.nvals;
        h->set_edges(o.ev, o.efilt, comm->rank, comm->world);
        if (h->K >= 2) {
            h->count[2] = (int64_t)o.T;
            h->local_off[2] = (int64_t)o.t0;
            h->local_n[2] = (int64_t)o.Tl;
            h->verts[2] = o.tv;
            h->filt[2] = o.tf;
            h->rows[2] = o.trows;
        }
        if (h->K >= 3) {
            h->count[3] = (int64_t)o.Q;
            h->local_off[3] = (int64_t)o.q0;
            h->local_n[3] = (int64_t)o.Ql;
            h->verts[3] = o.qv;
            h->filt[3] = o.qf;
            h->rows[3] = o.qrows;
        }
        VRB_CUDA(cudaStreamSynchronize(s));
        VRB_CUDA(cudaGetLastError());
        timer.finish();
        *out = h;
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaGetLastError();
        h->release_all();
        delete h;
        throw;
    }
}

}  // namespace

extern "C" {

int vrb_abi_version(void) { return VRB_ABI_VERSION; }

const char* vrb_last_error(void) { return vrb::t_last_error.c_str(); }

vrb_status vrb_set_allocator(vrb_alloc_fn alloc, vrb_free_fn free_fn, void* ctx) {
    return guarded([&] {
        if ((alloc == nullptr) != (free_fn == nullptr)) fail(VRB_EINVAL, "alloc and free hooks must be set together");
        vrb::g_alloc = alloc;
        vrb::g_free = free_fn;
        vrb::g_ctx = ctx;
    });
}

vrb_status vrb_build(const double* X, int64_t n, int32_t d, const vrb_opts* opts, void* stream, vrb_handle* out) {
    return guarded([&] { build_impl(X, n, d, opts, (cudaStream_t)stream, out); });
}

vrb_status vrb_build_dm(const double* D, int64_t n, const vrb_opts* opts, void* stream, vrb_handle* out) {
    return guarded([&] {
        if (opts && (opts->flags & VRB_DIM_MAJOR)) fail(VRB_EINVAL, "VRB_DIM_MAJOR does not apply to a distance matrix");
        build_impl(D, n, 1, opts, (cudaStream_t)stream, out, true);
    });
}

vrb_status vrb_latlon2euc(const double* latlon_dev, int64_t n, double* xyz_dev, void* stream) {
    return guarded([&] {
        if (n < 0) fail(VRB_EINVAL, "n < 0");
        if (n > 0 && (!latlon_dev || !xyz_dev)) fail(VRB_EINVAL, "NULL pointer");
        vrb::latlon2euc(latlon_dev, n, xyz_dev, (cudaStream_t)stream);
        VRB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    });
}

vrb_status vrb_build_dist(const double* X, int64_t n, int32_t d, const vrb_opts* opts, const vrb_comm* comm,
                          void* stream, vrb_handle* out) {
    return guarded([&] { build_dist(X, n, d, opts, comm, (cudaStream_t)stream, out); });
}

vrb_status vrb_partition_bounds(const uint64_t* prefix, const uint32_t* efilt, int64_t E, int32_t world,
                                int64_t* bounds) {
    return guarded([&] {
        if (!prefix || !bounds || (E > 0 && !efilt)) fail(VRB_EINVAL, "NULL pointer");
        if (E < 0 || world < 1) fail(VRB_EINVAL, "E < 0 or world < 1");
        vrb::partition_bounds_host(prefix, efilt, E, world, bounds);
    });
}

vrb_status vrb_count(vrb_handle h, int32_t dim, int64_t* global_n, int64_t* local_off, int64_t* local_n) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (dim < 0 || dim > h->K) fail(VRB_EINVAL, "dim %d out of range 0..%d", dim, h->K);
        if (global_n) *global_n = h->count[dim];
        if (local_off) *local_off = h->local_off[dim];
        if (local_n) *local_n = h->local_n[dim];
    });
}

vrb_status vrb_simplices(vrb_handle h, int32_t dim, const uint32_t** verts_dev, const uint32_t** filt_dev) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (dim < 1 || dim > h->K) fail(VRB_EINVAL, "dim %d out of range 1..%d", dim, h->K);
        if (verts_dev) *verts_dev = h->verts[dim];
        if (filt_dev) *filt_dev = h->filt[dim];
    });
}

vrb_status vrb_rank_values(vrb_handle h, const double** value_of_rank_dev, int64_t* nvals) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (value_of_rank_dev) *value_of_rank_dev = h->vor;
        if (nvals) *nvals = h->nvals;
    });
}

vrb_status vrb_boundary(vrb_handle h, int32_t k, int64_t* nrows, int64_t* ncols, const uint32_t** rowval_dev) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (k < 1 || k > h->K) fail(VRB_EINVAL, "k %d out of range 1..%d", k, h->K);
        if (k >= 2 && (h->flags & VRB_SKIP_BOUNDARY)) fail(VRB_EINVAL, "boundary of dim %d was skipped", k);
        if (nrows) *nrows = h->count[k - 1];
        if (ncols) *ncols = h->local_n[k];
        if (rowval_dev) *rowval_dev = k == 1 ? h->verts[1] : h->rows[k];
    });
}

vrb_status vrb_boundary_colptr(vrb_handle h, int32_t k, uint64_t* colptr_dev, void* stream) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (k < 1 || k > h->K) fail(VRB_EINVAL, "k %d out of range 1..%d", k, h->K);
        if (!colptr_dev) fail(VRB_EINVAL, "colptr is NULL");
        const int64_t nc = h->local_n[k];
        k_colptr<<<grid_of(nc + 1), 256, 0, (cudaStream_t)stream>>>(colptr_dev, nc, (uint64_t)(k + 1),
                                                                     (uint64_t)h->local_off[k]);
        VRB_LAUNCH_CHECK();
    });
}

vrb_status vrb_free(vrb_handle h) {
    return guarded([&] {
        if (!h) return;
        h->release_all();
        delete h;
    });
}

namespace {
struct H0Alloc {
    vrb_result* h;
    cudaStream_t s;
};
uint32_t* h0_alloc(int64_t n, void* ctx) {
    auto* a = static_cast<H0Alloc*>(ctx);
    return a->h->own<uint32_t>((size_t)n, a->s);
}
}  // namespace

vrb_status vrb_h0(vrb_handle h, void* stream, const uint32_t** forest_pos, const uint32_t** death_filt,
                  int64_t* n_finite, int64_t* n_essential) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (!h->h0_done) {
            const cudaStream_t s = (cudaStream_t)stream;
            H0Alloc ctx{h, s};
            h->h0_nf = vrb::h0_forest(h->ev_all, h->efilt_all, h->n, h->count[1], s, h0_alloc, &ctx, &h->h0_pos,
                                      &h->h0_death);
            h->h0_done = true;
        }
        if (forest_pos) *forest_pos = h->h0_pos;
        if (death_filt) *death_filt = h->h0_death;
        if (n_finite) *n_finite = h->h0_nf;
        if (n_essential) *n_essential = h->n - h->h0_nf;
    });
}

vrb_status vrb_compress_d2(vrb_handle h, void* stream, int64_t* nrows, int64_t* nnz, const uint64_t** colptr,
                           const uint32_t** rowval, const uint32_t** rowmap) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (h->K < 2) fail(VRB_EINVAL, "the build has no dimension 2 (maxdim 0)");
        if (h->flags & VRB_SKIP_BOUNDARY) fail(VRB_EINVAL, "D_2 was not materialised (VRB_SKIP_BOUNDARY)");
        const cudaStream_t s = (cudaStream_t)stream;
        if (!h->h0_done) {
            H0Alloc ctx{h, s};
            h->h0_nf = vrb::h0_forest(h->ev_all, h->efilt_all, h->n, h->count[1], s, h0_alloc, &ctx, &h->h0_pos,
                                      &h->h0_death);
            h->h0_done = true;
        }
        if (!h->c2_done) {
            const int64_t nc = h->local_n[2];
            h->c2_colptr = h->own<uint64_t>((size_t)nc + 1, s);
            H0Alloc ctx{h, s};
            h->c2_nnz = vrb::compress_d2(h->h0_pos, h->h0_nf, h->count[1], h->rows[2], nc, s, h->c2_colptr, h0_alloc,
                                         &ctx, &h->c2_rowval, &h->c2_rowmap, &h->c2_nrows);
            h->c2_done = true;
        }
        if (nrows) *nrows = h->c2_nrows;
        if (nnz) *nnz = h->c2_nnz;
        if (colptr) *colptr = h->c2_colptr;
        if (rowval) *rowval = h->c2_rowval;
        if (rowmap) *rowmap = h->c2_rowmap;
    });
}

struct vrb_gf2 {
    int64_t ncols = 0, nnz = 0;
    uint64_t* colptr = nullptr;
    uint32_t* rowval = nullptr;
    std::vector<vrb::Alloc> owned;
    void release_all() {
        for (auto& a : owned) vrb::dfree_owned(a);
        owned.clear();
    }
};

namespace {
struct Gf2Alloc {
    vrb_gf2* g;
    cudaStream_t s;
};
uint32_t* gf2_alloc_rows(int64_t n, void* ctx) {
    auto* a = static_cast<Gf2Alloc*>(ctx);
    const vrb::Alloc al = vrb::dalloc_owned((size_t)n * sizeof(uint32_t), a->s);
    a->g->owned.push_back(al);
    return static_cast<uint32_t*>(al.p);
}
}  // namespace

vrb_status vrb_gf2_blockprodsum(int64_t nrows, int64_t ncols, int64_t k, const uint64_t* d_colptr,
                                const uint32_t* d_rowval, const uint64_t* c_colptr, const uint32_t* c_rowval,
                                const uint64_t* e_colptr, const uint32_t* e_rowval, void* stream,
                                vrb_gf2_handle* out) {
    return guarded([&] {
        if (!out) fail(VRB_EINVAL, "out is NULL");
        *out = nullptr;
        if (nrows < 0 || ncols < 0 || k < 0) fail(VRB_EINVAL, "negative dimension");
        if (nrows > 0xFFFFFFFFll || k > 0xFFFFFFFFll) fail(VRB_EOVERFLOW, "row indices must fit u32");
        if (!d_colptr || !c_colptr || !e_colptr) fail(VRB_EINVAL, "NULL colptr");
        const cudaStream_t s = (cudaStream_t)stream;
        vrb_gf2* g = new vrb_gf2();
        try {
            g->ncols = ncols;
            const vrb::Alloc al = vrb::dalloc_owned((size_t)(ncols + 1) * sizeof(uint64_t), s);
            g->colptr = static_cast<uint64_t*>(al.p);
            g->owned.push_back(al);
            VRB_CUDA(cudaMemsetAsync(g->colptr, 0, (size_t)(ncols + 1) * sizeof(uint64_t), s));
            Gf2Alloc ctx{g, s};
            g->nnz = vrb::gf2_blockprodsum(nrows, ncols, k, d_colptr, d_rowval, c_colptr, c_rowval, e_colptr,
                                           e_rowval, s, g->colptr, gf2_alloc_rows, &ctx, &g->rowval);
            VRB_CUDA(cudaStreamSynchronize(s));
        } catch (...) {
            cudaStreamSynchronize(s);
            g->release_all();
            delete g;
            throw;
        }
        *out = g;
    });
}

vrb_status vrb_gf2_csc(vrb_gf2_handle h, int64_t* nnz, const uint64_t** colptr_dev, const uint32_t** rowval_dev) {
    return guarded([&] {
        if (!h) fail(VRB_EINVAL, "NULL handle");
        if (nnz) *nnz = h->nnz;
        if (colptr_dev) *colptr_dev = h->colptr;
        if (rowval_dev) *rowval_dev = h->rowval;
    });
}

vrb_status vrb_gf2_free(vrb_gf2_handle h) {
    return guarded([&] {
        if (!h) return;
        h->release_all();
        delete h;
    });
}

vrb_status vrb_sortperm_f64(const double* keys_dev, int64_t n, int64_t* perm_dev, uint32_t* dense_rank_dev,
                            void* stream) {
    return guarded([&] {
        if (n < 0) fail(VRB_EINVAL, "n < 0");
        if (n == 0) return;
        if (!keys_dev || !perm_dev) fail(VRB_EINVAL, "NULL pointer");
        if (n >= (int64_t)0xFFFFFFFFll) fail(VRB_EOVERFLOW, "n exceeds u32 permutation indices");
        cudaStream_t s = (cudaStream_t)stream;
        DBuf<uint64_t> k0(n, s), k1(n, s);
        DBuf<uint32_t> v0(n, s), v1(n, s);
        DBuf<int> bad(1, s);
        VRB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
        k_sortable_keys<<<grid_of(n), 256, 0, s>>>(keys_dev, n, k0.get(), bad.get());
        VRB_LAUNCH_CHECK();
        int hbad = 0;
        VRB_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        if (hbad) fail(VRB_EINVAL, "NaN key");
        iota_u32(v0.get(), n, s);
        const uint64_t vary = varying_bits(k0.get(), n, s);
        const bool alt = radix_sort_pairs(k0.get(), k1.get(), v0.get(), v1.get(), n, vary, s);
        const uint64_t* sk = alt ? k1.get() : k0.get();
        const uint32_t* sp = alt ? v1.get() : v0.get();
        DBuf<uint32_t> head(n, s), rank(n, s);
        k_heads<<<grid_of(n), 256, 0, s>>>(sk, n, head.get());
        VRB_LAUNCH_CHECK();
        inclusive_scan_u32(head.get(), rank.get(), n, s);
        k_sortperm_out<<<grid_of(n), 256, 0, s>>>(sk, sp, rank.get(), n, perm_dev, dense_rank_dev);
        VRB_LAUNCH_CHECK();
        VRB_CUDA(cudaStreamSynchronize(s));
    });
}

unsigned long long vrb_launch_count(void) { return vrb::g_launches.load(); }

int32_t vrb_last_edge_path(void) { return vrb::last_edge_path(); }

vrb_status vrb_set_profiling(int32_t enable) {
    vrb::g_profiling = enable != 0;
    return VRB_OK;
}

vrb_status vrb_last_stage_ms(double* ms8) {
    return guarded([&] {
        if (!ms8) fail(VRB_EINVAL, "NULL output");
        for (int q = 0; q < 8; ++q) ms8[q] = vrb::t_stage_ms[q];
    });
}

vrb_status vrb_last_stage_ms_n(double* ms, int32_t n) {
    return guarded([&] {
        if (!ms || n < 0) fail(VRB_EINVAL, "NULL output or negative count");
        for (int q = 0; q < n && q < 10; ++q) ms[q] = vrb::t_stage_ms[q];
        for (int q = 10; q < n; ++q) ms[q] = 0.0;
    });
}

}  // extern "C"
