// gf2.cu -- SURVEY 8(f) F4: blockprodsum, S = D + C E over GF(2).
//
// Definition (sec. 4.6): inside Eirene's Schur-complement step
// ("S = D + C A^-1 B using the modulo-2 operation")
// blockprodsum computes D + C E with E = A^-1 B; all matrices are CSC
// (P:1014).  Column j of S is the mod-2 sum of D[:, j] and of C[:, i] for
// every i in E[:, j].
//
// B200 design.  The paper partitions the columns over pthreads and lets the
// master fix up the column pointers (Fig. BlkProdSum).  Here the
// columns are independent data-parallel work end to end:
//   1. candidates: per column, |D_j| + sum over E_j of |C_i| (one warp per
//      column), exclusive scan -> candidate offsets (the colptr fix-up of
//      the paper is this scan);
//   2. gather: each column's candidate rows as 64-bit keys (j << rowbits | r)
//      -- D_j, then every C_i of E_j, lanes copying a C column coalesced;
//   3. one radix sort of the keys (only the varying digits are passed), so
//      equal (column, row) pairs become adjacent runs;
//   4. parity: a run survives iff its length is odd (x + x = 0 mod 2);
//      survivors are compacted in order and counted per column -> colptr.
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

unsigned warp_grid(int64_t nwarps) {
    const int64_t g = ceil_div(nwarps * 32, 256), cap = (int64_t)device_sm_count() * 16;
    return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

// candidates per column (one warp per column)
__global__ void k_cand_count(int64_t nc, const uint64_t* __restrict__ dcp, const uint64_t* __restrict__ ccp,
                             const uint64_t* __restrict__ ecp, const uint32_t* __restrict__ erv,
                             uint64_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < nc; j += nw) {
        uint64_t c = 0;
        for (uint64_t q = ecp[j] + lane; q < ecp[j + 1]; q += 32) {
            const uint32_t i = erv[q];
            c += ccp[(uint64_t)i + 1] - ccp[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
        if (lane == 0) cnt[j] = c + (dcp[j + 1] - dcp[j]);
    }
}

__global__ void k_cand_fill(int64_t nc, int rowbits, const uint64_t* __restrict__ dcp,
                            const uint32_t* __restrict__ drv, const uint64_t* __restrict__ ccp,
                            const uint32_t* __restrict__ crv, const uint64_t* __restrict__ ecp,
                            const uint32_t* __restrict__ erv, const uint64_t* __restrict__ coff,
                            uint64_t* __restrict__ keys) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < nc; j += nw) {
        const uint64_t hi = (uint64_t)j << rowbits;
        uint64_t o = coff[j];
        const uint64_t d0 = dcp[j], d1 = dcp[j + 1];
        for (uint64_t q = d0 + lane; q < d1; q += 32) keys[o + (q - d0)] = hi | drv[q];
        o += d1 - d0;
        for (uint64_t q = ecp[j]; q < ecp[j + 1]; ++q) {
            const uint32_t i = erv[q];
            const uint64_t c0 = ccp[i], c1 = ccp[(uint64_t)i + 1];
            for (uint64_t t = c0 + lane; t < c1; t += 32) keys[o + (t - c0)] = hi | crv[t];
            o += c1 - c0;
        }
    }
}

// keep[p] = p starts a run of equal keys of odd length
__global__ void k_parity(const uint64_t* __restrict__ keys, int64_t M, uint32_t* __restrict__ keep) {
    GRID_STRIDE(p, M) {
        uint32_t k = 0;
        if (p == 0 || keys[p] != keys[p - 1]) {
            int64_t q = p + 1;
            while (q < M && keys[q] == keys[p]) ++q;
            k = (uint32_t)((q - p) & 1);
        }
        keep[p] = k;
    }
}

__global__ void k_emit(const uint64_t* __restrict__ keys, int64_t M, int rowbits, const uint32_t* __restrict__ keep,
                       const uint64_t* __restrict__ pos, uint32_t* __restrict__ rowval,
                       uint32_t* __restrict__ colcnt) {
    const uint64_t mask = (rowbits >= 64) ? ~0ull : ((1ull << rowbits) - 1ull);
    GRID_STRIDE(p, M) {
        if (!keep[p]) continue;
        const uint64_t k = keys[p];
        rowval[pos[p]] = (uint32_t)(k & mask);
        atomicAdd(&colcnt[k >> rowbits], 1u);
    }
}

// 1 + the largest index, accumulated in 64 bits (an index of 0xFFFFFFFF, an
// int32 -1, gives 2^32 and fails the range check instead of wrapping to 0)
__global__ void k_max_u32(const uint32_t* __restrict__ a, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long m = 0;
    GRID_STRIDE(i, n) m = max(m, (unsigned long long)a[i] + 1ull);   // + 1: 0 means empty
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// 1 + the largest index in a[0, n) (0 when n == 0)
uint64_t max_plus_one(const uint32_t* a, int64_t n, cudaStream_t s) {
    if (n <= 0) return 0;
    DBuf<unsigned long long> m(1, s);
    VRB_CUDA(cudaMemsetAsync(m.get(), 0, sizeof(unsigned long long), s));
    k_max_u32<<<grid_for(n), 256, 0, s>>>(a, n, m.get());
    VRB_LAUNCH_CHECK();
    unsigned long long h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, m.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return h;
}

// colptr must start at 0 and be non-decreasing (else the ranges it names are
// not columns of one array)
__global__ void k_colptr_ok(const uint64_t* __restrict__ cp, int64_t n, int* __restrict__ bad) {
    GRID_STRIDE(j, n) if ((j == 0 && cp[0] != 0) || cp[j] > cp[j + 1]) atomicOr(bad, 1);
}

bool colptr_ok(const uint64_t* cp, int64_t n, cudaStream_t s) {
    DBuf<int> bad(1, s);
    VRB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    if (n > 0) {
        k_colptr_ok<<<grid_for(n), 256, 0, s>>>(cp, n, bad.get());
        VRB_LAUNCH_CHECK();
    }
    int h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return h == 0;
}

uint64_t last_of(const uint64_t* colptr, int64_t n, cudaStream_t s) {
    uint64_t v = 0;
    VRB_CUDA(cudaMemcpyAsync(&v, colptr + n, sizeof(v), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    return v;
}

}  // namespace

int64_t gf2_blockprodsum(int64_t nrows, int64_t ncols, int64_t kdim, const uint64_t* dcp, const uint32_t* drv,
                         const uint64_t* ccp, const uint32_t* crv, const uint64_t* ecp, const uint32_t* erv,
                         cudaStream_t s, uint64_t* colptr_out, uint32_t* (*alloc_rows)(int64_t, void*), void* ctx,
                         uint32_t** rowval_out) {
    *rowval_out = nullptr;
    if (ncols == 0) return 0;
    if (!colptr_ok(dcp, ncols, s) || !colptr_ok(ccp, kdim, s) || !colptr_ok(ecp, ncols, s))
        fail(VRB_EINVAL, "blockprodsum: a colptr does not start at 0 or decreases");
    // index ranges (out-of-range rows would gather outside C): VRB_EINVAL
    if (max_plus_one(drv, (int64_t)last_of(dcp, ncols, s), s) > (uint64_t)nrows ||
        max_plus_one(crv, (int64_t)last_of(ccp, kdim, s), s) > (uint64_t)nrows ||
        max_plus_one(erv, (int64_t)last_of(ecp, ncols, s), s) > (uint64_t)kdim)
        fail(VRB_EINVAL, "blockprodsum: a row index is out of range");
    int rowbits = 1;
    while (rowbits < 32 && ((int64_t)1 << rowbits) < nrows) ++rowbits;
    DBuf<uint64_t> cnt(ncols, s), coff(ncols + 1, s);
    k_cand_count<<<warp_grid(ncols), 256, 0, s>>>(ncols, dcp, ccp, ecp, erv, cnt.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(cnt.get(), coff.get(), ncols, s);
    uint64_t M = 0;
    VRB_CUDA(cudaMemcpyAsync(&M, coff.get() + ncols, sizeof(M), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    DBuf<uint32_t> colcnt(ncols, s);
    VRB_CUDA(cudaMemsetAsync(colcnt.get(), 0, colcnt.bytes(), s));
    int64_t nnz = 0;
    if (M) {
        if (M >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu candidate entries exceed u32 sort values",
                                     (unsigned long long)M);
        DBuf<uint64_t> keys(M, s), keys_alt(M, s);
        DBuf<uint32_t> vals(M, s), vals_alt(M, s);
        k_cand_fill<<<warp_grid(ncols), 256, 0, s>>>(ncols, rowbits, dcp, drv, ccp, crv, ecp, erv, coff.get(),
                                                     keys.get());
        VRB_LAUNCH_CHECK();
        VRB_CUDA(cudaMemsetAsync(vals.get(), 0, vals.bytes(), s));   // the sort carries a dummy payload
        const uint64_t vary = varying_bits(keys.get(), (int64_t)M, s);
        const bool alt = radix_sort_pairs(keys.get(), keys_alt.get(), vals.get(), vals_alt.get(), (int64_t)M, vary, s);
        const uint64_t* sk = alt ? keys_alt.get() : keys.get();
        DBuf<uint32_t> keep(M, s);
        DBuf<uint64_t> pos(M + 1, s);
        k_parity<<<grid_for((int64_t)M), 256, 0, s>>>(sk, (int64_t)M, keep.get());
        VRB_LAUNCH_CHECK();
        exclusive_scan(keep.get(), pos.get(), (int64_t)M, s);
        uint64_t nz = 0;
        VRB_CUDA(cudaMemcpyAsync(&nz, pos.get() + M, sizeof(nz), cudaMemcpyDeviceToHost, s));
        VRB_CUDA(cudaStreamSynchronize(s));
        nnz = (int64_t)nz;
        if (nnz) {
            *rowval_out = alloc_rows(nnz, ctx);
            k_emit<<<grid_for((int64_t)M), 256, 0, s>>>(sk, (int64_t)M, rowbits, keep.get(), pos.get(), *rowval_out,
                                                        colcnt.get());
            VRB_LAUNCH_CHECK();
        }
    }
    exclusive_scan(colcnt.get(), colptr_out, ncols, s);
    VRB_CUDA(cudaStreamSynchronize(s));
    return nnz;
}

}  // namespace vrb
