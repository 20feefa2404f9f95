// distance.cu -- S1 (point placement) and S2 (pairwise distance + radius cap).
//
// Paper: sec. 2.1 P:107-113 ("any two points that are less than the distance
// epsilon from each other are connected by an edge"); the distance matrix is
// "the primary input" of Eirene.  Readings: A1 inclusive
// cap (len <= r; STRICT: len < r), A5 fixed-order fold
//     acc = +0.0; for c = 0..d-1: t = x_ic - x_jc; acc = acc + t*t; len = sqrt(acc)
// with every operation binary64 round-to-nearest and no FMA contraction
// (__dsub_rn / __dmul_rn / __dadd_rn / __dsqrt_rn).
//
// The cap is applied to d2 against a host-computed threshold T(r) = the
// largest double x with sqrt_rn(x) <= r (or < r): sqrt_rn is monotone, so
// "d2 <= T(r)" is exactly "sqrt_rn(d2) <= r" without a sqrt per pair.
//
// Two passes over 64x64 upper-triangular tiles of the pair matrix:
//   k_dist_mask : FP64 fold for every pair of the tile -> 64x64 kept bitmask
//                 + per (row, tile) kept counts            (FP64-ALU bound)
//   scan        : per (row, tile) counts -> lex slot bases
//   k_dist_fill : kept pairs only: recompute the fold, sqrt, write
//                 (len bits, i, j) at its lex slot          (write bound)
// Full filtration (r = inf, inclusive): every pair is kept, so the mask pass
// and the scan are skipped and k_dist_fill derives bits and slots in closed form.
// Output: the kept edges in lexicographic (i, j) order.
#include <cmath>

#include "vrb_internal.cuh"
#include "vrb_stages.cuh"

namespace vrb {
namespace {

constexpr int kT = 64;        // tile edge
constexpr int kDC = 16;       // coordinates staged per chunk
constexpr int kThreads = 256;
constexpr int kFillStageD = 16;   // k_dist_fill stages the tile's points for d <= 16 (16 KB)

__device__ __host__ __forceinline__ int64_t tile_index(int64_t ti, int64_t tj, int64_t nt) {
    return ti * nt - ti * (ti - 1) / 2 + (tj - ti);   // packed upper triangle (tj >= ti)
}

// The grid is 1-D over the upper-triangular tiles of tile rows [ti_lo, ti_hi)
// only (no block of the lower triangle is launched): block b is packed tile
// mask_base + b, whose row is found by a binary search of the row starts.
__device__ __forceinline__ void tile_of_block(int64_t b, int64_t nt, int64_t ti_lo, int64_t ti_hi, int64_t mask_base,
                                              int64_t& ti, int64_t& tj) {
    const int64_t q = mask_base + b;
    int64_t lo = ti_lo, hi = ti_hi;   // last row with tile_index(row, row) <= q
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (tile_index(mid, mid, nt) <= q) lo = mid; else hi = mid;
    }
    ti = lo;
    tj = ti + (q - tile_index(ti, ti, nt));
}

// The same, computed once per CTA (thread 0) and broadcast: the search is
// ~90 instructions per thread when every thread runs it.
__device__ __forceinline__ void tile_of_cta(int64_t nt, int64_t ti_lo, int64_t ti_hi, int64_t mask_base, int64_t& ti,
                                            int64_t& tj) {
    __shared__ int64_t s_tile[2];
    if (threadIdx.x == 0) tile_of_block(blockIdx.x, nt, ti_lo, ti_hi, mask_base, s_tile[0], s_tile[1]);
    __syncthreads();
    ti = s_tile[0];
    tj = s_tile[1];
}

// Tile rows [ti_lo, ti_lo + gridDim.y) (a rank's row block);
// masks are indexed from the block's first tile (mask_base) and the per
// (row, tile) counts from its first row.
// The cap decision per pair, d2 <= thr (thr = T(r), reading A1), taken on
// an FP32 fold of the coordinates rounded to float, with a rigorous error
// bound, and by the exact FP64 fold of the fixed RN sequence only when the
// FP32 value lies within the bound of thr:
//   x' = fl32(x): |x' - x| <= u|x|, u = 2^-24; t' = fl(x'_i - x'_j):
//   |t' - t| <= 2.1 u (|x_i| + |x_j|) <= 4.2 u M (M = max |coordinate| over
//   the tile's points); |t'^2 - t^2| <= 4.2 u M (4M + 1) <= 17 u M^2 + 4.2 u M;
//   FMA accumulation of d terms: |s' - sum t'^2| <= 1.01 d u sum t'^2.
//   So |s' - d2| <= d (17 u M^2 + 4.2 u M) + 1.05 d u s' (+ the FP64 fold's
//   own rounding, < 1e-15 d d2, and subnormal slack): B below doubles it.
// The FP32 fold costs 2 FP32 ops per coordinate against 3 FP64 ops (B200
// runs FP32 at twice the FP64 rate); undecided pairs are ~1e-5 of all.
__global__ void __launch_bounds__(kThreads) k_dist_mask(const double* __restrict__ X, int64_t n, int d,
                                                        int64_t nt, double thr, int all,
                                                        unsigned long long* __restrict__ masks,
                                                        uint32_t* __restrict__ rowtile_cnt, int64_t ti_lo,
                                                        int64_t ti_hi, int64_t mask_base) {
    int64_t ti, tj;
    tile_of_cta(nt, ti_lo, ti_hi, mask_base, ti, tj);
    __shared__ float fA[kDC][kT];
    __shared__ float fB[kDC][kT];
    __shared__ unsigned long long mrow[kT];
    __shared__ unsigned s_m;   // max |coordinate| of the tile's points (float bits)
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = ti * kT, j0 = tj * kT;
    if (threadIdx.x == 0) s_m = 0u;

    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
    float mloc = 0.0f;
    bool huge = false;
    if (!all) {
        for (int c0 = 0; c0 < d; c0 += kDC) {
            const int dc = min(kDC, d - c0);
            __syncthreads();
            for (int q = threadIdx.x; q < kT * kDC; q += kThreads) {
                const int r = q / kDC, c = q % kDC;
                double va = 0.0, vb = 0.0;
                if (c < dc) {
                    if (i0 + r < n) va = X[(i0 + r) * d + c0 + c];
                    if (j0 + r < n) vb = X[(j0 + r) * d + c0 + c];
                }
                huge |= !(fabs(va) < 1e15) || !(fabs(vb) < 1e15);
                fA[c][r] = __double2float_rn(va);
                fB[c][r] = __double2float_rn(vb);
                mloc = fmaxf(mloc, fmaxf(fabsf(fA[c][r]), fabsf(fB[c][r])));
            }
            __syncthreads();
            for (int c = 0; c < dc; ++c) {
                float a[4], b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) { a[q] = fA[c][ty + 16 * q]; b[q] = fB[c][tx + 16 * q]; }
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float t = __fsub_rn(a[p], b[q]);
                        acc[p][q] = __fmaf_rn(t, t, acc[p][q]);
                    }
            }
        }
    }
    // huge coordinates (float overflow / the bound's squares): every pair exact
    atomicMax(&s_m, huge ? 0x7F800000u : __float_as_uint(mloc));
    __syncthreads();
    const double M = (double)__uint_as_float(s_m) * (1.0 + 1e-6);   // |x'| <= M: |x| <= M (1 + u)
    const bool exact_all = s_m >= 0x7F800000u;
    const double u = 5.9604644775390625e-08;   // 2^-24
    const double Bc = 2.0 * (double)d * (17.0 * u * M * M + 4.2 * u * M) + 1e-30;
    const double Bs = 2.0 * 1.05 * (double)d * u + 1e-15 * (double)d;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int64_t i = i0 + ty + 16 * p;
        unsigned long long bits = 0ull;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t j = j0 + tx + 16 * q;
            if (!(i < n && j < n && j > i)) continue;
            bool keep = all != 0;
            if (!all) {
                const double s32 = (double)acc[p][q];
                const double B = Bc + Bs * s32;
                if (!exact_all && s32 + B <= thr) {
                    keep = true;
                } else if (!exact_all && s32 - B > thr) {
                    keep = false;
                } else {   // undecided: the exact FP64 fold (A5)
                    double e = 0.0;
                    for (int c = 0; c < d; ++c) {
                        const double t = __dsub_rn(X[i * d + c], X[j * d + c]);
                        e = __dadd_rn(e, __dmul_rn(t, t));
                    }
                    keep = e <= thr;
                }
            }
            if (keep) bits |= 1ull << (tx + 16 * q);
        }
        // the row's 16 threads are one half-warp (lanes tx): OR their bits
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
        if (tx == 0) mrow[ty + 16 * p] = bits;
    }
    __syncthreads();
    if (threadIdx.x < kT) {
        const int r = threadIdx.x;
        const unsigned long long m = mrow[r];
        masks[(tile_index(ti, tj, nt) - mask_base) * kT + r] = m;
        if (i0 + r < n) rowtile_cnt[(i0 + r - ti_lo * kT) * nt + tj] = (uint32_t)__popcll(m);
    }
}

// Full filtration (masks == null): every pair j > i is kept, so the row
// bits and the lex slot are closed-form and the mask pass is skipped.
__device__ __forceinline__ unsigned long long full_row_bits(int64_t i, int64_t j0, int64_t n) {
    const int64_t a = i + 1 - j0, b = n - j0;
    const int64_t lo = a > 0 ? a : 0, hi = b < kT ? b : kT;   // columns [lo, hi)
    if (lo >= hi) return 0ull;
    const unsigned long long upto = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
    return upto & ~((1ull << lo) - 1ull);
}

__global__ void __launch_bounds__(kThreads) k_dist_fill(const double* __restrict__ X, int64_t n, int d,
                                                        int64_t nt,
                                                        const unsigned long long* __restrict__ masks,
                                                        const uint64_t* __restrict__ slot_base,
                                                        uint64_t* __restrict__ key,
                                                        uint32_t* __restrict__ ei,
                                                        uint32_t* __restrict__ ej,
                                                        uint32_t* __restrict__ pij, int64_t ti_lo,
                                                        int64_t ti_hi, int64_t mask_base) {
    int64_t ti, tj;
    tile_of_cta(nt, ti_lo, ti_hi, mask_base, ti, tj);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i0 = ti * kT, j0 = tj * kT;
    const int64_t row_lo = ti_lo * kT;
    const unsigned long long* m = masks ? masks + (tile_index(ti, tj, nt) - mask_base) * kT : nullptr;
    // the tile's points, coordinate-major, when they fit (d <= kFillStageD):
    // the fold then reads shared memory (row point broadcast, column points
    // conflict-free) instead of strided global loads
    __shared__ double sA[kFillStageD][kT];
    __shared__ double sB[kFillStageD][kT];
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    if (threadIdx.x < kT && (m ? m[threadIdx.x] : full_row_bits(i0 + threadIdx.x, j0, n))) s_any = 1;
    __syncthreads();
    if (!s_any) return;
    const bool staged = d <= kFillStageD;
    if (staged) {
        for (int q = threadIdx.x; q < kT * d; q += kThreads) {
            const int r = q / d, c = q % d;
            sA[c][r] = i0 + r < n ? X[(i0 + r) * d + c] : 0.0;
            sB[c][r] = j0 + r < n ? X[(j0 + r) * d + c] : 0.0;
        }
        __syncthreads();
    }
    if (m && staged) {
        // capped build: the tile's kept pairs are sparse (C5B: ~5% of 4096),
        // so compact them first (row starts by a warp scan of the row
        // popcounts, then each row's set bits) and give every thread whole
        // pairs: no lane idles on a dropped pair
        __shared__ uint32_t rstart[kT + 1];
        __shared__ uint16_t plist[kT * kT];
        if (wid == 0) {
            uint32_t c0 = __popcll(m[lane]), c1 = __popcll(m[lane + 32]);
            uint32_t x0 = c0, x1 = c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
                if (lane >= o) { x0 += y0; x1 += y1; }
            }
            const uint32_t t0 = __shfl_sync(0xffffffffu, x0, 31);
            rstart[lane] = x0 - c0;
            rstart[lane + 32] = t0 + x1 - c1;
            if (lane == 31) rstart[kT] = t0 + x1;
        }
        __syncthreads();
        for (int r = wid; r < kT; r += kThreads / 32) {
            const unsigned long long bits = m[r];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = lane + 32 * h;
                if ((bits >> c) & 1ull)
                    plist[rstart[r] + __popcll(bits & ((1ull << c) - 1ull))] = (uint16_t)(r << 6 | c);
            }
        }
        __syncthreads();
        const uint32_t total = rstart[kT];
        for (uint32_t q = threadIdx.x; q < total; q += kThreads) {
            const int rc = plist[q], r = rc >> 6, c = rc & 63;
            const int64_t i = i0 + r, j = j0 + c;
            double acc = 0.0;
            for (int u = 0; u < d; ++u) {
                const double t = __dsub_rn(sA[u][r], sB[u][c]);
                acc = __dadd_rn(acc, __dmul_rn(t, t));
            }
            const double len = __dsqrt_rn(acc);
            const uint64_t slot = slot_base[(i - row_lo) * nt + tj] + (q - rstart[r]);
            key[slot] = (uint64_t)__double_as_longlong(len);
            if (pij) {
                pij[slot] = ((uint32_t)i << 16) | (uint32_t)j;
            } else {
                ei[slot] = (uint32_t)i;
                ej[slot] = (uint32_t)j;
            }
        }
        return;
    }
    for (int r = wid; r < kT; r += kThreads / 32) {
        const int64_t i = i0 + r;
        if (i >= n) break;
        const unsigned long long bits = m ? m[r] : full_row_bits(i, j0, n);
        if (!bits) continue;
        // full filtration: row i starts at lex slot i n - i (i + 1) / 2; its
        // columns j0 + c (c >= lo) follow from j = max(i + 1, j0)
        const uint64_t base = m ? slot_base[(i - row_lo) * nt + tj]
                                : (uint64_t)(i * n - i * (i + 1) / 2 + (j0 - i - 1 > 0 ? j0 - i - 1 : 0) -
                                             (row_lo * n - row_lo * (row_lo + 1) / 2));
        const double* xi = X + i * d;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            if (!((bits >> c) & 1ull)) continue;
            const int64_t j = j0 + c;
            const double* xj = X + j * d;
            double acc = 0.0;
            if (staged) {
                for (int q = 0; q < d; ++q) {
                    const double t = __dsub_rn(sA[q][r], sB[q][c]);
                    acc = __dadd_rn(acc, __dmul_rn(t, t));
                }
            } else {
                for (int q = 0; q < d; ++q) {
                    const double t = __dsub_rn(__ldg(xi + q), __ldg(xj + q));
                    acc = __dadd_rn(acc, __dmul_rn(t, t));
                }
            }
            const double len = __dsqrt_rn(acc);
            const uint64_t slot = base + __popcll(bits & ((1ull << c) - 1ull));
            key[slot] = (uint64_t)__double_as_longlong(len);
            if (pij) {
                pij[slot] = ((uint32_t)i << 16) | (uint32_t)j;
            } else {
                ei[slot] = (uint32_t)i;
                ej[slot] = (uint32_t)j;
            }
        }
    }
}

// Full filtration (r = inf, inclusive): every pair j > i is kept and the lex
// slot of (i, j) is closed-form, so one register-tiled pass computes and
// writes them (4 x 4 pairs per thread: 8 shared loads per coordinate serve
// 16 folds, as in k_dist_mask).  The fold is the same RN sequence
// (t = x_ic - x_jc; acc = acc + t * t; len = sqrt(acc)).  The pass also
// reduces min / max / OR of the length bits for the edge sort (key_range).
// The 4 x 4 register-tiled fold of the 64 x 64 tile (i0, j0): thread
// (tx, ty) holds the squared lengths of rows i0 + ty + 16 p, columns
// j0 + tx + 16 q (the same RN sequence t = x_ic - x_jc; acc = acc + t * t).
__device__ __forceinline__ void fold_tile(const double* __restrict__ X, int64_t n, int d, int64_t i0, int64_t j0,
                                          double (&sA)[kDC][kT], double (&sB)[kDC][kT], double (&acc)[4][4]) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int c0 = 0; c0 < d; c0 += kDC) {
        const int dc = min(kDC, d - c0);
        __syncthreads();
        for (int q = threadIdx.x; q < kT * kDC; q += kThreads) {
            const int r = q / kDC, c = q % kDC;
            double va = 0.0, vb = 0.0;
            if (c < dc) {
                if (i0 + r < n) va = X[(i0 + r) * d + c0 + c];
                if (j0 + r < n) vb = X[(j0 + r) * d + c0 + c];
            }
            sA[c][r] = va;
            sB[c][r] = vb;
        }
        __syncthreads();
        for (int c = 0; c < dc; ++c) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { a[q] = sA[c][ty + 16 * q]; b[q] = sB[c][tx + 16 * q]; }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double t = __dsub_rn(a[p], b[q]);
                    acc[p][q] = __dadd_rn(acc[p][q], __dmul_rn(t, t));
                }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_dist_full(const double* __restrict__ X, int64_t n, int d, int64_t nt,
                                                        uint64_t* __restrict__ key, uint32_t* __restrict__ ei,
                                                        uint32_t* __restrict__ ej, uint32_t* __restrict__ pij,
                                                        int64_t ti_lo, int64_t ti_hi, int64_t mask_base,
                                                        unsigned long long* __restrict__ range) {
    int64_t ti, tj;
    tile_of_cta(nt, ti_lo, ti_hi, mask_base, ti, tj);
    __shared__ double sA[kDC][kT];
    __shared__ double sB[kDC][kT];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = ti * kT, j0 = tj * kT;
    const int64_t row_lo = ti_lo * kT;
    double acc[4][4];
    fold_tile(X, n, d, i0, j0, sA, sB, acc);
    uint64_t mn = ~0ull, mx = 0ull, orr = 0ull;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int64_t i = i0 + ty + 16 * p;
        if (i >= n) continue;
        // row i starts at lex slot i n - i (i + 1) / 2 (less the block's first row)
        const uint64_t rbase = (uint64_t)(i * n - i * (i + 1) / 2 - (row_lo * n - row_lo * (row_lo + 1) / 2));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t j = j0 + tx + 16 * q;
            if (j <= i || j >= n) continue;
            const uint64_t bits = (uint64_t)__double_as_longlong(__dsqrt_rn(acc[p][q]));
            const uint64_t slot = rbase + (uint64_t)(j - i - 1);
            __stcs(reinterpret_cast<unsigned long long*>(key + slot), (unsigned long long)bits);
            if (pij) {
                __stcs(pij + slot, ((uint32_t)i << 16) | (uint32_t)j);
            } else {
                ei[slot] = (uint32_t)i;
                ej[slot] = (uint32_t)j;
            }
            mn = bits < mn ? bits : mn;
            mx = bits > mx ? bits : mx;
            orr |= bits;
        }
    }
    if (range) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t a = __shfl_down_sync(0xffffffffu, mn, o), b = __shfl_down_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
            orr |= __shfl_down_sync(0xffffffffu, orr, o);
        }
        if ((threadIdx.x & 31) == 0 && orr | mx) {
            atomicMin(&range[0], (unsigned long long)mn);
            atomicMax(&range[1], (unsigned long long)mx);
            atomicOr(&range[2], (unsigned long long)orr);
        }
    }
}

__global__ void k_check_points(const double* __restrict__ X, int64_t total, int* bad) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(X[q])) atomicOr(bad, 1);
}

__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, int64_t n, int d) {
    // in: d x n (dimension-major), out: n x d
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * d;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / d, c = q % d;
        out[q] = in[c * n + i];
    }
}

// ---------------------------------------------------------------------------
// F3: distance-matrix input ("a square symmetric matrix (typically a
// pairwise distance matrix)").  Edge (i, j), i < j, has length D[i][j] + 0.0
// (so -0.0 is +0.0).  Checked: off-diagonal entries finite, >= 0 and
// D[i][j] == D[j][i] (32 x 32 tiles staged through shared memory so both
// reads are coalesced); the diagonal is ignored.
// ---------------------------------------------------------------------------
__global__ void k_dm_check(const double* __restrict__ D, int64_t n, int* __restrict__ bad) {
    __shared__ double tile[32][33];
    const int64_t nt = (n + 31) / 32;
    for (int64_t t = blockIdx.x; t < nt * nt; t += gridDim.x) {
        const int64_t ti = t / nt, tj = t % nt;
        if (tj < ti) continue;
        // tile (tj, ti) transposed into shared memory
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t i = tj * 32 + r, j = ti * 32 + threadIdx.x;
            tile[r][threadIdx.x] = (i < n && j < n) ? D[i * n + j] : 0.0;
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t i = ti * 32 + r, j = tj * 32 + threadIdx.x;
            if (i < n && j < n && i != j) {
                const double a = D[i * n + j], b = tile[threadIdx.x][r];
                if (!(a >= 0.0) || isinf(a) || a != b) atomicOr(bad, 1);
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ bool dm_keep(double len, double r, int strict) { return strict ? len < r : len <= r; }

// kept pairs j > i of row i (one warp per row)
__global__ void k_dm_count(const double* __restrict__ D, int64_t n, double r, int strict, uint32_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        uint32_t c = 0;
        for (int64_t j = i + 1 + lane; j < n; j += 32) c += dm_keep(D[i * n + j] + 0.0, r, strict) ? 1u : 0u;
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) cnt[i] = c;
    }
}

// kept pairs of row i in lex order at [off[i], off[i+1]) (ballot compaction)
__global__ void k_dm_fill(const double* __restrict__ D, int64_t n, double r, int strict,
                          const uint64_t* __restrict__ off, uint64_t* __restrict__ key, uint32_t* __restrict__ ei,
                          uint32_t* __restrict__ ej, uint32_t* __restrict__ pij) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        uint64_t slot = off[i];
        for (int64_t j0 = i + 1; j0 < n; j0 += 32) {
            const int64_t j = j0 + lane;
            const double len = j < n ? D[i * n + j] + 0.0 : 0.0;
            const bool keep = j < n && dm_keep(len, r, strict);
            const uint32_t b = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint64_t q = slot + __popc(b & ((1u << lane) - 1u));
                key[q] = (uint64_t)__double_as_longlong(len);
                if (pij) {
                    pij[q] = ((uint32_t)i << 16) | (uint32_t)j;
                } else {
                    ei[q] = (uint32_t)i;
                    ej[q] = (uint32_t)j;
                }
            }
            slot += __popc(b);
        }
    }
}

// latlon2euc: degrees on the unit sphere -> xyz
__global__ void k_latlon2euc(const double* __restrict__ ll, int64_t n, double* __restrict__ xyz) {
    const double deg = 3.14159265358979323846 / 180.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double sla, cla, slo, clo;
        sincos(__dmul_rn(ll[2 * i], deg), &sla, &cla);
        sincos(__dmul_rn(ll[2 * i + 1], deg), &slo, &clo);
        xyz[3 * i] = __dmul_rn(cla, clo);
        xyz[3 * i + 1] = __dmul_rn(cla, slo);
        xyz[3 * i + 2] = sla;
    }
}

}  // namespace

void latlon2euc(const double* latlon, int64_t n, double* xyz, cudaStream_t s) {
    if (n <= 0) return;
    k_latlon2euc<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, s>>>(latlon, n, xyz);
    VRB_LAUNCH_CHECK();
}

void place_matrix(const double* D, int64_t n, uint32_t flags, cudaStream_t s, DBuf<double>& out) {
    const int64_t total = n * n;
    out.alloc((size_t)total, s);
    if (total == 0) return;
    VRB_CUDA(cudaMemcpyAsync(out.get(), D, total * sizeof(double),
                             (flags & VRB_POINTS_ON_DEVICE) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    DBuf<int> bad(1, s);
    VRB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    const int64_t nt = ceil_div(n, 32);
    k_dm_check<<<(unsigned)std::min<int64_t>(nt * nt, (int64_t)device_sm_count() * 16), dim3(32, 8), 0, s>>>(
        out.get(), n, bad.get());
    VRB_LAUNCH_CHECK();
    int h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h) fail(VRB_EINVAL, "distance matrix: an off-diagonal entry is negative, non-finite or asymmetric");
}

void build_kept_edges_dm(const double* D, int64_t n, double radius, bool strict, cudaStream_t s, KeptEdges& out) {
    out.E = 0;
    out.n = n;
    if (n < 2) return;
    DBuf<uint32_t> cnt(n, s);
    DBuf<uint64_t> off(n + 1, s);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n * 32, 256), (int64_t)device_sm_count() * 16);
    k_dm_count<<<g, 256, 0, s>>>(D, n, radius, strict ? 1 : 0, cnt.get());
    VRB_LAUNCH_CHECK();
    exclusive_scan(cnt.get(), off.get(), n, s);
    uint64_t E = 0;
    VRB_CUDA(cudaMemcpyAsync(&E, off.get() + n, sizeof(E), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (E >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu kept edges exceed u32 positions", (unsigned long long)E);
    out.E = (int64_t)E;
    if (E == 0) return;
    out.key.alloc(E, s);
    out.packed = n <= 65536;
    if (out.packed) {
        out.pij.alloc(E, s);
    } else {
        out.ei.alloc(E, s);
        out.ej.alloc(E, s);
    }
    k_dm_fill<<<g, 256, 0, s>>>(D, n, radius, strict ? 1 : 0, off.get(), out.key.get(), out.ei.get(), out.ej.get(),
                                out.pij.get());
    VRB_LAUNCH_CHECK();
}

// Threshold on d2 equivalent to the cap on len = sqrt_rn(d2) (reading A1).
double cap_threshold(double r, bool strict) {
    if (std::isinf(r)) return strict ? 1.79769313486231570815e308 : INFINITY;
    auto ok = [&](double x) { double s = std::sqrt(x); return strict ? s < r : s <= r; };
    if (!ok(0.0)) return -1.0;                    // nothing can be kept (strict, r == 0)
    double x = r * r;
    if (std::isinf(x)) x = 1.79769313486231570815e308;
    while (x > 0.0 && !ok(x)) x = std::nextafter(x, -INFINITY);
    while (!std::isinf(std::nextafter(x, INFINITY)) && ok(std::nextafter(x, INFINITY)))
        x = std::nextafter(x, INFINITY);
    return x;
}

bool place_points(const double* X, int64_t n, int d, uint32_t flags, cudaStream_t s, DBuf<double>& out, bool soft) {
    const int64_t total = n * d;
    if (out.size() != (size_t)total) out.alloc((size_t)total, s);
    if (total == 0) return true;
    DBuf<double> staged;
    const double* src = X;
    if (!(flags & VRB_POINTS_ON_DEVICE)) {
        if (flags & VRB_DIM_MAJOR) {
            staged.alloc((size_t)total, s);
            VRB_CUDA(cudaMemcpyAsync(staged.get(), X, total * sizeof(double), cudaMemcpyHostToDevice, s));
            src = staged.get();
        } else {
            VRB_CUDA(cudaMemcpyAsync(out.get(), X, total * sizeof(double), cudaMemcpyHostToDevice, s));
            src = nullptr;
        }
    }
    if (src) {
        const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 4096);
        if (flags & VRB_DIM_MAJOR) {
            k_transpose<<<g, 256, 0, s>>>(src, out.get(), n, d);
        } else {
            VRB_CUDA(cudaMemcpyAsync(out.get(), src, total * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
        VRB_LAUNCH_CHECK();
    }
    DBuf<int> bad(1, s);
    VRB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 4096);
    k_check_points<<<g, 256, 0, s>>>(out.get(), total, bad.get());
    VRB_LAUNCH_CHECK();
    int h = 0;
    VRB_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (h && !soft) fail(VRB_EINVAL, "non-finite coordinate in the point cloud");
    return h == 0;
}

int64_t edge_tile() { return kT; }


void build_kept_edges(const double* X, int64_t n, int d, double radius, bool strict, cudaStream_t s,
                      KeptEdges& out, int64_t row_lo, int64_t row_hi) {
    out.E = 0;
    out.n = n;
    if (row_hi < 0 || row_hi > n) row_hi = n;
    if (n < 2 || row_lo >= row_hi) return;
    if (row_lo % kT) fail(VRB_EINVAL, "row block must start at a multiple of %d", kT);
    const int64_t nt = ceil_div(n, kT);
    const int64_t ti_lo = row_lo / kT, ti_hi = ceil_div(row_hi, kT);
    if (row_hi != n && row_hi % kT) fail(VRB_EINVAL, "row block must end at a multiple of %d", kT);
    const int64_t nrows = std::min(row_hi, n) - row_lo;
    const double thr = cap_threshold(radius, strict);
    const int all = (!strict && std::isinf(radius)) ? 1 : 0;
    if (thr < 0.0) return;
    auto tidx = [&](int64_t ti) { return ti * nt - ti * (ti - 1) / 2; };   // first packed tile of tile row ti
    const int64_t mask_base = tidx(ti_lo);
    const int64_t ntiles = tidx(ti_hi) - mask_base;
    const unsigned grid = (unsigned)ntiles;
    if (all) {   // full filtration: no mask pass, closed-form slots
        auto start = [&](int64_t i) { return (uint64_t)(i * n - i * (i + 1) / 2); };   // lex slot of row i
        const uint64_t E = start(std::min(row_hi, n)) - start(row_lo);
        if (E >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu kept edges exceed u32 positions", (unsigned long long)E);
        out.E = (int64_t)E;
        out.key.alloc(E, s);
        out.packed = n <= 65536;
        if (out.packed) {
            out.pij.alloc(E, s);
        } else {
            out.ei.alloc(E, s);
            out.ej.alloc(E, s);
        }
        if (E == 0) return;
        // the key range (min, max, OR of the length bits) comes with the pass
        out.range.alloc(3, s);
        const unsigned long long init[3] = {~0ull, 0ull, 0ull};
        VRB_CUDA(cudaMemcpyAsync(out.range.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_dist_full<<<grid, kThreads, 0, s>>>(X, n, d, nt, out.key.get(), out.ei.get(), out.ej.get(), out.pij.get(),
                                              ti_lo, ti_hi, mask_base, out.range.get());
        VRB_LAUNCH_CHECK();
        return;
    }
    DBuf<unsigned long long> masks((size_t)ntiles * kT, s);
    DBuf<uint32_t> cnt((size_t)(nrows * nt), s);
    VRB_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
    k_dist_mask<<<grid, kThreads, 0, s>>>(X, n, d, nt, thr, all, masks.get(), cnt.get(), ti_lo, ti_hi, mask_base);
    VRB_LAUNCH_CHECK();
    DBuf<uint64_t> base((size_t)(nrows * nt + 1), s);
    exclusive_scan(cnt.get(), base.get(), nrows * nt, s);
    uint64_t E = 0;
    VRB_CUDA(cudaMemcpyAsync(&E, base.get() + nrows * nt, sizeof(E), cudaMemcpyDeviceToHost, s));
    VRB_CUDA(cudaStreamSynchronize(s));
    if (E >= 0xFFFFFFFFull) fail(VRB_EOVERFLOW, "%llu kept edges exceed u32 positions", (unsigned long long)E);
    out.E = (int64_t)E;
    if (E == 0) return;
    out.key.alloc(E, s);
    out.packed = n <= 65536;
    if (out.packed) {
        out.pij.alloc(E, s);
    } else {
        out.ei.alloc(E, s);
        out.ej.alloc(E, s);
    }
    k_dist_fill<<<grid, kThreads, 0, s>>>(X, n, d, nt, masks.get(), base.get(), out.key.get(),
                                          out.ei.get(), out.ej.get(), out.pij.get(), ti_lo, ti_hi, mask_base);
    VRB_LAUNCH_CHECK();
}

}  // namespace vrb
