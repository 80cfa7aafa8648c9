// Rank decision of Eigen's ColPivHouseholderQR (randevd.cpp:67-73, 89-92) on the device.
//
// Eigen counts the pivots |R_ii| > m eps max_k |R_kk| of a column-pivoted Householder QR.
// The fast probe in sketch.cu (a pivoted Cholesky of the double Gram Y^T Y) can only
// resolve |R_ii| / |R_00| down to ~sqrt(n eps): a Gram squares the condition number.  When
// it reports a deficient rank, this path decides with Eigen's own threshold instead:
//   * G = Y^T Y in double-double (exact products by FMA, compensated sums, fixed-order
//     split reduction), so G is accurate to ~n eps^2 |Y|^2;
//   * a diagonally pivoted Cholesky of G in double-double.  Its pivot order and |R_ii| are,
//     in exact arithmetic, those of the column-pivoted QR of Y (both pick the column of
//     largest remaining norm), so rank = #{R_ii > m eps R_00} is Eigen's rule.
// Only an ill-conditioned or exactly rank-deficient sample pays for it.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace w4 {
namespace {

struct dd {
    double hi, lo;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = a + b;
    const double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    double s, e;
    two_sum(a.hi, b.hi, s, e);
    e += a.lo + b.lo;
    dd r;
    r.hi = s + e;
    r.lo = e - (r.hi - s);
    return r;
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    const double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, e);
    e = fma(a.lo, b.hi, e);
    dd r;
    r.hi = p + e;
    r.lo = e - (r.hi - p);
    return r;
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
    const double q1 = a.hi / b.hi;
    const dd r = dd_add(a, dd_neg(dd_mul(dd{q1, 0.0}, b)));
    const double q2 = r.hi / b.hi;
    dd q;
    q.hi = q1 + q2;
    q.lo = q2 - (q.hi - q1);
    return q;
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
    if (!(a.hi > 0.0)) return dd{0.0, 0.0};
    const double s = sqrt(a.hi);
    const dd r = dd_add(a, dd_neg(dd_mul(dd{s, 0.0}, dd{s, 0.0})));
    const double c = r.hi / (2.0 * s);
    dd q;
    q.hi = s + c;
    q.lo = c - (q.hi - s);
    return q;
}

constexpr int TG = 16;   // Gram tile (TG x TG entries, one per thread)
constexpr int RB = 64;   // rows staged per step

// partial (split) of G tile (ti, tj): work[(split * m + j) * m + i] = {hi, lo}
__global__ void __launch_bounds__(TG* TG) dd_gram_kernel(int64_t n, int m, const double* __restrict__ Y, int64_t ld,
                                                          int64_t rows_per_split, int tiles, double2* __restrict__ work) {
    __shared__ double a[RB][TG + 1], b[RB][TG + 1];
    const int tile = blockIdx.x % (tiles * tiles);
    const int64_t split = blockIdx.x / (tiles * tiles);
    const int i0 = (tile % tiles) * TG, j0 = (tile / tiles) * TG;
    const int ti = threadIdx.x % TG, tj = threadIdx.x / TG;
    const int64_t r0 = split * rows_per_split, r1 = min(n, r0 + rows_per_split);
    dd acc{0.0, 0.0};
    for (int64_t rb = r0; rb < r1; rb += RB) {
        for (int e = threadIdx.x; e < RB * TG; e += TG * TG) {
            const int rr = e % RB, cc = e / RB;
            const int64_t r = rb + rr;
            a[rr][cc] = (r < r1 && i0 + cc < m) ? Y[r + (int64_t)(i0 + cc) * ld] : 0.0;
            b[rr][cc] = (r < r1 && j0 + cc < m) ? Y[r + (int64_t)(j0 + cc) * ld] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int rr = 0; rr < RB; ++rr) {
            const double x = a[rr][ti], y = b[rr][tj];
            const double p = x * y;
            const double pe = fma(x, y, -p);
            double s, e;
            two_sum(acc.hi, p, s, e);
            acc.lo += e + pe;
            acc.hi = s;
        }
        __syncthreads();
    }
    if (i0 + ti < m && j0 + tj < m) {
        double h = acc.hi + acc.lo;
        work[(split * m + j0 + tj) * m + i0 + ti] = make_double2(h, acc.lo - (h - acc.hi));
    }
}

__global__ void dd_reduce_kernel(int m, int64_t nsplit, const double2* __restrict__ work, double2* __restrict__ G) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)m * m) return;
    dd s{0.0, 0.0};
    for (int64_t k = 0; k < nsplit; ++k) {  // fixed order
        const double2 v = work[k * m * m + e];
        s = dd_add(s, dd{v.x, v.y});
    }
    G[e] = make_double2(s.hi, s.lo);
}

// Pivoted Cholesky of the dd Gram A (m x m, col-major, in place in global memory); rank by
// Eigen's rule R_ii > m eps R_00; perm[0 .. rank) = the pivot columns.
__global__ void __launch_bounds__(512) dd_pchol_kernel(int m, double2* __restrict__ A, double thr_factor,
                                                       int* rank, int* perm) {
    __shared__ int s_piv, s_stop;
    __shared__ double s_best[16];
    __shared__ int s_bidx[16];
    __shared__ dd s_r00;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < m; i += nt) perm[i] = i;
    __syncthreads();
    int r = m;
    for (int k = 0; k < m; ++k) {
        // pivot: largest remaining diagonal (lowest index on ties)
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < m; i += nt) {
            const double v = A[(int64_t)i * m + i].x;
            if (v > best) best = v, bi = i;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi;
        }
        if (lane == 0) s_best[warp] = best, s_bidx[warp] = bi;
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nt / 32; ++w)
                if (s_best[w] > best || (s_best[w] == best && s_bidx[w] < bi)) best = s_best[w], bi = s_bidx[w];
            const double2 pv = A[(int64_t)bi * m + bi];
            const dd piv{pv.x, pv.y};
            const dd rkk = dd_sqrt(piv);
            if (k == 0) s_r00 = rkk;
            s_stop = !(rkk.hi > thr_factor * s_r00.hi) || !isfinite(piv.hi);
            s_piv = bi;
            if (!s_stop && bi != k) {
                const int t = perm[k];
                perm[k] = perm[bi];
                perm[bi] = t;
            }
        }
        __syncthreads();
        if (s_stop) {
            r = k;
            break;
        }
        const int p = s_piv;
        if (p != k) {  // symmetric swap of rows and columns k, p
            for (int c = tid; c < m; c += nt) {
                const double2 t = A[(int64_t)c * m + k];
                A[(int64_t)c * m + k] = A[(int64_t)c * m + p];
                A[(int64_t)c * m + p] = t;
            }
            __syncthreads();
            for (int c = tid; c < m; c += nt) {
                const double2 t = A[(int64_t)k * m + c];
                A[(int64_t)k * m + c] = A[(int64_t)p * m + c];
                A[(int64_t)p * m + c] = t;
            }
            __syncthreads();
        }
        const double2 akk = A[(int64_t)k * m + k];
        const dd rkk = dd_sqrt(dd{akk.x, akk.y});
        __syncthreads();
        // row k of R: A[k, j] / R_kk for j > k (stored in column j, row k)
        for (int j = k + 1 + tid; j < m; j += nt) {
            const double2 v = A[(int64_t)j * m + k];
            const dd q = dd_div(dd{v.x, v.y}, rkk);
            A[(int64_t)j * m + k] = make_double2(q.hi, q.lo);
        }
        __syncthreads();
        // trailing update A[i, j] -= R_ki R_kj, i, j > k
        const int t = m - k - 1;
        for (int64_t e = tid; e < (int64_t)t * t; e += nt) {
            const int i = k + 1 + (int)(e % t), j = k + 1 + (int)(e / t);
            const double2 ri = A[(int64_t)i * m + k], rj = A[(int64_t)j * m + k];
            const double2 aij = A[(int64_t)j * m + i];
            const dd u = dd_add(dd{aij.x, aij.y}, dd_neg(dd_mul(dd{ri.x, ri.y}, dd{rj.x, rj.y})));
            A[(int64_t)j * m + i] = make_double2(u.hi, u.lo);
        }
        __syncthreads();
    }
    if (tid == 0) *rank = r;
}

}  // namespace

// rank (host) and perm (device, m ints) of Y (n x m, ld) by Eigen's ColPivHouseholderQR rule.
int colpiv_rank_dd(int64_t n, int m, const double* Y, int64_t ld, int* perm_dev, int* rank_dev, int* rank_host,
                   DevBuf& work, cudaStream_t st) {
    const int tiles = (m + TG - 1) / TG;
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * kSMs, (int64_t)tiles * tiles), cdiv(n, 4096)));
    const int64_t rows_per_split = cdiv(n, nsplit);
    nsplit = cdiv(n, rows_per_split);
    double2* w = work.get<double2>((size_t)(nsplit + 1) * m * m);
    double2* G = w + (size_t)nsplit * m * m;
    dd_gram_kernel<<<(unsigned)(nsplit * tiles * tiles), TG * TG, 0, st>>>(n, m, Y, ld, rows_per_split, tiles, w);
    W4_LAUNCH();
    dd_reduce_kernel<<<(unsigned)cdiv((int64_t)m * m, 256), 256, 0, st>>>(m, nsplit, w, G);
    W4_LAUNCH();
    const double thr = (double)m * 2.220446049250313e-16;  // Eigen: diagSize * epsilon
    dd_pchol_kernel<<<1, 512, 0, st>>>(m, G, thr, rank_dev, perm_dev);
    W4_LAUNCH();
    W4_CUDA(cudaMemcpyAsync(rank_host, rank_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    return *rank_host;
}

}  // namespace w4
