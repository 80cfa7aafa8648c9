// Single-CTA dense kernels on the (k+l)-dimension (see smallla.cuh).
#include "smallla.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace w4 {
namespace {

// Jacobi rotation (c, s) of the 2x2 problem (h = beta - alpha, g = 2 gamma or gamma): t =
// sgn(h) g / (|h| + sqrt(h^2 + g^2)), c = 1 / sqrt(1 + t^2), s = t c.  The IEEE sqrt and
// division sit on the serial path of every Jacobi step, so they are replaced by the MUFU
// approximations refined with two Newton steps (1-ulp class): c^2 + s^2 = 1 holds to working
// precision whatever the rounding of t, so the rotation stays orthogonal.
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double r = fma(-hx * y, y, 0.5);
    y = fma(y, r, y);
    r = fma(-hx * y, y, 0.5);
    return fma(y, r, y);
}
__device__ __forceinline__ void jacobi_rot(double h, double g, double& c, double& s) {
    const double x = fma(h, h, g * g);
    if (!(x > 1e-280 && x < 1e280)) {  // far outside the sketch range: IEEE path (no ftz / overflow)
        const double t = (h >= 0.0 ? g : -g) / (fabs(h) + sqrt(h * h + g * g));
        c = rsqrt(1.0 + t * t);
        s = t * c;
        return;
    }
    const double d = x * rsqrt_nr(x);
    const double t = (h >= 0.0 ? g : -g) * rcp_nr(fabs(h) + d);
    c = rsqrt_nr(fma(t, t, 1.0));
    s = t * c;
}


constexpr int kThreads = 1024;
constexpr size_t kSmemMax = 200 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// The single-CTA kernels take their working matrix in SMEM when it fits, else in a global
// work buffer.  SM is a template parameter so the SMEM variant compiles to LDS/STS instead
// of generic loads (which cost extra latency on every access of these latency-bound loops).

// ---------------------------------------------------------------- Cholesky
template <bool SM>
__global__ void __launch_bounds__(kThreads)
    chol_kernel(int m, const double* __restrict__ G, double* __restrict__ R, int* info,
                double* gwork, int use_smem) {
    extern __shared__ double sm[];
    double* A = SM ? sm : gwork;
    __shared__ int fail;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < m * m; e += nt) {
        const int i = e % m, j = e / m;
        A[e] = 0.5 * (G[i + j * m] + G[j + i * m]);
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    const int wid = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int j = 0; j < m; ++j) {
        // every thread reads the pivot after the previous barrier: uniform decision
        const double d = A[j + j * m];
        if (!(d > 0.0) || !isfinite(d)) {
            if (tid == 0) fail = j + 1;
            break;
        }
        const double ljj = sqrt(d);
        for (int i = j + 1 + tid; i < m; i += nt) A[i + j * m] /= ljj;
        __syncthreads();
        for (int k = j + 1 + wid; k < m; k += nw) {
            const double lk = A[k + j * m];
            for (int i = k + lane; i < m; i += 32) A[i + k * m] -= A[i + j * m] * lk;
        }
        if (tid == 0) A[j + j * m] = ljj;  // the trailing update never reads the diagonal
        __syncthreads();
    }
    __syncthreads();
    if (!fail)
        for (int e = tid; e < m * m; e += nt) {
            const int r = e % m, c = e / m;  // R(r, c) = L(c, r) for c >= r
            R[e] = (c >= r) ? A[c + r * m] : 0.0;
        }
    if (tid == 0) *info = fail;
}

// ---------------------------------------------------------------- Cholesky + inverse, fused
// R (upper, R^T R = sym(G)) and R^{-1} in one pass for m <= 128: symmetric Gaussian
// elimination of the augmented rows [G | I].  Step j subtracts m_ij = A(i,j) / A(j,j) times
// pivot row j from every row i > j, on the trailing lower triangle of A (the Schur
// complement) and on the lower triangle of X (which ends as L_unit^{-1}); then
// L = L_unit D^{1/2}, L^{-1} = D^{-1/2} L_unit^{-1}, R = L^T, R^{-1} = L^{-T}.
// Row i needs only i + 1 slots: slot c holds A(i,c) while c > j and X(i,c) once c <= j (the
// A entry retires, as pivot-column value, at exactly the step its X entry is born), so
// every update is v_c <- (c == j ? 0 : v_c) - m_ij p_c with p the compact pivot row
// [X(j, 0..j-1), 1, A(j+1..m-1, j)].  Slots live in registers of fixed owners (TPR threads
// per row, slot c at lane c % TPR); p is published to a double-buffered SMEM vector by its
// owners, so a step costs one barrier and at most NE FMAs per thread, instead of the two
// barriers and SMEM read-modify-writes of chol_kernel + tri_inv.
template <int TPR, int NP>
__global__ void __launch_bounds__(TPR * 128 < 1024 ? TPR * 128 : 1024)
    chol_inv_reg_kernel(int m, const double* __restrict__ G, double* __restrict__ R,
                        double* __restrict__ Rinv, int* info) {
    static_assert((NP & (NP - 1)) == 0, "NP must be a power of two");
    constexpr int SPAN = 2 * TPR;  // slots per register pair across a row's TPR threads
    __shared__ __align__(16) double pv[2][128];
    __shared__ double pd[2][2], rl_s[128];  // pd[b] = {sqrt(d_j), 1 / sqrt(d_j)}
    __shared__ int fail;
    const int tid = threadIdx.x;
    const int i = tid / TPR, lane = tid % TPR;
    const bool row_ok = i < m;
    const int c0 = 2 * lane;
    // Register pair s holds slots c0 + SPAN * ((s + k) % NP) + {0, 1} after k rotations: the
    // pair whose slots transition in the current block of SPAN steps is always v[0], so every
    // register index below is static.  Slots c > i are never read (no masks in the update).
    double v[NP][2];
#pragma unroll
    for (int s = 0; s < NP; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = c0 + SPAN * s + h;
            v[s][h] = (row_ok && c <= i) ? 0.5 * (G[i + (size_t)c * m] + G[c + (size_t)i * m]) : 0.0;
        }
    // The owner of the next pivot publishes its square root and reciprocal, so the sqrt /
    // division latency overlaps the other threads' updates.  A non-positive or non-finite
    // pivot publishes rl = NaN (every thread then sees the same breakdown).
    auto publish_pivot = [&](int b, double d) {
        const bool ok = d > 0.0 && isfinite(d);
        const double l = ok ? sqrt(d) : 0.0;
        pd[b][0] = l;
        pd[b][1] = ok ? 1.0 / l : __longlong_as_double(0x7ff8000000000000ll);
    };
    if (row_ok && lane == 0) {  // pivot row of step 0: p = [1, A(1..m-1, 0)], d = A(0, 0)
        if (i == 0) {
            pv[0][0] = 1.0;
            publish_pivot(0, v[0][0]);
        } else {
            pv[0][i] = v[0][0];
        }
    }
    if (tid == 0) fail = 0;
    __syncthreads();  // G fully read: R / Rinv may alias it from here on
    for (int e = tid; e < m * m; e += blockDim.x) {
        const int r = e % m, c = e / m;
        if (r > c) {
            R[e] = 0.0;
            Rinv[e] = 0.0;
        }
    }
    int f = 0, k = 0;
    for (int jb = 0; jb < m && !f; jb += SPAN, ++k) {
#pragma unroll
        for (int u = 0; u < SPAN; ++u) {
            const int j = jb + u;
            if (j >= m) break;
            const int b = j & 1;
            const double ljj = pd[b][0], rl = pd[b][1];
            if (rl != rl) {  // NaN: breakdown at pivot j (uniform)
                f = j + 1;
                break;
            }
            if (tid == 0) rl_s[j] = rl;
            if (row_ok && i >= j) {
                const double aij = pv[b][i];
                if (lane == 0) R[j + (size_t)i * m] = (i == j) ? ljj : aij * rl;
                if (i > j) {
                    const double mi = aij * (rl * rl);
                    // slot j (v[0][u & 1] of lane u / 2) turns from A(i, j) into X(i, j)
                    if (lane == (u >> 1)) v[0][u & 1] = 0.0;
#pragma unroll
                    for (int s = 0; s < NP; ++s) {
                        const int c = c0 + SPAN * ((s + k) & (NP - 1));
                        const double2 p2 = *reinterpret_cast<const double2*>(&pv[b][c]);
                        v[s][0] = fma(-mi, p2.x, v[s][0]);
                        v[s][1] = fma(-mi, p2.y, v[s][1]);
                    }
                    // publish the pivot row of step j + 1 into the other buffer
                    const int jn = j + 1;
                    if (i == jn) {  // X(jn, 0..j)
#pragma unroll
                        for (int s = 0; s < NP; ++s)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int c = c0 + SPAN * ((s + k) & (NP - 1)) + h;
                                if (c <= j) pv[b ^ 1][c] = v[s][h];
                            }
                    }
                    // slot jn: v[0][(u + 1) & 1] of lane (u + 1) / 2, or v[1][0] of lane 0
                    const int ln = (u + 1 < SPAN) ? ((u + 1) >> 1) : 0;
                    if (lane == ln) {
                        const double x = (u + 1 < SPAN) ? v[0][(u + 1) & 1] : v[1 % NP][0];
                        if (i == jn) {
                            pv[b ^ 1][jn] = 1.0;
                            publish_pivot(b ^ 1, x);
                        } else {
                            pv[b ^ 1][i] = x;
                        }
                    }
                }
            }
            __syncthreads();
        }
        // rotate: the finished pair moves to the back, the next block's pair to v[0]
        double t0 = v[0][0], t1 = v[0][1];
#pragma unroll
        for (int s = 0; s + 1 < NP; ++s) {
            v[s][0] = v[s + 1][0];
            v[s][1] = v[s + 1][1];
        }
        v[NP - 1][0] = t0;
        v[NP - 1][1] = t1;
    }
    if (tid == 0) {
        fail = f;
        *info = f;
    }
    __syncthreads();
    if (fail || !row_ok) return;
    const double ri = rl_s[i];
#pragma unroll
    for (int s = 0; s < NP; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = c0 + SPAN * ((s + k) & (NP - 1)) + h;
            if (c <= i) Rinv[c + (size_t)i * m] = (c == i ? 1.0 : v[s][h]) * ri;
        }
}

template <int TPR, int NP>
void launch_chol_inv(int m, const double* G, double* R, double* Rinv, int* info, cudaStream_t st) {
    chol_inv_reg_kernel<TPR, NP><<<1, TPR * m, 0, st>>>(m, G, R, Rinv, info);
    W4_LAUNCH();
}

// ---------------------------------------------------------------- pivoted Cholesky rank
template <bool SM>
__global__ void __launch_bounds__(kThreads)
    pchol_kernel(int m, const double* __restrict__ G, double tol_rel, int* rank, int* perm,
                 double* gwork, int use_smem) {
    extern __shared__ double sm[];
    double* A = SM ? sm : gwork;
    __shared__ int piv, stop;
    __shared__ double maxd;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < m * m; e += nt) {
        const int i = e % m, j = e / m;
        A[e] = 0.5 * (G[i + j * m] + G[j + i * m]);
    }
    for (int i = tid; i < m; i += nt) perm[i] = i;
    __syncthreads();
    if (tid == 0) {
        double mx = 0.0;
        for (int i = 0; i < m; ++i) mx = fmax(mx, A[i + i * m]);
        maxd = mx;
        stop = 0;
    }
    __syncthreads();
    const double tol = tol_rel * maxd;
    int r = m;
    for (int j = 0; j < m; ++j) {
        if (tid == 0) {
            int p = j;
            double best = A[j + j * m];
            for (int i = j + 1; i < m; ++i)
                if (A[i + i * m] > best) {
                    best = A[i + i * m];
                    p = i;
                }
            piv = p;
            stop = !(best > tol) || !isfinite(best);
            if (!stop && p != j) {
                const int t = perm[j];
                perm[j] = perm[p];
                perm[p] = t;
            }
        }
        __syncthreads();
        if (stop) {
            r = j;
            break;
        }
        const int p = piv;
        if (p != j) {
            for (int c = tid; c < m; c += nt) {
                const double t = A[j + c * m];
                A[j + c * m] = A[p + c * m];
                A[p + c * m] = t;
            }
            __syncthreads();
            for (int rr = tid; rr < m; rr += nt) {
                const double t = A[rr + j * m];
                A[rr + j * m] = A[rr + p * m];
                A[rr + p * m] = t;
            }
            __syncthreads();
        }
        const double ljj = sqrt(A[j + j * m]);
        __syncthreads();
        for (int i = j + tid; i < m; i += nt) A[i + j * m] = (i == j) ? ljj : A[i + j * m] / ljj;
        __syncthreads();
        const int w = m - j - 1;
        for (int e = tid; e < w * w; e += nt) {
            const int i = j + 1 + e % w, k = j + 1 + e / w;
            A[i + k * m] -= A[i + j * m] * A[k + j * m];
        }
        __syncthreads();
    }
    if (tid == 0) *rank = r;
}

// ---------------------------------------------------------------- triangular inverse
// Single CTA, R staged in SMEM: warp w solves R x = e_j for columns j = w, w + 32, ...
__global__ void __launch_bounds__(1024)
    tri_inv_smem_kernel(int m, const double* __restrict__ R, double* __restrict__ Rinv) {
    extern __shared__ double sm[];
    double* Rs = sm;                           // m x m
    const int tid = threadIdx.x, nt = blockDim.x;
    const int wid = tid >> 5, lane = tid & 31, nw = nt >> 5;
    double* x = sm + (size_t)m * m + (size_t)wid * m;
    for (int e = tid; e < m * m; e += nt) Rs[e] = R[e];
    __syncthreads();
    for (int j = wid; j < m; j += nw) {
        if (lane == 0) x[j] = 1.0 / Rs[j + j * m];
        __syncwarp();
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1 + lane; k <= j; k += 32) s += Rs[i + k * m] * x[k];
            s = warp_sum(s);
            if (lane == 0) x[i] = -s / Rs[i + i * m];
            __syncwarp();
        }
        for (int i = lane; i < m; i += 32) Rinv[i + j * m] = (i <= j) ? x[i] : 0.0;
        __syncwarp();
    }
}

__global__ void tri_inv_kernel(int m, const double* __restrict__ R, double* __restrict__ Rinv) {
    extern __shared__ double xs[];
    const int warps = blockDim.x / 32;
    const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int j = blockIdx.x * warps + wid;
    if (j >= m) return;
    double* x = xs + wid * m;
    if (lane == 0) x[j] = 1.0 / R[j + j * m];
    __syncwarp();
    for (int i = j - 1; i >= 0; --i) {
        double s = 0.0;
        for (int k = i + 1 + lane; k <= j; k += 32) s += R[i + k * m] * x[k];
        s = warp_sum(s);
        if (lane == 0) x[i] = -s / R[i + i * m];
        __syncwarp();
    }
    for (int i = lane; i < m; i += 32) Rinv[i + j * m] = (i <= j) ? x[i] : 0.0;
}

// ---------------------------------------------------------------- round-robin pairs
__device__ __forceinline__ void rr_pair(int k, int r, int mp, int& p, int& q) {
    auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + r) % (mp - 1); };
    p = player(k);
    q = player(mp - 1 - k);
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}

// ---------------------------------------------------------------- two-sided Jacobi EVD, 2x2 blocks
// Parallel cyclic Jacobi (round-robin pairs).  All m/2 rotations of a round act on
// disjoint index pairs, so A' = J^T A J factors into independent 2x2 blocks
// A'_{PQ} = J_P^T A_{PQ} J_Q: each thread reads, rotates and writes whole blocks, and a
// round costs two barriers (rotation parameters, block update) instead of three.  The
// matrix is padded to even order with a zero row/column that no rotation ever touches.
constexpr int kEvdThreads = 512;

template <bool SM>
__global__ void __launch_bounds__(kEvdThreads)
    jacobi_evd_blk_kernel(int m, const double* __restrict__ K, double* __restrict__ vals,
                          double* __restrict__ W, double* gwork, int use_smem, int debug,
                          const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // the Cholesky + one-sided path succeeded (sym_evd_desc)
    extern __shared__ double sm[];
    const int mp = m + (m & 1);
    double* A = SM ? sm : gwork;
    double* V = A + (size_t)mp * mp;
    __shared__ double cs_c[256], cs_s[256];
    __shared__ int cs_p[256], cs_q[256];
    __shared__ int rank_of[512];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < mp * mp; e += nt) {
        const int i = e % mp, j = e / mp;
        A[e] = (i < m && j < m) ? 0.5 * (K[i + j * m] + K[j + i * m]) : 0.0;
        V[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    const int npairs = mp / 2;
    // fixed per-thread roles of the block-update phase (see below)
    const int aTQ = nt / npairs > 0 ? nt / npairs : 1;
    const int aP = tid < aTQ * npairs ? tid % npairs : npairs;  // npairs: no A role
    const int aQ0 = tid / npairs;
    const int vTQ = nt / mp > 0 ? nt / mp : 1;
    const int vI = tid < vTQ * mp ? tid % mp : mp;  // mp: no V role
    const int vQ0 = tid / mp;
    for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
        int rotated = 0;
        for (int r = 0; r < mp - 1; ++r) {
            for (int k = tid; k < npairs; k += nt) {
                int p, q;
                rr_pair(k, r, mp, p, q);
                double c = 1.0, s = 0.0;
                const double apq = A[p + q * mp];
                const double app = A[p + p * mp], aqq = A[q + q * mp];
                // Rotation threshold m*eps*sqrt|a_pp a_qq| (relative accuracy m*eps); a
                // pure eps threshold lets roundoff re-create above-threshold entries so the
                // sweep never goes quiet.
                // (squared test, no sqrt).  Rotation t = sgn(tau)/(|tau| + sqrt(1 + tau^2)),
                // tau = h / g, rewritten as sgn(h) g / (|h| + sqrt(h^2 + g^2)), c = 1 / sqrt(1
                // + t^2) (jacobi_rot: Newton-refined MUFU reciprocal / rsqrt on this serial path).
                const double thr = mp * DBL_EPSILON;
                if (apq != 0.0 && apq * apq > thr * thr * fabs(app * aqq)) {
                    const double h = aqq - app, g = 2.0 * apq;
                    jacobi_rot(h, g, c, s);
                    rotated = 1;
                }
                cs_c[k] = c;
                cs_s[k] = s;
                cs_p[k] = p;
                cs_q[k] = q;
            }
            __syncthreads();
            // 2x2 block updates A <- J_P^T A J_Q for all pair blocks (P, Q) and V <- V J_Q.
            // Each thread's roles were fixed before the sweep (no per-item index division):
            // A blocks (P = aP, Q = aQ0 + k aTQ), V entries (row vI, pair Q = vQ0 + k vTQ).
            // Two items per step with both loads issued before either store (the blocks are
            // disjoint).  A pair with (c, s) = (1, 0) leaves its entries bit-identical.
            if (aP < npairs) {
                const int p1 = cs_p[aP], p2 = cs_q[aP];
                const double cP = cs_c[aP], sP = cs_s[aP];
                auto rot_blk = [&](int Q, double& a11, double& a12, double& a21, double& a22) {
                    const double cQ = cs_c[Q], sQ = cs_s[Q];
                    const double b11 = cQ * a11 - sQ * a12, b12 = sQ * a11 + cQ * a12;
                    const double b21 = cQ * a21 - sQ * a22, b22 = sQ * a21 + cQ * a22;
                    a11 = cP * b11 - sP * b21;
                    a21 = sP * b11 + cP * b21;
                    a12 = cP * b12 - sP * b22;
                    a22 = sP * b12 + cP * b22;
                };
                int Q = aQ0;
                for (; Q + aTQ < npairs; Q += 2 * aTQ) {
                    const int Qb = Q + aTQ;
                    const int qa1 = cs_p[Q] * mp, qa2 = cs_q[Q] * mp, qb1 = cs_p[Qb] * mp, qb2 = cs_q[Qb] * mp;
                    double x11 = A[p1 + qa1], x12 = A[p1 + qa2], x21 = A[p2 + qa1], x22 = A[p2 + qa2];
                    double y11 = A[p1 + qb1], y12 = A[p1 + qb2], y21 = A[p2 + qb1], y22 = A[p2 + qb2];
                    rot_blk(Q, x11, x12, x21, x22);
                    rot_blk(Qb, y11, y12, y21, y22);
                    A[p1 + qa1] = x11;
                    A[p1 + qa2] = x12;
                    A[p2 + qa1] = x21;
                    A[p2 + qa2] = x22;
                    A[p1 + qb1] = y11;
                    A[p1 + qb2] = y12;
                    A[p2 + qb1] = y21;
                    A[p2 + qb2] = y22;
                }
                if (Q < npairs) {
                    const int qa1 = cs_p[Q] * mp, qa2 = cs_q[Q] * mp;
                    double x11 = A[p1 + qa1], x12 = A[p1 + qa2], x21 = A[p2 + qa1], x22 = A[p2 + qa2];
                    rot_blk(Q, x11, x12, x21, x22);
                    A[p1 + qa1] = x11;
                    A[p1 + qa2] = x12;
                    A[p2 + qa1] = x21;
                    A[p2 + qa2] = x22;
                }
            }
            if (vI < mp) {
                int Q = vQ0;
                for (; Q + vTQ < npairs; Q += 2 * vTQ) {
                    const int Qb = Q + vTQ;
                    const int oa1 = vI + cs_p[Q] * mp, oa2 = vI + cs_q[Q] * mp;
                    const int ob1 = vI + cs_p[Qb] * mp, ob2 = vI + cs_q[Qb] * mp;
                    const double va1 = V[oa1], va2 = V[oa2], vb1 = V[ob1], vb2 = V[ob2];
                    const double ca = cs_c[Q], sa = cs_s[Q], cb = cs_c[Qb], sb = cs_s[Qb];
                    V[oa1] = ca * va1 - sa * va2;
                    V[oa2] = sa * va1 + ca * va2;
                    V[ob1] = cb * vb1 - sb * vb2;
                    V[ob2] = sb * vb1 + cb * vb2;
                }
                if (Q < npairs) {
                    const int oa1 = vI + cs_p[Q] * mp, oa2 = vI + cs_q[Q] * mp;
                    const double va1 = V[oa1], va2 = V[oa2];
                    const double ca = cs_c[Q], sa = cs_s[Q];
                    V[oa1] = ca * va1 - sa * va2;
                    V[oa2] = sa * va1 + ca * va2;
                }
            }
            __syncthreads();
        }
        const int any = __syncthreads_or(rotated);
        if (debug && tid == 0) printf("jacobi_evd m=%d sweep %d rotated %d\n", m, sweep, any);
        if (!any) break;
    }
    for (int i = tid; i < m; i += nt) {
        const double di = A[i + i * mp];
        int rk = 0;
        for (int j = 0; j < m; ++j) {
            const double dj = A[j + j * mp];
            rk += (dj > di) || (dj == di && j < i);
        }
        rank_of[i] = rk;
        vals[rk] = di;
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += nt) {
        const int i = e % m, j = e / m;
        W[i + rank_of[j] * m] = V[i + j * mp];
    }
}

// ---------------------------------------------------------------- tridiagonal-QL EVD
// Symmetric EVD for the Rayleigh-Ritz / ritzit / Nystrom small problems
// (SelfAdjointEigenSolver, randevd.cpp:37-43): Householder tridiagonalisation (m-2
// reflections, each one SMEM mat-vec + rank-2 update), implicit-shift QL on the
// tridiagonal (the scalar recurrence runs on one thread; each QL sweep's Givens rotations
// are recorded and then applied to the eigenvector rows by all threads at once), and the
// back-transform by the stored reflectors.  ~6 barriers per reflection + 2 per QL sweep
// instead of the 2 per round x (m-1) rounds x ~9 sweeps of cyclic Jacobi.  Absolute
// accuracy ~ m eps ||K|| (LAPACK steqr class).
__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();  // red[] may still be read by a previous call
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];  // fixed order: deterministic
    return t;
}

constexpr int kTqlThreads = 512;

template <bool SM>
__global__ void __launch_bounds__(kTqlThreads)
    sym_evd_tql_kernel(int m, const double* __restrict__ K, double* __restrict__ vals,
                       double* __restrict__ W, double* gwork, int use_smem, int* info) {
    extern __shared__ double sm[];
    double* base = SM ? sm : gwork;
    double* A = base;                      // m x m column-major; reflectors below the subdiagonal
    double* Z = A + (size_t)m * m;         // eigenvectors of T, column-major Z[i + k m]
    double* d = Z + (size_t)m * m;         // diagonal
    double* e = d + m;                     // subdiagonal e[i] = T(i+1, i), e[m-1] = 0
    double* tau = e + m;
    double* pv = tau + m;
    double* rc = pv + m;                   // recorded rotations of one QL sweep
    double* rs = rc + m;
    int* ri = reinterpret_cast<int*>(rs + m);
    __shared__ double red[32];
    __shared__ int s_ctl[4];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;

    for (int idx = tid; idx < m * m; idx += nt) {
        const int i = idx % m, j = idx / m;
        A[idx] = 0.5 * (K[i + j * m] + K[j + i * m]);
        Z[idx] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();

    // 1. Householder tridiagonalisation: H_k = I - tau_k u u^T zeroes A[k+2:, k]
    for (int k = 0; k + 2 < m; ++k) {
        const int n2 = m - k - 1;
        double* x = A + (k + 1) + (size_t)k * m;  // column k below the diagonal, length n2
        double part = 0.0;
        for (int i = 1 + tid; i < n2; i += nt) part += x[i] * x[i];
        const double sig = block_sum(part, red);
        const double x0 = x[0];
        if (sig == 0.0) {  // already tridiagonal in this column
            if (tid == 0) {
                tau[k] = 0.0;
                e[k] = x0;
            }
            continue;
        }
        const double alpha = -copysign(sqrt(x0 * x0 + sig), x0);
        const double u0 = x0 - alpha;
        const double tk = 2.0 / (u0 * u0 + sig);
        __syncthreads();  // everyone has read x0
        if (tid == 0) {
            x[0] = u0;  // u = [u0, x1, ...] stored in place
            tau[k] = tk;
            e[k] = alpha;
        }
        __syncthreads();
        // p = tau A22 u (rows of A22 via symmetry: consecutive threads, consecutive rows)
        double* A22 = A + (k + 1) + (size_t)(k + 1) * m;
        for (int i = tid; i < n2; i += nt) {
            double s = 0.0;
            for (int j = 0; j < n2; ++j) s += A22[i + (size_t)j * m] * x[j];
            pv[i] = tk * s;
        }
        __syncthreads();
        part = 0.0;
        for (int i = tid; i < n2; i += nt) part += x[i] * pv[i];
        const double Kc = 0.5 * tk * block_sum(part, red);
        for (int i = tid; i < n2; i += nt) pv[i] -= Kc * x[i];  // w = p - K u
        __syncthreads();
        for (int idx = tid; idx < n2 * n2; idx += nt) {  // A22 -= u w^T + w u^T
            const int i = idx % n2, j = idx / n2;
            A22[i + (size_t)j * m] -= x[i] * pv[j] + pv[i] * x[j];
        }
        __syncthreads();
    }
    for (int i = tid; i < m; i += nt) {
        d[i] = A[i + (size_t)i * m];
        if (i + 2 >= m) tau[i] = 0.0;
    }
    if (tid == 0) {
        if (m >= 2) e[m - 2] = A[(m - 1) + (size_t)(m - 2) * m];
        e[m - 1] = 0.0;
    }
    __syncthreads();

    // 2. implicit-shift QL on (d, e); thread 0 runs the recurrence, everyone rotates Z rows
    int l = 0, iter = 0;
    while (true) {
        if (tid == 0) {
            int nrot = 0, done = 0;
            while (l < m) {
                int mm;
                for (mm = l; mm < m - 1; ++mm) {
                    const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
                    if (fabs(e[mm]) <= DBL_EPSILON * dd) break;
                }
                if (mm == l) {  // d[l] converged
                    ++l;
                    iter = 0;
                    continue;
                }
                if (++iter > 60) {  // no convergence: poison the values (caught by validation)
                    if (info) *info = 1;
                    for (int q = 0; q < m; ++q) d[q] = nan("");
                    done = 1;
                    break;
                }
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = hypot(g, 1.0);
                g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = mm - 1; i >= l; --i) {
                    const double ei = e[i];
                    const double f = s * ei;
                    const double b = c * ei;
                    // r = hypot(f, g) via one rsqrt (values here are far from over/underflow)
                    const double h2 = f * f + g * g;
                    if (h2 == 0.0) {
                        e[i + 1] = 0.0;
                        r = 0.0;
                        d[i + 1] -= p;
                        e[mm] = 0.0;
                        break;
                    }
                    const double rinv = rsqrt(h2);
                    r = h2 * rinv;
                    e[i + 1] = r;
                    s = f * rinv;
                    c = g * rinv;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    d[i + 1] = g + (p = s * r);
                    g = c * r - b;
                    rc[nrot] = c;
                    rs[nrot] = s;
                    ri[nrot] = i;
                    ++nrot;
                }
                if (r == 0.0 && i >= l) break;  // split: rotations so far are recorded
                d[l] -= p;
                e[l] = g;
                e[mm] = 0.0;
                break;
            }
            if (l >= m) done = 1;
            s_ctl[0] = nrot;
            s_ctl[1] = done;
        }
        __syncthreads();
        const int nrot = s_ctl[0], done = s_ctl[1];
        // z[row][i], z[row][i+1]; one sweep's rotations visit i = i0, i0-1, ..., so the
        // updated z[row][i] is carried in a register into the next rotation
        if (nrot > 0)
            for (int row = tid; row < m; row += nt) {
                const int i0 = ri[0];
                double f = Z[row + (size_t)(i0 + 1) * m];
                for (int q = 0; q < nrot; ++q) {
                    const int i = i0 - q;
                    const double c = rc[q], s = rs[q];
                    const double zi = Z[row + (size_t)i * m];
                    Z[row + (size_t)(i + 1) * m] = s * zi + c * f;
                    f = c * zi - s * f;
                }
                Z[row + (size_t)(i0 + 1 - nrot) * m] = f;
            }
        __syncthreads();
        if (done) break;
    }

    // 3. back-transform: eigvecs = H_0 H_1 ... H_{m-3} Z
    for (int k = m - 3; k >= 0; --k) {
        const double tk = tau[k];
        if (tk == 0.0) continue;
        const int n2 = m - k - 1;
        const double* u = A + (k + 1) + (size_t)k * m;
        for (int c = wid; c < m; c += nw) {  // s_c = u^T Z[k+1:, c]
            double s = 0.0;
            for (int i = lane; i < n2; i += 32) s += u[i] * Z[(k + 1 + i) + (size_t)c * m];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) pv[c] = tk * s;
        }
        __syncthreads();
        for (int idx = tid; idx < n2 * m; idx += nt) {
            const int i = idx % n2, c = idx / n2;
            Z[(k + 1 + i) + (size_t)c * m] -= u[i] * pv[c];
        }
        __syncthreads();
    }

    // 4. decreasing order (sorted_symmetric_evd, randevd.cpp:37-43)
    for (int i = tid; i < m; i += nt) {
        const double di = d[i];
        int rk = 0;
        for (int j = 0; j < m; ++j) {
            const double dj = d[j];
            rk += (dj > di) || (dj == di && j < i);
        }
        ri[i] = rk;
        vals[rk] = di;
    }
    __syncthreads();
    for (int idx = tid; idx < m * m; idx += nt) {
        const int i = idx % m, j = idx / m;
        W[i + (size_t)ri[j] * m] = Z[i + (size_t)j * m];
    }
}

// ---------------------------------------------------------------- one-sided Jacobi SVD
template <bool SM>
__global__ void __launch_bounds__(kThreads)
    jacobi_svd_kernel(int m, const double* __restrict__ Xin, double* __restrict__ sigma,
                      double* __restrict__ U, double* gwork, int use_smem) {
    extern __shared__ double sm[];
    double* X = SM ? sm : gwork;
    __shared__ double cs_c[512], cs_s[512];
    __shared__ int cs_p[512], cs_q[512];
    __shared__ double nrm[512];
    __shared__ int rank_of[512];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int wid = tid / 32, lane = tid % 32, nw = nt / 32;
    for (int e = tid; e < m * m; e += nt) X[e] = Xin[e];
    __syncthreads();
    const int mp = m + (m & 1);
    const int npairs = mp / 2;
    const int uTK = nt / m > 0 ? nt / m : 1;  // update roles, fixed for all rounds
    const int uI = tid < uTK * m ? tid % m : m;
    const int uK0 = tid / m;
    for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
        int rotated = 0;
        for (int r = 0; r < mp - 1; ++r) {
            // 8-lane groups per column pair (4 pairs per warp, all pairs of a round at once);
            // the warp iterates uniformly so the width-8 shuffles see every lane
            const int gl = lane & 7, grp = lane >> 3;
            for (int base = wid * 4; base < npairs; base += nw * 4) {
                const int k = base + grp;
                int p = 0, q = m;
                if (k < npairs) rr_pair(k, r, mp, p, q);
                double c = 1.0, s = 0.0;
                double al = 0.0, be = 0.0, ga = 0.0;
                if (q < m)
                    for (int i = gl; i < m; i += 8) {
                        const double xp = X[i + p * m], xq = X[i + q * m];
                        al += xp * xp;
                        be += xq * xq;
                        ga += xp * xq;
                    }
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o, 8);
                    be += __shfl_xor_sync(0xffffffffu, be, o, 8);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o, 8);
                }
                if (k >= npairs) continue;
                if (q < m) {
                    // |ga| > mp eps sqrt(al be), squared; t as in the two-sided kernel
                    const double thr = mp * DBL_EPSILON;
                    if (ga != 0.0 && ga * ga > thr * thr * (al * be)) {
                        const double h = be - al, g = 2.0 * ga;
                        jacobi_rot(h, g, c, s);
                        rotated = 1;
                    }
                }
                if (gl == 0) {
                    cs_c[k] = c;
                    cs_s[k] = s;
                    cs_p[k] = p;
                    cs_q[k] = q;
                }
            }
            __syncthreads();
            if (uI < m)  // fixed roles: row uI of pairs k = uK0, uK0 + uTK, ...
                for (int k = uK0; k < npairs; k += uTK) {
                    const double s = cs_s[k];
                    if (s == 0.0) continue;
                    const double c = cs_c[k];
                    const int op = uI + cs_p[k] * m, oq = uI + cs_q[k] * m;
                    const double xp = X[op], xq = X[oq];
                    X[op] = c * xp - s * xq;
                    X[oq] = s * xp + c * xq;
                }
            __syncthreads();
        }
        if (!__syncthreads_or(rotated)) break;
    }
    for (int j = wid; j < m; j += nw) {
        double a = 0.0;
        for (int i = lane; i < m; i += 32) a += X[i + j * m] * X[i + j * m];
        a = warp_sum(a);
        if (lane == 0) nrm[j] = sqrt(a);
    }
    __syncthreads();
    for (int i = tid; i < m; i += nt) {
        int rk = 0;
        for (int j = 0; j < m; ++j) rk += (nrm[j] > nrm[i]) || (nrm[j] == nrm[i] && j < i);
        rank_of[i] = rk;
        sigma[rk] = nrm[i];
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += nt) {
        const int i = e % m, j = e / m;
        const double sj = nrm[j];
        U[i + rank_of[j] * m] = sj > 0.0 ? X[e] / sj : 0.0;
    }
}

// ---------------------------------------------------------------- one-sided Jacobi, one barrier
// Left singular vectors / values of X (m <= 128), or of X^T (trans), by one-sided Jacobi in
// the odd-even transposition ordering (Brent-Luk): positions 0..mp-1 on a line; even steps
// rotate the column pairs at positions (2k, 2k+1), odd steps (2k+1, 2k+2), and every rotated
// pair swaps positions, so after mp steps every pair of columns has met exactly once (a
// sweep).  Group k (8 lanes) owns the pair of step parity; a column pair lives in
// REGISTERS (lane l holds row pairs 2l + 16t: LDS.128 / STS.128) and between steps each
// group keeps one of its columns and trades the other with one neighbour through a
// double-buffered SMEM mailbox: one column out and one in per step (the round-robin order
// moves both) and one barrier per step.  The group reduces the three dot products with
// width-8 shuffles and rotates in registers; rotation and threshold as jacobi_svd_kernel
// (m eps relative, squared test).  gate (optional): run only if *gate == 0 (the Cholesky
// feeding sym_evd_desc succeeded).  square: write sigma^2 (eigenvalues of X X^T).
template <int RP>  // row pairs per lane: rows covered = 16 RP >= m
__global__ void __launch_bounds__(512)
    svd_reg_kernel(int m, const double* __restrict__ Xin, int trans, double* __restrict__ sigma,
                   double* __restrict__ U, const int* __restrict__ gate, int square, int debug) {
    if (gate && *gate != 0) return;
    extern __shared__ __align__(16) double sm[];
    constexpr int ld = 16 * RP;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int mp = m + (m & 1), np = mp / 2, L = np - 1;
    double* X = sm;                              // ld x mp staging (load / final), zero padded
    double* mbox = sm;                           // [2][np][ld] mailboxes, aliasing X (unused
                                                 // while the columns live in registers)
    double* park = sm + (size_t)ld * mp;         // [2][ld]: group 0's and group L's parked column
    __shared__ double nrm[128];
    __shared__ int rank_of[128];
    __shared__ int mid[2][64];
    for (int e = tid; e < ld * mp; e += nt) {
        const int i = e % ld, j = e / ld;
        X[e] = (i < m && j < m) ? (trans ? Xin[j + (size_t)i * m] : Xin[i + (size_t)j * m]) : 0.0;
    }
    __syncthreads();
    const int k = tid >> 3, gl = tid & 7;
    const bool active = k < np;
    double2 a[RP], b[RP];
    int ia = 2 * k, ib = 2 * k + 1, ipk = -1;  // column ids (id m = odd-m phantom)
#pragma unroll
    for (int t = 0; t < RP; ++t) {
        a[t] = active ? *reinterpret_cast<const double2*>(X + (size_t)ia * ld + 2 * gl + 16 * t)
                      : make_double2(0.0, 0.0);
        b[t] = active ? *reinterpret_cast<const double2*>(X + (size_t)ib * ld + 2 * gl + 16 * t)
                      : make_double2(0.0, 0.0);
    }
    __syncthreads();  // X is read: the mailboxes may overwrite it
    const double thr = mp * DBL_EPSILON;
    int step = 0;
    for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
        int rotated = 0;
        for (int ss = 0; ss < mp; ++ss, ++step) {
            const bool odd = step & 1;
            const bool work = active && !(odd && k == L);
            double al0 = 0.0, al1 = 0.0, be0 = 0.0, be1 = 0.0, ga0 = 0.0, ga1 = 0.0;
#pragma unroll
            for (int t = 0; t < RP; ++t) {
                al0 = fma(a[t].x, a[t].x, al0);
                al1 = fma(a[t].y, a[t].y, al1);
                be0 = fma(b[t].x, b[t].x, be0);
                be1 = fma(b[t].y, b[t].y, be1);
                ga0 = fma(a[t].x, b[t].x, ga0);
                ga1 = fma(a[t].y, b[t].y, ga1);
            }
            double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                al += __shfl_xor_sync(0xffffffffu, al, o, 8);
                be += __shfl_xor_sync(0xffffffffu, be, o, 8);
                ga += __shfl_xor_sync(0xffffffffu, ga, o, 8);
            }
            if (work && ga != 0.0 && ga * ga > thr * thr * (al * be)) {
                const double h = be - al, g2 = 2.0 * ga;
                double c, sn;
                jacobi_rot(h, g2, c, sn);
                rotated = 1;
#pragma unroll
                for (int t = 0; t < RP; ++t) {
                    const double2 x = a[t], y = b[t];
                    a[t] = make_double2(c * x.x - sn * y.x, c * x.y - sn * y.y);
                    b[t] = make_double2(sn * x.x + c * y.x, sn * x.y + c * y.y);
                }
            }
            if (np == 1) continue;  // a single pair never moves
            // positions swap after the step; then hand one column to a neighbour:
            //   even -> odd: keep a, send b left (group 0 parks it), receive b from the right
            //                (the last group parks a and idles);
            //   odd -> even: keep b, send a right (the last group takes its park as b),
            //                receive a from the left (group 0 takes its park as a).
            const int par = step & 1;
            double* mb = mbox + (size_t)par * np * ld;
            if (active) {
                // even: every group but 0 sends b to k - 1; odd: every group but L sends a to k + 1
                const int dst = !odd ? (k > 0 ? k - 1 : -1) : (k < L ? k + 1 : -1);
                if (dst >= 0) {
                    double* o = mb + (size_t)dst * ld + 2 * gl;
                    if (!odd) {
#pragma unroll
                        for (int t = 0; t < RP; ++t) *reinterpret_cast<double2*>(o + 16 * t) = b[t];
                    } else {
#pragma unroll
                        for (int t = 0; t < RP; ++t) *reinterpret_cast<double2*>(o + 16 * t) = a[t];
                    }
                    if (gl == 0) mid[par][dst] = !odd ? ib : ia;
                }
            }
            __syncthreads();
            if (active) {
                const double2* in = reinterpret_cast<const double2*>(mb + (size_t)k * ld + 2 * gl);
                double2* pkb = reinterpret_cast<double2*>(park + (k == 0 ? 0 : ld) + 2 * gl);
                if (!odd) {
                    if (k == 0) {  // park b (position 0 idles in odd steps)
#pragma unroll
                        for (int t = 0; t < RP; ++t) pkb[8 * t] = b[t];
                        ipk = ib;
                    }
                    if (k == L) {  // park a, idle
#pragma unroll
                        for (int t = 0; t < RP; ++t) pkb[8 * t] = a[t];
                        ipk = ia;
                    } else {       // receive b from the right
#pragma unroll
                        for (int t = 0; t < RP; ++t) b[t] = in[8 * t];
                        ib = mid[par][k];
                    }
                } else {
                    if (k == L) {  // b <- park, receive a from the left
#pragma unroll
                        for (int t = 0; t < RP; ++t) b[t] = pkb[8 * t];
                        ib = ipk;
                    }
                    if (k == 0) {  // a <- park
#pragma unroll
                        for (int t = 0; t < RP; ++t) a[t] = pkb[8 * t];
                        ia = ipk;
                    } else {
#pragma unroll
                        for (int t = 0; t < RP; ++t) a[t] = in[8 * t];
                        ia = mid[par][k];
                    }
                }
            }
        }
        const int any = __syncthreads_or(rotated);
        if (debug && tid == 0) printf("svd_reg m=%d sweep %d rotated %d\n", m, sweep, any);
        if (!any) break;
    }
    // back to X by column id (the odd-m phantom column is dropped); a parked column (odd
    // sweep end never happens: mp is even, so every sweep ends after an odd step) is none
    if (active) {
#pragma unroll
        for (int t = 0; t < RP; ++t) {
            if (ia < m) *reinterpret_cast<double2*>(X + (size_t)ia * ld + 2 * gl + 16 * t) = a[t];
            if (ib < m) *reinterpret_cast<double2*>(X + (size_t)ib * ld + 2 * gl + 16 * t) = b[t];
        }
    }
    __syncthreads();
    const int wid = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int j = wid; j < m; j += nw) {
        double s2 = 0.0;
        for (int i = lane; i < m; i += 32) s2 += X[i + j * ld] * X[i + j * ld];
        s2 = warp_sum(s2);
        if (lane == 0) nrm[j] = sqrt(s2);
    }
    __syncthreads();
    for (int i = tid; i < m; i += nt) {
        int rk = 0;
        for (int j = 0; j < m; ++j) rk += (nrm[j] > nrm[i]) || (nrm[j] == nrm[i] && j < i);
        rank_of[i] = rk;
        sigma[rk] = square ? nrm[i] * nrm[i] : nrm[i];
    }
    __syncthreads();
    for (int e = tid; e < m * m; e += nt) {
        const int i = e % m, j = e / m;
        const double sj = nrm[j];
        U[i + rank_of[j] * m] = sj > 0.0 ? X[i + j * ld] / sj : 0.0;
    }
}

// ---------------------------------------------------------------- one-sided Jacobi on a cluster
// The same Brent-Luk odd-even transposition Jacobi as svd_reg_kernel for 128 < m <= 256: one
// WARP per column pair (lane l holds rows 2l + 64t, 2l + 1 + 64t, t < 4: 16 doubles), 128
// warps on a cluster of four 1024-thread CTAs.  Between steps a group keeps one column and
// hands the other to its neighbour group through a double-buffered mailbox in the
// destination CTA's shared memory (distributed shared memory: st.shared::cluster through
// map_shared_rank), then one cluster barrier (arrive.release / wait.acquire).  The whole
// 256 x 256 problem stays on chip: no global-memory traffic per step (the single-CTA
// jacobi kernels stream a 512 KB matrix through L2 every round at these sizes).
constexpr int kCjCtas = 4, kCjWarps = 32, kCjRP = 4, kCjLd = 256;

__global__ void __cluster_dims__(kCjCtas, 1, 1) __launch_bounds__(kCjWarps * 32, 1)
    svd_cluster_kernel(int m, const double* __restrict__ Xin, int trans, double* __restrict__ sigma,
                       double* __restrict__ U, const int* __restrict__ gate, int square,
                       double* __restrict__ Xs, double* __restrict__ nrm, int* __restrict__ rank_of,
                       int debug) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    if (gate && *gate != 0) return;  // uniform across the cluster
    extern __shared__ __align__(16) double csm[];
    double* mbox = csm;                                  // [2][kCjWarps][kCjLd] (this CTA's groups)
    double* park = csm + 2 * kCjWarps * kCjLd;           // [2][kCjLd]: groups 0 / L park a column
    __shared__ int mid[2][kCjWarps];
    __shared__ int any_s;
    const int crank = (int)cluster.block_rank();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int k = crank * kCjWarps + w;                  // this warp's group (column pair)
    const int mp = m + (m & 1), np = mp / 2, L = np - 1;
    const bool active = k < np;
    double2 a[kCjRP], b[kCjRP];
    int ia = 2 * k, ib = 2 * k + 1, ipk = -1;            // column ids (id m: odd-m phantom)
    auto elem = [&](int i, int j) -> double {
        if (i >= m || j >= m) return 0.0;
        return trans ? Xin[j + (size_t)i * m] : Xin[i + (size_t)j * m];
    };
#pragma unroll
    for (int t = 0; t < kCjRP; ++t) {
        const int i = 2 * lane + 64 * t;
        a[t] = active ? make_double2(elem(i, ia), elem(i + 1, ia)) : make_double2(0.0, 0.0);
        b[t] = active ? make_double2(elem(i, ib), elem(i + 1, ib)) : make_double2(0.0, 0.0);
    }
    const double thr = mp * DBL_EPSILON;
    int step = 0;
    for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
        int rotated = 0;
        for (int ss = 0; ss < mp; ++ss, ++step) {
            const bool odd = step & 1;
            const bool work = active && !(odd && k == L);
            double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
            for (int t = 0; t < kCjRP; ++t) {
                al = fma(a[t].x, a[t].x, fma(a[t].y, a[t].y, al));
                be = fma(b[t].x, b[t].x, fma(b[t].y, b[t].y, be));
                ga = fma(a[t].x, b[t].x, fma(a[t].y, b[t].y, ga));
            }
            al = warp_sum(al);
            be = warp_sum(be);
            ga = warp_sum(ga);
            if (work && ga != 0.0 && ga * ga > thr * thr * (al * be)) {
                double c, sn;
                jacobi_rot(be - al, 2.0 * ga, c, sn);
                rotated = 1;
#pragma unroll
                for (int t = 0; t < kCjRP; ++t) {
                    const double2 x = a[t], y = b[t];
                    a[t] = make_double2(c * x.x - sn * y.x, c * x.y - sn * y.y);
                    b[t] = make_double2(sn * x.x + c * y.x, sn * x.y + c * y.y);
                }
            }
            if (np == 1) continue;
            // even -> odd: keep a, send b to k - 1 (group 0 parks b), receive b from k + 1 (group L
            // parks a); odd -> even: keep b, send a to k + 1 (group L takes its park as b),
            // receive a from k - 1 (group 0 takes its park as a) -- as svd_reg_kernel
            const int par = step & 1;
            if (active) {
                const int dst = !odd ? (k > 0 ? k - 1 : -1) : (k < L ? k + 1 : -1);
                if (dst >= 0) {
                    const int dr = dst / kCjWarps, dl = dst % kCjWarps;
                    double* o = cluster.map_shared_rank(mbox + ((size_t)par * kCjWarps + dl) * kCjLd, dr);
#pragma unroll
                    for (int t = 0; t < kCjRP; ++t)
                        *reinterpret_cast<double2*>(o + 2 * lane + 64 * t) = !odd ? b[t] : a[t];
                    if (lane == 0) *cluster.map_shared_rank(&mid[par][dl], dr) = !odd ? ib : ia;
                }
            }
            cluster.sync();
            if (active) {
                const double* in = mbox + ((size_t)par * kCjWarps + w) * kCjLd + 2 * lane;
                double* pk = park + (k == 0 ? 0 : kCjLd) + 2 * lane;
                if (!odd) {
                    if (k == 0) {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) *reinterpret_cast<double2*>(pk + 64 * t) = b[t];
                        ipk = ib;
                    }
                    if (k == L) {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) *reinterpret_cast<double2*>(pk + 64 * t) = a[t];
                        ipk = ia;
                    } else {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) b[t] = *reinterpret_cast<const double2*>(in + 64 * t);
                        ib = mid[par][w];
                    }
                } else {
                    if (k == L) {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) b[t] = *reinterpret_cast<const double2*>(pk + 64 * t);
                        ib = ipk;
                    }
                    if (k == 0) {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) a[t] = *reinterpret_cast<const double2*>(pk + 64 * t);
                        ia = ipk;
                    } else {
#pragma unroll
                        for (int t = 0; t < kCjRP; ++t) a[t] = *reinterpret_cast<const double2*>(in + 64 * t);
                        ia = mid[par][w];
                    }
                }
            }
        }
        // cluster-wide "any rotation this sweep": OR into CTA 0's flag
        if (threadIdx.x == 0) any_s = 0;
        cluster.sync();
        const int anyc = __syncthreads_or(rotated);
        if (threadIdx.x == 0 && anyc) atomicOr(cluster.map_shared_rank(&any_s, 0), 1);
        cluster.sync();
        const int any = *cluster.map_shared_rank(&any_s, 0);
        if (debug && crank == 0 && threadIdx.x == 0) printf("svd_cluster m=%d sweep %d rotated %d\n", m, sweep, any);
        cluster.sync();  // every CTA has read the flag before it is reset
        if (!any) break;
    }
    // columns back by id (the phantom column dropped), then norms, ranks and the output
    if (active) {
#pragma unroll
        for (int t = 0; t < kCjRP; ++t) {
            const int i = 2 * lane + 64 * t;
            if (ia < m) {
                if (i < m) Xs[i + (size_t)ia * m] = a[t].x;
                if (i + 1 < m) Xs[i + 1 + (size_t)ia * m] = a[t].y;
            }
            if (ib < m) {
                if (i < m) Xs[i + (size_t)ib * m] = b[t].x;
                if (i + 1 < m) Xs[i + 1 + (size_t)ib * m] = b[t].y;
            }
        }
    }
    cluster.sync();
    const int gw = k, nw = kCjCtas * kCjWarps;
    for (int j = gw; j < m; j += nw) {
        double s2 = 0.0;
        for (int i = lane; i < m; i += 32) s2 += Xs[i + (size_t)j * m] * Xs[i + (size_t)j * m];
        s2 = warp_sum(s2);
        if (lane == 0) nrm[j] = sqrt(s2);
    }
    cluster.sync();
    const int gt = crank * blockDim.x + threadIdx.x, gn = kCjCtas * blockDim.x;
    for (int i = gt; i < m; i += gn) {
        const double ni = nrm[i];
        int rk = 0;
        for (int j = 0; j < m; ++j) rk += (nrm[j] > ni) || (nrm[j] == ni && j < i);
        rank_of[i] = rk;
        sigma[rk] = square ? ni * ni : ni;
    }
    cluster.sync();
    for (int e = gt; e < m * m; e += gn) {
        const int i = e % m, j = e / m;
        const double sj = nrm[j];
        U[i + (size_t)rank_of[j] * m] = sj > 0.0 ? Xs[e] / sj : 0.0;
    }
}

// ws: m^2 + 2 m + 8 doubles of device scratch
void launch_svd_cluster(int m, const double* X, int trans, double* sigma, double* U, const int* gate, int square,
                        double* ws, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)(2 * kCjWarps * kCjLd + 2 * kCjLd);
    static bool attr = false;
    if (!attr) {
        W4_CUDA(cudaFuncSetAttribute(svd_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    double* Xs = ws;
    double* nrm = Xs + (size_t)m * m;
    int* rank_of = reinterpret_cast<int*>(nrm + m);
    static const int debug = std::getenv("WC4DVAR_DEBUG_JACOBI") ? 1 : 0;
    svd_cluster_kernel<<<kCjCtas, kCjWarps * 32, smem, st>>>(m, X, trans, sigma, U, gate, square, Xs, nrm, rank_of,
                                                            debug);
    W4_LAUNCH();
}

template <int RP>
void launch_svd_reg(int m, const double* X, int trans, double* sigma, double* U, const int* gate,
                    int square, cudaStream_t st) {
    const int mp = m + (m & 1);
    const size_t smem = sizeof(double) * (size_t)(16 * RP) * (mp + 2);
    auto kern = svd_reg_kernel<RP>;
    cudaFuncAttributes fa;
    W4_CUDA(cudaFuncGetAttributes(&fa, kern));
    if (smem + fa.sharedSizeBytes > 48 * 1024)
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = std::max(32, ((mp / 2) * 8 + 31) / 32 * 32);
    static const int debug = std::getenv("WC4DVAR_DEBUG_JACOBI") ? 1 : 0;
    kern<<<1, threads, smem, st>>>(m, X, trans, sigma, U, gate, square, debug);
    W4_LAUNCH();
}

void svd_reg(int m, const double* X, int trans, double* sigma, double* U, const int* gate, int square,
             cudaStream_t st) {
    const int rp = (m + 15) / 16;
    if (rp <= 2) return launch_svd_reg<2>(m, X, trans, sigma, U, gate, square, st);
    if (rp <= 4) return launch_svd_reg<4>(m, X, trans, sigma, U, gate, square, st);
    if (rp <= 7) return launch_svd_reg<7>(m, X, trans, sigma, U, gate, square, st);
    return launch_svd_reg<8>(m, X, trans, sigma, U, gate, square, st);
}

__global__ void small_gemm_kernel(bool ta, bool tb, int M, int N, int K, double alpha,
                                  const double* __restrict__ A, int lda,
                                  const double* __restrict__ B, int ldb, double beta,
                                  double* __restrict__ C, int ldc) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int i = e % M, j = e / M;
    double s = 0.0;
    for (int k = 0; k < K; ++k) {
        const double a = ta ? A[k + (size_t)i * lda] : A[i + (size_t)k * lda];
        const double b = tb ? B[j + (size_t)k * ldb] : B[k + (size_t)j * ldb];
        s += a * b;
    }
    C[i + (size_t)j * ldc] = alpha * s + (beta != 0.0 ? beta * C[i + (size_t)j * ldc] : 0.0);
}

__global__ void gather_cols_kernel(int64_t R, int r, const double* __restrict__ in, int64_t ldi,
                                   const int* __restrict__ perm, double* __restrict__ out,
                                   int64_t ldo) {
    const int j = blockIdx.y;
    const double* src = in + (int64_t)perm[j] * ldi;
    double* dst = out + (int64_t)j * ldo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

size_t setup_smem(const void* kern, size_t bytes, int& use_smem) {
    use_smem = bytes <= kSmemMax;
    if (!use_smem) return 0;
    // the kernels' static SMEM counts toward the 48 KB default too, so opt in whenever the
    // total exceeds it (e.g. the SVD's 18 KB of rotation tables + a 32 KB matrix at m = 64)
    cudaFuncAttributes fa;
    W4_CUDA(cudaFuncGetAttributes(&fa, kern));
    if (bytes + fa.sharedSizeBytes > 48 * 1024)
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return bytes;
}

}  // namespace

// gws: m^2 doubles of device scratch, used when the matrix does not fit shared memory
void chol_upper_ws(int m, const double* G, double* R, int* info, double* gws, cudaStream_t st) {
    int use = 0;
    const size_t bytes = sizeof(double) * m * m;
    const size_t sh = setup_smem(reinterpret_cast<const void*>(chol_kernel<true>), bytes, use);
    (use ? chol_kernel<true> : chol_kernel<false>)<<<1, kThreads, sh, st>>>(m, G, R, info, use ? nullptr : gws, use);
    W4_LAUNCH();
}

void chol_upper(int m, const double* G, double* R, int* info, DevBuf& work, cudaStream_t st) {
    int use = 0;
    setup_smem(reinterpret_cast<const void*>(chol_kernel<true>), sizeof(double) * m * m, use);
    chol_upper_ws(m, G, R, info, use ? nullptr : work.get<double>((size_t)m * m), st);
}

void chol_inv_upper(int m, const double* G, double* R, double* Rinv, int* info, DevBuf& work,
                    cudaStream_t st) {
    if (m <= 32) return launch_chol_inv<16, 1>(m, G, R, Rinv, info, st);
    if (m <= 64) return launch_chol_inv<16, 2>(m, G, R, Rinv, info, st);
    if (m <= 128) {
        static const int tpr = std::getenv("WC4DVAR_CHOLINV_TPR") ? std::atoi(std::getenv("WC4DVAR_CHOLINV_TPR")) : 8;
        if (tpr == 4) return launch_chol_inv<4, 16>(m, G, R, Rinv, info, st);  // 512 threads
        return launch_chol_inv<8, 8>(m, G, R, Rinv, info, st);
    }
    chol_upper(m, G, R, info, work, st);
    tri_inv_upper(m, R, Rinv, st);  // garbage after a breakdown; callers check info first
}

void pivoted_chol_rank(int m, const double* G, double tol_rel, int* rank, int* perm, DevBuf& work,
                       cudaStream_t st) {
    int use = 0;
    const size_t bytes = sizeof(double) * m * m;
    const size_t sh = setup_smem(reinterpret_cast<const void*>(pchol_kernel<true>), bytes, use);
    double* g = use ? nullptr : work.get<double>((size_t)m * m);
    (use ? pchol_kernel<true> : pchol_kernel<false>)<<<1, kThreads, sh, st>>>(m, G, tol_rel, rank, perm, g,
                                                                              use);
    W4_LAUNCH();
}

void tri_inv_upper(int m, const double* R, double* Rinv, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)m * m + 32 * (size_t)m);
    if (smem <= kSmemMax) {
        if (smem > 48 * 1024)
            W4_CUDA(cudaFuncSetAttribute(tri_inv_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        tri_inv_smem_kernel<<<1, 1024, smem, st>>>(m, R, Rinv);
        W4_LAUNCH();
        return;
    }
    const int warps = 8;
    tri_inv_kernel<<<(unsigned)cdiv(m, warps), warps * 32, sizeof(double) * warps * m, st>>>(m, R,
                                                                                           Rinv);
    W4_LAUNCH();
}

void sym_evd_desc(int m, const double* K, double* vals, double* W, DevBuf& work,
                  cudaStream_t st) {
    require(m <= 512, "sym_evd_desc: m too large");
    // Default: cyclic block-Jacobi (high relative accuracy; the LMP / PCG parity tests are
    // tuned to it).  WC4DVAR_EVD=tql selects the tridiagonal-QL kernel (absolute accuracy;
    // not yet faster at m ~ 100 because the QL recurrence is serial).
    static const bool jacobi = [] {
        const char* e = std::getenv("WC4DVAR_EVD");
        return !(e && std::strcmp(e, "tql") == 0);
    }();
    if (!jacobi) {
        const size_t tb = sizeof(double) * (2 * (size_t)m * m + 7 * (size_t)m) + sizeof(int) * m;
        int use_t = 0;
        const size_t sh_t = setup_smem(reinterpret_cast<const void*>(sym_evd_tql_kernel<true>), tb, use_t);
        double* gw = use_t ? nullptr : work.get<double>(tb / sizeof(double) + 1);
        (use_t ? sym_evd_tql_kernel<true> : sym_evd_tql_kernel<false>)<<<1, kTqlThreads, sh_t, st>>>(
            m, K, vals, W, gw, use_t, nullptr);
        W4_LAUNCH();
        return;
    }
    // Default for m <= 128 and SPD K (every sketch: Z^T A Z with A >= I, R R^T): K = R^T R by
    // the fused Cholesky, then the register one-sided Jacobi on R^T gives the eigenvectors as
    // its left singular vectors and the eigenvalues as sigma^2, with no eigenvector
    // accumulation and one barrier per round.  If the Cholesky breaks down (indefinite K) the
    // two-sided block-Jacobi kernel runs instead; the device info word gates both kernels, so
    // there is no host round trip.  WC4DVAR_EVD=jacobi forces the two-sided kernel.
    static const bool two_sided = [] {
        const char* e = std::getenv("WC4DVAR_EVD");
        return e && std::strcmp(e, "jacobi") == 0;
    }();
    const int mp = m + (m & 1);
    const size_t bytes2 = sizeof(double) * 2 * mp * mp;
    int use = 0;
    const size_t sh = setup_smem(reinterpret_cast<const void*>(jacobi_evd_blk_kernel<true>), bytes2, use);
    // cluster-Jacobi scratch (128 < m <= 256): m^2 + 2m + 8, then m^2 for the Cholesky
    const size_t cl_ws = 2 * (size_t)m * m + 2 * (size_t)m + 8;
    double* scratch = work.get<double>(2 * (size_t)m * m + 2 * (size_t)mp * mp + 8 + cl_ws);
    const int* gate = nullptr;
    if (m > 128 && m <= 256 && !two_sided) {
        // K = R^T R (Cholesky), eigenvectors = left singular vectors of R^T by the cluster
        // one-sided Jacobi (eigenvalues sigma^2); the two-sided kernel below runs only if the
        // Cholesky broke down (indefinite K)
        double* R = scratch;
        int* info = reinterpret_cast<int*>(scratch + 2 * (size_t)m * m + 2 * (size_t)mp * mp);
        double* cws = scratch + 2 * (size_t)m * m + 2 * (size_t)mp * mp + 8;
        chol_upper_ws(m, K, R, info, cws + (size_t)m * m + 2 * (size_t)m + 8, st);
        launch_svd_cluster(m, R, /*trans=*/1, vals, W, info, /*square=*/1, cws, st);
        gate = info;
    }
    if (m <= 128 && !two_sided) {
        double* R = scratch;
        double* Ri = R + (size_t)m * m;
        int* info = reinterpret_cast<int*>(scratch + 2 * (size_t)m * m + 2 * (size_t)mp * mp);
        chol_inv_upper(m, K, R, Ri, info, work, st);  // m <= 128: no work-buffer use
        svd_reg(m, R, /*trans=*/1, vals, W, info, /*square=*/1, st);
        gate = info;
    }
    double* g = use ? nullptr : scratch + 2 * (size_t)m * m;
    static const int debug = std::getenv("WC4DVAR_DEBUG_JACOBI") ? 1 : 0;
    (use ? jacobi_evd_blk_kernel<true> : jacobi_evd_blk_kernel<false>)<<<1, kEvdThreads, sh, st>>>(
        m, K, vals, W, g, use, debug, gate);
    W4_LAUNCH();
}

void svd_left_desc(int m, const double* X, double* sigma, double* U, DevBuf& work,
                   cudaStream_t st) {
    require(m <= 512, "svd_left_desc: m too large");
    static const bool two_phase = [] {
        const char* e = std::getenv("WC4DVAR_SVD");
        return e && std::strcmp(e, "jacobi") == 0;
    }();
    if (m <= 128 && !two_phase) return svd_reg(m, X, 0, sigma, U, nullptr, 0, st);
    if (m <= 256 && !two_phase)
        return launch_svd_cluster(m, X, 0, sigma, U, nullptr, 0, work.get<double>((size_t)m * m + 2 * (size_t)m + 8),
                                  st);
    int use = 0;
    const size_t bytes = sizeof(double) * m * m;
    const size_t sh = setup_smem(reinterpret_cast<const void*>(jacobi_svd_kernel<true>), bytes, use);
    double* g = use ? nullptr : work.get<double>((size_t)m * m);
    (use ? jacobi_svd_kernel<true> : jacobi_svd_kernel<false>)<<<1, kThreads, sh, st>>>(m, X, sigma, U, g, use);
    W4_LAUNCH();
}

void small_gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                const double* B, int ldb, double beta, double* C, int ldc, cudaStream_t st) {
    if (M * N == 0) return;
    small_gemm_kernel<<<(unsigned)cdiv((int64_t)M * N, 256), 256, 0, st>>>(
        ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    W4_LAUNCH();
}

void gather_cols(int64_t R, int r, const double* in, int64_t ldi, const int* perm, double* out,
                 int64_t ldo, cudaStream_t st) {
    if (r == 0 || R == 0) return;
    dim3 grid((unsigned)std::min<int64_t>(cdiv(R, 256), 1024), (unsigned)r);
    gather_cols_kernel<<<grid, 256, 0, st>>>(R, r, in, ldi, perm, out, ldo);
    W4_LAUNCH();
}

}  // namespace w4
