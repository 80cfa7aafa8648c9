// Resident window sweeps: one CTA owns one sketch column for the whole window; the
// n-point state lives in shared memory (ping-pong), so the only HBM traffic is the
// compulsory read of the forcing blocks and the write of the swept blocks.
//
// Reference semantics (operators.cpp:79-101):
//   forward  x_0 = X_0,  x_{i+1} = M_i x_i + X_{i+1},   M_i = (sub-step)^s
//   adjoint  s_N = v_N + H_N^T y,  s_i = v_i + H_i^T y + M_i^T s_{i+1}
// with the observation selection (models.cpp:184-201) fused into the sweeps.
#include "sweep.cuh"

#include <cooperative_groups.h>

#include <cstdlib>

namespace w4 {
namespace {

// One TL sub-step of a single-phase stencil model (models.cpp:27-45 + EXTENSION).
template <int KIND>
__device__ __forceinline__ double tl_point(const double* __restrict__ u, int64_t j, int64_t n,
                                           double c, double d) {
    if (KIND == WC4DVAR_MODEL_IDENTITY) return u[j];
    const int64_t jm = (j == 0) ? n - 1 : j - 1;
    if (KIND == WC4DVAR_MODEL_ADVECTION) return u[j] - c * (u[j] - u[jm]);
    const int64_t jp = (j + 1 == n) ? 0 : j + 1;
    return u[j] - c * (u[j] - u[jm]) + d * (u[jp] - 2.0 * u[j] + u[jm]);
}

template <int KIND>
__device__ __forceinline__ double adj_point(const double* __restrict__ l, int64_t j, int64_t n,
                                            double c, double d) {
    if (KIND == WC4DVAR_MODEL_IDENTITY) return l[j];
    const int64_t jp = (j + 1 == n) ? 0 : j + 1;
    if (KIND == WC4DVAR_MODEL_ADVECTION) return (1.0 - c) * l[j] + c * l[jp];
    const int64_t jm = (j == 0) ? n - 1 : j - 1;
    return l[j] - c * (l[j] - l[jp]) + d * (l[jm] - 2.0 * l[j] + l[jp]);
}

template <int KIND>
__global__ void __launch_bounds__(1024)
    sweep_resident_kernel(const ModelDev md, const NetDev net, const SweepArgs a,
                          unsigned* __restrict__ status) {
    extern __shared__ double sm[];
    const int64_t n = md.n;
    const int N = md.N, s = md.s;
    const double c = md.c, d = md.d;
    double* buf0 = sm;
    double* buf1 = sm + n;
    const int64_t col = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int np = net.n_points;
    bool bad_f = false, bad_a = false;

    if (a.do_fwd) {
        const double* X = a.X + col * a.ldx;
        double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
        // x_0 = X_0
        {
            const int sl = net.slot[0];
            for (int64_t j = tid; j < n; j += nt) {
                const double v = X[j];
                buf0[j] = v;
                bad_f |= !isfinite(v);
                if (tr) tr[j] = v;
                if (a.fwd_obs && sl >= 0) {
                    const int b = net.pmap[j];
                    if (b >= 0) Yc[(int64_t)sl * np + b] = a.scale_fwd * v;
                }
            }
        }
        __syncthreads();
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = 0; i < N; ++i) {
            const double* Xn = X + (int64_t)(i + 1) * n;
            const int sl = net.slot[i + 1];
            for (int k = 0; k < s; ++k) {
                if (k + 1 < s) {
                    for (int64_t j = tid; j < n; j += nt) nxt[j] = tl_point<KIND>(cur, j, n, c, d);
                } else {
                    double* trn = tr ? tr + (int64_t)(i + 1) * n : nullptr;
                    for (int64_t j = tid; j < n; j += nt) {
                        const double v = tl_point<KIND>(cur, j, n, c, d) + Xn[j];
                        nxt[j] = v;
                        bad_f |= !isfinite(v);
                        if (trn) trn[j] = v;
                        if (a.fwd_obs && sl >= 0) {
                            const int b = net.pmap[j];
                            if (b >= 0) Yc[(int64_t)sl * np + b] = a.scale_fwd * v;
                        }
                    }
                }
                __syncthreads();
                double* t = cur;
                cur = nxt;
                nxt = t;
            }
            if (s == 0) {  // no sub-steps: M_i = I
                for (int64_t j = tid; j < n; j += nt) cur[j] += Xn[j];
                __syncthreads();
            }
        }
    }

    if (a.do_adj) {
        const double* V = a.V ? a.V + col * a.ldv : nullptr;
        const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* S = a.S + col * a.lds;
        // s_N = v_N + H_N^T y
        {
            const int sl = net.slot[N];
            const int64_t off = (int64_t)N * n;
            for (int64_t j = tid; j < n; j += nt) {
                double v = V ? V[off + j] : 0.0;
                if (a.adj_obs && sl >= 0) {
                    const int b = net.pmap[j];
                    if (b >= 0) v = V ? v + Yc[(int64_t)sl * np + b] : Yc[(int64_t)sl * np + b];
                }
                buf0[j] = v;
                S[off + j] = v;
                bad_a |= !isfinite(v);
            }
        }
        __syncthreads();
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = N - 1; i >= 0; --i) {
            const int sl = net.slot[i];
            const int64_t off = (int64_t)i * n;
            for (int k = 0; k < s; ++k) {
                if (k + 1 < s) {
                    for (int64_t j = tid; j < n; j += nt) nxt[j] = adj_point<KIND>(cur, j, n, c, d);
                } else {
                    for (int64_t j = tid; j < n; j += nt) {
                        // s_i = v_i + H_i^T y + M_i^T s_{i+1}  (operators.cpp:99: v + back)
                        double add = V ? V[off + j] : 0.0;
                        if (a.adj_obs && sl >= 0) {
                            const int b = net.pmap[j];
                            if (b >= 0) add = V ? add + Yc[(int64_t)sl * np + b]
                                                : Yc[(int64_t)sl * np + b];
                        }
                        const double v = add + adj_point<KIND>(cur, j, n, c, d);
                        nxt[j] = v;
                        S[off + j] = v;
                        bad_a |= !isfinite(v);
                    }
                }
                __syncthreads();
                double* t = cur;
                cur = nxt;
                nxt = t;
            }
            if (s == 0) {
                for (int64_t j = tid; j < n; j += nt) {
                    double add = V ? V[off + j] : 0.0;
                    if (a.adj_obs && sl >= 0) {
                        const int b = net.pmap[j];
                        if (b >= 0) add += Yc[(int64_t)sl * np + b];
                    }
                    cur[j] += add;
                    S[off + j] = cur[j];
                }
                __syncthreads();
            }
        }
    }

    const int any_f = __syncthreads_or(bad_f);
    const int any_a = __syncthreads_or(bad_a);
    if (tid == 0 && (any_f || any_a))
        atomicOr(status, (any_f ? ST_FWD_NONFINITE : 0u) | (any_a ? ST_ADJ_NONFINITE : 0u));
}

// ---------------------------------------------------------------------------
// Register-blocked variant (temporal blocking): each thread owns P consecutive grid
// points and gathers a halo of S points per side from shared memory once per window
// interval, then applies all S sub-steps at once as one fused (2S+1)-tap stencil in
// registers.  One __syncthreads per interval instead of one per sub-step; redundant halo
// loads are 2S/P.  Radius-1 stencils (identity, upwind advection, advection-diffusion).
// ---------------------------------------------------------------------------
// SMEM state rows use a point-major ("transposed") layout: grid point j lives at
// (j % P) * ntp + j / P, ntp = ceil(n / P).  Thread t owns points [tP, tP + P), so when a warp
// reads its u-th halo/centre value the 32 addresses are consecutive -- conflict-free -- where
// the natural layout (stride P doubles between threads) is a 16-way bank conflict.
template <int P>
__device__ __forceinline__ int pm_slot(int j, int ntp) { return (j % P) * ntp + j / P; }

// One interval as the fused (2S+1)-tap stencil (see StencilTaps, built by stencil_power from
// the S-fold product of the 3-point step); results land in v[S .. S+P).
template <int S, int P>
__device__ __forceinline__ void conv_interval(const double* __restrict__ cur, int b, int n, int ntp,
                                              const StencilTaps& tp, double (&v)[P + 2 * S]) {
    constexpr int L = P + 2 * S;
    int j = (b - S) % n;
    if (j < 0) j += n;
#pragma unroll
    for (int u = 0; u < L; ++u) {
        v[u] = cur[pm_slot<P>(j, ntp)];
        j = (j + 1 == n) ? 0 : j + 1;
    }
    double o[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        double acc = tp.t[0] * v[p];
#pragma unroll
        for (int k = 1; k <= 2 * S; ++k) acc = fma(tp.t[k], v[p + k], acc);
        o[p] = acc;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) v[S + p] = o[p];
}

template <int KIND, int S, int P>
__global__ void __launch_bounds__(512)
    sweep_blocked_kernel(const ModelDev md, const NetDev net, const SweepArgs a, const StencilTaps tf,
                         const StencilTaps tb, unsigned* __restrict__ status) {
    extern __shared__ double sm[];
    const int n = (int)md.n;
    const int N = md.N;
    const int ntp = (n + P - 1) / P;  // point-major rows (see pm_slot)
    double* buf0 = sm;
    double* buf1 = sm + P * ntp;
    int* pmap = reinterpret_cast<int*>(sm + 2 * P * ntp);  // observation tables staged in SMEM
    int* slot = pmap + n;
    const int64_t col = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int b = tid * P;
    const bool owner = b < n;
    const int np = net.n_points;
    bool bad_f = false, bad_a = false;
    double v[P + 2 * S];
    for (int j = tid; j < n; j += nt) pmap[j] = net.pmap[j];
    for (int t = tid; t <= N; t += nt) slot[t] = net.slot[t];
    __syncthreads();

    if (a.do_fwd) {
        const double* X = a.X + col * a.ldx;
        double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
        {
            const int sl = slot[0];
            for (int j = tid; j < n; j += nt) {
                const double x = X[j];
                buf0[pm_slot<P>(j, ntp)] = x;
                bad_f |= !isfinite(x);
                if (tr) tr[j] = x;
                if (a.fwd_obs && sl >= 0) {
                    const int bb = pmap[j];
                    if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                }
            }
        }
        // forcing of the next interval, prefetched one interval ahead into registers
        double xin[P];
#pragma unroll
        for (int p = 0; p < P; ++p) xin[p] = (owner && N > 0 && b + p < n) ? X[(int64_t)n + b + p] : 0.0;
        __syncthreads();
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = 0; i < N; ++i) {
            const int sl = slot[i + 1];
            double* trn = tr ? tr + (int64_t)(i + 1) * n : nullptr;
            double xnx[P];
            const double* Xnn = X + (int64_t)(i + 2) * n;
#pragma unroll
            for (int p = 0; p < P; ++p) xnx[p] = (owner && i + 1 < N && b + p < n) ? Xnn[b + p] : 0.0;
            if (owner) {
                conv_interval<S, P>(cur, b, n, ntp, tf, v);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int j = b + p;
                    if (j < n) {
                        const double x = v[S + p] + xin[p];
                        nxt[p * ntp + tid] = x;
                        bad_f |= !isfinite(x);
                        if (trn) trn[j] = x;
                        if (a.fwd_obs && sl >= 0) {
                            const int bb = pmap[j];
                            if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                        }
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) xin[p] = xnx[p];
            __syncthreads();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }

    if (a.do_adj) {
        const double* V = a.V ? a.V + col * a.ldv : nullptr;
        const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* Sv = a.S + col * a.lds;
        // s_i = v_i + H_i^T y + M_i^T s_{i+1}: the addend of interval i, prefetched
        auto addend = [&](int i, int j) -> double {
            double x = V ? V[(int64_t)i * n + j] : 0.0;
            if (a.adj_obs) {
                const int sl = slot[i];
                if (sl >= 0) {
                    const int bb = pmap[j];
                    if (bb >= 0) x = V ? x + Yc[(int64_t)sl * np + bb] : Yc[(int64_t)sl * np + bb];
                }
            }
            return x;
        };
        {
            const int64_t off = (int64_t)N * n;
            for (int j = tid; j < n; j += nt) {
                const double x = addend(N, j);
                buf0[pm_slot<P>(j, ntp)] = x;
                Sv[off + j] = x;
                bad_a |= !isfinite(x);
            }
        }
        double ain[P];
#pragma unroll
        for (int p = 0; p < P; ++p) ain[p] = (owner && N > 0 && b + p < n) ? addend(N - 1, b + p) : 0.0;
        __syncthreads();
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = N - 1; i >= 0; --i) {
            const int64_t off = (int64_t)i * n;
            double anx[P];
#pragma unroll
            for (int p = 0; p < P; ++p) anx[p] = (owner && i > 0 && b + p < n) ? addend(i - 1, b + p) : 0.0;
            if (owner) {
                conv_interval<S, P>(cur, b, n, ntp, tb, v);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int j = b + p;
                    if (j < n) {
                        const double x = ain[p] + v[S + p];  // operators.cpp:99 (v_i + back)
                        nxt[p * ntp + tid] = x;
                        Sv[off + j] = x;
                        bad_a |= !isfinite(x);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) ain[p] = anx[p];
            __syncthreads();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }

    const int any_f = __syncthreads_or(bad_f);
    const int any_a = __syncthreads_or(bad_a);
    if (tid == 0 && (any_f || any_a))
        atomicOr(status, (any_f ? ST_FWD_NONFINITE : 0u) | (any_a ? ST_ADJ_NONFINITE : 0u));
}

// ---------------------------------------------------------------------------
// Cluster-split resident sweep for few columns (PCG's single-vector applies): the CL CTAs
// of a thread-block cluster each own n/CL points of the column; per interval every CTA
// pulls the S-point halos of its two neighbours from their SMEM over DSMEM after one
// cluster barrier, then advances its segment with the fused stencil.  One column runs on
// CL SMs instead of one (the resident sweep is latency-bound at one CTA per column).
// Region layout per CTA: e in [0, Lseg + 2S), e = S + local point, point-major slots.
// ---------------------------------------------------------------------------
template <int KIND, int S, int P, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(512)
    sweep_cluster_kernel(const ModelDev md, const NetDev net, const SweepArgs a, const StencilTaps tf,
                         const StencilTaps tb, unsigned* __restrict__ status) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double sm[];
    const int n = (int)md.n;
    const int N = md.N;
    const int Lseg = n / CL;
    const int R = Lseg + 2 * S;
    const int ntp = (R + P - 1) / P;
    double* buf0 = sm;
    double* buf1 = sm + P * ntp;
    int* pm = reinterpret_cast<int*>(sm + 2 * P * ntp);  // pmap of the own segment
    int* slot = pm + Lseg;
    const int rank = (int)cluster.block_rank();
    const int64_t col = blockIdx.x / CL;
    const int seg0 = rank * Lseg;
    const int left = (rank + CL - 1) % CL, right = (rank + 1) % CL;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int b = tid * P;  // own local points [b, b + P), region e = S + b + p
    const bool owner = b < Lseg;
    const int np = net.n_points;
    bool bad_f = false, bad_a = false;
    double v[P + 2 * S];
    auto sl_of = [&](int e) { return (e % P) * ntp + e / P; };
    for (int j = tid; j < Lseg; j += nt) pm[j] = net.pmap[seg0 + j];
    for (int t = tid; t <= N; t += nt) slot[t] = net.slot[t];
    __syncthreads();  // the staged tables are read by other threads below
    // halos of buffer `cur`: e in [0, S) <- left's own tail, e in [Lseg + S, R) <- right's head
    auto pull_halos = [&](double* cur) {
        if (tid < 2 * S) {
            const bool lft = tid < S;
            const int e_dst = lft ? tid : Lseg + S + (tid - S);
            const int e_src = lft ? Lseg + tid : S + (tid - S);
            const double* nb = cluster.map_shared_rank(cur, lft ? left : right);
            cur[sl_of(e_dst)] = nb[sl_of(e_src)];
        }
    };
    auto advance = [&](const double* cur, const StencilTaps& tp) {
#pragma unroll
        for (int u = 0; u < P + 2 * S; ++u) v[u] = cur[sl_of(b + u)];
        double o[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            double acc = tp.t[0] * v[p];
#pragma unroll
            for (int k = 1; k <= 2 * S; ++k) acc = fma(tp.t[k], v[p + k], acc);
            o[p] = acc;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) v[S + p] = o[p];
    };

    if (a.do_fwd) {
        const double* X = a.X + col * a.ldx;
        double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
        {
            const int sl = slot[0];
            for (int j = tid; j < Lseg; j += nt) {
                const int g = seg0 + j;
                const double x = X[g];
                buf0[sl_of(S + j)] = x;
                bad_f |= !isfinite(x);
                if (tr) tr[g] = x;
                if (a.fwd_obs && sl >= 0) {
                    const int bb = pm[j];
                    if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                }
            }
        }
        double xin[P];
#pragma unroll
        for (int p = 0; p < P; ++p) xin[p] = (owner && N > 0) ? X[(int64_t)n + seg0 + b + p] : 0.0;
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = 0; i < N; ++i) {
            cluster.sync();  // every segment of x_i is in SMEM (and the old halos are read)
            pull_halos(cur);
            __syncthreads();
            const int sl = slot[i + 1];
            double* trn = tr ? tr + (int64_t)(i + 1) * n : nullptr;
            double xnx[P];
            const double* Xnn = X + (int64_t)(i + 2) * n + seg0;
#pragma unroll
            for (int p = 0; p < P; ++p) xnx[p] = (owner && i + 1 < N) ? Xnn[b + p] : 0.0;
            if (owner) {
                advance(cur, tf);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int j = b + p;
                    const double x = v[S + p] + xin[p];  // operators.cpp:88
                    nxt[sl_of(S + j)] = x;
                    bad_f |= !isfinite(x);
                    if (trn) trn[seg0 + j] = x;
                    if (a.fwd_obs && sl >= 0) {
                        const int bb = pm[j];
                        if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) xin[p] = xnx[p];
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }

    if (a.do_adj) {
        cluster.sync();  // the forward's last halo reads of buf0 / buf1 are done
        const double* V = a.V ? a.V + col * a.ldv : nullptr;
        const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
        double* Sv = a.S + col * a.lds;
        auto addend = [&](int i, int j) -> double {  // j: local point
            double x = V ? V[(int64_t)i * n + seg0 + j] : 0.0;
            if (a.adj_obs) {
                const int sl = slot[i];
                if (sl >= 0) {
                    const int bb = pm[j];
                    if (bb >= 0) x = V ? x + Yc[(int64_t)sl * np + bb] : Yc[(int64_t)sl * np + bb];
                }
            }
            return x;
        };
        {
            const int64_t off = (int64_t)N * n + seg0;
            for (int j = tid; j < Lseg; j += nt) {
                const double x = addend(N, j);
                buf0[sl_of(S + j)] = x;
                Sv[off + j] = x;
                bad_a |= !isfinite(x);
            }
        }
        double ain[P];
#pragma unroll
        for (int p = 0; p < P; ++p) ain[p] = (owner && N > 0) ? addend(N - 1, b + p) : 0.0;
        double* cur = buf0;
        double* nxt = buf1;
        for (int i = N - 1; i >= 0; --i) {
            cluster.sync();
            pull_halos(cur);
            __syncthreads();
            const int64_t off = (int64_t)i * n + seg0;
            double anx[P];
#pragma unroll
            for (int p = 0; p < P; ++p) anx[p] = (owner && i > 0) ? addend(i - 1, b + p) : 0.0;
            if (owner) {
                advance(cur, tb);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int j = b + p;
                    const double x = ain[p] + v[S + p];  // operators.cpp:99
                    nxt[sl_of(S + j)] = x;
                    Sv[off + j] = x;
                    bad_a |= !isfinite(x);
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) ain[p] = anx[p];
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    cluster.sync();  // no CTA exits while a neighbour may still read its SMEM
    const int any_f = __syncthreads_or(bad_f);
    const int any_a = __syncthreads_or(bad_a);
    if (tid == 0 && (any_f || any_a))
        atomicOr(status, (any_f ? ST_FWD_NONFINITE : 0u) | (any_a ? ST_ADJ_NONFINITE : 0u));
}

template <int KIND, int S, int P, int CL>
bool launch_cluster_sp(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                       cudaStream_t stream) {
    if (md.n % (CL * P) != 0) return false;
    const int Lseg = (int)(md.n / CL);
    if (Lseg < 2 * S || Lseg / P > 512) return false;
    const int R = Lseg + 2 * S, ntp = (R + P - 1) / P;
    const size_t smem = sizeof(double) * 2 * P * ntp + sizeof(int) * (Lseg + md.N + 1);
    if (smem > 48 * 1024) return false;
    const int nt = ((Lseg / P + 31) / 32) * 32;
    const StencilTaps tf = stencil_power(KIND, md.c, md.d, S, false);
    const StencilTaps tb = stencil_power(KIND, md.c, md.d, S, true);
    sweep_cluster_kernel<KIND, S, P, CL><<<(unsigned)(a.m * CL), nt, smem, stream>>>(md, net, a, tf, tb, status);
    W4_LAUNCH();
    return true;
}

template <int KIND, int S, int P>
bool launch_blocked_sp(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                       cudaStream_t stream) {
    const int64_t owners = (md.n + P - 1) / P;
    if (owners > 512) return false;
    int nt = (int)((owners + 31) / 32) * 32;
    const size_t smem = sizeof(double) * 2 * P * owners + sizeof(int) * (md.n + md.N + 1);
    if (smem > 200 * 1024) return false;
    auto kern = sweep_blocked_kernel<KIND, S, P>;
    if (smem > 48 * 1024)
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const StencilTaps tf = stencil_power(KIND, md.c, md.d, S, false);
    const StencilTaps tb = stencil_power(KIND, md.c, md.d, S, true);
    kern<<<(unsigned)a.m, nt, smem, stream>>>(md, net, a, tf, tb, status);
    W4_LAUNCH();
    return true;
}

// Points per thread: P = 4 when a column fits 512 threads that way (twice the warps per
// column to hide the per-interval latency chain; the sweep is latency-bound at one CTA per
// column), else P = 8.  WC4DVAR_SWEEP_P=8 forces the wider blocking.
template <int KIND, int S>
bool launch_blocked_s(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                      cudaStream_t stream) {
    static const int pref = [] {
        const char* e = std::getenv("WC4DVAR_SWEEP_P");
        return e ? std::atoi(e) : 4;
    }();
    // few columns (PCG): split each column over a 4-CTA cluster (WC4DVAR_SWEEP_CLUSTER=0 off)
    static const int clus = [] {
        const char* e = std::getenv("WC4DVAR_SWEEP_CLUSTER");
        return e ? std::atoi(e) : 4;
    }();
    if (clus == 4 && a.m * 4 <= kSMs && launch_cluster_sp<KIND, S, 4, 4>(md, net, a, status, stream)) return true;
    if (pref == 4 && launch_blocked_sp<KIND, S, 4>(md, net, a, status, stream)) return true;
    return launch_blocked_sp<KIND, S, 8>(md, net, a, status, stream);
}

template <int KIND>
bool launch_blocked(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                    cudaStream_t stream) {
    switch (md.s) {
        case 1: return launch_blocked_s<KIND, 1>(md, net, a, status, stream);
        case 5: return launch_blocked_s<KIND, 5>(md, net, a, status, stream);
        case 10: return launch_blocked_s<KIND, 10>(md, net, a, status, stream);
        default: return false;
    }
}

template <int KIND>
void launch_resident(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                     cudaStream_t stream) {
    if (launch_blocked<KIND>(md, net, a, status, stream)) return;
    const size_t smem = sizeof(double) * 2 * md.n;
    auto kern = sweep_resident_kernel<KIND>;
    if (smem > 48 * 1024)
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nt = (int)((md.n + 3) / 4);
    nt = ((nt + 31) / 32) * 32;
    if (nt < 128) nt = 128;
    if (nt > 1024) nt = 1024;
    kern<<<(unsigned)a.m, nt, smem, stream>>>(md, net, a, status);
    W4_LAUNCH();
}

}  // namespace

int64_t sweep_resident_max_n() { return (227 * 1024) / (2 * sizeof(double)); }

StencilTaps stencil_power(int kind, double c, double d, int s, bool adjoint) {
    require(s >= 1 && s <= kMaxFusedS, "stencil_power: sub-steps out of range");
    // one step: coefficients of x_{j-1}, x_j, x_{j+1} (models.cpp:27-45; adjoint mirrored)
    long double lft = 0, mid = 1, rgt = 0;
    if (kind == WC4DVAR_MODEL_ADVECTION) {
        lft = c;
        mid = 1.0L - c;
    } else if (kind == WC4DVAR_MODEL_ADVDIFF) {
        lft = (long double)c + d;
        mid = 1.0L - c - 2.0L * d;
        rgt = d;
    }
    if (adjoint) std::swap(lft, rgt);
    long double poly[2 * kMaxFusedS + 1] = {1.0L};
    int len = 1;
    for (int k = 0; k < s; ++k) {  // poly <- poly * (lft z^-1 + mid + rgt z)
        long double nx[2 * kMaxFusedS + 1] = {};
        for (int i = 0; i < len; ++i) {
            nx[i] += poly[i] * lft;
            nx[i + 1] += poly[i] * mid;
            nx[i + 2] += poly[i] * rgt;
        }
        len += 2;
        for (int i = 0; i < len; ++i) poly[i] = nx[i];
    }
    StencilTaps t{};
    for (int i = 0; i < len; ++i) t.t[i] = (double)poly[i];
    return t;
}

void sweep(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
           cudaStream_t stream, DevBuf* ws) {
    if (a.m == 0) return;
    // WC4DVAR_SWEEP_TILE=T forces the tiled path with tile size T (test hook: lets the
    // halo / multi-launch logic run on problem sizes the oracle can check quickly).
    static const int forced_tile = [] {
        const char* e = std::getenv("WC4DVAR_SWEEP_TILE");
        return e ? std::atoi(e) : 0;
    }();
    if (md.kind == WC4DVAR_MODEL_LORENZ96 || md.n > sweep_resident_max_n() || forced_tile > 0) {
        static thread_local DevBuf local;
        sweep_tiled(md, net, a, status, stream, ws ? *ws : local, forced_tile);
        return;
    }
    switch (md.kind) {
        case WC4DVAR_MODEL_IDENTITY:
            launch_resident<WC4DVAR_MODEL_IDENTITY>(md, net, a, status, stream);
            break;
        case WC4DVAR_MODEL_ADVECTION:
            launch_resident<WC4DVAR_MODEL_ADVECTION>(md, net, a, status, stream);
            break;
        case WC4DVAR_MODEL_ADVDIFF:
            launch_resident<WC4DVAR_MODEL_ADVDIFF>(md, net, a, status, stream);
            break;
        default:
            throw InvalidArgument("sweep: model kind not supported by the resident sweep");
    }
}

}  // namespace w4
