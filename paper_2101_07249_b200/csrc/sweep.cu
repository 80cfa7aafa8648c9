// Resident window sweeps: one CTA owns one sketch column for the whole window; the
// n-point state lives in shared memory (ping-pong), so the only HBM traffic is the
// compulsory read of the forcing blocks and the write of the swept blocks.
//
// Reference semantics (operators.cpp:79-101):
//   forward  x_0 = X_0,  x_{i+1} = M_i x_i + X_{i+1},   M_i = (sub-step)^s
//   adjoint  s_N = v_N + H_N^T y,  s_i = v_i + H_i^T y + M_i^T s_{i+1}
// with the observation selection (models.cpp:184-201) fused into the sweeps.
#include "sweep.cuh"

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

template <int KIND>
void launch_resident(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                     cudaStream_t stream) {
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

void sweep(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
           cudaStream_t stream) {
    if (a.m == 0) return;
    require(md.n <= sweep_resident_max_n(),
            "sweep: n exceeds the resident-sweep limit (tiled sweep not built yet)");
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
