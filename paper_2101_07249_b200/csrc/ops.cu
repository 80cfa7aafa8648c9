// Operator, LMP and cost handles plus their C-ABI entry points.
#include "ops.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "fft4.cuh"
#include "lmp_pcg.cuh"
#include "spectral.cuh"

namespace w4 {

std::atomic<long long> g_launch_count{0};

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

}  // namespace w4

extern "C" int64_t wc4dvar_gpu_launch_count(void) { return w4::g_launch_count.load(); }

using namespace w4;

// ----------------------------------------------------------------------------- base op
wc4dvar_op::~wc4dvar_op() {
    DeviceGuard g(device);
    for (cudaEvent_t e : pev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : pipe_ev)
        if (e) cudaEventDestroy(e);
    if (pipe_in) cudaStreamDestroy(pipe_in);
    if (pipe_out) cudaStreamDestroy(pipe_out);
    if (h_int) cudaFreeHost(h_int);
    if (d_status) cudaFree(d_status);
    if (h_status) cudaFreeHost(h_status);
    if (stream) cudaStreamDestroy(stream);
}

void wc4dvar_op::init_common(int dev, int64_t n) {
    device = dev;
    dim = n;
    W4_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    W4_CUDA(cudaMalloc(&d_status, sizeof(unsigned)));
    W4_CUDA(cudaMallocHost(&h_status, sizeof(unsigned)));
    W4_CUDA(cudaMallocHost(&h_int, 16 * sizeof(int)));
    W4_CUDA(cudaMemset(d_status, 0, sizeof(unsigned)));
}

void wc4dvar_op::ensure_pipeline() {
    if (pipe_in) return;
    W4_CUDA(cudaStreamCreateWithFlags(&pipe_in, cudaStreamNonBlocking));
    W4_CUDA(cudaStreamCreateWithFlags(&pipe_out, cudaStreamNonBlocking));
    for (cudaEvent_t& e : pipe_ev) W4_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void wc4dvar_op::collect_profile() {
    if (!prof || !prof_pending) return;
    prof_pending = false;
    for (int i = 0; i < 3; ++i) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, pev[i], pev[i + 1]) == cudaSuccess) prof_ms[i] += ms;
    }
    ++prof_calls;
}

void wc4dvar_op::reset_status(cudaStream_t st) {
    W4_CUDA(cudaMemsetAsync(d_status, 0, sizeof(unsigned), st));
}

void wc4dvar_op::check_status(cudaStream_t st) {
    W4_CUDA(cudaMemcpyAsync(h_status, d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    const unsigned s = *h_status;
    collect_profile();
    // operators.cpp:133-143, in the reference's order of checks
    if (s & ST_FWD_NONFINITE)
        throw NumericalError("hessian apply: non-finite value after forward sweep");
    if (s & ST_ADJ_NONFINITE)
        throw NumericalError("hessian apply: non-finite value after adjoint sweep");
    if (s & ST_OUT_NONFINITE) throw NumericalError("hessian apply: non-finite result");
}

namespace w4 {

// ----------------------------------------------------------------------------- Hessian
HessianOp::~HessianOp() {
    DeviceGuard g(device);
    for (double* p : {b_half, b_half_inv, q_half, q_half_inv, d_stages})
        if (p) cudaFree(p);
    if (d_slot) cudaFree(d_slot);
    if (d_pmap) cudaFree(d_pmap);
    if (d_times) cudaFree(d_times);
    if (d_points) cudaFree(d_points);
    if (d_mhat) cudaFree(d_mhat);
    delete circ;
}

// The Fourier-space apply needs: a fused transform with the in-place pass B, a TL step that
// is a periodic constant-coefficient stencil, and the regular network of
// ObservationNetwork::build (models.cpp:159-176) with a stride that divides n and the last
// row radix.  WC4DVAR_SPECTRAL=0 keeps the grid-space path (two convolutions + sweeps).
void HessianOp::setup_spectral(cudaStream_t st) {
    spectral = false;
    static const bool enabled = [] {
        const char* e = std::getenv("WC4DVAR_SPECTRAL");
        return !e || std::atoi(e) != 0;
    }();
    if (cov_kind != WC4DVAR_COV_CIRCULANT || !circ) return;
    Fft4* f4 = circ->spectral_fft();
    if (!f4) return;
    if (md.kind != WC4DVAR_MODEL_IDENTITY && md.kind != WC4DVAR_MODEL_ADVECTION && md.kind != WC4DVAR_MODEL_ADVDIFF)
        return;
    if (nd.q == 0 || nd.sx <= 0 || n % nd.sx != 0) return;
    if (!spectral_window_supported(nd.sx, f4->last_radix(), N + 1)) return;
    // one sub-step: coefficients of x_{j-1}, x_j, x_{j+1} (models.cpp:27-45), as stencil_power
    double lft = 0.0, mid = 1.0, rgt = 0.0;
    if (md.kind == WC4DVAR_MODEL_ADVECTION) {
        lft = md.c;
        mid = 1.0 - md.c;
    } else if (md.kind == WC4DVAR_MODEL_ADVDIFF) {
        lft = md.c + md.d;
        mid = 1.0 - md.c - 2.0 * md.d;
        rgt = md.d;
    }
    W4_CUDA(cudaMalloc(&d_mhat, sizeof(double2) * (size_t)n));
    f4->build_symbol(lft, mid, rgt, md.kind == WC4DVAR_MODEL_IDENTITY ? 1 : md.s, d_mhat, st);
    spectral = enabled;  // d_mhat != nullptr marks the operator eligible (wc4dvar_gpu_op_spectral)
}

void HessianOp::d_half(bool inv, const double* V, int64_t ldv, int64_t m, double* out,
                       int64_t ldo, const double* add, int64_t ldadd, unsigned* status,
                       cudaStream_t st) {
    if (cov_kind == WC4DVAR_COV_CIRCULANT) {
        circ->apply(inv, N, V, ldv, m, out, ldo, add, ldadd, status, circ_z, circ_x, st);
        return;
    }
    const double* B = inv ? b_half_inv : b_half;
    const double* Q = inv ? q_half_inv : q_half;
    require(B && Q, "apply_D_half_inv: inverse factors were not provided");
    GemmPass ps[2];
    int np = 0;
    if (N > 0) {
        GemmPass& p = ps[np++];
        p.A = Q;
        p.lda = n;
        p.M = n;
        p.K = n;
        p.ncols = (int64_t)N * m;
        p.in = ColMap{V, ldv, n, N, 1};
        p.out = ColMap{out, ldo, n, N, 1};
        if (add) p.add = ColMap{add, ldadd, n, N, 1};
        p.symA = sym[inv ? 3 : 1];
    }
    {
        GemmPass& p = ps[np++];
        p.A = B;
        p.lda = n;
        p.M = n;
        p.K = n;
        p.ncols = m;
        p.in = ColMap{V, ldv, n, 1, 0};
        p.out = ColMap{out, ldo, n, 1, 0};
        if (add) p.add = ColMap{add, ldadd, n, 1, 0};
        p.symA = sym[inv ? 2 : 0];
    }
    gemm_nn(ps, np, status, st);
}

void HessianOp::factor_apply(int which, bool inv, const double* X, int64_t ldx, int64_t c, double* out,
                             int64_t ldo, cudaStream_t st) {
    if (c == 0) return;
    if (cov_kind == WC4DVAR_COV_CIRCULANT) {
        circ->apply(inv, 0, X, ldx, c, out, ldo, nullptr, 0, nullptr, circ_z, circ_x, st, which);
        return;
    }
    const double* F = which == 0 ? (inv ? b_half_inv : b_half) : (inv ? q_half_inv : q_half);
    require(F, "apply_D_half_inv: inverse factors were not provided");
    GemmPass p;
    p.A = F;
    p.lda = n;
    p.M = n;
    p.K = n;
    p.ncols = c;
    p.in = ColMap::plain(X, ldx);
    p.out = ColMap::plain(out, ldo);
    p.symA = sym[which == 0 ? (inv ? 2 : 0) : (inv ? 3 : 1)];
    gemm_nn(&p, 1, nullptr, st);
}

void HessianOp::apply_block_dev(const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                                cudaStream_t st) {
    if (m == 0) return;
    if (spectral) {
        // DFT -> window recurrences per frequency class -> inverse DFT (+ v); see spectral.cu
        Fft4* f4 = circ->spectral_fft();
        // one column (PCG, Lanczos): pack its window blocks in pairs instead of leaving every
        // transform half empty (WC4DVAR_SPECTRAL_PACK1=0: the generic form)
        static const bool pack1 = [] {
            const char* e = std::getenv("WC4DVAR_SPECTRAL_PACK1");
            return !e || std::atoi(e) != 0;
        }();
        if (m == 1 && pack1 && N >= 1) {
            const int64_t npk = (N + 2) / 2;
            double2* Zin = t_ws.get<double2>((size_t)2 * npk * n);
            double2* Zout = Zin + npk * n;
            prof_mark(0, st);
            f4->forward(N, V, ldv, 1, Zin, circ_z, st, true);
            prof_mark(1, st);
            SpectralArgs sa;
            sa.N = n;
            sa.per = N + 1;
            sa.lamB = f4->lam(0);
            sa.lamQ = f4->lam(1);
            sa.mhat = d_mhat;
            sa.slot = nd.slot;
            sa.RL = f4->last_radix();
            sa.sx = nd.sx;
            sa.r_inv = 1.0 / (sigma_obs * sigma_obs);
            sa.status = d_status;
            int rad[4], nrad = 0;
            f4->row_radices(rad, nrad);
            spectral_window1(sa, Zin, Zout, (int)f4->n1(), (int)f4->n2(), rad, nrad, st);
            prof_mark(2, st);
            f4->inverse(N, Zout, 1, out, ldo, V, ldv, d_status, circ_z, st, true);
            prof_mark(3, st);
            prof_pending = prof;
            return;
        }
        const int64_t npc = (m + 1) / 2;
        double2* Z = t_ws.get<double2>((size_t)npc * (N + 1) * n);
        prof_mark(0, st);
        f4->forward(N, V, ldv, m, Z, circ_z, st);
        prof_mark(1, st);
        SpectralArgs sa;
        sa.Z = Z;
        sa.N = n;
        sa.per = N + 1;
        sa.npc = npc;
        sa.lamB = f4->lam(0);
        sa.lamQ = f4->lam(1);
        sa.mhat = d_mhat;
        sa.slot = nd.slot;
        sa.RL = f4->last_radix();
        sa.sx = nd.sx;
        sa.r_inv = 1.0 / (sigma_obs * sigma_obs);
        sa.status = d_status;
        spectral_window(sa, st);
        prof_mark(2, st);
        f4->inverse(N, Z, m, out, ldo, V, ldv, d_status, circ_z, st);
        prof_mark(3, st);
        prof_pending = prof;
        return;
    }
    const int64_t q = nd.q;
    double* T = t_ws.get<double>((size_t)dim * m);
    double* Y = q > 0 ? y_ws.get<double>((size_t)q * m) : nullptr;
    prof_mark(0, st);
    // t = D^{1/2} v  (operators.cpp:131)
    d_half(false, V, ldv, m, T, dim, nullptr, 0, nullptr, st);
    prof_mark(1, st);
    // traj = L^{-1} t; y = R^{-1} H traj; s = L^{-T} H^T y  (operators.cpp:132-141)
    SweepArgs a;
    a.X = T;
    a.ldx = dim;
    a.Y = Y;
    a.scale_fwd = 1.0 / (sigma_obs * sigma_obs);
    a.do_fwd = true;
    a.fwd_obs = q > 0;
    a.S = T;  // in place: the adjoint runs after the forward sweep of the same column
    a.lds = dim;
    a.do_adj = true;
    a.adj_obs = q > 0;
    a.m = m;
    sweep(md, nd, a, d_status, st, &sweep_ws);
    prof_mark(2, st);
    // out = v + D^{1/2} s  (operators.cpp:141)
    d_half(false, T, dim, m, out, ldo, V, ldv, d_status, st);
    prof_mark(3, st);
    prof_pending = prof;
}

namespace {
__global__ void identity_kernel(int64_t q, double* Y) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q * q; e += (int64_t)gridDim.x * blockDim.x)
        Y[e] = (e % (q + 1) == 0) ? 1.0 : 0.0;
}
}  // namespace

namespace {
// y[a np + b] = traj[times[a] n + points[b]]  (network order, models.cpp:184-192)
__global__ void observe_kernel(int64_t n, int np, int64_t q, const int* __restrict__ times,
                               const int* __restrict__ points, const double* __restrict__ traj,
                               double* __restrict__ y) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e / np, b = e - a * np;
        y[e] = traj[(int64_t)times[a] * n + points[b]];
    }
}
}  // namespace

void HessianOp::observe_dev(const double* traj, double* y, cudaStream_t st) {
    const int64_t q = nd.q;
    if (q == 0) return;
    observe_kernel<<<(unsigned)std::min<int64_t>(cdiv(q, 256), 4096), 256, 0, st>>>(n, nd.n_points, q, d_times,
                                                                                      d_points, traj, y);
    W4_LAUNCH();
}

void HessianOp::observation_range_dev(double* W, int64_t ldw, cudaStream_t st) {
    const int64_t q = nd.q;
    if (q == 0) return;
    double* Y = y_ws.get<double>((size_t)q * q);
    identity_kernel<<<(unsigned)std::min<int64_t>(cdiv(q * q, 256), 4096), 256, 0, st>>>(q, Y);
    W4_LAUNCH();
    double* S = t_ws.get<double>((size_t)dim * q);
    // s = L^{-T} H^T e_r for all r at once (observe_adjoint, models.cpp:193-201)
    SweepArgs a;
    a.Y = Y;
    a.S = S;
    a.lds = dim;
    a.do_adj = true;
    a.adj_obs = true;
    a.m = q;
    sweep(md, nd, a, d_status, st, &sweep_ws);
    d_half(false, S, dim, q, W, ldw, nullptr, 0, d_status, st);
}

void HessianOp::piece_dev(int which, const double* V, int64_t ldv, int64_t m, double* out,
                          int64_t ldo, cudaStream_t st) {
    if (m == 0) return;
    SweepArgs a;
    a.m = m;
    switch (which) {
        case WC4DVAR_LINV:
            a.X = V;
            a.ldx = ldv;
            a.traj = out;
            a.ldtraj = ldo;
            a.do_fwd = true;
            sweep(md, nd, a, d_status, st, &sweep_ws);
            break;
        case WC4DVAR_LINVT:
            a.V = V;
            a.ldv = ldv;
            a.S = out;
            a.lds = ldo;
            a.do_adj = true;
            sweep(md, nd, a, d_status, st, &sweep_ws);
            break;
        case WC4DVAR_SWEEPS: {  // L^{-T} H^T R^{-1} H L^{-1} v (operators.cpp:132-141)
            const int64_t q = nd.q;
            a.X = V;
            a.ldx = ldv;
            a.Y = q > 0 ? y_ws.get<double>((size_t)q * m) : nullptr;
            a.scale_fwd = 1.0 / (sigma_obs * sigma_obs);
            a.do_fwd = true;
            a.fwd_obs = q > 0;
            a.S = out;
            a.lds = ldo;
            a.do_adj = true;
            a.adj_obs = q > 0;
            sweep(md, nd, a, d_status, st, &sweep_ws);
            break;
        }
        case WC4DVAR_D_HALF:
        case WC4DVAR_D_HALF_INV:
            d_half(which == WC4DVAR_D_HALF_INV, V, ldv, m, out, ldo, nullptr, 0, nullptr, st);
            break;
        default:
            throw InvalidArgument("hessian piece: unknown selector");
    }
}

// ----------------------------------------------------------------------------- Dense
DenseOp::~DenseOp() {
    DeviceGuard g(device);
    if (A) cudaFree(A);
}

void DenseOp::apply_block_dev(const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                              cudaStream_t st) {
    if (m == 0) return;
    GemmPass p;
    p.A = A;
    p.lda = dim;
    p.M = dim;
    p.K = dim;
    p.ncols = m;
    p.in = ColMap::plain(V, ldv);
    p.out = ColMap::plain(out, ldo);
    gemm_nn(&p, 1, nullptr, st);
}

}  // namespace w4

// ----------------------------------------------------------------------------- LMP / cost dtors
wc4dvar_lmp::~wc4dvar_lmp() {
    DeviceGuard g(device);
    if (U) cudaFree(U);
    if (theta) cudaFree(theta);
    if (T) cudaFree(T);
    if (counter) cudaFree(counter);
    if (stream) cudaStreamDestroy(stream);
}

wc4dvar_cost::~wc4dvar_cost() {
    if (b_tilde) cudaFree(b_tilde);
    if (d) cudaFree(d);
    if (counter) cudaFree(counter);
    if (d_val) cudaFree(d_val);
}

double wc4dvar_cost::eval_dev(const double* x, cudaStream_t st) {
    HessianOp& h = *op;
    const int64_t dim = h.dim, q = h.nd.q;
    double* t = ws_t.get<double>((size_t)dim);
    double* y = q > 0 ? ws_y.get<double>((size_t)q) : nullptr;
    double* part = partial.get<double>(2 * kSMs);
    // J(x) = 1/2 |x - b~|^2 + 1/2 r_inv |H L^{-1} D^{1/2} x - d|^2  (assimilation.cpp:135-140)
    h.d_half(false, x, dim, 1, t, dim, nullptr, 0, nullptr, st);
    SweepArgs a;
    a.X = t;
    a.ldx = dim;
    a.Y = y;
    a.scale_fwd = 1.0;
    a.do_fwd = true;
    a.fwd_obs = q > 0;
    a.m = 1;
    sweep(h.md, h.nd, a, h.d_status, st, &h.sweep_ws);
    sqdist(dim, x, b_tilde, d_val, part, counter, st);
    if (q > 0) sqdist(q, y, d, d_val + 1, part, counter, st);
    else W4_CUDA(cudaMemsetAsync(d_val + 1, 0, sizeof(double), st));
    double hv[2];
    W4_CUDA(cudaMemcpyAsync(hv, d_val, sizeof(hv), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    const double r_inv = 1.0 / (h.sigma_obs * h.sigma_obs);
    return 0.5 * hv[0] + 0.5 * r_inv * hv[1];
}

