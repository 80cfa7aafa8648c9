// Deterministic (previous-loop) LMP eigenpairs on the device:
//   lanczos_eigenpairs   krylov.cpp:178-278  matrix-free Lanczos, full re-orthogonalisation
//   ritz_from_tridiagonal krylov.cpp:136-176 Ritz pairs from the CG-Lanczos tridiagonal and
//                                            the stored normalised CG residuals
//
// The n-long work -- operator applies, the two Gram-Schmidt passes against the whole
// basis (one DMMA Gram GEMV + one tall x small DMMA GEMM each), the Ritz vectors -- runs on
// the device; the basis lives in HBM as one n x (max_iter + 1) block.  The per-iteration
// convergence test needs only the top-k eigenvalues of the small tridiagonal T_m and the
// last row of its eigenvectors: an implicit-QL sweep on the host that tracks that one row
// (O(m^2)).  The final eigendecomposition of T_m uses the device Jacobi EVD.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>
#include <vector>

#include "gemm.cuh"
#include "lanczos.cuh"
#include "lmp_pcg.cuh"
#include "smallla.cuh"

namespace w4 {
void gaussian_fill(int64_t count, uint64_t seed, double* out);

namespace {

__global__ void scale_kernel(int64_t n, const double* __restrict__ x, double s, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] * s;
}

// columns of X (n x k, ld n) scaled to unit 2-norm; one CTA per column, fixed-order sums
__global__ void __launch_bounds__(512) normalize_cols_kernel(int64_t n, double* X) {
    __shared__ double red[512];
    double* x = X + (int64_t)blockIdx.x * n;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 512) s += x[i] * x[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 256; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double inv = 1.0 / sqrt(red[0]);
    for (int64_t i = threadIdx.x; i < n; i += 512) x[i] *= inv;
}

// F (n x j) with column i scaled by (-1)^i (the Lanczos basis hiding in CG, krylov.cpp:143-146)
__global__ void alt_sign_kernel(int64_t n, int64_t j, const double* __restrict__ F, int64_t ldf,
                                double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * j; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / n, r = e - c * n;
        const double v = F[c * ldf + r];
        out[e] = (c & 1) ? -v : v;
    }
}

unsigned grid1d(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4 * kSMs)); }

// Eigenvalues of the symmetric tridiagonal (d, e) (e[i] couples i and i+1) by implicit QL
// with Wilkinson shifts, tracking only the last row z of the eigenvector matrix.  Returns
// the pairs (value, |z|) sorted by decreasing value.
std::vector<std::pair<double, double>> tridiag_values_lastrow(std::vector<double> d, const std::vector<double>& off) {
    const int m = (int)d.size();
    std::vector<double> e(m, 0.0), z(m, 0.0);
    for (int i = 0; i + 1 < m; ++i) e[i] = off[i];
    z[m - 1] = 1.0;
    const double eps = 2.220446049250313e-16;
    for (int l = 0; l < m; ++l) {
        int iter = 0;
        int mm;
        do {
            for (mm = l; mm < m - 1; ++mm) {
                const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
                if (std::fabs(e[mm]) <= eps * dd) break;
            }
            if (mm != l) {
                if (iter++ == 100) throw NumericalError("lanczos_eigenpairs: tridiagonal QL did not converge");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = mm - 1; i >= l; --i) {
                    double f = s * e[i];
                    const double b = c * e[i];
                    e[i + 1] = (r = std::hypot(f, g));
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[mm] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    d[i + 1] = g + (p = s * r);
                    g = c * r - b;
                    f = z[i + 1];
                    z[i + 1] = s * z[i] + c * f;
                    z[i] = c * z[i] - s * f;
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[mm] = 0.0;
            }
        } while (mm != l);
    }
    std::vector<std::pair<double, double>> out(m);
    for (int i = 0; i < m; ++i) out[i] = {d[i], std::fabs(z[i])};
    std::sort(out.begin(), out.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    return out;
}

struct Work {
    wc4dvar_op& op;
    cudaStream_t st;
    int64_t n;
    DevBuf gemm_ws, small_ws, part, cnt, scal;
    double* pinned = nullptr;
    explicit Work(wc4dvar_op& o, cudaStream_t s) : op(o), st(s), n(o.dim) {
        W4_CUDA(cudaMallocHost(&pinned, 8 * sizeof(double)));
    }
    ~Work() {
        if (pinned) cudaFreeHost(pinned);
    }
    // a . b (deterministic row pass) -> host
    double dot(const double* a, const double* b) {
        const int64_t maxgrid = std::min<int64_t>(cdiv(n, 32) + 1, 2048);
        RowPassCtx c{n, 0, nullptr, n, 0, nullptr, part.get<double>((size_t)maxgrid),
                     cnt.get<unsigned>(4), scal.get<double>(SC_N), nullptr, nullptr};
        W4_CUDA(cudaMemsetAsync(c.counter, 0, 4 * sizeof(unsigned), st));
        double* out = scal.get<double>(SC_N) + SC_N - 1;
        rowpass_utv(c, a, a, b, out, st);
        W4_CUDA(cudaMemcpyAsync(pinned, out, sizeof(double), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        return pinned[0];
    }
    // w -= V[:, 0..cols) (V^T w), twice (classical Gram-Schmidt with re-orthogonalisation)
    void reorth(const double* V, int64_t cols, double* w, double* h) {
        for (int pass = 0; pass < 2; ++pass) {
            gemm_tn(n, cols, 1, V, n, w, n, 1.0, h, cols, gemm_ws, st);
            GemmPass gp;
            gp.A = V;
            gp.lda = n;
            gp.M = n;
            gp.K = cols;
            gp.ncols = 1;
            gp.alpha = -1.0;
            gp.in = ColMap::plain(h, cols);
            gp.out = ColMap::plain(w, n);
            gp.add = ColMap::plain(w, n);
            gemm_nn(&gp, 1, nullptr, st);
        }
    }
};

}  // namespace

int64_t lanczos_eigenpairs_dev(wc4dvar_op& op, int64_t k, int max_iter, double tol, uint64_t seed,
                               double* U_out, int64_t ldu, double* values_out, cudaStream_t st) {
    const int64_t n = op.dim;
    require(k >= 1 && k <= n, "lanczos_eigenpairs: k out of range");
    require(ldu == n, "lanczos_eigenpairs: U must be contiguous (ldu = dim)");
    const int M = max_iter > 0 ? max_iter : (int)std::min<int64_t>(n, 8 * k + 120);
    require(M <= 512, "lanczos_eigenpairs: more than 512 Lanczos steps is not supported by the device "
                      "small-matrix kernels");
    Work wk(op, st);
    DevBuf vb, wb, hb;
    double* V = vb.get<double>((size_t)n * (M + 1));
    double* w = wb.get<double>(n);
    double* h = hb.get<double>(M + 2);
    // v_0 = NormalStream(seed).draw(n).normalized()  (krylov.cpp:186-188)
    std::vector<double> host((size_t)n);
    uint64_t draws = 0;  // normals consumed from the stream (restarts continue it)
    auto draw = [&](std::vector<double>& buf) {
        // NormalStream is sequential: regenerate the prefix and keep the next n normals
        std::vector<double> all((size_t)(draws + n));
        gaussian_fill((int64_t)all.size(), seed, all.data());
        std::copy(all.begin() + (int64_t)draws, all.end(), buf.begin());
        draws += n;
    };
    draw(host);
    double nrm = 0.0;
    for (double x : host) nrm += x * x;
    nrm = std::sqrt(nrm);
    for (double& x : host) x /= nrm;
    W4_CUDA(cudaMemcpyAsync(V, host.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    W4_CUDA(cudaStreamSynchronize(st));

    std::vector<double> diag, off;
    int converged_at = -1;
    int nb = 1;  // basis vectors stored
    for (int j = 0; j < M; ++j) {
        double* vj = V + (int64_t)j * n;
        op.applies += 1;
        op.reset_status(st);
        op.apply_block_dev(vj, n, 1, w, n, st);
        op.check_status(st);
        if (j > 0) axpby(n, 1.0, w, -off[j - 1], V + (int64_t)(j - 1) * n, w, st);
        const double a = wk.dot(vj, w);
        diag.push_back(a);
        axpby(n, 1.0, w, -a, vj, w, st);
        wk.reorth(V, nb, w, h);  // full re-orthogonalisation, twice (krylov.cpp:199-201)
        const double b = std::sqrt(wk.dot(w, w));
        const int64_t m = (int64_t)diag.size();
        if (m >= k) {
            const auto vz = tridiag_values_lastrow(diag, off);
            const double scale = std::fabs(vz[0].first);
            bool all = true;
            for (int64_t i = 0; i < k; ++i)
                if (b * vz[i].second > tol * scale) {
                    all = false;
                    break;
                }
            if (all) {
                converged_at = (int)m;
                break;
            }
        }
        double* vn = V + (int64_t)(j + 1) * n;
        if (b <= 1e-14) {
            // invariant subspace: restart with a fresh orthogonal direction (krylov.cpp:233-242)
            draw(host);
            W4_CUDA(cudaMemcpyAsync(w, host.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
            wk.reorth(V, nb, w, h);
            const double fn = std::sqrt(wk.dot(w, w));
            if (fn <= 1e-14) break;
            off.push_back(0.0);
            scale_kernel<<<grid1d(n), 256, 0, st>>>(n, w, 1.0 / fn, vn);
        } else {
            off.push_back(b);
            scale_kernel<<<grid1d(n), 256, 0, st>>>(n, w, 1.0 / b, vn);
        }
        W4_LAUNCH();
        ++nb;
    }
    const int64_t m = converged_at > 0 ? converged_at : (int64_t)diag.size();
    if (m < k) throw NumericalError("lanczos_eigenpairs: Krylov space exhausted before k pairs");
    // T_m on the device, Jacobi EVD (values decreasing), U = normalise(V_m W[:, :k])
    std::vector<double> T((size_t)m * m, 0.0);
    for (int64_t i = 0; i < m; ++i) {
        T[i * m + i] = diag[i];
        if (i + 1 < m) T[i * m + i + 1] = T[(i + 1) * m + i] = off[i];
    }
    DevBuf tb, vals, wv;
    double* dT = tb.get<double>((size_t)m * m);
    double* dvals = vals.get<double>(m);
    double* dW = wv.get<double>((size_t)m * m);
    W4_CUDA(cudaMemcpyAsync(dT, T.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st));
    sym_evd_desc((int)m, dT, dvals, dW, wk.small_ws, st);
    GemmPass gp;
    gp.A = V;
    gp.lda = n;
    gp.M = n;
    gp.K = m;
    gp.ncols = k;
    gp.in = ColMap::plain(dW, m);
    gp.out = ColMap::plain(U_out, ldu);
    gemm_nn(&gp, 1, nullptr, st);
    normalize_cols_kernel<<<(unsigned)k, 512, 0, st>>>(n, U_out);
    W4_LAUNCH();
    W4_CUDA(cudaMemcpyAsync(values_out, dvals, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    return m;
}

int64_t ritz_from_tridiagonal_dev(int64_t n, int64_t j, const double* gammas, const double* taus, const double* F,
                                  int64_t ldf, int64_t k, double* U_out, int64_t ldu, double* values_out,
                                  cudaStream_t st) {
    require(k >= 1 && k <= j, "ritz_from_tridiagonal: k out of range");
    require(j <= 512, "ritz_from_tridiagonal: T above 512 is not supported by the device small-matrix kernels");
    DevBuf fb, gb, ws, small, tb, vals, wv, pb;
    double* Fs = fb.get<double>((size_t)n * j);
    alt_sign_kernel<<<grid1d(n * j), 256, 0, st>>>(n, j, F, ldf, Fs);
    W4_LAUNCH();
    // orthogonality of the residual basis (krylov.cpp:147-151)
    double* G = gb.get<double>((size_t)j * j + 1);
    gemm_tn(n, j, j, Fs, n, Fs, n, 1.0, G, j, ws, st);
    defect_max((int)j, G, G + j * j, st);
    double defect = 0.0;
    W4_CUDA(cudaMemcpyAsync(&defect, G + j * j, sizeof(double), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    if (!(defect <= 1e-8))
        throw NumericalError("ritz_from_tridiagonal: residual basis lost orthogonality; "
                             "run CG with reorthogonalization");
    std::vector<double> T((size_t)j * j, 0.0);
    for (int64_t i = 0; i < j; ++i) {
        T[i * j + i] = gammas[i];
        if (i + 1 < j) T[i * j + i + 1] = T[(i + 1) * j + i] = taus[i];
    }
    double* dT = tb.get<double>((size_t)j * j);
    double* dv = vals.get<double>(j);
    double* dW = wv.get<double>((size_t)j * j);
    W4_CUDA(cudaMemcpyAsync(dT, T.data(), sizeof(double) * j * j, cudaMemcpyHostToDevice, st));
    sym_evd_desc((int)j, dT, dv, dW, small, st);
    std::vector<double> hv(j);
    W4_CUDA(cudaMemcpyAsync(hv.data(), dv, sizeof(double) * j, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    // collapse suspected ghosts (near-duplicate values), keeping the first (krylov.cpp:157-163)
    const double ghost_tol = 1e-10 * std::fabs(hv[0]);
    std::vector<int> keep;
    for (int i = 0; i < (int)j; ++i) {
        if (!keep.empty() && std::fabs(hv[keep.back()] - hv[i]) <= ghost_tol) continue;
        keep.push_back(i);
    }
    if ((int64_t)keep.size() < k)
        throw NumericalError("ritz_from_tridiagonal: fewer distinct Ritz values than requested");
    keep.resize(k);
    int* dperm = pb.get<int>(k);
    W4_CUDA(cudaMemcpyAsync(dperm, keep.data(), sizeof(int) * k, cudaMemcpyHostToDevice, st));
    double* Wk = tb.get<double>((size_t)j * j);  // dT is consumed by the EVD
    gather_cols(j, (int)k, dW, j, dperm, Wk, j, st);
    GemmPass gp;
    gp.A = Fs;
    gp.lda = n;
    gp.M = n;
    gp.K = j;
    gp.ncols = k;
    gp.in = ColMap::plain(Wk, j);
    gp.out = ColMap::plain(U_out, ldu);
    gemm_nn(&gp, 1, nullptr, st);
    for (int64_t i = 0; i < k; ++i) values_out[i] = hv[keep[i]];
    W4_CUDA(cudaStreamSynchronize(st));
    return k;
}

}  // namespace w4
