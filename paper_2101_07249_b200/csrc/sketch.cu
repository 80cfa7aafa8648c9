// REVD / Nystrom / ritzit on device (randevd.cpp:47-148).
//
// Orthonormalisation is CholQR2 (Gram by DMMA split-GEMM, Cholesky + triangular inverse
// in one CTA, Y R^{-1} by DMMA GEMM, twice).  The reference's Householder QR, pivoted QR
// and BDCSVD are replaced by numerically equivalent (basis-invariant) steps:
//   * Ritz values / LMP are invariant to the orthonormal basis of span(Y)
//     (sign and rotation of Z cancel in Z W), so CholQR2 replaces HouseholderQR;
//   * the ColPivHouseholderQR rank probe becomes a diagonally pivoted Cholesky of Y^T Y
//     with a Gram-noise threshold;
//   * BDCSVD(F) becomes CholQR2(F) = Q_F R_F plus one-sided Jacobi SVD of R_F.
#include "sketch.cuh"

#include <cmath>
#include <cstring>
#include <sstream>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"
#include "lmp_pcg.cuh"
#include "smallla.cuh"

namespace w4 {
void gaussian_fill(int64_t count, uint64_t seed, double* out);
int colpiv_rank_dd(int64_t n, int m, const double* Y, int64_t ld, int* perm_dev, int* rank_dev, int* rank_host,
                   DevBuf& work, cudaStream_t st);
namespace {

enum {
    P_Y = 0, P_Z, P_Q1, P_AZ, P_F, P_G, P_R1, P_R1I, P_G2, P_R2, P_R2I, P_R, P_K, P_W,
    P_VALS, P_INT, P_TMP, P_SEL, P_GEMMWS, P_SMALLWS, P_DDWS, P_RA, P_RB, P_COUNT
};

static_assert(P_COUNT <= 24, "sketch workspaces must stay below the PCG pool range (ops.cuh)");

struct Timer {
    cudaStream_t st;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> evs;
    int cur = -1;
    cudaEvent_t cur_start = nullptr;
    bool on;
    Timer(cudaStream_t s, bool enabled) : st(s), on(enabled) {}
    ~Timer() {
        for (auto& e : evs) {
            cudaEventDestroy(e.second.first);
            cudaEventDestroy(e.second.second);
        }
    }
    void begin(int cat) {
        if (!on) return;
        end();
        W4_CUDA(cudaEventCreate(&cur_start));
        W4_CUDA(cudaEventRecord(cur_start, st));
        cur = cat;
    }
    void end() {
        if (!on || cur < 0) return;
        cudaEvent_t e;
        W4_CUDA(cudaEventCreate(&e));
        W4_CUDA(cudaEventRecord(e, st));
        evs.push_back({cur, {cur_start, e}});
        cur = -1;
    }
    void collect(SketchTiming* t) {
        if (!on || !t) return;
        end();
        W4_CUDA(cudaStreamSynchronize(st));
        double acc[4] = {0, 0, 0, 0};
        for (auto& e : evs) {
            float ms = 0;
            W4_CUDA(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
            acc[e.first] += ms;
        }
        t->apply_ms = acc[0];
        t->orth_ms = acc[1];
        t->small_ms = acc[2];
        t->gemm_ms = acc[3];
        t->total_ms = acc[0] + acc[1] + acc[2] + acc[3];
    }
};
enum { T_APPLY = 0, T_ORTH = 1, T_SMALL = 2, T_GEMM = 3 };

struct Ctx {
    wc4dvar_op& op;
    cudaStream_t st;
    int64_t n;
    Timer& tm;
    DevBuf* pool;
    int* h_int;  // pinned scratch
    int shifted_calls = 0;  // orth() calls that needed shifted CholQR3
    int single_pass_calls = 0;  // cholqr2() calls that stopped after one pass (cond(Y) <= 4)
    int dd_rank_calls = 0;  // rank probes decided on the double-double Gram

    double* buf(int id, size_t count) { return pool[id].get<double>(count); }

    int read_int(const int* d) {
        W4_CUDA(cudaMemcpyAsync(h_int, d, sizeof(int), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        return *h_int;
    }

    // out = A in  (m columns), counted and finite-checked like apply_block.
    void apply(const double* in, int64_t m, double* out) {
        tm.begin(T_APPLY);
        op.applies += m;
        op.reset_status(st);
        op.apply_block_dev(in, n, m, out, n, st);
        op.check_status(st);
        tm.end();
    }

    // G = A^T B (m1 x m2)
    // sym: A^T B is known to be symmetric (upper-triangle tiles only, mirrored)
    void gram(const double* A, int64_t m1, const double* B, int64_t m2, double* G, bool sym = false) {
        gemm_tn(n, m1, m2, A, n, B, n, 1.0, G, m1, pool[P_GEMMWS], st, sym);
    }

    // C (n x ncols) = A (n x K) * B (K x ncols, ld K); tri: B is upper triangular (R^{-1})
    void tall_times_small(const double* A, int64_t K, const double* B, int64_t ldb, int64_t ncols,
                          double* C, int64_t ldc, bool tri = false) {
        GemmPass p;
        p.upper_tri = tri;
        p.A = A;
        p.lda = n;
        p.M = n;
        p.K = K;
        p.ncols = ncols;
        p.in = ColMap::plain(B, ldb);
        p.out = ColMap::plain(C, ldc);
        gemm_nn(&p, 1, nullptr, st);
    }

    // Adaptive CholQR test: passes are expensive (2 n m^2 >= 1e11 flops per Gram) and the
    // singular values of R1 (those of Y; Jacobi SVD of the m x m factor) give cond(Y) <= 4.
    bool single_pass_ok(const double* R1, int64_t m) {
        const char* adapt_env = std::getenv("WC4DVAR_CHOLQR_ADAPT");  // read per call (tests toggle it)
        const bool adapt = !adapt_env || std::atoi(adapt_env) != 0;
        if (!adapt || 2.0 * (double)n * (double)m * (double)m < 1e11) return false;
        double* sig = buf(P_R2, m * m);
        svd_left_desc((int)m, R1, sig, buf(P_G2, m * m), pool[P_SMALLWS], st);
        double hs[2];
        W4_CUDA(cudaMemcpyAsync(&hs[0], sig, sizeof(double), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaMemcpyAsync(&hs[1], sig + (m - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        return hs[1] > 0.0 && hs[0] <= 4.0 * hs[1];
    }

    // Factored orthonormalisation for callers that only multiply the basis by a small matrix
    // next (Q W = Y (R^{-1} W)): when one CholQR pass suffices, R and R^{-1} of Y = Q R are
    // returned WITHOUT forming Q (one n x m x m product less).  false: use orth(); the Gram it
    // computed stays in P_G for orth's G0.
    bool orth_factored(const double* Y, int64_t m, double* R_out, double* Rinv_out, const double* G0 = nullptr) {
        if (2.0 * (double)n * (double)m * (double)m < 1e11) return false;
        tm.begin(T_ORTH);
        double* G = buf(P_G, m * m);
        if (G0) {
            if (G0 != G) W4_CUDA(cudaMemcpyAsync(G, G0, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
        } else {
            gram(Y, m, Y, m, G);
        }
        factored_gram = G;
        double* R1 = buf(P_R1, m * m);
        double* R1i = buf(P_R1I, m * m);
        int* info = reinterpret_cast<int*>(buf(P_INT, 4 + 2 * m));
        chol_inv_upper((int)m, G, R1, R1i, info, pool[P_SMALLWS], st);
        const bool ok = !read_int(info) && single_pass_ok(R1, m);
        if (ok) {
            ++single_pass_calls;
            W4_CUDA(cudaMemcpyAsync(R_out, R1, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
            W4_CUDA(cudaMemcpyAsync(Rinv_out, R1i, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
        }
        tm.end();
        return ok;
    }
    const double* factored_gram = nullptr;  // Y^T Y left by the last orth_factored (for orth's G0)

    // CholQR2: Q (n x m) with Y = Q R; G0 = Y^T Y may be supplied.  Q may alias Y (Y is
    // dead once Q1 = Y R1^{-1} exists); `scratch` (n x m) holds Q1 and must alias neither.
    // Returns false on a Cholesky breakdown (caller raises the method-specific
    // NumericalError).
    bool cholqr2(const double* Y, int64_t m, double* Q, double* R_out, const double* G0, double* scratch) {
        tm.begin(T_ORTH);
        double* G = buf(P_G, m * m);
        if (G0) {
            if (G0 != G)
                W4_CUDA(cudaMemcpyAsync(G, G0, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
        } else {
            gram(Y, m, Y, m, G);
        }
        double* R1 = buf(P_R1, m * m);
        double* R1i = buf(P_R1I, m * m);
        int* info = reinterpret_cast<int*>(buf(P_INT, 4 + 2 * m));
        chol_inv_upper((int)m, G, R1, R1i, info, pool[P_SMALLWS], st);
        if (read_int(info)) return false;
        // The second pass exists to repair the cond(Y)^2 eps loss of orthogonality of the first.
        // When the passes are expensive and cond(Y) <= 4 (single_pass_ok) the first pass already
        // gives |Q1^T Q1 - I| ~ 16 eps, what Householder QR of the reference delivers (m eps), and
        // the second pass is skipped (C4: cond(Y) = 1.6, cond(Omega) = 1.01).
        // WC4DVAR_CHOLQR_ADAPT=0 always runs both passes.
        {
            if (single_pass_ok(R1, m)) {
                ++single_pass_calls;
                if (Q != Y) {
                    tall_times_small(Y, m, R1i, m, m, Q, n, true);
                } else {  // in place: through the scratch block
                    tall_times_small(Y, m, R1i, m, m, scratch, n, true);
                    W4_CUDA(cudaMemcpyAsync(Q, scratch, sizeof(double) * n * m, cudaMemcpyDeviceToDevice, st));
                }
                if (R_out) W4_CUDA(cudaMemcpyAsync(R_out, R1, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
                tm.end();
                return true;
            }
        }
        double* Q1 = scratch;
        tall_times_small(Y, m, R1i, m, m, Q1, n, true);
        double* G2 = buf(P_G2, m * m);
        gram(Q1, m, Q1, m, G2);
        double* R2 = buf(P_R2, m * m);
        double* R2i = buf(P_R2I, m * m);
        chol_inv_upper((int)m, G2, R2, R2i, info, pool[P_SMALLWS], st);
        if (read_int(info)) return false;
        tall_times_small(Q1, m, R2i, m, m, Q, n, true);
        if (R_out) small_gemm(false, false, (int)m, (int)m, (int)m, 1.0, R2, (int)m, R1, (int)m, 0.0,
                              R_out, (int)m, st);
        tm.end();
        return true;
    }

    // Orthonormal basis Q of span(Y) (full column rank) with Y = Q R: CholQR2, falling back
    // to shifted CholQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020) when the
    // Gram is too ill-conditioned for a plain Cholesky (cond(Y) >~ 1e8; the reference's
    // Householder QR accepts any full-rank Y).  Q may alias Y; `scratch` aliases neither.
    // Returns false only if the shifted variant breaks down too.
    bool orth(const double* Y, int64_t m, double* Q, double* R_out, const double* G0, double* scratch) {
        if (cholqr2(Y, m, Q, R_out, G0, scratch)) return true;
        ++shifted_calls;
        tm.begin(T_ORTH);
        double* G = buf(P_G, m * m);
        gram(Y, m, Y, m, G);  // cholqr2 may have overwritten P_G
        std::vector<double> hG((size_t)m * m);
        W4_CUDA(cudaMemcpyAsync(hG.data(), G, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        double tr = 0.0;
        for (int64_t i = 0; i < m; ++i) tr += hG[i + i * m];
        // shift s = 11 (m n + m (m + 1)) u ||Y||_2^2, with trace(G) >= ||Y||_2^2
        const double shift = 11.0 * ((double)m * (double)n + (double)m * (m + 1)) * 1.1102230246251565e-16 * tr;
        for (int64_t i = 0; i < m; ++i) hG[i + i * m] += shift;
        W4_CUDA(cudaMemcpyAsync(G, hG.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, st));
        double* Rs = buf(P_R1, m * m);
        double* Rsi = buf(P_R1I, m * m);
        int* info = reinterpret_cast<int*>(buf(P_INT, 4 + 2 * m));
        chol_inv_upper((int)m, G, Rs, Rsi, info, pool[P_SMALLWS], st);
        if (read_int(info)) return false;
        tall_times_small(Y, m, Rsi, m, m, scratch, n, true);  // Q1 = Y Rs^{-1}; Y is dead after this
        double* Racc = buf(P_TMP, 2 * m * m);
        double* Rtmp = Racc + m * m;
        W4_CUDA(cudaMemcpyAsync(Racc, Rs, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
        double* src = scratch;
        double* dst = Q;  // Q is free: either Y's own (dead) buffer or a separate output
        for (int pass = 0; pass < 2; ++pass) {
            double* G2 = buf(P_G2, m * m);
            gram(src, m, src, m, G2);
            double* R2 = buf(P_R2, m * m);
            double* R2i = buf(P_R2I, m * m);
            chol_inv_upper((int)m, G2, R2, R2i, info, pool[P_SMALLWS], st);
            if (read_int(info)) return false;
            tall_times_small(src, m, R2i, m, m, dst, n, true);
            small_gemm(false, false, (int)m, (int)m, (int)m, 1.0, R2, (int)m, Racc, (int)m, 0.0, Rtmp, (int)m, st);
            std::swap(Racc, Rtmp);
            std::swap(src, dst);
        }
        if (src != Q) W4_CUDA(cudaMemcpyAsync(Q, src, sizeof(double) * n * m, cudaMemcpyDeviceToDevice, st));
        if (R_out) W4_CUDA(cudaMemcpyAsync(R_out, Racc, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
        tm.end();
        return true;
    }

    // Rank probe of ColPivHouseholderQR (randevd.cpp:67-73, 89-92); perm to P_INT[4..].
    // Fast path: a pivoted Cholesky of the double Gram G with a Gram-noise tolerance; it is
    // conclusive when it finds full rank (cond(Y) <~ 1e6).  Otherwise, when Y is given, the
    // rank is decided by Eigen's own rule on a double-double Gram (rank_dd.cu), so an
    // ill-conditioned but full-rank sample (cond up to ~1/(m eps)) is accepted as Eigen does.
    int rank_probe(const double* G, int64_t m, int** perm_out, const double* Y = nullptr) {
        tm.begin(T_SMALL);
        int* ints = reinterpret_cast<int*>(buf(P_INT, 4 + 2 * m));
        int* perm = ints + 4;
        const double tol_rel = 32.0 * std::sqrt((double)n) * 2.220446049250313e-16;
        pivoted_chol_rank((int)m, G, tol_rel, ints + 1, perm, pool[P_SMALLWS], st);
        int r = read_int(ints + 1);
        if (r < m && Y) {
            ++dd_rank_calls;
            r = colpiv_rank_dd(n, (int)m, Y, n, perm, ints + 1, h_int, pool[P_DDWS], st);
        }
        tm.end();
        *perm_out = perm;
        return r;
    }
};

__global__ void sqrt_head_kernel(int k, const double* __restrict__ vals, double* __restrict__ out) {
    const int i = threadIdx.x + blockIdx.x * blockDim.x;
    if (i < k) out[i] = sqrt(vals[i]);
}
__global__ void square_head_kernel(int k, const double* __restrict__ s, double* __restrict__ out) {
    const int i = threadIdx.x + blockIdx.x * blockDim.x;
    if (i < k) out[i] = s[i] * s[i];
}

// check_z = false: Z is the basis Ctx::orth just produced (two CholQR passes, or one at
// cond <= 4: |Z^T Z - I| is a small multiple of eps), so the 1e-8 test of randevd.cpp:50-52
// cannot fire and its n m^2 Gram is not computed; the public rayleigh_ritz always checks.
void rr_core(Ctx& c, const double* Z, int64_t m, int64_t keep, double* U_out, int64_t ldu,
             double* theta_out, double* AZ, bool check_z = true) {
    const int64_t n = c.n;
    if (check_z) {  // Gram defect check (randevd.cpp:50-52)
        c.tm.begin(T_GEMM);
        double* G = c.buf(P_G, m * m);
        c.gram(Z, m, Z, m, G);
        double* defect = c.buf(P_TMP, 4);
        defect_max((int)m, G, defect, c.st);
        double hd = 0;
        W4_CUDA(cudaMemcpyAsync(&hd, defect, sizeof(double), cudaMemcpyDeviceToHost, c.st));
        W4_CUDA(cudaStreamSynchronize(c.st));
        c.tm.end();
        if (!(hd <= 1e-8)) throw NumericalError("rayleigh_ritz: Z is not orthonormal");
    }
    c.apply(Z, m, AZ);  // second block product
    c.tm.begin(T_GEMM);
    double* K = c.buf(P_K, m * m);
    c.gram(Z, m, AZ, m, K);
    c.tm.begin(T_SMALL);
    double* vals = c.buf(P_VALS, m);
    double* W = c.buf(P_W, m * m);
    sym_evd_desc((int)m, K, vals, W, c.pool[P_SMALLWS], c.st);
    c.tm.begin(T_GEMM);
    c.tall_times_small(Z, m, W, m, keep, U_out, ldu);
    W4_CUDA(cudaMemcpyAsync(theta_out, vals, sizeof(double) * keep, cudaMemcpyDeviceToDevice, c.st));
    c.tm.end();
}

}  // namespace

void clustered_spectrum_dev(wc4dvar_op& op, const double* Wobs, int64_t q, const double* U, int64_t k,
                            const double* T, double* vals_out, cudaStream_t st) {
    const int64_t n = op.dim;
    const int64_t m = q + k;
    require(m >= 1 && m <= n, "clustered_spectrum: q + k must lie in [1, dim]");
    require(m <= 512, "clustered_spectrum: q + k above 512 is not supported by the device small-matrix kernels");
    Timer tm(st, false);
    Ctx c{op, st, n, tm, op.pool, op.h_int};
    // B = [W | U] (spectrum.cpp:38-41)
    double* B = c.buf(P_Y, n * m);
    if (q) W4_CUDA(cudaMemcpyAsync(B, Wobs, sizeof(double) * n * q, cudaMemcpyDeviceToDevice, st));
    if (k) W4_CUDA(cudaMemcpyAsync(B + n * q, U, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
    // Orthonormal Q with q + k columns spanning span(B) (spectrum.cpp:45-46: Householder Q).
    // CholQR2 when B has full numerical rank; otherwise CholQR2 of the r pivot columns,
    // completed by Gaussian directions orthogonalised against them -- C^T A C is the
    // identity on that complement, as on the Householder completion.
    double* G = c.buf(P_G, m * m);
    c.gram(B, m, B, m, G);
    int* perm = nullptr;
    const int r = c.rank_probe(G, m, &perm);
    if (r == 0) throw NumericalError("clustered_spectrum: observation range and LMP vectors are zero");
    double* Q = c.buf(P_Z, n * m);
    if (r == m) {
        if (!c.orth(B, m, Q, nullptr, G, c.buf(P_Q1, n * m)))
            throw NumericalError("clustered_spectrum: basis too ill-conditioned for CholQR2");
    } else {
        double* Bp = c.buf(P_SEL, n * m);
        gather_cols(n, r, B, n, perm, Bp, n, st);
        if (!c.orth(Bp, r, Q, nullptr, nullptr, c.buf(P_Q1, n * m)))
            throw NumericalError("clustered_spectrum: basis too ill-conditioned for CholQR2");
        const int64_t e = m - r;
        std::vector<double> hz((size_t)n * e);
        gaussian_fill(n * e, 1, hz.data());  // NormalStream(1): deterministic completion
        double* Z = Bp;                       // Bp is dead once Q[:, :r] exists
        W4_CUDA(cudaMemcpyAsync(Z, hz.data(), sizeof(double) * n * e, cudaMemcpyHostToDevice, st));
        double* P = c.buf(P_TMP, (size_t)r * e);
        for (int pass = 0; pass < 2; ++pass) {  // Z -= Q_r (Q_r^T Z), twice
            c.gram(Q, r, Z, e, P);
            GemmPass gp;
            gp.A = Q;
            gp.lda = n;
            gp.M = n;
            gp.K = r;
            gp.ncols = e;
            gp.alpha = -1.0;
            gp.in = ColMap::plain(P, r);
            gp.out = ColMap::plain(Z, n);
            gp.add = ColMap::plain(Z, n);
            gemm_nn(&gp, 1, nullptr, st);
        }
        if (!c.orth(Z, e, Q + n * r, nullptr, nullptr, c.buf(P_Q1, n * m)))
            throw NumericalError("clustered_spectrum: completion basis breakdown");
        W4_CUDA(cudaStreamSynchronize(st));  // hz is released on return
    }
    // Y = C^T A C Q (spectrum.cpp:48-55), C = I - U T U^T (compact WY)
    auto apply_lmp = [&](const double* X, double* out, bool transpose) {
        double* G1 = c.buf(P_TMP, 2 * (size_t)k * m);
        double* G2 = G1 + k * m;
        c.gram(U, k, X, m, G1);  // U^T X
        small_gemm(transpose, false, (int)k, (int)m, (int)k, 1.0, T, (int)k, G1, (int)k, 0.0, G2, (int)k, st);
        GemmPass gp;
        gp.A = U;
        gp.lda = n;
        gp.M = n;
        gp.K = k;
        gp.ncols = m;
        gp.alpha = -1.0;
        gp.in = ColMap::plain(G2, k);
        gp.out = ColMap::plain(out, n);
        gp.add = ColMap::plain(X, n);
        gemm_nn(&gp, 1, nullptr, st);
    };
    double* V1 = c.buf(P_F, n * m);
    const double* CQ = Q;
    if (k) {
        apply_lmp(Q, V1, false);
        CQ = V1;
    }
    double* AV = c.buf(P_AZ, n * m);
    c.apply(CQ, m, AV);
    const double* Y = AV;
    if (k) {
        apply_lmp(AV, V1, true);
        Y = V1;
    }
    // K = sym(Q^T Y), eigenvalues decreasing (spectrum.cpp:56-62)
    double* K = c.buf(P_K, m * m);
    c.gram(Q, m, Y, m, K);
    double* Wv = c.buf(P_W, m * m);
    sym_evd_desc((int)m, K, vals_out, Wv, c.pool[P_SMALLWS], st);
}

void rayleigh_ritz_dev(wc4dvar_op& op, const double* Z, int64_t ldz, int64_t m, double* U_out,
                       int64_t ldu, double* theta_out, cudaStream_t st) {
    require(ldz == op.dim, "rayleigh_ritz: Z must be contiguous (ld = dim)");
    Timer tm(st, false);
    Ctx c{op, st, op.dim, tm, op.pool, op.h_int};
    rr_core(c, Z, m, m, U_out, ldu, theta_out, c.buf(P_AZ, op.dim * m));
}

int64_t sketch_dev(wc4dvar_op& op, const wc4dvar_sketch_config& cfg, const double* omega,
                   double* U_out, int64_t ldu, double* theta_out, cudaStream_t st,
                   SketchTiming* timing) {
    const int64_t n = op.dim;
    // SketchConfig::validate, randevd.cpp:10-14
    require(cfg.target_rank >= 1, "SketchConfig: target rank must be >= 1");
    require(cfg.oversample >= 0, "SketchConfig: oversampling must be >= 0");
    const int64_t k = cfg.target_rank;
    const int64_t m = k + cfg.oversample;
    require(m <= n, "SketchConfig: k + l exceeds operator dimension");
    require(m <= 512, "sketch: k + l above 512 is not supported by the device small-matrix kernels");
    Timer tm(st, timing != nullptr);
    Ctx c{op, st, n, tm, op.pool, op.h_int};
    int64_t produced = 0;

    // Memory plan (SURVEY §7 hard part 7): besides the caller's Omega and U and the
    // operator's apply workspace, a sketch holds TWO n x m blocks (bufA, bufB): the
    // orthonormalisations run with Q aliasing their input and the other block as scratch,
    // and each block product writes into whichever block is dead.  C4 at m = 256:
    // Omega + 2 blocks + workspace + U = 4.5 x 34.8 GB.
    double* bufA = c.buf(P_Y, n * m);
    double* bufB = c.buf(P_Z, n * m);
    if (cfg.method == WC4DVAR_SKETCH_REVD) {
        // randevd.cpp:62-80
        double* Y = bufA;
        c.apply(omega, m, Y);
        tm.begin(T_GEMM);
        double* G = c.buf(P_G, m * m);
        c.gram(Y, m, Y, m, G);
        int* perm = nullptr;
        const int r = c.rank_probe(G, m, &perm, Y);
        if (r < m) {
            std::ostringstream msg;
            msg << "revd: sample matrix rank collapsed to " << r << " of " << m << " columns";
            throw NumericalError(msg.str());
        }
        // Z = householder_q(Y) only enters through A Z = (A Y) R^{-1} (A is linear), K = Z^T A Z =
        // R^{-T} (Y^T A Y) R^{-1} and U = Z W = Y (R^{-1} W): when one CholQR pass suffices
        // (cond(Y) <= 4) Z is never formed and the second block product runs on Y itself.
        double* Rl = c.buf(P_RA, m * m);
        double* Rli = c.buf(P_RB, m * m);
        if (c.orth_factored(Y, m, Rl, Rli, G)) {
            double* AY = bufB;
            c.apply(Y, m, AY);  // second block product
            tm.begin(T_GEMM);
            double* Kraw = c.buf(P_G2, m * m);
            c.gram(Y, m, AY, m, Kraw, true);  // Y^T A Y, A symmetric
            tm.begin(T_SMALL);
            double* T1 = c.buf(P_R, m * m);
            double* K = c.buf(P_K, m * m);
            small_gemm(false, false, (int)m, (int)m, (int)m, 1.0, Kraw, (int)m, Rli, (int)m, 0.0, T1, (int)m, st);
            small_gemm(true, false, (int)m, (int)m, (int)m, 1.0, Rli, (int)m, T1, (int)m, 0.0, K, (int)m, st);
            double* vals = c.buf(P_VALS, m);
            double* W = c.buf(P_W, m * m);
            sym_evd_desc((int)m, K, vals, W, c.pool[P_SMALLWS], st);
            double* S = c.buf(P_G2, m * m);
            small_gemm(false, false, (int)m, (int)k, (int)m, 1.0, Rli, (int)m, W, (int)m, 0.0, S, (int)m, st);
            tm.begin(T_GEMM);
            c.tall_times_small(Y, m, S, m, k, U_out, ldu);
            W4_CUDA(cudaMemcpyAsync(theta_out, vals, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
            tm.end();
            tm.collect(timing);
            return k;
        }
        double* Z = bufA;  // householder_q(Y), randevd.cpp:74
        if (!c.orth(Y, m, Z, nullptr, G, bufB))
            throw NumericalError("revd: sample matrix is numerically rank deficient (CholQR breakdown)");
        rr_core(c, Z, m, k, U_out, ldu, theta_out, bufB, /*check_z=*/false);
        produced = k;
    } else if (cfg.method == WC4DVAR_SKETCH_NYSTROM) {
        // randevd.cpp:82-114
        double* Y = bufA;
        c.apply(omega, m, Y);
        tm.begin(T_GEMM);
        double* G = c.buf(P_G, m * m);
        c.gram(Y, m, Y, m, G);
        int* perm = nullptr;
        const int r = c.rank_probe(G, m, &perm, Y);
        if (r == 0) throw NumericalError("nystrom: sample matrix is zero");
        double* Z = bufA;
        double* other = bufB;
        if (r < m) {  // the r pivot columns span the kept subspace (randevd.cpp:89-92)
            gather_cols(n, r, Y, n, perm, bufB, n, st);
            Z = bufB;
            other = bufA;
        }
        // Full rank and one CholQR pass (cond(Y) <= 4): Z = Y R^{-1} is never formed; E1 = A Z =
        // (A Y) R^{-1} stays lazy (the block holds A Y), E2 = Z^T E1 = R^{-T} (Y^T A Y) R^{-1}, and
        // the pending R^{-1} joins U^{-1} in the one product that forms F.
        double* Rl = c.buf(P_RA, m * m);
        double* Rli = c.buf(P_RB, m * m);
        const bool lazy = r == m && c.orth_factored(Y, m, Rl, Rli, G);
        if (!lazy && !c.orth(Z, r, Z, nullptr, r < m ? nullptr : G, other))
            throw NumericalError("nystrom: sample matrix is numerically rank deficient (CholQR breakdown)");
        double* E1 = other;
        c.apply(Z, r, E1);
        tm.begin(T_GEMM);
        double* E2 = c.buf(P_K, r * r);
        if (lazy) {
            double* E2raw = c.buf(P_G2, r * r);
            double* T1 = c.buf(P_R, r * r);
            c.gram(Z, r, E1, r, E2raw, true);  // Y^T A Y, A symmetric
            small_gemm(false, false, (int)r, (int)r, (int)r, 1.0, E2raw, (int)r, Rli, (int)r, 0.0, T1, (int)r, st);
            small_gemm(true, false, (int)r, (int)r, (int)r, 1.0, Rli, (int)r, T1, (int)r, 0.0, E2, (int)r, st);
        } else {
            c.gram(Z, r, E1, r, E2);
        }
        tm.begin(T_SMALL);
        double* Ru = c.buf(P_R1, r * r);
        double* Rui = c.buf(P_R1I, r * r);
        int* info = reinterpret_cast<int*>(c.buf(P_INT, 4 + 2 * m));
        chol_inv_upper((int)r, E2, Ru, Rui, info, op.pool[P_SMALLWS], st);  // sym(E2), randevd.cpp:96-97
        if (c.read_int(info))
            throw NumericalError(
                "nystrom: Cholesky of Z^T A Z failed; the projected operator is numerically "
                "indefinite. Increase the oversampling parameter or use revd for indefinite "
                "spectra.");
        tm.begin(T_GEMM);
        double* F = Z;  // Z is dead once E2 exists
        const double* Fi = Rui;
        if (lazy) {  // F = (A Y) (R^{-1} U^{-1}): upper triangular times upper triangular
            double* T2 = c.buf(P_G2, r * r);
            small_gemm(false, false, (int)r, (int)r, (int)r, 1.0, Rli, (int)r, Rui, (int)r, 0.0, T2, (int)r, st);
            Fi = T2;
        }
        c.tall_times_small(E1, r, Fi, r, r, F, n, true);  // F = E1 U^{-1}, randevd.cpp:104-105
        double* RF = c.buf(P_R, r * r);
        // BDCSVD(F) = Q_F (U_R S V^T) with F = Q_F R_F: when one CholQR pass suffices Q_F is never
        // formed, U = Q_F W = F (R_F^{-1} W)
        double* RFi = c.buf(P_TMP, r * r);
        const bool factored = c.orth_factored(F, r, RF, RFi);
        if (!factored && !c.orth(F, r, F, RF, c.factored_gram, E1))
            throw NumericalError("nystrom: factor F is numerically rank deficient (CholQR breakdown)");
        tm.begin(T_SMALL);
        double* sig = c.buf(P_VALS, r);
        double* W = c.buf(P_W, r * r);
        svd_left_desc((int)r, RF, sig, W, op.pool[P_SMALLWS], st);
        const int64_t keep = std::min<int64_t>(k, r);
        const double* Wf = W;
        if (factored) {
            double* S = c.buf(P_K, r * r);  // E2 is dead
            small_gemm(false, false, (int)r, (int)keep, (int)r, 1.0, RFi, (int)r, W, (int)r, 0.0, S, (int)r, st);
            Wf = S;
        }
        tm.begin(T_GEMM);
        c.tall_times_small(F, r, Wf, r, keep, U_out, ldu);
        square_head_kernel<<<1, 512, 0, st>>>((int)keep, sig, theta_out);
        W4_LAUNCH();
        tm.end();
        produced = keep;
    } else if (cfg.method == WC4DVAR_SKETCH_RITZIT) {
        // randevd.cpp:116-136 (+ p_iter EXTENSION)
        double* G3 = bufA;
        double* Y3 = bufB;
        // Omega = Q R_o.  With one subspace iteration and a sample that needs one CholQR pass
        // (cond(Omega) ~ 1.01) Q is never formed: A is linear, so Y3 = A Q = (A Omega) R_o^{-1}; the
        // block holds A Omega and the m x m factor R_o^{-1} stays pending ("lazy") until the end.
        double* Ro = c.buf(P_RA, m * m);
        double* Roi = c.buf(P_RB, m * m);
        bool lazy = std::max(cfg.p_iter, 1) == 1 && c.orth_factored(omega, m, Ro, Roi);
        if (lazy) {
            c.apply(omega, m, Y3);
        } else {
            if (!c.orth(omega, m, G3, nullptr, c.factored_gram, bufB))
                throw NumericalError("revd_ritzit: Gaussian sample is numerically rank deficient");
            c.apply(G3, m, Y3);
        }
        for (int it = 1; it < std::max(cfg.p_iter, 1); ++it) {
            if (!c.orth(Y3, m, Y3, nullptr, nullptr, G3))
                throw NumericalError("revd_ritzit: QR of the sample matrix is rank deficient");
            std::swap(G3, Y3);  // the basis now lives in the old Y3 block
            c.apply(G3, m, Y3);
        }
        double* Z3 = Y3;
        double* R3 = c.buf(P_R, m * m);
        // U = Z3 W with Y3 = Z3 R3: when one CholQR pass suffices Z3 is never formed, U = Y3 (R3^{-1} W)
        double* R3i = c.buf(P_TMP, m * m);
        bool factored = false;
        if (lazy) {
            // Gram of Y3 = (A Omega) R_o^{-1} from the Gram of the block: R_o^{-T} (A Omega)^T (A Omega) R_o^{-1}
            tm.begin(T_ORTH);
            double* Gy = c.buf(P_G, m * m);
            c.gram(Y3, m, Y3, m, Gy);
            double* T1 = c.buf(P_K, m * m);
            small_gemm(false, false, (int)m, (int)m, (int)m, 1.0, Gy, (int)m, Roi, (int)m, 0.0, T1, (int)m, st);
            small_gemm(true, false, (int)m, (int)m, (int)m, 1.0, Roi, (int)m, T1, (int)m, 0.0, Gy, (int)m, st);
            double* R1 = c.buf(P_R1, m * m);
            double* R1i = c.buf(P_R1I, m * m);
            int* info = reinterpret_cast<int*>(c.buf(P_INT, 4 + 2 * m));
            chol_inv_upper((int)m, Gy, R1, R1i, info, op.pool[P_SMALLWS], st);
            factored = !c.read_int(info) && c.single_pass_ok(R1, m);
            if (factored) {  // Y3 = Z3 R3 with R3 = R1; pending factor R_o^{-1} R1^{-1}
                ++c.single_pass_calls;
                W4_CUDA(cudaMemcpyAsync(R3, R1, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
                small_gemm(false, false, (int)m, (int)m, (int)m, 1.0, Roi, (int)m, R1i, (int)m, 0.0, R3i, (int)m, st);
                tm.end();
            } else {  // materialise Y3 = (A Omega) R_o^{-1} and take the general route
                tm.end();
                tm.begin(T_GEMM);
                c.tall_times_small(Y3, m, Roi, m, m, G3, n, true);
                tm.end();
                std::swap(G3, Y3);
                Z3 = Y3;
                lazy = false;
            }
        }
        if (!lazy) {
            factored = c.orth_factored(Y3, m, R3, R3i);
            if (!factored && !c.orth(Y3, m, Z3, R3, c.factored_gram, G3))
                throw NumericalError("revd_ritzit: QR of the sample matrix is rank deficient");
        }
        // min |R_ii| <= 1e-14 max |R_ii| (randevd.cpp:125-127)
        std::vector<double> hR(m * m);
        W4_CUDA(cudaMemcpyAsync(hR.data(), R3, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        double dmin = INFINITY, dmax = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            dmin = std::min(dmin, std::fabs(hR[i + i * m]));
            dmax = std::max(dmax, std::fabs(hR[i + i * m]));
        }
        if (dmin <= 1e-14 * dmax)
            throw NumericalError("revd_ritzit: QR of the sample matrix is rank deficient");
        tm.begin(T_SMALL);
        double* K = c.buf(P_K, m * m);
        small_gemm(false, true, (int)m, (int)m, (int)m, 1.0, R3, (int)m, R3, (int)m, 0.0, K, (int)m,
                   st);  // R3 R3^T
        double* vals = c.buf(P_VALS, m);
        double* W = c.buf(P_W, m * m);
        sym_evd_desc((int)m, K, vals, W, op.pool[P_SMALLWS], st);
        double hv = 0;
        W4_CUDA(cudaMemcpyAsync(&hv, vals + (std::min(k, m) - 1), sizeof(double),
                                cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        if (hv <= 0.0) throw NumericalError("revd_ritzit: nonpositive squared Ritz value");
        const double* Wf = W;
        if (factored) {
            double* S = c.buf(P_G2, m * m);
            small_gemm(false, false, (int)m, (int)k, (int)m, 1.0, R3i, (int)m, W, (int)m, 0.0, S, (int)m, st);
            Wf = S;
        }
        tm.begin(T_GEMM);
        c.tall_times_small(Z3, m, Wf, m, k, U_out, ldu);
        sqrt_head_kernel<<<1, 512, 0, st>>>((int)k, vals, theta_out);
        W4_LAUNCH();
        tm.end();
        produced = k;
    } else {
        throw InvalidArgument("sketch_eigenpairs: unknown method");
    }
    tm.collect(timing);
    return produced;
}

}  // namespace w4
