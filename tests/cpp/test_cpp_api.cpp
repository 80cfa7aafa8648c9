// The C++ host side (include/wc4dvar_gpu.hpp) driven the way the reference's doctest suites
// drive wc4dvar (test_operators.cpp, test_randevd.cpp, test_lmp.cpp, test_krylov.cpp,
// test_models.cpp), with the CPU oracle (oracle/liboracle.so, test infrastructure) as the
// parity checker for the Hessian apply.  Built and run by tests/test_gpu_cpp_api.py:
//   g++ -std=c++17 -Iinclude tests/cpp/test_cpp_api.cpp -Lpaper_2101_07249_b200 -lwc4dvar_gpu
//       -Loracle -loracle
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "wc4dvar_gpu.hpp"

using namespace wc4dvar_gpu;

// ---- the oracle's C interface (oracle/wc4dvar_oracle.c) ------------------------------------
extern "C" {
typedef struct {
    int model;
    int64_t n;
    int N;
    int substeps;
    double courant, diffusion, dt;
    const double* stages;
    int n_times;
    const int* times;
    int n_points;
    const int* points;
    int cov_kind;
    const double *b_half, *b_half_inv, *q_half, *q_half_inv;
    double sigma_obs;
} orc_hessian;
int orc_hessian_apply_block(const orc_hessian* h, int64_t m, const double* V, double* out, int threads);
void orc_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);
}

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                      \
    } while (0)
template <class E, class F>
static bool throws_as(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double d = 0.0, s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        d = std::fmax(d, std::fabs(a[i] - b[i]));
        s = std::fmax(s, std::fabs(b[i]));
    }
    return d / s;
}

// symmetric circulant square root from a SOAR first column, by a naive real DFT (small n)
static CovarianceFactor circulant_soar_sqrt(int n, double sigma, double L) {
    const double pi = 3.14159265358979323846;
    std::vector<double> c(n), lam(n);
    for (int j = 0; j < n; ++j) {  // covariance.cpp:36-41 chordal distance
        const int d = std::min(j, n - j);
        const double r = (n / pi) * std::sin(pi * d / n);
        c[j] = sigma * sigma * (1.0 + r / L) * std::exp(-r / L);
    }
    for (int k = 0; k < n; ++k) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += c[j] * std::cos(2.0 * pi * j * k / n);
        lam[k] = s;
    }
    CovarianceFactor f;
    f.kind = WC4DVAR_COV_CIRCULANT;
    f.half.assign(n, 0.0);
    f.half_inv.assign(n, 0.0);
    for (int j = 0; j < n; ++j) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < n; ++k) {
            const double w = std::cos(2.0 * pi * j * k / n) / n;
            a += std::sqrt(lam[k]) * w;
            b += w / std::sqrt(lam[k]);
        }
        f.half[j] = a;
        f.half_inv[j] = b;
    }
    return f;
}

static void test_network() {  // test_models.cpp:167-179
    const ObservationNetwork net = ObservationNetwork::build(8, 7, 2, 3);
    CHECK((net.times == std::vector<int32_t>{1, 4, 7}));
    CHECK(net.q == 12);
    CHECK(throws_as<std::invalid_argument>([] { ObservationNetwork::build(8, 7, 9, 1); }));
}

static void test_hessian_vs_oracle() {
    const int n = 40, N = 10;
    LinearizedModel model;
    model.kind = WC4DVAR_MODEL_ADVECTION;
    model.n = n;
    model.N = N;
    model.courant = 0.8;
    const ObservationNetwork net = ObservationNetwork::build(n, N, 4, 2);
    const CovarianceFactor b = circulant_soar_sqrt(n, 1.0, 3.0), q = circulant_soar_sqrt(n, 0.3, 3.0);
    HessianOperator op(model, net, b, q, 0.1);
    CHECK(op.dim() == n * (N + 1));
    // n = 40 has no fused transform: the Fourier-space form is not eligible and cannot be forced
    CHECK(!op.spectral());
    bool refused = false;
    try {
        op.spectral(1);
    } catch (const std::invalid_argument&) {
        refused = true;
    }
    CHECK(refused);
    const Index m = 5;
    Matrix V(op.dim(), m);
    orc_gaussian_matrix(op.dim(), m, 7, V.data());
    op.reset_apply_count();
    const Matrix AV = op.apply_block(V);
    CHECK(op.apply_count() == m);  // count(m) per block (operators.cpp:9-19)
    orc_hessian h{};
    h.model = 1;
    h.n = n;
    h.N = N;
    h.substeps = 1;
    h.courant = 0.8;
    std::vector<int> times(net.times.begin(), net.times.end()), points(net.points.begin(), net.points.end());
    h.n_times = (int)times.size();
    h.times = times.data();
    h.n_points = (int)points.size();
    h.points = points.data();
    h.cov_kind = 1;
    h.b_half = b.half.data();
    h.b_half_inv = b.half_inv.data();
    h.q_half = q.half.data();
    h.q_half_inv = q.half_inv.data();
    h.sigma_obs = 0.1;
    Matrix ref(op.dim(), m);
    CHECK(orc_hessian_apply_block(&h, m, V.data(), ref.data(), 4) == 0);
    CHECK(max_rel(AV.data_, ref.data_) <= 1e-13);
    // block apply == column-wise apply, bitwise (test_operators.cpp:188-209)
    Vector col;
    op.apply(V.col(2), col);
    CHECK(col == AV.col(2));
    CHECK(op.apply_count() == m + 1);
    // pieces: L^{-1} then L^{-T} adjoint identity (test_operators.cpp:91-120)
    const Vector p = V.col(0), v = V.col(1);
    const Vector Lp = op.apply_Linv(p), LTv = op.apply_LinvT(v);
    double a = 0.0, c = 0.0;
    for (Index i = 0; i < op.dim(); ++i) {
        a += Lp[i] * v[i];
        c += p[i] * LTv[i];
    }
    CHECK(std::fabs(a - c) <= 1e-12 * (1.0 + std::fabs(a)));
    // error types: bad construction, non-finite input (operators.cpp:133-143)
    CHECK(throws_as<std::invalid_argument>([&] { HessianOperator bad(model, net, b, q, -1.0); }));
    Vector nan_in = V.col(0), out;
    nan_in[3] = std::nan("");
    CHECK(throws_as<NumericalError>([&] { op.apply(nan_in, out); }));
    // clustered spectrum without a preconditioner: the unit cluster is n_A - q
    const ClusteredSpectrum cs = clustered_spectrum(op);
    CHECK(cs.unit_multiplicity == op.dim() - net.q);
    CHECK(cs.min_eigenvalue() >= 1.0 - 1e-12);
    // QuadraticCost recorded every PCG iteration (record_cost, assimilation.hpp:112,
    // assimilation.cpp:235): the cost of the CG iterates never increases (test_krylov.cpp:100-115)
    Vector bg((size_t)op.dim()), d((size_t)net.q);
    orc_gaussian_matrix(op.dim(), 1, 21, bg.data());
    orc_gaussian_matrix(net.q, 1, 22, d.data());
    const QuadraticCost J(op, bg, d);
    PcgOptions co;
    co.max_iter = 40;
    co.rel_tol = 1e-10;
    co.cost_eval = &J;
    const PcgResult pr = pcg_split(op, J.rhs(), nullptr, {}, co);
    CHECK(pr.history.quadratic_costs.size() == (size_t)pr.history.iterations + 1);
    bool mono = true;
    for (size_t j = 1; j < pr.history.quadratic_costs.size(); ++j)
        mono = mono && pr.history.quadratic_costs[j] <= pr.history.quadratic_costs[j - 1] * (1 + 1e-12);
    CHECK(mono);
    CHECK(std::fabs(J(pr.x) - pr.history.quadratic_costs.back()) <= 1e-12 * std::fabs(J(pr.x)));
    CHECK(throws_as<std::invalid_argument>([&] { QuadraticCost bad(op, bg, Vector(3)); }));
}

static void test_sketches_and_pcg() {
    const Index n = 60;
    // identity operator: every method returns theta = 1 (test_randevd.cpp:82-95), with the
    // reference's apply counts {2m, 2m, m} (test_randevd.cpp:186-206)
    Matrix I(n, n);
    for (Index i = 0; i < n; ++i) I(i, i) = 1.0;
    DenseOperator eye(I);
    for (SketchMethod meth : {SketchMethod::Revd, SketchMethod::Nystrom, SketchMethod::Ritzit}) {
        SketchConfig cfg;
        cfg.target_rank = 4;
        cfg.oversample = 6;
        cfg.seed = 3;
        cfg.method = meth;
        eye.reset_apply_count();
        const RitzPairs p = sketch_eigenpairs(eye, cfg);
        CHECK(p.k() == 4);
        for (int i = 0; i < 4; ++i) CHECK(std::fabs(p.values[i] - 1.0) <= 1e-12);
        CHECK(p.orthonormality_defect() <= 1e-10);
        CHECK(eye.apply_count() == (meth == SketchMethod::Ritzit ? 10 : 20));
    }
    SketchConfig bad;
    bad.target_rank = 0;
    CHECK(throws_as<std::invalid_argument>([&] { sketch_eigenpairs(eye, bad); }));
    // Nystrom on a rank-3 PSD operator caps k at the rank and recovers it exactly
    // (test_randevd.cpp:153-168)
    Matrix R3(n, n);
    R3(0, 0) = 50.0;
    R3(1, 1) = 20.0;
    R3(2, 2) = 10.0;
    DenseOperator rank3(R3);
    SketchConfig ny;
    ny.target_rank = 6;
    ny.oversample = 4;
    ny.method = SketchMethod::Nystrom;
    const RitzPairs p3 = sketch_eigenpairs(rank3, ny);
    CHECK(p3.k() == 3);
    CHECK(p3.k() == 3 && std::fabs(p3.values[0] - 50.0) <= 1e-10 * 50.0 &&
          std::fabs(p3.values[2] - 10.0) <= 1e-10 * 10.0);
    // Lanczos on A = diag(50, 20, 10, 5, 1, ...) (krylov.cpp:178-278)
    Matrix A(n, n);
    const double top[4] = {50.0, 20.0, 10.0, 5.0};
    for (Index i = 0; i < n; ++i) A(i, i) = i < 4 ? top[i] : 1.0;
    DenseOperator op(A);
    LanczosOptions lo;
    lo.tol = 1e-12;
    const RitzPairs lz = lanczos_eigenpairs(op, 4, lo);
    for (int i = 0; i < 4; ++i) CHECK(std::fabs(lz.values[i] - top[i]) <= 1e-9 * top[i]);
    // the LMP of the exact top pairs is a perfect preconditioner here (C^T A C = I):
    // PCG converges in one iteration (test_krylov.cpp:43-55)
    auto lmp = build_spectral_lmp(lz);
    Vector b(n, 0.0);
    b[0] = 1.0;
    b[2] = -2.0;
    b[10] = 0.5;
    PcgOptions opts;
    opts.max_iter = 50;
    opts.rel_tol = 1e-8;
    const PcgResult none = pcg_split(op, b, nullptr, {}, opts);
    const PcgResult pre = pcg_split(op, b, lmp.get(), {}, opts);
    CHECK(none.history.converged && pre.history.converged);
    CHECK(pre.history.iterations == 1 && none.history.iterations > 1);
    Vector Ax;
    op.apply(pre.x, Ax);
    double r = 0.0, nb = 0.0;
    for (Index i = 0; i < n; ++i) {
        r += (Ax[i] - b[i]) * (Ax[i] - b[i]);
        nb += b[i] * b[i];
    }
    CHECK(std::sqrt(r / nb) <= 1e-8);
    // C^T = C for the spectral LMP (test_lmp.cpp:93-110)
    const Vector u = lmp->apply(b), ut = lmp->apply_transpose(b);
    CHECK(max_rel(u, ut) <= 1e-13);
}

int main() {
    std::printf("%s\n", wc4dvar_gpu_version());
    test_network();
    test_hessian_vs_oracle();
    test_sketches_and_pcg();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
