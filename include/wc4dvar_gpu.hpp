// C++ host side above the C-ABI: the reference's operator / sketch / LMP / PCG interface
// (proj/include/wc4dvar/{operators,randevd,ritz,lmp,krylov,spectrum}.hpp) with the same names,
// argument meaning and exception types, over libwc4dvar_gpu.so.  Header-only; the dense
// types are plain column-major std::vector<double> (Eigen's MatrixXd layout) so it compiles
// without Eigen -- a reference build swaps them for Eigen::VectorXd / MatrixXd.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "wc4dvar_gpu.h"

namespace wc4dvar_gpu {

using Index = std::int64_t;
using Vector = std::vector<double>;

// Column-major dense matrix (types.hpp:9-11 layout).
struct Matrix {
    Index rows_ = 0, cols_ = 0;
    std::vector<double> data_;
    Matrix() = default;
    Matrix(Index r, Index c) : rows_(r), cols_(c), data_((size_t)(r * c), 0.0) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    double& operator()(Index i, Index j) { return data_[(size_t)(i + j * rows_)]; }
    double operator()(Index i, Index j) const { return data_[(size_t)(i + j * rows_)]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    Vector col(Index j) const { return Vector(data_.begin() + j * rows_, data_.begin() + (j + 1) * rows_); }
};

// types.hpp:14-30
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DenseCapError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == WC4DVAR_OK) return;
    const std::string msg = wc4dvar_gpu_last_error();
    switch (rc) {
        case WC4DVAR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case WC4DVAR_NUMERICAL: throw NumericalError(msg);
        case WC4DVAR_DENSE_CAP: throw DenseCapError(msg);
        default: throw DeviceError(msg);
    }
}

// ---------------------------------------------------------------- operators.hpp
class LinearOperator {
public:
    virtual ~LinearOperator() {
        if (h_) wc4dvar_gpu_op_destroy(h_);
    }
    LinearOperator(const LinearOperator&) = delete;
    LinearOperator& operator=(const LinearOperator&) = delete;
    Index dim() const { return wc4dvar_gpu_op_dim(h_); }
    void apply(const Vector& v, Vector& out) const {
        if ((Index)v.size() != dim()) throw std::invalid_argument("LinearOperator::apply: dimension mismatch");
        out.resize(v.size());
        check(wc4dvar_gpu_op_apply(h_, v.data(), out.data()));
    }
    Matrix apply_block(const Matrix& V) const {
        Matrix out(V.rows(), V.cols());
        check(wc4dvar_gpu_op_apply_block(h_, V.data(), V.rows(), V.cols(), out.data(), V.rows()));
        return out;
    }
    long apply_count() const { return (long)wc4dvar_gpu_op_apply_count(h_); }
    void reset_apply_count() { wc4dvar_gpu_op_reset_apply_count(h_); }
    wc4dvar_op* handle() const { return h_; }

protected:
    LinearOperator() = default;
    wc4dvar_op* h_ = nullptr;
};

// operators.hpp:42-53
class DenseOperator : public LinearOperator {
public:
    explicit DenseOperator(const Matrix& A, int device = 0) {
        if (A.rows() != A.cols()) throw std::invalid_argument("DenseOperator: matrix must be square");
        check(wc4dvar_gpu_dense_create(A.rows(), A.data(), A.rows(), device, &h_));
    }
};

// models.hpp:45-56 / models.cpp:159-176
struct ObservationNetwork {
    int n = 0, N = 0, space_stride = 1, time_stride = 1;
    std::vector<int32_t> times, points;
    int q = 0;
    static ObservationNetwork build(int n, int N, int space_stride, int time_stride) {
        if (n < 1 || N < 1) throw std::invalid_argument("ObservationNetwork: grid must be nonempty");
        if (space_stride < 1 || space_stride > n)
            throw std::invalid_argument("ObservationNetwork: space stride inconsistent with grid");
        if (time_stride < 1 || time_stride > N)
            throw std::invalid_argument("ObservationNetwork: time stride inconsistent with window");
        ObservationNetwork net;
        net.n = n;
        net.N = N;
        net.space_stride = space_stride;
        net.time_stride = time_stride;
        for (int t = N; t >= 1; t -= time_stride) net.times.insert(net.times.begin(), t);
        for (int j = 0; j < n; j += space_stride) net.points.push_back(j);
        net.q = (int)(net.times.size() * net.points.size());
        return net;
    }
};

// covariance.hpp:31-38 (dense) plus the circulant representation (first columns)
struct CovarianceFactor {
    int kind = WC4DVAR_COV_DENSE;
    Vector half, half_inv;  // dense: n x n col-major; circulant: n
};

// operators.hpp:57-111 (+ the BASELINE extensions: adv-diff, sub-steps)
struct LinearizedModel {
    int kind = WC4DVAR_MODEL_IDENTITY;
    Index n = 0;
    int N = 0, substeps = 1;
    double courant = 0.0, diffusion = 0.0, dt = 0.0, forcing = 8.0;
    Matrix trajectory;  // Lorenz-96: n x (N substeps + 1); stages are built on the device
};

// operators.hpp:116-152
class HessianOperator : public LinearOperator {
public:
    HessianOperator(const LinearizedModel& model, const ObservationNetwork& net, const CovarianceFactor& b_half,
                    const CovarianceFactor& q_half, double sigma_obs, int device = 0)
        : net_(net), sigma_obs_(sigma_obs) {
        wc4dvar_model_desc md{};
        md.kind = model.kind;
        md.N = model.N;
        md.n = model.n;
        md.substeps = model.substeps;
        md.courant = model.courant;
        md.diffusion = model.diffusion;
        md.dt = model.dt;
        md.forcing = model.forcing;
        if (model.kind == WC4DVAR_MODEL_LORENZ96) {
            md.trajectory = model.trajectory.data();
            md.ld_trajectory = model.trajectory.rows();
        }
        wc4dvar_network_desc nd{};
        nd.n = net.n;
        nd.N = net.N;
        nd.n_times = (int32_t)net.times.size();
        nd.times = net.times.data();
        nd.n_points = (int32_t)net.points.size();
        nd.points = net.points.data();
        wc4dvar_cov_desc b{b_half.kind, 0, b_half.half.data(), b_half.half_inv.empty() ? nullptr : b_half.half_inv.data()};
        wc4dvar_cov_desc q{q_half.kind, 0, q_half.half.data(), q_half.half_inv.empty() ? nullptr : q_half.half_inv.data()};
        check(wc4dvar_gpu_hessian_create(&md, &nd, &b, &q, sigma_obs, device, &h_));
    }
    const ObservationNetwork& network() const { return net_; }
    double sigma_obs() const { return sigma_obs_; }
    // Fourier-space form of apply / apply_block (wc4dvar_gpu_op_spectral): mode 1 / 0 switches it
    // on / off, -1 queries; returns whether it is active (an execution strategy, same result).
    bool spectral(int mode = -1) {
        int active = 0;
        check(wc4dvar_gpu_op_spectral(h_, mode, &active));
        return active != 0;
    }
    // operators.hpp:127-135 (not counted as applies, as in the reference)
    Vector apply_Linv(const Vector& p) const { return piece(WC4DVAR_LINV, p); }
    Vector apply_LinvT(const Vector& v) const { return piece(WC4DVAR_LINVT, v); }
    Vector apply_D_half(const Vector& v) const { return piece(WC4DVAR_D_HALF, v); }
    Vector apply_D_half_inv(const Vector& v) const { return piece(WC4DVAR_D_HALF_INV, v); }
    // operators.cpp:146-154
    Matrix observation_range() const {
        Matrix W(dim(), net_.q);
        check(wc4dvar_gpu_observation_range(h_, W.data(), dim()));
        return W;
    }

private:
    Vector piece(int which, const Vector& v) const {
        Vector out(v.size());
        check(wc4dvar_gpu_hessian_piece(h_, which, v.data(), (Index)v.size(), 1, out.data(), (Index)v.size()));
        return out;
    }
    ObservationNetwork net_;
    double sigma_obs_;
};

// ---------------------------------------------------------------- randevd.hpp / ritz.hpp
enum class SketchMethod { Revd = WC4DVAR_SKETCH_REVD, Nystrom = WC4DVAR_SKETCH_NYSTROM, Ritzit = WC4DVAR_SKETCH_RITZIT };

struct SketchConfig {  // randevd.hpp:13-21
    Index target_rank = 10;
    Index oversample = 5;
    std::uint64_t seed = 1;
    SketchMethod method = SketchMethod::Revd;
    int p_iter = 1;  // ritzit EXTENSION
};

struct RitzPairs {  // ritz.hpp:9-27
    Matrix vectors;  // n x k, orthonormal columns
    Vector values;   // k, decreasing
    Index k() const { return (Index)values.size(); }
    double orthonormality_defect() const {
        double d = 0.0;
        for (Index i = 0; i < k(); ++i)
            for (Index j = 0; j < k(); ++j) {
                double s = 0.0;
                for (Index r = 0; r < vectors.rows(); ++r) s += vectors(r, i) * vectors(r, j);
                d = std::fmax(d, std::fabs(s - (i == j ? 1.0 : 0.0)));
            }
        return d;
    }
};

// randevd.cpp:138-148 (omega: dim x (k + l), or empty to draw gaussian_matrix(seed))
inline RitzPairs sketch_eigenpairs(const LinearOperator& op, const SketchConfig& cfg, const Matrix* omega = nullptr) {
    wc4dvar_sketch_config c{(int32_t)cfg.target_rank, (int32_t)cfg.oversample, cfg.seed, (int32_t)cfg.method,
                            cfg.p_iter};
    RitzPairs p;
    p.vectors = Matrix(op.dim(), cfg.target_rank);
    p.values.assign((size_t)cfg.target_rank, 0.0);
    int64_t k = 0;
    check(wc4dvar_gpu_sketch(op.handle(), &c, omega ? omega->data() : nullptr, p.vectors.data(), op.dim(),
                             p.values.data(), &k));
    p.values.resize((size_t)k);
    p.vectors.cols_ = k;
    p.vectors.data_.resize((size_t)(op.dim() * k));
    return p;
}

// ---------------------------------------------------------------- lmp.hpp
class LmpFactor {  // lmp.hpp:12-26, compact-WY on the device
public:
    LmpFactor(const RitzPairs& pairs, int device = 0) : n_(pairs.vectors.rows()), k_(pairs.k()) {
        check(wc4dvar_gpu_lmp_build(n_, k_, pairs.vectors.data(), n_, pairs.values.data(), device, &h_));
    }
    ~LmpFactor() {
        if (h_) wc4dvar_gpu_lmp_destroy(h_);
    }
    LmpFactor(const LmpFactor&) = delete;
    LmpFactor& operator=(const LmpFactor&) = delete;
    Index k() const { return k_; }
    Vector apply(const Vector& v) const { return run(0, v); }
    Vector apply_transpose(const Vector& v) const { return run(1, v); }
    wc4dvar_lmp* handle() const { return h_; }

private:
    Vector run(int t, const Vector& v) const {
        Vector out(v.size());
        check(wc4dvar_gpu_lmp_apply(h_, t, v.data(), out.data()));
        return out;
    }
    Index n_, k_;
    wc4dvar_lmp* h_ = nullptr;
};

// lmp.cpp:35-52
inline std::unique_ptr<LmpFactor> build_spectral_lmp(const RitzPairs& pairs, int device = 0) {
    return std::unique_ptr<LmpFactor>(new LmpFactor(pairs, device));
}

// ---------------------------------------------------------------- assimilation.hpp
// QuadraticCost (assimilation.hpp:82-97, assimilation.cpp:130-150): J(x) = 1/2 |x - D^{-1/2} b|^2
// + 1/2 sigma_o^-2 |H L^{-1} D^{1/2} x - d|^2, evaluated on the device.  Passed to pcg_split
// through PcgOptions::cost_eval it records the cost every iteration, as run_inner_loop does
// with record_cost = true (assimilation.hpp:112, assimilation.cpp:235).
class QuadraticCost {
public:
    QuadraticCost(const HessianOperator& op, const Vector& b, const Vector& d) : dim_(op.dim()) {
        if ((Index)b.size() != op.dim()) throw std::invalid_argument("QuadraticCost: background length mismatch");
        if ((Index)d.size() != op.network().q) throw std::invalid_argument("QuadraticCost: innovation length mismatch");
        check(wc4dvar_gpu_cost_create(op.handle(), b.data(), d.data(), &h_));
    }
    ~QuadraticCost() {
        if (h_) wc4dvar_gpu_cost_destroy(h_);
    }
    QuadraticCost(const QuadraticCost&) = delete;
    QuadraticCost& operator=(const QuadraticCost&) = delete;
    double operator()(const Vector& x) const {
        if ((Index)x.size() != dim_) throw std::invalid_argument("QuadraticCost: dimension mismatch");
        double v = 0.0;
        check(wc4dvar_gpu_cost_eval(h_, x.data(), &v));
        return v;
    }
    // rhs = D^{-1/2} b + sigma_o^-2 D^{1/2} L^{-T} H^T d (assimilation.cpp:142-146)
    Vector rhs() const {
        Vector r((size_t)dim_);
        check(wc4dvar_gpu_cost_rhs(h_, r.data()));
        return r;
    }
    wc4dvar_cost* handle() const { return h_; }

private:
    Index dim_;
    wc4dvar_cost* h_ = nullptr;
};

// ---------------------------------------------------------------- krylov.hpp
struct PcgOptions {  // krylov.hpp:32-38
    int max_iter = 100;
    double rel_tol = 1e-6;
    bool reorthogonalize = false;
    bool store_residual_vectors = false;
    const QuadraticCost* cost_eval = nullptr;  // krylov.hpp:37 (the reference's std::function hook)
};

struct CgHistory {  // krylov.hpp:17-30
    std::vector<double> alphas, betas, residual_norms, quadratic_costs;
    int iterations = 0;
    bool converged = false;
    std::string stop_reason;
    double relative_residual(int j) const { return residual_norms.at(j) / residual_norms.at(0); }
};

struct PcgResult {
    Vector x;
    CgHistory history;
};

// krylov.cpp:22-108 (precond null = identity LMP; x0 empty = zero guess)
inline PcgResult pcg_split(const LinearOperator& op, const Vector& b, const LmpFactor* precond, const Vector& x0,
                           const PcgOptions& opts) {
    const Index n = op.dim();
    if ((Index)b.size() != n) throw std::invalid_argument("pcg_split: right-hand side dimension mismatch");
    if (!x0.empty() && (Index)x0.size() != n)
        throw std::invalid_argument("pcg_split: initial guess dimension mismatch");
    const int mi = opts.max_iter > 0 ? opts.max_iter : 0;
    std::vector<double> al(mi + 1), be(mi + 1), rn(mi + 2), qc(mi + 2);
    wc4dvar_pcg_history h{};
    h.alphas = al.data();
    h.betas = be.data();
    h.residual_norms = rn.data();
    h.quadratic_costs = qc.data();
    wc4dvar_pcg_options o{};
    o.max_iter = opts.max_iter;
    o.reorthogonalize = opts.reorthogonalize ? 1 : 0;
    o.rel_tol = opts.rel_tol;
    o.store_residual_vectors = opts.store_residual_vectors ? 1 : 0;
    PcgResult r;
    r.x.resize((size_t)n);
    check(wc4dvar_gpu_pcg(op.handle(), b.data(), precond ? precond->handle() : nullptr,
                          x0.empty() ? nullptr : x0.data(), &o, opts.cost_eval ? opts.cost_eval->handle() : nullptr,
                          r.x.data(), &h));
    if (opts.cost_eval) r.history.quadratic_costs.assign(qc.begin(), qc.begin() + h.iterations + 1);
    r.history.alphas.assign(al.begin(), al.begin() + h.iterations);
    r.history.betas.assign(be.begin(), be.begin() + h.iterations);
    r.history.residual_norms.assign(rn.begin(), rn.begin() + h.iterations + 1);
    r.history.iterations = h.iterations;
    r.history.converged = h.converged != 0;
    static const char* reasons[] = {"zero initial residual", "relative residual tolerance reached",
                                    "maximum iterations reached"};
    r.history.stop_reason = reasons[h.stop_reason >= 0 && h.stop_reason <= 2 ? h.stop_reason : 2];
    return r;
}

// krylov.hpp:81-91
struct LanczosOptions {
    int max_iter = 0;
    double tol = 1e-10;
    std::uint64_t seed = 0x5eed0f4dULL;
};

inline RitzPairs lanczos_eigenpairs(const LinearOperator& op, Index k, const LanczosOptions& opts = {}) {
    wc4dvar_lanczos_options o{opts.max_iter, 0, opts.tol, opts.seed};
    RitzPairs p;
    p.vectors = Matrix(op.dim(), k);
    p.values.assign((size_t)k, 0.0);
    check(wc4dvar_gpu_lanczos_eigenpairs(op.handle(), k, &o, p.vectors.data(), op.dim(), p.values.data(), nullptr));
    return p;
}

// ---------------------------------------------------------------- spectrum.hpp
struct ClusteredSpectrum {  // spectrum.hpp:13-24
    Vector nonunit;
    Index unit_multiplicity = 0;
    double min_eigenvalue() const {
        double m = unit_multiplicity > 0 ? 1.0 : INFINITY;
        for (double v : nonunit) m = std::fmin(m, v);
        return m;
    }
    double max_eigenvalue() const {
        double m = unit_multiplicity > 0 ? 1.0 : -INFINITY;
        for (double v : nonunit) m = std::fmax(m, v);
        return m;
    }
};

// spectrum.cpp:31-64
inline ClusteredSpectrum clustered_spectrum(const HessianOperator& op, const LmpFactor* precond = nullptr,
                                            const Matrix* obs_range = nullptr) {
    const Index q = obs_range ? obs_range->cols() : op.network().q;
    const Index k = precond ? precond->k() : 0;
    ClusteredSpectrum cs;
    cs.nonunit.assign((size_t)(q + k > 0 ? q + k : 1), 0.0);
    int64_t nn = 0, unit = 0;
    check(wc4dvar_gpu_clustered_spectrum(op.handle(), precond ? precond->handle() : nullptr,
                                         obs_range ? obs_range->data() : nullptr, op.dim(), cs.nonunit.data(), &nn,
                                         &unit));
    cs.nonunit.resize((size_t)nn);
    cs.unit_multiplicity = unit;
    return cs;
}

}  // namespace wc4dvar_gpu
