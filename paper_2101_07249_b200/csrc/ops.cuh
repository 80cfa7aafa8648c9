// Operator handles behind the C-ABI (include/wc4dvar_gpu.h).
#pragma once

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "circulant.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "sweep.cuh"

// LinearOperator (operators.hpp:15-40): dim, apply_block, atomic apply counter.
struct wc4dvar_op {
    int device = 0;
    int64_t dim = 0;
    std::atomic<int64_t> applies{0};
    std::recursive_mutex mu;
    cudaStream_t stream = nullptr;
    unsigned* d_status = nullptr;  // device status word (finite checks)
    unsigned* h_status = nullptr;  // pinned mirror
    int* h_int = nullptr;          // pinned scratch for small device->host reads
    w4::DevBuf in_buf, out_buf;
    w4::DevBuf pool[40];           // [0,24) sketch, [24,40) PCG workspaces

    // Stage profiling (wc4dvar_gpu_op_profile): events around the apply's kernels.
    bool prof = false;
    bool prof_pending = false;
    cudaEvent_t pev[4] = {nullptr, nullptr, nullptr, nullptr};
    double prof_ms[3] = {0, 0, 0};
    int64_t prof_calls = 0;
    void prof_mark(int i, cudaStream_t st) {
        if (prof) cudaEventRecord(pev[i], st);
    }
    void collect_profile();  // after a synchronising call

    // Host-buffer block apply pipeline (api.cu): H2D of chunk c+1 and D2H of chunk c-1 run
    // on their own streams while chunk c computes on `stream`.
    cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
    cudaEvent_t pipe_ev[8] = {};
    void ensure_pipeline();

    virtual ~wc4dvar_op();
    // Frees every grow-only workspace (they re-grow on the next call).
    virtual void release_workspaces() {
        in_buf.release();
        out_buf.release();
        for (auto& b : pool) b.release();
    }
    // Block apply on device pointers; does not count and does not synchronise.
    virtual void apply_block_dev(const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                                 cudaStream_t st) = 0;
    virtual const char* kind_name() const = 0;

    void init_common(int dev, int64_t n);
    void reset_status(cudaStream_t st);
    // Synchronises st and throws NumericalError with the reference's stage message.
    void check_status(cudaStream_t st);
};

namespace w4 {

// HessianOperator (operators.hpp:116-152), Eq. 12 of the paper.
struct HessianOp final : wc4dvar_op {
    ModelDev md;
    NetDev nd;
    int cov_kind = WC4DVAR_COV_DENSE;
    int64_t n = 0;
    int N = 0;
    double sigma_obs = 1.0;
    double* b_half = nullptr;
    double* b_half_inv = nullptr;
    double* q_half = nullptr;
    double* q_half_inv = nullptr;
    bool sym[4] = {false, false, false, false};  // b_half, q_half, b_half_inv, q_half_inv == ^T
    int* d_slot = nullptr;
    int* d_pmap = nullptr;
    int* d_times = nullptr;   // network times / points (device copies, observe)
    int* d_points = nullptr;
    double* d_stages = nullptr;
    std::vector<int> times, points;
    DevBuf t_ws, y_ws, sweep_ws;
    void release_workspaces() override {
        wc4dvar_op::release_workspaces();
        t_ws.release();
        y_ws.release();
        sweep_ws.release();
    }
    CirculantPlan* circ = nullptr;  // WC4DVAR_COV_CIRCULANT factors
    DevBuf circ_z, circ_x;
    // Fourier-space apply (spectral.cu): periodic constant-coefficient model, circulant factors
    // and a regular observation network; d_mhat = symbol of one window interval
    bool spectral = false;
    double2* d_mhat = nullptr;
    void setup_spectral(cudaStream_t st);

    ~HessianOp() override;
    const char* kind_name() const override { return "HessianOperator"; }
    void apply_block_dev(const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                         cudaStream_t st) override;
    // which: WC4DVAR_LINV / LINVT / D_HALF / D_HALF_INV (block forms).
    void piece_dev(int which, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                   cudaStream_t st);
    // HessianOperator::observation_range (operators.cpp:146-154): W (n_A x q, ldw) =
    // D^{1/2} L^{-T} H^T [e_1 .. e_q], one block adjoint sweep of the q unit observations.
    void observation_range_dev(double* W, int64_t ldw, cudaStream_t st);
    // observe (models.cpp:184-192): y = H traj (window trajectory, network order)
    void observe_dev(const double* traj, double* y, cudaStream_t st);
    // out = D^{1/2} V (+ add) for an n_A x m block; inverse factors when inv.
    // One covariance factor (which = 0: B^{1/2}, 1: Q^{1/2}; their inverses when inv) on c
    // n-vectors: the block-sharded D^{1/2} of the row-sharded apply (distributed.py).
    void factor_apply(int which, bool inv, const double* X, int64_t ldx, int64_t c, double* out, int64_t ldo,
                      cudaStream_t st);
    void d_half(bool inv, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                const double* add, int64_t ldadd, unsigned* status, cudaStream_t st);
};

// DenseOperator (operators.hpp:42-53).
struct DenseOp final : wc4dvar_op {
    double* A = nullptr;
    ~DenseOp() override;
    const char* kind_name() const override { return "DenseOperator"; }
    void apply_block_dev(const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                         cudaStream_t st) override;
};

// Thread-local error message for the C-ABI.
void set_last_error(const std::string& msg);
const char* last_error_cstr();

}  // namespace w4

// LmpFactor (lmp.hpp:12-26) in compact-WY form.
struct wc4dvar_lmp {
    int device = 0;
    int64_t n = 0;
    int k = 0;
    double* U = nullptr;      // n x k (ld n)
    double* theta = nullptr;  // k
    double* T = nullptr;      // k x k upper
    cudaStream_t stream = nullptr;
    std::mutex mu;
    w4::DevBuf partial, gbuf, tmp;
    unsigned* counter = nullptr;
    ~wc4dvar_lmp();
};

// QuadraticCost (assimilation.hpp:82-97).
struct wc4dvar_cost {
    w4::HessianOp* op = nullptr;
    double* b_tilde = nullptr;  // n_A
    double* d = nullptr;        // q
    w4::DevBuf ws_t, ws_y, partial;
    unsigned* counter = nullptr;
    double* d_val = nullptr;    // 2 doubles
    ~wc4dvar_cost();
    // value on device pointer x (n_A); synchronises op stream.
    double eval_dev(const double* x, cudaStream_t st);
};
