// Split-preconditioned CG on device (krylov.cpp:22-99, Algorithm 1 of the paper).
//
// Per iteration: one operator apply (w = A p) and three fused row passes over the LMP
// vectors U (lmp_pcg.cuh); scalars alpha/beta/rho stay on device and the host reads one
// small pinned record per iteration for the reference's checks and stopping test.
#include "pcg.cuh"

#include <cmath>
#include <cstdlib>
#include <sstream>
#include <vector>

#include "gemm.cuh"
#include "lmp_pcg.cuh"

namespace w4 {
namespace {

__global__ void reorth_fix_kernel(double* scal, const double* h, int k) {
    // after MGS re-orthogonalisation: rho_next = |r|^2 recomputed (krylov.cpp:71-76)
    const double rn = h[k];
    scal[SC_RHO_NEXT] = rn;
    scal[SC_BETA] = rn / scal[SC_DOT];
    scal[SC_RHO] = rn;
}

__global__ void scale_copy_kernel(int64_t n, const double* __restrict__ r, const double* rho,
                                  double* __restrict__ f) {
    const double inv = 1.0 / sqrt(*rho);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        f[i] = r[i] * inv;
}

// Device-side loop control for iterations 2.. of the unpreconditioned-cost path: record
// alpha / beta / |r| of iteration j, stop (condition 0) on an error, on convergence or at
// max_iter.  state = {j, err, status, converged}.
__global__ void pcg_loop_check_kernel(cudaGraphConditionalHandle h, const double* __restrict__ scal,
                                      const unsigned* __restrict__ status, int* state, double* alphas,
                                      double* betas, double* res, double r0, double tol, int max_iter) {
    const int j = state[0] + 1;
    state[0] = j;
    const unsigned s = *status;
    const double curv = scal[SC_CURV], alpha = scal[SC_ALPHA], rn = scal[SC_RHO_NEXT], beta = scal[SC_BETA];
    int err = 0;
    if (s) err = 1;
    else if (!isfinite(curv) || curv <= 0.0 || !isfinite(alpha) || !isfinite(beta)) err = 2;
    if (err) {
        state[1] = err;
        state[2] = (int)s;
        cudaGraphSetConditional(h, 0);
        return;
    }
    alphas[j - 1] = alpha;
    betas[j - 1] = beta;
    res[j] = sqrt(rn);
    const bool conv = sqrt(rn) / r0 <= tol;
    if (conv) state[3] = 1;
    cudaGraphSetConditional(h, (conv || j >= max_iter) ? 0u : 1u);
}

void check_finite(double v, const char* what, int it) {
    if (!std::isfinite(v)) {
        std::ostringstream m;
        m << "pcg_split: non-finite " << what << " at iteration " << it;
        throw NumericalError(m.str());
    }
}

}  // namespace

void pcg_dev(wc4dvar_op& op, const double* b, wc4dvar_lmp* pre, const double* x0,
             const wc4dvar_pcg_options& opts, wc4dvar_cost* cost, double* x,
             PcgRecord& rec, cudaStream_t st) {
    const int64_t n = op.dim;
    const int k = pre ? pre->k : 0;
    require(!pre || pre->k == 0 || pre->n == n, "pcg_split: preconditioner dimension mismatch");
    enum { B_R = 0, B_P, B_W, B_TMP, B_PART, B_SCAL, B_G, B_H, B_F, B_CNT, B_GWS, B_HF };
    DevBuf* pool = op.pool + 24;  // pool[0..23] belong to the sketch workspaces
    double* r = pool[B_R].get<double>(n);
    double* p = pool[B_P].get<double>(n);
    double* w = pool[B_W].get<double>(n);
    double* tmp = pool[B_TMP].get<double>(n);
    const int64_t maxgrid = std::min<int64_t>(cdiv(n, 32) + 1, 2048);
    double* part = pool[B_PART].get<double>((size_t)maxgrid * (k + 1));
    double* scal = pool[B_SCAL].get<double>(SC_N + 2);
    double* g = pool[B_G].get<double>(k + 1);
    double* h = pool[B_H].get<double>(k + 1);
    unsigned* counter = pool[B_CNT].get<unsigned>(4);
    W4_CUDA(cudaMemsetAsync(counter, 0, 4 * sizeof(unsigned), st));
    W4_CUDA(cudaMemsetAsync(scal, 0, (SC_N + 2) * sizeof(double), st));
    double* F = nullptr;
    // CgHistory::normalized_residuals are kept for re-orthogonalisation or on request
    // (krylov.cpp:30)
    if (opts.reorthogonalize || opts.store_residual_vectors) {
        // the n x (max_iter + 1) residual store must fit beside the operator's workspaces
        size_t free_b = 0, total_b = 0;
        W4_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const double need = 8.0 * (double)n * (double)(opts.max_iter + 1);
        if (need > 0.9 * (double)(free_b + pool[B_F].bytes)) {
            std::ostringstream m;
            m << "pcg_split: the stored residual basis (" << need / 1e9 << " GB for " << opts.max_iter + 1
              << " vectors of " << n << ") does not fit in device memory; lower max_iter";
            throw InvalidArgument(m.str());
        }
        F = pool[B_F].get<double>((size_t)n * (opts.max_iter + 1));
    }
    const bool reorth = opts.reorthogonalize != 0;
    static thread_local double* pinned = nullptr;
    if (!pinned) W4_CUDA(cudaMallocHost(&pinned, 16 * sizeof(double)));

    RowPassCtx c;
    c.n = n;
    c.k = k;
    c.U = pre ? pre->U : nullptr;
    c.ldu = n;
    c.blk_rb = pre && pre->k ? lmp_tile_rows(pre->k) : 0;
    c.T = pre ? pre->T : nullptr;
    c.partial = part;
    c.counter = counter;
    c.scal = scal;
    c.g = g;
    c.h = h;

    auto read_scal = [&]() {
        W4_CUDA(cudaMemcpyAsync(pinned, scal, SC_N * sizeof(double), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
    };

    // x = x0 or 0; r = C^T (b - A x0)   (krylov.cpp:32-38)
    bool x0_zero = true;
    if (x0) {
        // isZero(0.0): every entry exactly zero (checked on device)
        rowpass_utv(RowPassCtx{n, 0, nullptr, n, 0, nullptr, part, counter, scal, g, h}, x0, x0, x0,
                    tmp, st);  // tmp[0] = x0 . x0
        double hv = 0;
        W4_CUDA(cudaMemcpyAsync(&hv, tmp, sizeof(double), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        x0_zero = (hv == 0.0);
    }
    if (x0 && !x0_zero) {
        W4_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        op.applies += 1;
        op.reset_status(st);
        op.apply_block_dev(x, n, 1, w, n, st);
        op.check_status(st);
        axpby(n, 1.0, b, -1.0, w, tmp, st);  // b - A x0
    } else {
        if (x0) W4_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        else W4_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
        W4_CUDA(cudaMemcpyAsync(tmp, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    rowpass_utv(c, tmp, nullptr, nullptr, g, st);        // g = U^T rhs
    rowpass_apply(c, true, tmp, g, r, st);               // r = C^T rhs
    rowpass_utv(c, r, r, r, h, st);                      // h = [U^T r ; r.r]
    rowpass_apply(c, false, r, h, p, st);                // p = C r  (krylov.cpp:39)
    W4_CUDA(cudaMemcpyAsync(scal + SC_RHO, h + k, sizeof(double), cudaMemcpyDeviceToDevice, st));
    read_scal();
    const double rho0 = pinned[SC_RHO];
    const double r0 = std::sqrt(rho0);
    rec.residual_norms.push_back(r0);
    if (cost) rec.costs.push_back(cost->eval_dev(x, st));
    rec.iterations = 0;
    rec.converged = false;
    if (r0 == 0.0) {
        rec.converged = true;
        rec.stop_reason = 0;
        return;
    }
    int nf = 0;
    if (F) {
        scale_copy_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 1184), 256, 0, st>>>(
            n, r, scal + SC_RHO, F);
        W4_LAUNCH();
        nf = 1;
    }
    // Without re-orthogonalisation every iteration issues the same device work on the same
    // buffers: capture it once as a CUDA graph (apply + 3 row passes + the scalar read-back)
    // and replay it, so the host's per-iteration sync is followed by one graph launch instead
    // of ~10 kernel launches.  WC4DVAR_PCG_GRAPH=0 disables.
    static const bool graph_env = [] {
        const char* e = std::getenv("WC4DVAR_PCG_GRAPH");
        return !(e && std::atoi(e) == 0);
    }();
    const bool use_graph = graph_env && !F && !op.prof;
    cudaGraphExec_t gexec = nullptr;
    struct GraphGuard {
        cudaGraphExec_t& e;
        ~GraphGuard() {
            if (e) cudaGraphExecDestroy(e);
        }
    } gguard{gexec};
    auto body = [&]() {
        op.reset_status(st);
        op.apply_block_dev(p, n, 1, w, n, st);
        pcg_pass1(c, p, w, st);        // curvature, alpha
        pcg_pass2(c, x, r, p, w, st);  // x, r, rho_next, beta
        pcg_pass3(c, r, p, st);        // p = C r + beta p (speculative; unused on exit)
        W4_CUDA(cudaMemcpyAsync(op.h_status, op.d_status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaMemcpyAsync(pinned, scal, SC_N * sizeof(double), cudaMemcpyDeviceToHost, st));
    };
    // Iterations 2.. can run as ONE graph launch: a conditional WHILE node whose body is the
    // iteration plus a check kernel that records alpha / beta / |r| on the device and stops
    // the loop; the host reads the history once at the end.  Used when nothing needs the
    // host per iteration (no cost recorder, no re-orthogonalisation, no profiling).
    // WC4DVAR_PCG_DEVLOOP=0 keeps the per-iteration graph + host check.
    static const bool devloop_env = [] {
        const char* e = std::getenv("WC4DVAR_PCG_DEVLOOP");
        return !(e && std::atoi(e) == 0);
    }();
    const bool dev_loop = use_graph && devloop_env && !cost;
    // returns false when the loop graph could not be built (the host loop then continues)
    auto run_dev_loop = [&](int j0) -> bool {
        const int left = opts.max_iter - j0 + 1;
        DevBuf rec_buf;
        double* hist = rec_buf.get<double>((size_t)3 * (opts.max_iter + 2) + 4);
        double* d_al = hist;
        double* d_be = hist + (opts.max_iter + 2);
        double* d_rs = hist + 2 * (opts.max_iter + 2);
        int* state = reinterpret_cast<int*>(hist + 3 * (opts.max_iter + 2));
        std::vector<int> st0 = {j0 - 1, 0, 0, 0};
        W4_CUDA(cudaMemcpyAsync(state, st0.data(), sizeof(int) * 4, cudaMemcpyHostToDevice, st));
        W4_CUDA(cudaStreamSynchronize(st));
        cudaGraph_t g = nullptr, bodyg = nullptr;
        cudaGraphExec_t ex = nullptr;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
        cudaGraphConditionalHandle h{};
        if (ok) ok = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        cudaGraphNode_t node;
        cudaGraphNodeParams cp = {};
        if (ok) {
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
        }
        if (ok) {
            bodyg = cp.conditional.phGraph_out[0];
            ok = cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) ==
                 cudaSuccess;
            if (ok) {
                try {
                    op.reset_status(st);
                    op.apply_block_dev(p, n, 1, w, n, st);
                    pcg_pass1(c, p, w, st);
                    pcg_pass2(c, x, r, p, w, st);
                    pcg_pass3(c, r, p, st);
                    pcg_loop_check_kernel<<<1, 1, 0, st>>>(h, scal, op.d_status, state, d_al, d_be, d_rs, r0,
                                                           opts.rel_tol, opts.max_iter);
                } catch (...) {
                    ok = false;
                }
                cudaGraph_t cap = nullptr;
                if (cudaStreamEndCapture(st, &cap) != cudaSuccess) ok = false;
            }
        }
        if (ok) ok = cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();  // clear a sticky capture / instantiate error
            if (ex) cudaGraphExecDestroy(ex);
            if (g) cudaGraphDestroy(g);
            return false;
        }
        W4_CUDA(cudaGraphLaunch(ex, st));
        std::vector<int> hs(4);
        W4_CUDA(cudaMemcpyAsync(hs.data(), state, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
        W4_CUDA(cudaStreamSynchronize(st));
        cudaGraphExecDestroy(ex);
        cudaGraphDestroy(g);
        const int jl = hs[0];  // last iteration executed
        const int done_ok = hs[1] ? jl - 1 : jl;
        op.applies += jl - j0 + 1;
        std::vector<double> ha(left + 1), hb(left + 1), hr(left + 2);
        if (done_ok >= j0) {
            W4_CUDA(cudaMemcpyAsync(ha.data(), d_al + j0 - 1, sizeof(double) * (done_ok - j0 + 1),
                                    cudaMemcpyDeviceToHost, st));
            W4_CUDA(cudaMemcpyAsync(hb.data(), d_be + j0 - 1, sizeof(double) * (done_ok - j0 + 1),
                                    cudaMemcpyDeviceToHost, st));
            W4_CUDA(cudaMemcpyAsync(hr.data(), d_rs + j0, sizeof(double) * (done_ok - j0 + 1),
                                    cudaMemcpyDeviceToHost, st));
        }
        W4_CUDA(cudaStreamSynchronize(st));
        for (int jj = j0; jj <= done_ok; ++jj) {
            rec.alphas.push_back(ha[jj - j0]);
            rec.betas.push_back(hb[jj - j0]);
            rec.residual_norms.push_back(hr[jj - j0]);
            rec.iterations = jj;
        }
        if (hs[1]) {  // reproduce the host loop's checks and messages for iteration jl
            const unsigned s = (unsigned)hs[2];
            if (s & ST_FWD_NONFINITE) throw NumericalError("hessian apply: non-finite value after forward sweep");
            if (s & ST_ADJ_NONFINITE) throw NumericalError("hessian apply: non-finite value after adjoint sweep");
            if (s & ST_OUT_NONFINITE) throw NumericalError("hessian apply: non-finite result");
            read_scal();
            const double curv = pinned[SC_CURV];
            check_finite(curv, "curvature", jl);
            if (curv <= 0.0) {
                std::ostringstream m;
                m << "pcg_split: p^T A p = " << curv << " at iteration " << jl
                  << "; operator lost positive definiteness";
                throw NumericalError(m.str());
            }
            check_finite(pinned[SC_ALPHA], "alpha", jl);
            check_finite(pinned[SC_BETA], "beta", jl);
        }
        if (hs[3]) {
            rec.converged = true;
            rec.stop_reason = 1;
        }
        return true;
    };
    for (int j = 1; j <= opts.max_iter; ++j) {
        if (dev_loop && j == 2 && run_dev_loop(j)) break;
        op.applies += 1;  // the single operator apply of this iteration (krylov.cpp:56)
        // iteration 1 runs eagerly (it grows the workspaces; no allocation under capture)
        const bool graph_it = use_graph && j > 1;
        if (graph_it) {
            if (!gexec) {
                cudaGraph_t graph = nullptr;
                W4_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
                try {
                    body();
                } catch (...) {
                    cudaStreamEndCapture(st, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                W4_CUDA(cudaStreamEndCapture(st, &graph));
                W4_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
                W4_CUDA(cudaGraphDestroy(graph));
            }
            W4_CUDA(cudaGraphLaunch(gexec, st));
            W4_CUDA(cudaStreamSynchronize(st));
        } else {
            op.reset_status(st);
            op.apply_block_dev(p, n, 1, w, n, st);
            pcg_pass1(c, p, w, st);  // curvature, alpha
            if (reorth) W4_CUDA(cudaMemcpyAsync(scal + SC_DOT, scal + SC_RHO, sizeof(double),
                                                cudaMemcpyDeviceToDevice, st));
            pcg_pass2(c, x, r, p, w, st);  // x, r, rho_next, beta
        }
        if (!graph_it && reorth) {
            // re-orthogonalisation against the stored normalised residuals (krylov.cpp:71-74):
            // the reference's modified Gram-Schmidt becomes classical Gram-Schmidt applied
            // twice (CGS2, as stable as MGS) -- per pass one DMMA Gram h = F^T r and one
            // DMMA update r -= F h over the whole n x nf store, instead of 2 nf launches
            double* hf = pool[B_HF].get<double>((size_t)nf + 1);
            for (int pass = 0; pass < 2 && nf > 0; ++pass) {
                gemm_tn(n, nf, 1, F, n, r, n, 1.0, hf, nf, pool[B_GWS], st);
                GemmPass gp;
                gp.A = F;
                gp.lda = n;
                gp.M = n;
                gp.K = nf;
                gp.ncols = 1;
                gp.alpha = -1.0;
                gp.in = ColMap::plain(hf, nf);
                gp.out = ColMap::plain(r, n);
                gp.add = ColMap::plain(r, n);
                gemm_nn(&gp, 1, nullptr, st);
            }
            rowpass_utv(c, r, r, r, h, st);
            reorth_fix_kernel<<<1, 1, 0, st>>>(scal, h, k);
            W4_LAUNCH();
        }
        if (!graph_it) {
            pcg_pass3(c, r, p, st);  // p = C r + beta p (speculative; unused on exit)
            W4_CUDA(cudaMemcpyAsync(op.h_status, op.d_status, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                    st));
            read_scal();
        }
        const unsigned s = *op.h_status;
        if (s & ST_FWD_NONFINITE)
            throw NumericalError("hessian apply: non-finite value after forward sweep");
        if (s & ST_ADJ_NONFINITE)
            throw NumericalError("hessian apply: non-finite value after adjoint sweep");
        if (s & ST_OUT_NONFINITE) throw NumericalError("hessian apply: non-finite result");
        const double curv = pinned[SC_CURV];
        check_finite(curv, "curvature", j);
        if (curv <= 0.0) {
            std::ostringstream m;
            m << "pcg_split: p^T A p = " << curv << " at iteration " << j
              << "; operator lost positive definiteness";
            throw NumericalError(m.str());
        }
        const double alpha = pinned[SC_ALPHA];
        check_finite(alpha, "alpha", j);
        const double rho_next = pinned[SC_RHO_NEXT];
        const double beta = pinned[SC_BETA];
        check_finite(beta, "beta", j);
        rec.alphas.push_back(alpha);
        rec.betas.push_back(beta);
        rec.residual_norms.push_back(std::sqrt(rho_next));
        if (cost) rec.costs.push_back(cost->eval_dev(x, st));
        if (F && rho_next > 0.0) {
            scale_copy_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 1184), 256, 0, st>>>(
                n, r, scal + SC_RHO_NEXT, F + (int64_t)nf * n);
            W4_LAUNCH();
            ++nf;
        }
        rec.iterations = j;
        if (std::sqrt(rho_next) / r0 <= opts.rel_tol) {
            rec.converged = true;
            rec.stop_reason = 1;
            break;
        }
    }
    if (!rec.converged) rec.stop_reason = 2;
    rec.F = F;
    rec.nf = nf;
    W4_CUDA(cudaStreamSynchronize(st));
}

}  // namespace w4
