// Spectral LMP in compact-WY form and the fused split-PCG row passes.
//
// The reference applies C = prod_{i} (I - c_i u_i u_i^T), c_i = 1 - theta_i^{-1/2}, as k
// sequential rank-1 updates (lmp.cpp:8-26): 2k passes over U per apply, 4k per PCG
// iteration.  Algebraically (no orthonormality assumed)
//     C   = H_0 H_1 ... H_{k-1} = I - U T U^T,   C^T = I - U T^T U^T,
// with T upper triangular, T_ii = c_i, T[0:i, i] = -c_i T[0:i,0:i] (U^T U)[0:i, i]
// (the compact-WY recurrence).  Each apply is then two streaming passes over U, and the
// PCG iteration (krylov.cpp:55-95) fuses into three row passes that read U once each.
#pragma once

#include "common.cuh"

namespace w4 {

// T (k x k, upper) from S = U^T U (k x k) and theta; single CTA.
void lmp_build_T(int k, const double* S, const double* theta, double* T, cudaStream_t st);

// Device scalars used by the PCG passes.
enum { SC_RHO = 0, SC_CURV = 1, SC_ALPHA = 2, SC_RHO_NEXT = 3, SC_BETA = 4, SC_DOT = 5, SC_N = 8 };

struct RowPassCtx {
    int64_t n = 0;
    int k = 0;
    const double* U = nullptr;
    int64_t ldu = 0;
    int blk_rb = 0;             // > 0: U is row-tile blocked (lmp_block_U with rb = blk_rb)
    const double* T = nullptr;  // k x k upper
    double* partial = nullptr;  // grid x (k+1)
    unsigned* counter = nullptr;
    double* scal = nullptr;     // SC_N doubles
    double* g = nullptr;        // k+1 reduction result
    double* h = nullptr;        // k+1 reduction result
};

// Row-tile height of the PCG row passes for rank k, and the LMP factor's blocked copy of
// U: tile t (rows [t rb, (t+1) rb), zero-padded past n) is the contiguous rb x k
// column-major block at Ublk + t k rb, so a pass streams each tile with ONE bulk copy.
int lmp_tile_rows(int k);
int64_t lmp_blocked_size(int64_t n, int k);
void lmp_block_U(int64_t n, int k, const double* U, int64_t ldu, double* Ublk, cudaStream_t st);
void lmp_unblock_U(int64_t n, int k, const double* Ublk, double* U, int64_t ldu, cudaStream_t st);

// out[k] = U^T v, out[k] (dot) = a . b (a/b may be NULL -> 0); deterministic.
void rowpass_utv(const RowPassCtx& c, const double* v, const double* a, const double* b,
                 double* out, cudaStream_t st);
// out = v - U (op(T) g[0:k]), op = T (C v) or T^T (C^T v).
void rowpass_apply(const RowPassCtx& c, bool transpose, const double* v, const double* g,
                   double* out, cudaStream_t st);
// PCG pass 1: g = [U^T w ; p.w]; scal[CURV] = p.w, scal[ALPHA] = rho / curv.
void pcg_pass1(const RowPassCtx& c, const double* p, const double* w, cudaStream_t st);
// PCG pass 2: x += alpha p; r -= alpha (w - U T^T g); h = [U^T r ; r.r];
//             scal[RHO_NEXT] = r.r, scal[BETA] = rho_next / rho.
void pcg_pass2(const RowPassCtx& c, double* x, double* r, const double* p, const double* w,
               cudaStream_t st);
// PCG pass 3: p = (r - U T h) + beta p.
void pcg_pass3(const RowPassCtx& c, const double* r, double* p, cudaStream_t st);

// Squared-norm style reductions: out = sum_i (a_i - b_i)^2 (b may be NULL).
void sqdist(int64_t n, const double* a, const double* b, double* out, double* partial,
            unsigned* counter, cudaStream_t st);
// x = a*x + b*y elementwise helpers.
void axpby(int64_t n, double a, const double* x, double b, const double* y, double* out,
           cudaStream_t st);
// max |S - I| over a k x k matrix -> out (device).
void defect_max(int k, const double* S, double* out, cudaStream_t st);

}  // namespace w4
