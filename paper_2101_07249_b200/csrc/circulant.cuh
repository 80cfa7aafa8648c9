// Circulant D^{1/2} (EXTENSION for BASELINE configs 3-5; see circulant.cu).
#pragma once

#include "common.cuh"

namespace w4 {

class Fft4;

struct CirculantPlan {
    struct Impl;
    Impl* impl;
    double2* spec[4] = {nullptr, nullptr, nullptr, nullptr};  // DFT of b, q, b_inv, q_inv columns

    CirculantPlan();
    ~CirculantPlan();
    CirculantPlan(const CirculantPlan&) = delete;
    CirculantPlan& operator=(const CirculantPlan&) = delete;

    // First columns (host) of B^{1/2}, Q^{1/2} and (optional) their inverses.
    void init(int64_t n, const double* h_b, const double* h_q, const double* h_bi, const double* h_qi,
              cudaStream_t st);
    // out = D^{1/2} V (+ add) for an n(N+1) x m block (inverse factors when inv).
    void apply(bool inv, int N, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
               const double* add, int64_t ldadd, unsigned* status, DevBuf& zbuf, DevBuf& xbuf,
               cudaStream_t st, int only = -1);
    // the fused four-step transform when it can run the spectral modes (spectral.cu), else null
    Fft4* spectral_fft();
};

}  // namespace w4
