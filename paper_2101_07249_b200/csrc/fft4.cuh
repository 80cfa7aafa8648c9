// Fused four-step FFT for the circulant D^{1/2} (see fft4.cu).
#pragma once

#include "common.cuh"

namespace w4 {

// Stockham plan of one SMEM-resident sequence length L (radices 2,3,4,5,8; L <= 4096).
struct SeqPlan {
    int L = 0, nst = 0, cnt = 1;  // cnt: sequences per CTA (cnt * L <= 4096)
    int radix[12] = {}, ns[12] = {};
    const double2* tw[12] = {};  // per stage: tw[(j % Ns) * R + r] = exp(-2 pi i r (j % Ns) / (Ns R))
};

class Fft4 {
public:
    Fft4() = default;
    ~Fft4();
    Fft4(const Fft4&) = delete;
    Fft4& operator=(const Fft4&) = delete;

    // false if N has no split N = N1 N2 into Stockham-friendly factors <= 4096
    bool init(int64_t N, const double2* const spec_half[4], cudaStream_t st);
    bool ready() const { return N_ > 0; }

    // out = D^{1/2} V (+ add) for an N(Nsw+1) x m block; spectra 0/1 (2/3 when inv) = B / Q.
    void apply(bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
               const double* add, int64_t ldadd, unsigned* status, DevBuf& ybuf, DevBuf& pairbuf,
               cudaStream_t st);

private:
    int64_t N_ = 0;
    int N1_ = 0, N2_ = 0;
    SeqPlan p1_, p2_;
    double2* tables_ = nullptr;  // stage twiddles of both lengths + the four-step tables
    const double2* tw_lo_ = nullptr;
    const double2* tw_hi_ = nullptr;
    double* lam_[4] = {nullptr, nullptr, nullptr, nullptr};  // real spectra, full length N
    int64_t pairs_m_ = -1;  // shape of the uploaded column-pair table
    int pairs_per_ = -1;
    const void* pairs_ptr_ = nullptr;
};

}  // namespace w4
