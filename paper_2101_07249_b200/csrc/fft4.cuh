// Fused four-step FFT convolution for the circulant D^{1/2} (see fft4.cu).
#pragma once

#include "common.cuh"

namespace w4 {

class Fft4 {
public:
    Fft4() = default;
    ~Fft4();
    Fft4(const Fft4&) = delete;
    Fft4& operator=(const Fft4&) = delete;

    // false (and unready) when N has no compiled split N = N1 N2
    bool init(int64_t N, const double2* const spec_half[4], cudaStream_t st);
    bool ready() const { return plan_ >= 0; }

    // out = D^{1/2} V (+ add) for an N(Nsw+1) x m block; spectra 0/1 (2/3 when inv) = B / Q.
    void apply(bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
               const double* add, int64_t ldadd, unsigned* status, DevBuf& ybuf, DevBuf& pairbuf,
               cudaStream_t st, int only = -1);

    // Spectral modes (see spectral.cu).  forward: Z[(jj (Nsw+1) + i) N + t] = unscaled DFT of
    // window block i of sketch columns 2 jj (real part) and 2 jj + 1 (imaginary part), t the
    // row order of pass B' (frequency k2 + N2 f(e) at t = e + N1 k2).  inverse: out = add +
    // IDFT of such spectra (unnormalised).
    bool spectral_ready() const { return plan_ >= 0 && ipb_; }
    // pack_blocks (m = 1): pair a packs window blocks 2a / 2a + 1 of the ONE column instead,
    // Z[a N + t], a < (Nsw + 2) / 2 (see spectral_window1 for the Hermitian unpacking).
    void forward(int Nsw, const double* V, int64_t ldv, int64_t m, double2* Z, DevBuf& ybuf, cudaStream_t st,
                 bool pack_blocks = false);
    void inverse(int Nsw, const double2* Z, int64_t m, double* out, int64_t ldo, const double* add, int64_t ldadd,
                 unsigned* status, DevBuf& ybuf, cudaStream_t st, bool pack_blocks = false);
    void row_radices(int (&r)[4], int& n) const;  // DIF row radices, first stage first
    int64_t n1() const { return N1_; }
    int64_t n2() const { return N2_; }
    int last_radix() const;  // radix of the last DIF row stage: its outputs are contiguous in t
    // forward-factor spectra / N in the same row order (0: B^{1/2}, 1: Q^{1/2})
    const double* lam(int which) const { return lam_[which]; }
    // Fourier symbol of s sub-steps of the 3-point TL step, in the same row order
    void build_symbol(double lft, double mid, double rgt, int s, double2* mhat, cudaStream_t st) const;

private:
    void run(int mode, bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
             const double* add, int64_t ldadd, unsigned* status, double2* Z, DevBuf& ybuf, DevBuf& pairbuf,
             cudaStream_t st, int only);
    int plan_ = -1;
    int ipb_ = 1;                // pass B in place (the lam tables are in its digit-reversed order)
    int64_t N_ = 0, N1_ = 0, N2_ = 0;
    double2* tables_ = nullptr;  // w_N1^e, w_N2^e (stage twiddles) + two-level w_N^p
    const double2* tw1_ = nullptr;
    const double2* tw2_ = nullptr;
    const double2* tlo_ = nullptr;
    const double2* thi_ = nullptr;
    double* lam_[4] = {nullptr, nullptr, nullptr, nullptr};  // real spectra / N, transposed order
    DevBuf ctr_;                 // ticket + per-group completion counters
    int64_t pairs_m_[3] = {-1, -1, -1};  // shape of the uploaded pair tables (convolution / spectral / block-packed)
    int pairs_per_[3] = {-1, -1, -1};
    const void* pairs_ptr_[3] = {nullptr, nullptr, nullptr};
    DevBuf spair_, hpair_;       // pair tables of the spectral modes
};

}  // namespace w4
