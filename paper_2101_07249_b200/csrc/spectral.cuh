// Window sweeps in Fourier space for periodic constant-coefficient models (see spectral.cu).
#pragma once

#include "common.cuh"

namespace w4 {

struct SpectralArgs {
    double2* Z = nullptr;        // npc x (Nsw+1) x N spectra (Fft4::forward layout), updated in place
    int64_t N = 0;               // grid points
    int per = 0;                 // Nsw + 1 window blocks
    int64_t npc = 0;             // packed sketch-column pairs
    const double* lamB = nullptr;  // B^{1/2} / Q^{1/2} spectra (over N), row order of Z
    const double* lamQ = nullptr;
    const double2* mhat = nullptr;  // symbol of one window interval of the TL model, same order
    const int* slot = nullptr;   // Nsw+1: observation slot of time i, or -1 (NetDev::slot)
    int RL = 0;                  // last row radix (Fft4::last_radix)
    int sx = 0;                  // spatial observation stride (points 0, sx, 2 sx, ...)
    double r_inv = 1.0;          // 1 / sigma_obs^2
    unsigned* status = nullptr;
};

// strides the kernel is compiled for, and the SMEM limit on the window length
bool spectral_window_supported(int sx, int RL, int per);
void spectral_window(const SpectralArgs& a, cudaStream_t st);
// One column with its window blocks packed in pairs (Fft4::forward(pack_blocks)): Zin -> Zout,
// (per + 1) / 2 spectra each; a.Z / a.npc are unused.
void spectral_window1(const SpectralArgs& a, const double2* Zin, double2* Zout, int N1, int N2, const int (&rad)[4],
                      int nrad, cudaStream_t st);

}  // namespace w4
