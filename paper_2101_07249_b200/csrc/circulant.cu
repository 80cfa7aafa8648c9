// Circulant covariance factors (EXTENSION): on the periodic grid SOAR
// with chordal distance is circulant (covariance.cpp:36-41, test_covariance.cpp:41-43), so
// its symmetric square root is the circulant matrix whose eigenvalues are the square
// roots of the DFT of the first column.  D^{1/2} of an n_A x m block is then a batched
// real FFT over the (N+1)m n-columns, a pointwise product with the B^{1/2} or Q^{1/2}
// spectrum (picked per column; the 1/n normalisation and the optional identity term
// v + D^{1/2}s fused into the product / final pass), and a batched inverse FFT.
// The FFTs are cuFFT (library); the spectrum product and epilogues are our kernels.
#include "circulant.cuh"
#include "fft4.cuh"

#include <cufft.h>

#include <cstdlib>
#include <map>
#include <mutex>

namespace w4 {
namespace {

#define W4_CUFFT(expr)                                                                      \
    do {                                                                                    \
        cufftResult _r = (expr);                                                            \
        if (_r != CUFFT_SUCCESS)                                                            \
            throw DeviceError(std::string(#expr) + ": cuFFT error " + std::to_string((int)_r)); \
    } while (0)

__global__ void spectrum_mul_kernel(int64_t nh, int64_t ncols, int64_t c0, int per, const double2* __restrict__ sb,
                                    const double2* __restrict__ sq, double scale, double2* __restrict__ Z) {
    // column c0 + c of the (N+1)m view: block i = (c0 + c) % per; i == 0 -> B spectrum, else Q
    const int64_t total = nh * ncols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / nh, f = e % nh;
        const double2 h = (((c0 + c) % per) == 0) ? sb[f] : sq[f];
        const double2 z = Z[e];
        Z[e] = make_double2(scale * (z.x * h.x - z.y * h.y), scale * (z.x * h.y + z.y * h.x));
    }
}

// n-column chunk [c0, c0 + nc) of the (N+1)m view: view column c is window block
// i = c % per of sketch column j = c / per, i.e. element j*ld + i*n + r of a block.
__global__ void emit_chunk_kernel(int64_t n, int64_t nc, int64_t c0, int per, const double* __restrict__ tmp,
                                  const double* __restrict__ add, int64_t ldadd, double* __restrict__ out,
                                  int64_t ldo, unsigned* status) {
    bool bad = false;
    const int64_t total = n * nc;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = c0 + e / n, r = e % n;
        const int64_t j = c / per, i = c % per;
        double v = tmp[e];
        if (add) {
            v = add[j * ldadd + i * n + r] + v;  // out = v + D^{1/2} s
            bad |= !isfinite(v);
        }
        out[j * ldo + i * n + r] = v;
    }
    if (status && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, ST_OUT_NONFINITE);
}

__global__ void copy_cols_kernel(int64_t rows, int64_t m, const double* __restrict__ a, int64_t lda,
                                 double* __restrict__ out, int64_t ldo) {
    const int64_t total = rows * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / rows, r = e % rows;
        out[c * ldo + r] = a[c * lda + r];
    }
}

unsigned grid_for(int64_t total) {
    int64_t g = cdiv(total, 256);
    if (g > 16 * kSMs) g = 16 * kSMs;
    return (unsigned)std::max<int64_t>(g, 1);
}

}  // namespace

struct CirculantPlan::Impl {
    int64_t n = 0;
    Fft4 f4;          // fused four-step path (when n splits into SMEM-sized smooth factors)
    DevBuf pairbuf;   // its column-pair table
    std::mutex mu;
    std::map<int64_t, std::pair<cufftHandle, cufftHandle>> plans;  // batch -> (R2C, C2R)
    ~Impl() {
        for (auto& kv : plans) {
            cufftDestroy(kv.second.first);
            cufftDestroy(kv.second.second);
        }
    }
    std::pair<cufftHandle, cufftHandle> get(int64_t batch) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = plans.find(batch);
        if (it != plans.end()) return it->second;
        cufftHandle f, b;
        long long nn = n;
        W4_CUFFT(cufftCreate(&f));
        W4_CUFFT(cufftCreate(&b));
        size_t ws = 0;
        long long inembed = n, onembed = n / 2 + 1;
        W4_CUFFT(cufftMakePlanMany64(f, 1, &nn, &inembed, 1, n, &onembed, 1, n / 2 + 1, CUFFT_D2Z, batch, &ws));
        W4_CUFFT(cufftMakePlanMany64(b, 1, &nn, &onembed, 1, n / 2 + 1, &inembed, 1, n, CUFFT_Z2D, batch, &ws));
        plans[batch] = {f, b};
        return plans[batch];
    }
};

CirculantPlan::CirculantPlan() : impl(new Impl) {}
CirculantPlan::~CirculantPlan() {
    for (double2*& p : spec)
        if (p) cudaFree(p);
    delete impl;
}

void CirculantPlan::init(int64_t n, const double* h_b, const double* h_q, const double* h_bi,
                         const double* h_qi, cudaStream_t st) {
    impl->n = n;
    const int64_t nh = n / 2 + 1;
    auto spectrum = [&](const double* host_col, double2*& dst) {
        if (!host_col) {
            dst = nullptr;
            return;
        }
        double* d = nullptr;
        W4_CUDA(cudaMalloc(&d, sizeof(double) * n));
        W4_CUDA(cudaMalloc(&dst, sizeof(double2) * nh));
        W4_CUDA(cudaMemcpyAsync(d, host_col, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        auto pl = impl->get(1);
        W4_CUFFT(cufftSetStream(pl.first, st));
        W4_CUFFT(cufftExecD2Z(pl.first, d, reinterpret_cast<cufftDoubleComplex*>(dst)));
        W4_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
    };
    spectrum(h_b, spec[0]);
    spectrum(h_q, spec[1]);
    spectrum(h_bi, spec[2]);
    spectrum(h_qi, spec[3]);
    const double2* const sp[4] = {spec[0], spec[1], spec[2], spec[3]};
    impl->f4.init(n, sp, st);  // leaves f4 unready when n has no suitable split
}

Fft4* CirculantPlan::spectral_fft() { return impl->f4.spectral_ready() ? &impl->f4 : nullptr; }

void CirculantPlan::apply(bool inv, int N, const double* V, int64_t ldv, int64_t m, double* out,
                          int64_t ldo, const double* add, int64_t ldadd, unsigned* status,
                          DevBuf& zbuf, DevBuf& xbuf, cudaStream_t st, int only) {
    const int64_t n = impl->n, nh = n / 2 + 1;
    // only = 0 / 1: every column uses the B / Q factor (callers pass N = 0)
    const double2* sb = spec[inv ? (only == 1 ? 3 : 2) : (only == 1 ? 1 : 0)];
    const double2* sq = spec[inv ? 3 : 1];
    require(sb && sq, "apply_D_half_inv: inverse factors were not provided");
    const int64_t dim = n * (N + 1);
    const int64_t ncols = (int64_t)(N + 1) * m;
    // The fused four-step path (fft4.cu) runs whenever n has a compiled split; WC4DVAR_FFT4=0
    // forces batched cuFFT (the fallback for every other n).
    static const bool use_f4 = [] {
        const char* e = std::getenv("WC4DVAR_FFT4");
        return !e || std::atoi(e) != 0;
    }();
    if (use_f4 && impl->f4.ready()) {
        impl->f4.apply(inv, N, V, ldv, m, out, ldo, add, ldadd, status, zbuf, impl->pairbuf, st, only);
        return;
    }
    // contiguous real input (the FFT plan assumes column distance n)
    const double* X = V;
    if (ldv != dim) {
        double* xb = xbuf.get<double>((size_t)dim * m);
        copy_cols_kernel<<<grid_for(dim * m), 256, 0, st>>>(dim, m, V, ldv, xb, dim);
        W4_LAUNCH();
        X = xb;
    }
    // WC4DVAR_FFT_CHUNK=c runs the columns in L2-sized chunks of c (D2Z -> product -> Z2D
    // per chunk).  Measured at C4 (n = 1e6) this is SLOWER than one batched plan (chunk 1:
    // 72 ms, 8: 31 ms, all 1088 columns: 25 ms per D^1/2): small batches leave cuFFT's
    // kernels under-occupied.  Default: one chunk.
    static const int64_t chunk_env = [] {
        const char* e = std::getenv("WC4DVAR_FFT_CHUNK");
        return e ? (int64_t)std::atoll(e) : (int64_t)0;
    }();
    const int64_t chunk = chunk_env > 0 ? std::min(chunk_env, ncols) : ncols;
    const bool direct = !add && ldo == dim;  // Z2D straight into the output block
    // spectrum chunk and (if needed) the real chunk before the epilogue share zbuf; xbuf may
    // hold the contiguous copy of V
    double2* Z = zbuf.get<double2>((size_t)nh * chunk + (direct ? 0 : (size_t)(n * chunk + 1) / 2));
    double* tmp = direct ? nullptr : reinterpret_cast<double*>(Z + (size_t)nh * chunk);
    for (int64_t c0 = 0; c0 < ncols; c0 += chunk) {
        const int64_t nc = std::min(chunk, ncols - c0);
        auto pl = impl->get(nc);
        W4_CUFFT(cufftSetStream(pl.first, st));
        W4_CUFFT(cufftSetStream(pl.second, st));
        W4_CUFFT(cufftExecD2Z(pl.first, const_cast<double*>(X) + c0 * n, reinterpret_cast<cufftDoubleComplex*>(Z)));
        spectrum_mul_kernel<<<grid_for(nh * nc), 256, 0, st>>>(nh, nc, c0, N + 1, sb, sq, 1.0 / (double)n, Z);
        W4_LAUNCH();
        if (direct) {
            W4_CUFFT(cufftExecZ2D(pl.second, reinterpret_cast<cufftDoubleComplex*>(Z), out + c0 * n));
            continue;
        }
        W4_CUFFT(cufftExecZ2D(pl.second, reinterpret_cast<cufftDoubleComplex*>(Z), tmp));
        emit_chunk_kernel<<<grid_for(n * nc), 256, 0, st>>>(n, nc, c0, N + 1, tmp, add, ldadd, out, ldo, status);
        W4_LAUNCH();
    }
}

}  // namespace w4
