// The sweeps of HessianOperator::apply (operators.cpp:132-141) in Fourier space.
//
// For a periodic constant-coefficient TL model (advection / advection-diffusion,
// models.cpp:27-45) every operator between the two D^{1/2} of
//     A v = v + D^{1/2} L^{-T} H^T R^{-1} H L^{-1} D^{1/2} v
// is diagonal in the DFT basis except the observation mask, and the mask of a regular network
// (points 0, sx, 2 sx, ...; models.cpp:159-176) only couples the sx frequencies
// k, k + n/sx, ..., k + (sx-1) n/sx:  (mask x)^(k) = (1/sx) sum_a x^(k + a n/sx).  With circulant
// covariance factors the whole product is therefore
//     forward DFT -> [ per frequency class: lam, forward recurrence x_i = Mhat x_{i-1} + t_i,
//                      class sums at the observed times, adjoint recurrence
//                      z_i = conj(Mhat) z_{i+1} + H^T y_i, lam ] -> inverse DFT,
// ONE forward and ONE inverse transform per column instead of the two full convolutions and
// the two stencil sweeps of the grid-space path (half the FFT work, and a (2s+1)-tap stencil
// per interval becomes one complex multiply).  This file is the bracketed middle step.
//
// Layout (Fft4::forward): the spectrum of window block i of the packed sketch-column pair jj
// is Z[(jj per + i) N + t]; the last DIF row stage of pass B has radix RL and span 1, and its
// output digit is the MOST significant digit of the frequency, so the sx coupled frequencies
// of a class are the entries t = b RL + c + a (RL / sx), a < sx, of one butterfly b: a class is
// a short strided run inside one 16 RL-byte segment.  One thread owns one frequency for the
// whole window (consecutive threads, consecutive t: every load and store is a full coalesced
// line): it streams the per blocks once forwards, keeping the state x in registers, and once
// backwards, writing lam z_i in place.  The class sums of the forward pass go through SMEM:
// every thread publishes x_i, and after the interval's one barrier the first T / sx threads
// add up one class each into sums[i][class], which the backward pass reads back.  HBM
// traffic: one read and one write of Z.  Both packed columns ride through as real /
// imaginary parts: every step is complex-linear with real grid-space operators.
#include "spectral.cuh"

#include <cstdlib>

#include "bulk.cuh"

namespace w4 {
namespace {

constexpr int kSpecThreads = 320;  // a multiple of 32 and of every row radix (10, 20)
constexpr int kDepth = 8;          // window blocks in flight per CTA (forward pass; a power of two)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) b
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}

__global__ void __launch_bounds__(kSpecThreads, 3) spectral_window_kernel(const SpectralArgs a) {
    extern __shared__ double2 sm[];
    __shared__ uint64_t bars[kDepth];
    const int T = kSpecThreads, t = threadIdx.x;
    const int cps = a.RL / a.sx;  // classes per butterfly
    const int ncl = T / a.sx;     // classes per CTA
    double2* ring = sm;                   // [kDepth][T] window blocks in flight (bulk copies)
    double2* xbuf = sm + kDepth * T;      // [2][T] states of the current / previous interval
    double2* sums = sm + (kDepth + 2) * T;  // [per][ncl] class sums
    const int64_t pos0 = blockIdx.x * (int64_t)T, pos = pos0 + t;
    const bool act = pos < a.N;   // T and N are multiples of RL: classes are wholly in or out
    double2* Zc = a.Z + (int64_t)blockIdx.y * a.per * a.N + pos0;  // this CTA's segment of block 0
    double2* Z = Zc + t;
    const unsigned seg_bytes = (unsigned)(min((int64_t)T, a.N - pos0) * sizeof(double2));
    if (t == 0) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // the forward pass streams the window through a kDepth-stage ring of bulk copies: thread 0
    // issues one 16 T-byte copy per block, every thread waits on the stage's mbarrier
    if (t == 0) {
        for (int d = 0; d < kDepth && d < a.per; ++d) {
            mbar_arrive_expect_tx(&bars[d], seg_bytes);
            bulk_g2s(ring + d * T, Zc + (int64_t)d * a.N, seg_bytes, &bars[d]);
        }
    }
    double2 M = make_double2(0.0, 0.0);
    double lq = 0.0, lb = 0.0;
    if (act) {
        M = __ldg(a.mhat + pos);
        lq = __ldg(a.lamQ + pos);
        lb = __ldg(a.lamB + pos);
    }
    // scale of H^T R^{-1} H in this basis: 1 / sx from the mask, r_inv, and N because both lam
    // tables carry the 1 / N of the transform pair
    const double scale = a.r_inv * (double)a.N / (double)a.sx;
    bool bad_f = false;
    // traj = L^{-1} D^{1/2} v (operators.cpp:131-132); sums = H traj per class
    double2 x = make_double2(0.0, 0.0);
    const int sb = (t / cps) * a.RL + t % cps;  // first member of the class thread t < ncl adds up
    for (int i = 0; i < a.per; ++i) {
        const int st = i & (kDepth - 1);
        mbar_wait(&bars[st], (unsigned)(i / kDepth) & 1u);
        const double2 y = act ? ring[st * T + t] : make_double2(0.0, 0.0);
        const double l = i == 0 ? lb : lq;
        const double2 mx = cmul(M, x);  // x is zero before the first block
        x = make_double2(fma(l, y.x, mx.x), fma(l, y.y, mx.y));
        xbuf[(i & 1) * T + t] = x;
        __syncthreads();  // x_i published; every thread has read its ring entry
        if (t == 0 && i + kDepth < a.per) {
            mbar_arrive_expect_tx(&bars[st], seg_bytes);
            bulk_g2s(ring + st * T, Zc + (int64_t)(i + kDepth) * a.N, seg_bytes, &bars[st]);
        }
        if (t < ncl) {
            const double2* xb = xbuf + (i & 1) * T + sb;
            double2 s0 = make_double2(0.0, 0.0), s1 = s0;  // two chains
            int e = 0;
            for (; e + 1 < a.sx; e += 2) {
                const double2 v0 = xb[e * cps], v1 = xb[(e + 1) * cps];
                s0.x += v0.x;
                s0.y += v0.y;
                s1.x += v1.x;
                s1.y += v1.y;
            }
            if (e < a.sx) {
                const double2 v0 = xb[e * cps];
                s0.x += v0.x;
                s0.y += v0.y;
            }
            const double2 sum = make_double2(s0.x + s1.x, s0.y + s1.y);
            bad_f |= !isfinite(sum.x + sum.y);
            sums[i * ncl + t] = sum;
        }
    }
    __syncthreads();
    // s = L^{-T} H^T R^{-1} H traj (operators.cpp:136-140), then D^{1/2} s per block
    const int r = t % a.RL;
    const int mycl = (t / a.RL) * cps + r % cps;
    double2 z = make_double2(0.0, 0.0);
    for (int i = a.per - 1; i >= 0; --i) {
        const double2 mz = cmulc(M, z);  // z is zero before the last block
        z = mz;
        if (__ldg(a.slot + i) >= 0) {
            const double2 sum = sums[i * ncl + mycl];
            z = make_double2(fma(scale, sum.x, mz.x), fma(scale, sum.y, mz.y));
        }
        const double l = i == 0 ? lb : lq;
        if (act) __stcs(Z + (int64_t)i * a.N, make_double2(l * z.x, l * z.y));
    }
    const bool bad_a = !isfinite(z.x + z.y);  // a non-finite z_i propagates down to z_0
    if (a.status && (bad_f || bad_a))
        atomicOr(a.status, (bad_f ? ST_FWD_NONFINITE : 0u) | (bad_a ? ST_ADJ_NONFINITE : 0u));
}

// ---- one column (PCG / Lanczos applies): window blocks packed in pairs --------------------
// A single column would leave the imaginary half of every packed transform empty.  Instead
// Fft4::forward(pack_blocks) packs window blocks 2a and 2a + 1 of the column as real /
// imaginary part, P_a = v_2a + i v_2a+1, and this kernel separates the two real spectra by
// Hermitian symmetry, v^_2a(k) = (P^_a(k) + conj P^_a(-k)) / 2, v^_2a+1(k) = (P^_a(k) -
// conj P^_a(-k)) / (2 i), runs the same recurrences and class sums, and writes
// lam z^_2a + i lam z^_2a+1 for the inverse transform: half the transforms of the unpacked form.
// In the row order of pass B' (t = e + N1 k2, k = k2 + N2 f(e)) the mirror of row k2 > 0 is row
// N2 - k2 read backwards (digit-wise complement: e' = N1 - 1 - e); row 0 mirrors into itself
// through f.  Out of place (Zin -> Zout): a thread reads its mirror's entries.
struct Window1Args {
    const double2* Zin;
    double2* Zout;
    int npk;     // packed pairs, (per + 1) / 2
    int N1, N2;
    int rad[4];  // DIF row radices, first stage first
    int nrad;
};

__device__ __forceinline__ int64_t mirror_pos(const Window1Args& w, int64_t t) {
    const int e = (int)(t % w.N1), k2 = (int)(t / w.N1);
    if (k2 > 0) return (int64_t)(w.N2 - k2) * w.N1 + (w.N1 - 1 - e);
    int span = w.N1, pw = 1, k1 = 0;  // k1 = f(e)
    for (int i = 0; i < w.nrad; ++i) {
        span /= w.rad[i];
        k1 += ((e / span) % w.rad[i]) * pw;
        pw *= w.rad[i];
    }
    k1 = (w.N1 - k1) % w.N1;
    span = w.N1;
    pw = 1;
    int em = 0;  // f^{-1}(k1)
    for (int i = 0; i < w.nrad; ++i) {
        span /= w.rad[i];
        em += ((k1 / pw) % w.rad[i]) * span;
        pw *= w.rad[i];
    }
    return em;
}

__global__ void __launch_bounds__(kSpecThreads) spectral_window1_kernel(const SpectralArgs a, const Window1Args w) {
    extern __shared__ double2 sm[];
    const int T = (int)blockDim.x, t = threadIdx.x;  // 160 or kSpecThreads: a multiple of RL
    const int cps = a.RL / a.sx, ncl = T / a.sx;
    double2* xbuf = sm;          // [2][T]
    double2* sums = sm + 2 * T;  // [per][ncl]
    const int64_t pos = blockIdx.x * (int64_t)T + t;
    const bool act = pos < a.N;
    const int64_t mpos = act ? mirror_pos(w, pos) : 0;
    double2 M = make_double2(0.0, 0.0);
    double lq = 0.0, lb = 0.0;
    if (act) {
        M = __ldg(a.mhat + pos);
        lq = __ldg(a.lamQ + pos);
        lb = __ldg(a.lamB + pos);
    }
    const double scale = a.r_inv * (double)a.N / (double)a.sx;
    const int sb = (t / cps) * a.RL + t % cps;
    bool bad_f = false;
    double2 x = make_double2(0.0, 0.0);
    double2 p = make_double2(0.0, 0.0), pm = p;
    if (act) {
        p = __ldg(w.Zin + pos);
        pm = __ldg(w.Zin + mpos);
    }
    for (int i = 0; i < a.per; ++i) {
        double2 y;
        if ((i & 1) == 0) {
            y = make_double2(0.5 * (p.x + pm.x), 0.5 * (p.y - pm.y));  // (P + conj Pm) / 2
        } else {
            y = make_double2(0.5 * (p.y + pm.y), 0.5 * (pm.x - p.x));  // (P - conj Pm) / (2 i)
            if (act && i + 1 < a.per) {  // next pair
                p = __ldg(w.Zin + (int64_t)((i + 1) >> 1) * a.N + pos);
                pm = __ldg(w.Zin + (int64_t)((i + 1) >> 1) * a.N + mpos);
            }
        }
        const double l = i == 0 ? lb : lq;
        const double2 mx = cmul(M, x);
        x = make_double2(fma(l, y.x, mx.x), fma(l, y.y, mx.y));
        xbuf[(i & 1) * T + t] = x;
        __syncthreads();
        if (t < ncl) {
            const double2* xb = xbuf + (i & 1) * T + sb;
            double2 sum = make_double2(0.0, 0.0);
            for (int e = 0; e < a.sx; ++e) {
                const double2 v = xb[e * cps];
                sum.x += v.x;
                sum.y += v.y;
            }
            bad_f |= !isfinite(sum.x + sum.y);
            sums[i * ncl + t] = sum;
        }
    }
    __syncthreads();
    const int r = t % a.RL;
    const int mycl = (t / a.RL) * cps + r % cps;
    double2 z = make_double2(0.0, 0.0), odd = z;
    for (int i = a.per - 1; i >= 0; --i) {
        const double2 mz = cmulc(M, z);
        z = mz;
        if (__ldg(a.slot + i) >= 0) {
            const double2 sum = sums[i * ncl + mycl];
            z = make_double2(fma(scale, sum.x, mz.x), fma(scale, sum.y, mz.y));
        }
        const double l = i == 0 ? lb : lq;
        const double2 o = make_double2(l * z.x, l * z.y);
        if (i & 1) {
            odd = o;
        } else {  // lam z_2a + i lam z_2a+1
            if (act) w.Zout[(int64_t)(i >> 1) * a.N + pos] = make_double2(o.x - odd.y, o.y + odd.x);
            odd = make_double2(0.0, 0.0);
        }
    }
    const bool bad_a = !isfinite(z.x + z.y);
    if (a.status && (bad_f || bad_a)) atomicOr(a.status, (bad_f ? ST_FWD_NONFINITE : 0u) | (bad_a ? ST_ADJ_NONFINITE : 0u));
}

size_t smem_for(int sx, int per) {
    return sizeof(double2) * ((size_t)(kDepth + 2) * kSpecThreads + (size_t)per * (kSpecThreads / sx));
}

}  // namespace

bool spectral_window_supported(int sx, int RL, int per) {
    if (sx < 1 || RL <= 0 || RL % sx != 0 || kSpecThreads % RL != 0) return false;
    return smem_for(sx, per) <= 200 * 1024;
}

void spectral_window(const SpectralArgs& a, cudaStream_t st) {
    require(spectral_window_supported(a.sx, a.RL, a.per) && a.N % a.RL == 0,
            "spectral window: unsupported network or window");
    require(a.npc <= 65535, "spectral window: too many columns");
    if (a.npc == 0) return;
    const size_t smem = smem_for(a.sx, a.per);
    static bool attr = false;
    if (!attr) {
        W4_CUDA(cudaFuncSetAttribute(spectral_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    const dim3 grid((unsigned)cdiv(a.N, (int64_t)kSpecThreads), (unsigned)a.npc);
    spectral_window_kernel<<<grid, kSpecThreads, smem, st>>>(a);
    W4_LAUNCH();
}

void spectral_window1(const SpectralArgs& a, const double2* Zin, double2* Zout, int N1, int N2, const int (&rad)[4],
                      int nrad, cudaStream_t st) {
    require(spectral_window_supported(a.sx, a.RL, a.per) && a.N % a.RL == 0,
            "spectral window: unsupported network or window");
    Window1Args w;
    w.Zin = Zin;
    w.Zout = Zout;
    w.npk = (a.per + 1) / 2;
    w.N1 = N1;
    w.N2 = N2;
    for (int i = 0; i < 4; ++i) w.rad[i] = rad[i];
    w.nrad = nrad;
    // 160-thread CTAs where the row radix allows (five warps hold whole frequency-class groups
    // for RL = 10 and 20): the per-block barrier then spans half as many warps; the class sums
    // and recurrences are per thread / per class, so the CTA width never changes a bit
    static const int t_env = [] {
        const char* e = std::getenv("WC4DVAR_SPECTRAL_W1T");
        return e ? std::atoi(e) : 0;
    }();
    int T1 = (160 % a.RL == 0 && 160 % a.sx == 0) ? 160 : kSpecThreads;
    if (t_env == kSpecThreads) T1 = kSpecThreads;
    const size_t smem = sizeof(double2) * ((size_t)2 * T1 + (size_t)a.per * (T1 / a.sx));
    static bool attr = false;
    if (!attr) {
        W4_CUDA(cudaFuncSetAttribute(spectral_window1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    spectral_window1_kernel<<<(unsigned)cdiv(a.N, (int64_t)T1), T1, smem, st>>>(a, w);
    W4_LAUNCH();
}

}  // namespace w4
