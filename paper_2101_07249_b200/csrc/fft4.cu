// Fused four-step FFT for the circulant D^{1/2} (EXTENSION, BASELINE configs 3-5).
//
// D^{1/2} of a periodic-grid SOAR factor is a circulant convolution whose spectrum lam is
// real and even.  Two real window columns x1, x2 that use the same factor therefore go
// through ONE complex transform: z = x1 + i x2, D^{1/2}x1 = Re IFFT(lam FFT z),
// D^{1/2}x2 = Im IFFT(lam FFT z).  The length-N transform is the four-step split
// N = N1 N2 (index n = n1 + N1 n2, frequency k = k2 + N2 k1):
//   pass A   : per n1, FFT_N2 over n2 (strided gather), times w_N^{n1 k2}        -> Y
//   pass B   : per k2, FFT_N1 over n1, times lam[k2 + N2 k1], IFFT_N1, times
//              w_N^{-n1 k2}                                                      -> Y (in place)
//   pass A^-1: per n1, IFFT_N2 over k2, / N, real / imaginary parts (+ v) -> two outputs
// Every FFT of length <= 4096 runs in SMEM as Stockham radix-{8,5,4,3,2} stages.  HBM sees
// three read + write passes over the (complex) pair data instead of the ~7 of
// D2Z -> product -> Z2D with multi-pass library FFTs.
#include "fft4.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace w4 {
namespace {

constexpr int kFftThreads = 512;
constexpr int kFftMaxElems = 4096;  // cnt * L per CTA (bounds the per-thread butterflies)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
__device__ __forceinline__ double2 rot(double2 a, bool inv) {
    return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// DFT_R of v in place: X_k = sum_r v_r exp(-+2 pi i r k / R)  (- forward, + inverse)
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R], bool inv);

template <>
__device__ __forceinline__ void dft<2>(double2 (&v)[2], bool) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}
template <>
__device__ __forceinline__ void dft<4>(double2 (&v)[4], bool inv) {
    const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const double2 t2 = cadd(v[1], v[3]), t3 = rot(csub(v[1], v[3]), inv);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
}
template <>
__device__ __forceinline__ void dft<8>(double2 (&v)[8], bool inv) {
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft<4>(e, inv);
    dft<4>(o, inv);
    constexpr double h = 0.70710678118654752440;  // 1/sqrt(2)
    // o_k *= w8^k, w8 = exp(-+ i pi / 4)
    const double sg = inv ? 1.0 : -1.0;
    o[1] = make_double2(h * (o[1].x - sg * o[1].y), h * (o[1].y + sg * o[1].x));
    o[2] = rot(o[2], inv);
    o[3] = make_double2(h * (-o[3].x - sg * o[3].y), h * (-o[3].y + sg * o[3].x));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 4] = csub(e[k], o[k]);
    }
}
template <>
__device__ __forceinline__ void dft<3>(double2 (&v)[3], bool inv) {
    constexpr double s = 0.86602540378443864676;  // sin(2 pi / 3)
    const double2 t1 = cadd(v[1], v[2]), t2 = csub(v[1], v[2]);
    const double2 m1 = make_double2(v[0].x - 0.5 * t1.x, v[0].y - 0.5 * t1.y);
    const double2 m2 = rot(make_double2(s * t2.x, s * t2.y), inv);
    v[0] = cadd(v[0], t1);
    v[1] = cadd(m1, m2);
    v[2] = csub(m1, m2);
}
template <>
__device__ __forceinline__ void dft<5>(double2 (&v)[5], bool inv) {
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;  // cos 2pi/5, cos 4pi/5
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;   // sin 2pi/5, sin 4pi/5
    const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    const double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const double2 x0 = v[0];
    const double2 a1 = make_double2(x0.x + c1 * t1.x + c2 * t2.x, x0.y + c1 * t1.y + c2 * t2.y);
    const double2 a2 = make_double2(x0.x + c2 * t1.x + c1 * t2.x, x0.y + c2 * t1.y + c1 * t2.y);
    const double2 b1 = rot(make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y), inv);
    const double2 b2 = rot(make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y), inv);
    v[0] = make_double2(x0.x + t1.x + t2.x, x0.y + t1.y + t2.y);
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
}

// SMEM slot of sequence element i: one pad slot per 8 elements, so the stride-R writes of
// a Stockham stage (Ns = 1: consecutive butterflies write 8 R bytes apart) spread over all
// eight 16-byte bank groups instead of piling on one.
__device__ __forceinline__ int pd(int i) { return i + (i >> 3); }

// One Stockham stage over cnt SMEM sequences (row stride LS): read every butterfly's
// inputs, barrier, write the outputs in place.  MAXB bounds butterflies per thread:
// cnt * L / R <= MAXB * kFftThreads.
template <int R, int MAXB>
__device__ __noinline__ void fft_stage(double2* buf, int cnt, int L, int LS, int Ns,
                                          const double2* __restrict__ tw, bool inv) {
    const int tid = threadIdx.x;
    const int nb = L / R, total = cnt * nb;
    double2 v[MAXB][R];
    int dst[MAXB], row[MAXB];
#pragma unroll
    for (int b = 0; b < MAXB; ++b) {
        const int q = tid + b * kFftThreads;
        dst[b] = -1;
        if (q < total) {
            const int s = q / nb, j = q - s * nb;
            const int jm = j % Ns;
            const double2* src = buf + s * LS;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double2 x = src[pd(j + r * nb)];
                if (r > 0 && Ns > 1) {
                    double2 w = __ldg(tw + jm * R + r);
                    if (inv) w.y = -w.y;
                    x = cmul(x, w);
                }
                v[b][r] = x;
            }
            dft<R>(v[b], inv);
            dst[b] = (j - jm) * R + jm;  // (j / Ns) Ns R + j % Ns
            row[b] = s * LS;
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < MAXB; ++b)
        if (dst[b] >= 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) buf[row[b] + pd(dst[b] + r * Ns)] = v[b][r];
        }
    __syncthreads();
}

__device__ void fft_seq(double2* buf, const SeqPlan& p, int LS, bool inv) {
    for (int s = 0; s < p.nst; ++s) {
        const int R = p.radix[s], Ns = p.ns[s];
        const double2* tw = p.tw[s];
        switch (R) {
            // MAXB = ceil(kFftMaxElems / (R kFftThreads))
            case 8: fft_stage<8, 1>(buf, p.cnt, p.L, LS, Ns, tw, inv); break;
            case 5: fft_stage<5, 2>(buf, p.cnt, p.L, LS, Ns, tw, inv); break;
            case 4: fft_stage<4, 2>(buf, p.cnt, p.L, LS, Ns, tw, inv); break;
            case 3: fft_stage<3, 3>(buf, p.cnt, p.L, LS, Ns, tw, inv); break;
            default: fft_stage<2, 4>(buf, p.cnt, p.L, LS, Ns, tw, inv); break;
        }
    }
}

// w_N^{p}, p in [0, N): hi[p >> 10] * lo[p & 1023]
__device__ __forceinline__ double2 twiddle_n(int64_t p, const double2* __restrict__ lo,
                                             const double2* __restrict__ hi, bool conj) {
    double2 w = cmul(__ldg(hi + (p >> 10)), __ldg(lo + (p & 1023)));
    if (conj) w.y = -w.y;
    return w;
}

// window column c of the (Nsw+1)m view
__device__ __forceinline__ int64_t vcol(int64_t c, int per, int64_t ld, int64_t n) {
    return (c / per) * ld + (c % per) * n;
}

struct PassArgs {
    SeqPlan p;        // the length this pass transforms
    int N1, N2;
    int64_t N;
    const int2* pairs;
    int per;
    const double2* tlo;
    const double2* thi;
};

// Element loops run in batches of kB per thread with every load of the batch issued before
// the first use (kB * kFftThreads = kFftMaxElems covers a whole CTA tile in one batch), so
// each thread keeps kB global requests in flight instead of one.
constexpr int kB = kFftMaxElems / kFftThreads;

__global__ void __launch_bounds__(kFftThreads, 1) fft4_pass_a(const PassArgs pa, const double* __restrict__ V,
                                                            int64_t ldv, double2* __restrict__ Y) {
    extern __shared__ double2 fsm[];
    __shared__ SeqPlan sp;
    if (threadIdx.x == 0) sp = pa.p;
    const int cnt = pa.p.cnt, L = pa.p.L, LS = pd(L) + 1, total = cnt * L;
    const int a0 = blockIdx.x * cnt, na = min(cnt, pa.N1 - a0);
    const int2 cp = pa.pairs[blockIdx.y];
    const double* x1 = V + vcol(cp.x, pa.per, ldv, pa.N);
    const double* x2 = cp.y >= 0 ? V + vcol(cp.y, pa.per, ldv, pa.N) : x1;
    const bool two = cp.y >= 0;
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double2 z[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int a = idx % cnt, n2 = idx / cnt;
            const bool ok = idx < total && a < na;
            const int64_t g = ok ? a0 + a + (int64_t)pa.N1 * n2 : 0;
            z[u] = make_double2(ok ? x1[g] : 0.0, ok && two ? x2[g] : 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            if (idx < total) fsm[(idx % cnt) * LS + pd(idx / cnt)] = z[u];
        }
    }
    __syncthreads();
    fft_seq(fsm, sp, LS, false);
    double2* Yp = Y + (int64_t)blockIdx.y * pa.N;
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double2 w[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {  // n1 k2 < N: no reduction needed
            const int idx = base + u * kFftThreads;
            const int64_t a = idx % cnt, k2 = idx / cnt;
            w[u] = idx < total ? twiddle_n((a0 + a) * k2, pa.tlo, pa.thi, false) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int a = idx % cnt, k2 = idx / cnt;
            if (idx < total && a < na) Yp[a0 + a + (int64_t)pa.N1 * k2] = cmul(fsm[a * LS + pd(k2)], w[u]);
        }
    }
}

__global__ void __launch_bounds__(kFftThreads, 1) fft4_pass_b(const PassArgs pa, const double* __restrict__ lamB,
                                                            const double* __restrict__ lamQ, double2* __restrict__ Y) {
    extern __shared__ double2 fsm[];
    __shared__ SeqPlan sp;
    if (threadIdx.x == 0) sp = pa.p;
    const int cnt = pa.p.cnt, L = pa.p.L, LS = pd(L) + 1, total = cnt * L;  // L = N1
    const int k0 = blockIdx.x * cnt, nk = min(cnt, pa.N2 - k0);
    const int2 cp = pa.pairs[blockIdx.y];
    const double* lam = (cp.x % pa.per == 0) ? lamB : lamQ;  // transposed: lamT[k1 + N1 k2]
    double2* Yp = Y + (int64_t)blockIdx.y * pa.N;
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double2 z[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int r = idx / L, n1 = idx - r * L;
            z[u] = (idx < total && r < nk) ? Yp[n1 + (int64_t)L * (k0 + r)] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            if (idx < total) fsm[(idx / L) * LS + pd(idx % L)] = z[u];
        }
    }
    __syncthreads();
    fft_seq(fsm, sp, LS, false);
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double l[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int r = idx / L, k1 = idx - r * L;
            l[u] = (idx < total && r < nk) ? __ldg(lam + k1 + (int64_t)L * (k0 + r)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            if (idx >= total) continue;
            double2& zz = fsm[(idx / L) * LS + pd(idx % L)];
            zz = make_double2(l[u] * zz.x, l[u] * zz.y);
        }
    }
    __syncthreads();
    fft_seq(fsm, sp, LS, true);
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double2 w[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int64_t r = idx / L, n1 = idx - r * L;
            w[u] = idx < total ? twiddle_n(n1 * (k0 + r), pa.tlo, pa.thi, true) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int r = idx / L, n1 = idx - r * L;
            if (idx < total && r < nk) Yp[n1 + (int64_t)L * (k0 + r)] = cmul(fsm[r * LS + pd(n1)], w[u]);
        }
    }
}

__global__ void __launch_bounds__(kFftThreads, 1) fft4_pass_a_inv(const PassArgs pa, const double2* __restrict__ Y,
                                                                double* __restrict__ out, int64_t ldo,
                                                                const double* __restrict__ add, int64_t ldadd,
                                                                unsigned* status) {
    extern __shared__ double2 fsm[];
    __shared__ SeqPlan sp;
    if (threadIdx.x == 0) sp = pa.p;
    const int cnt = pa.p.cnt, L = pa.p.L, LS = pd(L) + 1, total = cnt * L;  // L = N2
    const int a0 = blockIdx.x * cnt, na = min(cnt, pa.N1 - a0);
    const int2 cp = pa.pairs[blockIdx.y];
    const double2* Yp = Y + (int64_t)blockIdx.y * pa.N;
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double2 z[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int a = idx % cnt, k2 = idx / cnt;
            z[u] = (idx < total && a < na) ? Yp[a0 + a + (int64_t)pa.N1 * k2] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            if (idx < total) fsm[(idx % cnt) * LS + pd(idx / cnt)] = z[u];
        }
    }
    __syncthreads();
    fft_seq(fsm, sp, LS, true);
    double* o1 = out + vcol(cp.x, pa.per, ldo, pa.N);
    double* o2 = cp.y >= 0 ? out + vcol(cp.y, pa.per, ldo, pa.N) : nullptr;
    const double* d1 = add ? add + vcol(cp.x, pa.per, ldadd, pa.N) : nullptr;
    const double* d2 = (add && cp.y >= 0) ? add + vcol(cp.y, pa.per, ldadd, pa.N) : nullptr;
    const double inv_n = 1.0 / (double)pa.N;
    bool bad = false;
    for (int base = threadIdx.x; base < total; base += kB * kFftThreads) {
        double ad1[kB], ad2[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {  // addend loads first (out = v + D^{1/2} s, operators.cpp:141)
            const int idx = base + u * kFftThreads;
            const int a = idx % cnt, n2 = idx / cnt;
            const bool ok = idx < total && a < na;
            const int64_t g = ok ? a0 + a + (int64_t)pa.N1 * n2 : 0;
            ad1[u] = (ok && d1) ? d1[g] : 0.0;
            ad2[u] = (ok && d2) ? d2[g] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kFftThreads;
            const int a = idx % cnt, n2 = idx / cnt;
            if (idx >= total || a >= na) continue;
            const int64_t g = a0 + a + (int64_t)pa.N1 * n2;
            const double2 z = fsm[a * LS + pd(n2)];
            double y1 = z.x * inv_n, y2 = z.y * inv_n;
            if (d1) {
                y1 = ad1[u] + y1;
                bad |= !isfinite(y1);
            }
            o1[g] = y1;
            if (o2) {
                if (d2) {
                    y2 = ad2[u] + y2;
                    bad |= !isfinite(y2);
                }
                o2[g] = y2;
            }
        }
    }
    if (status && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, ST_OUT_NONFINITE);
}

// lamT[k1 + N1 k2] = Re spec[min(k, N - k)], k = k2 + N2 k1 (real even spectrum)
__global__ void build_lam_kernel(int64_t N, int N1, int N2, const double2* __restrict__ spec, double* __restrict__ lamT) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k1 = e % N1, k2 = e / N1;
        const int64_t k = k2 + (int64_t)N2 * k1;
        lamT[e] = spec[k <= N - k ? k : N - k].x;
    }
}

bool smooth(int64_t L) {
    for (int r : {2, 3, 5})
        while (L % r == 0) L /= r;
    return L == 1;
}

// radices 8, 5, 4, 3, 2 greedily (largest butterflies first)
bool build_seq(int L, SeqPlan& p, std::vector<double2>& tab, std::vector<int64_t>& offs) {
    p.L = L;
    p.nst = 0;
    p.cnt = std::max(1, std::min(8, kFftMaxElems / L));
    int rem = L, Ns = 1;
    for (int r : {8, 5, 4, 3, 2}) {
        while (rem % r == 0) {
            if (p.nst >= 12) return false;
            p.radix[p.nst] = r;
            p.ns[p.nst] = Ns;
            offs.push_back((int64_t)tab.size());
            const long double two_pi = 6.283185307179586476925286766559L;
            for (int jm = 0; jm < Ns; ++jm)
                for (int q = 0; q < r; ++q) {
                    const int64_t k = ((int64_t)q * jm) % ((int64_t)Ns * r);
                    const long double ang = -two_pi * (long double)k / (long double)(Ns * r);
                    tab.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
                }
            ++p.nst;
            Ns *= r;
            rem /= r;
        }
    }
    return rem == 1;
}

}  // namespace

Fft4::~Fft4() {
    if (tables_) cudaFree(tables_);
    for (double*& l : lam_)
        if (l) cudaFree(l);
}

bool Fft4::init(int64_t N, const double2* const spec_half[4], cudaStream_t st) {
    if (N < 64 || !smooth(N)) return false;
    int best1 = 0;
    const double rt = std::sqrt((double)N);
    for (int64_t d = 2; d <= kFftMaxElems && d < N; ++d) {
        if (N % d) continue;
        const int64_t e = N / d;
        if (e > kFftMaxElems || !smooth(d) || !smooth(e)) continue;
        if (!best1 || std::fabs((double)d - rt) < std::fabs((double)best1 - rt)) best1 = (int)d;
    }
    if (!best1) return false;
    const int N1 = best1, N2 = (int)(N / best1);
    std::vector<double2> tab;
    std::vector<int64_t> o1, o2;
    SeqPlan p1, p2;
    if (!build_seq(N1, p1, tab, o1) || !build_seq(N2, p2, tab, o2)) return false;
    // four-step twiddles w_N^p = hi[p >> 10] * lo[p & 1023]
    const int64_t off_lo = (int64_t)tab.size();
    const long double two_pi = 6.283185307179586476925286766559L;
    for (int q = 0; q < 1024; ++q) {
        const long double ang = -two_pi * (long double)(q % N) / (long double)N;
        tab.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
    const int64_t off_hi = (int64_t)tab.size();
    for (int64_t h = 0; h <= N / 1024; ++h) {
        const long double ang = -two_pi * (long double)((h * 1024) % N) / (long double)N;
        tab.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
    W4_CUDA(cudaMalloc(&tables_, sizeof(double2) * tab.size()));
    W4_CUDA(cudaMemcpyAsync(tables_, tab.data(), sizeof(double2) * tab.size(), cudaMemcpyHostToDevice, st));
    for (int s = 0; s < p1.nst; ++s) p1.tw[s] = tables_ + o1[s];
    for (int s = 0; s < p2.nst; ++s) p2.tw[s] = tables_ + o2[s];
    tw_lo_ = tables_ + off_lo;
    tw_hi_ = tables_ + off_hi;
    for (int i = 0; i < 4; ++i) {
        if (!spec_half[i]) continue;
        W4_CUDA(cudaMalloc(&lam_[i], sizeof(double) * N));
        build_lam_kernel<<<(unsigned)std::min<int64_t>(cdiv(N, 256), 4096), 256, 0, st>>>(N, N1, N2, spec_half[i],
                                                                                            lam_[i]);
        W4_LAUNCH();
    }
    W4_CUDA(cudaStreamSynchronize(st));  // tab is freed on return
    N_ = N;
    N1_ = N1;
    N2_ = N2;
    p1_ = p1;
    p2_ = p2;
    return true;
}

void Fft4::apply(bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                 const double* add, int64_t ldadd, unsigned* status, DevBuf& ybuf, DevBuf& pairbuf,
                 cudaStream_t st) {
    const double* lamB = lam_[inv ? 2 : 0];
    const double* lamQ = lam_[inv ? 3 : 1];
    require(lamB && lamQ, "apply_D_half_inv: inverse factors were not provided");
    const int per = Nsw + 1;
    const int64_t ncols = (int64_t)per * m;
    // pair window columns that use the same factor: the i = 0 blocks (B) and the rest (Q)
    std::vector<int2> pairs;
    for (int kind = 0; kind < 2; ++kind) {
        int64_t pend = -1;
        for (int64_t c = 0; c < ncols; ++c) {
            if ((c % per == 0) != (kind == 0)) continue;
            if (pend < 0) {
                pend = c;
            } else {
                pairs.push_back(make_int2((int)pend, (int)c));
                pend = -1;
            }
        }
        if (pend >= 0) pairs.push_back(make_int2((int)pend, -1));
    }
    const int64_t np = (int64_t)pairs.size();
    require(ncols < (int64_t)1 << 31, "circulant apply: too many columns");
    // the pair table depends only on (m, Nsw): upload once per shape (the caller holds the
    // operator lock, so the cache is not shared between concurrent applies)
    int2* dpairs = pairbuf.get<int2>((size_t)np);
    if (pairs_m_ != m || pairs_per_ != per || pairs_ptr_ != dpairs) {
        W4_CUDA(cudaMemcpyAsync(dpairs, pairs.data(), sizeof(int2) * np, cudaMemcpyHostToDevice, st));
        W4_CUDA(cudaStreamSynchronize(st));  // pairs (pageable) is consumed before it goes away
        pairs_m_ = m;
        pairs_per_ = per;
        pairs_ptr_ = dpairs;
    }
    double2* Y = ybuf.get<double2>((size_t)np * N_);
    PassArgs pa{p2_, N1_, N2_, N_, dpairs, per, tw_lo_, tw_hi_};
    const size_t sm2 = sizeof(double2) * (size_t)p2_.cnt * (p2_.L + p2_.L / 8 + 1);
    const size_t sm1 = sizeof(double2) * (size_t)p1_.cnt * (p1_.L + p1_.L / 8 + 1);
    static bool attr = false;
    if (!attr) {
        W4_CUDA(cudaFuncSetAttribute(fft4_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        W4_CUDA(cudaFuncSetAttribute(fft4_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        W4_CUDA(cudaFuncSetAttribute(fft4_pass_a_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        attr = true;
    }
    const dim3 ga((unsigned)cdiv(N1_, p2_.cnt), (unsigned)np);
    fft4_pass_a<<<ga, kFftThreads, sm2, st>>>(pa, V, ldv, Y);
    W4_LAUNCH();
    PassArgs pb = pa;
    pb.p = p1_;
    const dim3 gb((unsigned)cdiv(N2_, p1_.cnt), (unsigned)np);
    fft4_pass_b<<<gb, kFftThreads, sm1, st>>>(pb, lamB, lamQ, Y);
    W4_LAUNCH();
    fft4_pass_a_inv<<<ga, kFftThreads, sm2, st>>>(pa, Y, out, ldo, add, ldadd, add ? status : nullptr);
    W4_LAUNCH();
}

}  // namespace w4
