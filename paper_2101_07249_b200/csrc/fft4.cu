// Fused four-step FFT convolution for the circulant D^{1/2} (EXTENSION, BASELINE configs 3-5).
//
// D^{1/2} of a periodic-grid SOAR factor is a circulant convolution whose spectrum lam is
// real and even.  Two real window columns x1, x2 that use the same factor therefore go
// through ONE complex transform: z = x1 + i x2, D^{1/2}x1 = Re IFFT(lam FFT z),
// D^{1/2}x2 = Im IFFT(lam FFT z).  The length-N transform is the four-step split
// N = N1 N2 (index j = j1 + N1 j2, frequency k = k2 + N2 k1):
//   pass A : per j1, FFT_N2 over j2 (strided), times w_N^{j1 k2}                  -> Y[j1 + N1 k2]
//   pass B : per k2, FFT_N1 over j1 (contiguous), times lam[k2 + N2 k1] / N,
//            IFFT_N1, times w_N^{-j1 k2}                                           -> Y (in place)
//   pass C : per j1, IFFT_N2 over k2, real / imaginary parts (+ v)                 -> two outputs
//
// B200 design:
//  * ONE persistent kernel runs all three passes as a ticketed dataflow.  Work items are
//    issued in steps {A(g), B(g-1), C(g-2)} over groups g of column pairs; an item waits on
//    a per-group completion counter of the pass before it (all such items hold smaller
//    tickets, so the wait never deadlocks).  Four Y slots rotate, so the working set of
//    a step (4 groups x 16 N bytes) stays in L2: HBM sees one read of V (and of the add
//    term) and one write of the output per column; Y round-trips through L2 only.
//  * Every FFT is a Stockham sequence of register-resident radix-R stages (R in 5..20,
//    composite radices as in-register Cooley-Tukey over hard-coded radix-2/4/5/8
//    butterflies).  The first stage loads straight from global memory and the last stage
//    stores straight to global memory, so a length-L sequence with s stages costs s - 1
//    SMEM exchanges; pass B turns around in registers (forward last stage, spectrum
//    product, inverse first stage) without an exchange.
//  * Stage twiddles w_M^{r jm} come from one w_L^e table per length (only e < ~400 is
//    touched, so it stays in L1) raised to the r-th power in registers; the four-step
//    twiddles w_N^p come from a two-level (p >> 10, p & 1023) table.
//  * 200 threads and <= 64000 B of SMEM per CTA for every item kind; two CTAs per SM (the
//    128-register budget of a radix-20 stage).
#include "fft4.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace w4 {
namespace {

constexpr int kNT = 200;       // threads per CTA (butterfly mapping, every item kind)
constexpr int kThreads = kNT;
constexpr int kCtaPerSm = 2;  // CTAs per SM (register budget)
constexpr int kSlots = 4;     // Y slots in flight (default): A(g) reuses the slot of C(g - 4), two steps earlier

__device__ __forceinline__ void cbar() { __syncthreads(); }

__constant__ double2 c_w400[400];  // exp(-2 pi i e / 400): every in-register DFT twiddle

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// w_R^{e} (conjugated for the inverse), e a compile-time constant after unrolling
template <int R, bool INV>
__device__ __forceinline__ double2 wr(int e) {
    double2 w = c_w400[(e % R) * (400 / R)];
    if (INV) w.y = -w.y;
    return w;
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&v)[R]);

// In-register Cooley-Tukey DFT_{R1 R2}: input n = R2 n1 + n2, output k = k1 + R1 k2.
template <int R1, int R2, bool INV>
__device__ __forceinline__ void dft_ct(double2 (&v)[R1 * R2]) {
    constexpr int R = R1 * R2;
    double2 a[R2][R1];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) a[n2][n1] = v[R2 * n1 + n2];
        dft<R1, INV>(a[n2]);
        if (n2 > 0) {
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) a[n2][k1] = cmul(a[n2][k1], wr<R, INV>(n2 * k1));
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
        double2 b[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) b[n2] = a[n2][k1];
        dft<R2, INV>(b);
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2) v[k1 + R1 * k2] = b[k2];
    }
}

// X_k = sum_r v_r exp(-+2 pi i r k / R)  (- forward, + inverse), in place
template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&v)[R]) {
    if constexpr (R == 2) {
        const double2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
        const double2 t2 = cadd(v[1], v[3]), t3 = rot<INV>(csub(v[1], v[3]));
        v[0] = cadd(t0, t2);
        v[2] = csub(t0, t2);
        v[1] = cadd(t1, t3);
        v[3] = csub(t1, t3);
    } else if constexpr (R == 5) {
        constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;  // cos 2pi/5, cos 4pi/5
        constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;   // sin 2pi/5, sin 4pi/5
        const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
        const double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
        const double2 x0 = v[0];
        const double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, x0.x)), fma(c2, t2.y, fma(c1, t1.y, x0.y)));
        const double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, x0.x)), fma(c1, t2.y, fma(c2, t1.y, x0.y)));
        const double2 b1 = rot<INV>(make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y)));
        const double2 b2 = rot<INV>(make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y)));
        v[0] = make_double2(x0.x + t1.x + t2.x, x0.y + t1.y + t2.y);
        v[1] = cadd(a1, b1);
        v[4] = csub(a1, b1);
        v[2] = cadd(a2, b2);
        v[3] = csub(a2, b2);
    } else if constexpr (R == 8) {
        double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
        dft<4, INV>(e);
        dft<4, INV>(o);
        constexpr double h = 0.70710678118654752440;  // 1/sqrt(2)
        const double sg = INV ? 1.0 : -1.0;           // o_k *= w8^k, w8 = exp(-+ i pi / 4)
        o[1] = make_double2(h * (o[1].x - sg * o[1].y), h * (o[1].y + sg * o[1].x));
        o[2] = rot<INV>(o[2]);
        o[3] = make_double2(h * (-o[3].x - sg * o[3].y), h * (-o[3].y + sg * o[3].x));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = cadd(e[k], o[k]);
            v[k + 4] = csub(e[k], o[k]);
        }
    } else if constexpr (R == 10) {
        dft_ct<2, 5, INV>(v);
    } else if constexpr (R == 16) {
        dft_ct<4, 4, INV>(v);
    } else if constexpr (R == 20) {
        dft_ct<4, 5, INV>(v);
    } else if constexpr (R == 25) {
        dft_ct<5, 5, INV>(v);
    } else {
        static_assert(R == 0, "unsupported radix");
    }
}

// v[r] *= w^r, r = 1..R-1 (w^r by repeated multiplication: <= R ulp, far inside the
// 1e-12 parity tolerance)
template <int R>
__device__ __forceinline__ void twiddle_pow(double2 (&v)[R], double2 w) {
    double2 c = w;
#pragma unroll
    for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], c);
        if (r + 1 < R) c = cmul(c, w);
    }
}

// ---- tile views --------------------------------------------------------------------
// Column tile (passes A / C): TC sequences (consecutive j1), length L along the strided
// index; SMEM i-major, lanes sequence-fast, so every access is a contiguous run.
template <int L_, int TC>
struct ColView {
    static constexpr int L = L_, S = TC, SMEM = L_ * TC;
    template <int R>
    __device__ static __forceinline__ void map(int q, int& seq, int& j) {
        seq = q % TC;
        j = q / TC;
    }
    __device__ static __forceinline__ int addr(int seq, int i) { return i * TC + seq; }
};
// Row tile (pass B): S contiguous rows of length L; lanes index-fast.  One pad slot per 32
// elements breaks the stride-R store pattern of the first stages.
template <int L_, int S_>
struct RowView {
    static constexpr int L = L_, S = S_, LP = L_ + L_ / 32 + 1, SMEM = S_ * LP;
    template <int R>
    __device__ static __forceinline__ void map(int q, int& seq, int& j) {
        seq = q / (L_ / R);
        j = q - seq * (L_ / R);
    }
    __device__ static __forceinline__ int addr(int seq, int i) { return seq * LP + i + (i >> 5); }
};

template <class V, int R>
struct Shape {
    static constexpr int LR = V::L / R;
    static constexpr int NB = V::S * LR;  // butterflies per stage
    static constexpr int BPT = (NB + kNT - 1) / kNT;
    static constexpr bool FULL = NB % kNT == 0;
};

// ---- Stockham stages ---------------------------------------------------------------
// Stage of radix R after NS = R_0 ... R_{s-1}: butterfly j reads x[j + r L/R], multiplies
// by w_{NS R}^{r (j % NS)}, DFT_R, writes y[(j - j % NS) R + j % NS + r NS].

// first stage (NS = 1): inputs from ld(seq, index)
template <class V, int R, bool INV, class Ld>
__device__ __forceinline__ void stage_first(double2* sm, Ld ld) {
    using SH = Shape<V, R>;
    double2 v[SH::BPT][R];
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
#pragma unroll
            for (int r = 0; r < R; ++r) v[b][r] = ld(seq, j + r * SH::LR);
        }
    }
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
            dft<R, INV>(v[b]);
#pragma unroll
            for (int r = 0; r < R; ++r) sm[V::addr(seq, j * R + r)] = v[b][r];
        }
    }
    cbar();
}

// read + twiddle + DFT of one stage into registers; tw = w_L^e table (w_{NS R}^{jm} =
// w_L^{jm L / (NS R)})
template <class V, int R, int NS, bool INV>
__device__ __forceinline__ void stage_read(const double2* sm, const double2* __restrict__ tw,
                                           double2 (&v)[Shape<V, R>::BPT][R]) {
    using SH = Shape<V, R>;
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
#pragma unroll
            for (int r = 0; r < R; ++r) v[b][r] = sm[V::addr(seq, j + r * SH::LR)];
        }
    }
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
            if (NS > 1) {
                const int jm = j % NS;
                double2 w = __ldg(tw + jm * (V::L / (NS * R)));
                if (INV) w.y = -w.y;
                twiddle_pow<R>(v[b], w);
            }
            dft<R, INV>(v[b]);
        }
    }
}

template <class V, int R, int NS>
__device__ __forceinline__ void stage_write(double2* sm, const double2 (&v)[Shape<V, R>::BPT][R]) {
    using SH = Shape<V, R>;
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
            const int jm = j % NS, base = (j - jm) * R + jm;
#pragma unroll
            for (int r = 0; r < R; ++r) sm[V::addr(seq, base + r * NS)] = v[b][r];
        }
    }
}

template <class V, int R, int NS, bool INV>
__device__ __forceinline__ void stage_mid(double2* sm, const double2* __restrict__ tw) {
    double2 v[Shape<V, R>::BPT][R];
    stage_read<V, R, NS, INV>(sm, tw, v);
    cbar();
    stage_write<V, R, NS>(sm, v);
    cbar();
}

template <int... R>
struct RL {};

template <class V, bool INV, int NS, class List>
struct Mids;
template <class V, bool INV, int NS>
struct Mids<V, INV, NS, RL<>> {
    __device__ static __forceinline__ void run(double2*, const double2*) {}
};
template <class V, bool INV, int NS, int R, int... Rest>
struct Mids<V, INV, NS, RL<R, Rest...>> {
    __device__ static __forceinline__ void run(double2* sm, const double2* tw) {
        stage_mid<V, R, NS, INV>(sm, tw);
        Mids<V, INV, NS * R, RL<Rest...>>::run(sm, tw);
    }
};

// last stage (NS R = L): outputs at index j + r L/R go to st(seq, j, v[R])
template <class V, int R, bool INV, class St>
__device__ __forceinline__ void stage_last(const double2* sm, const double2* __restrict__ tw, St st) {
    using SH = Shape<V, R>;
    double2 v[SH::BPT][R];
    stage_read<V, R, SH::LR, INV>(sm, tw, v);
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
            st(seq, j, v[b]);
        }
    }
}

// forward last stage, spectrum product mul(seq, j, v[R]) on index j + r L/R, inverse first
// stage (same butterfly positions), exchange
template <class V, int R, class Mul>
__device__ __forceinline__ void stage_turn(double2* sm, const double2* __restrict__ tw, Mul mul) {
    using SH = Shape<V, R>;
    double2 v[SH::BPT][R];
    stage_read<V, R, SH::LR, false>(sm, tw, v);
#pragma unroll
    for (int b = 0; b < SH::BPT; ++b) {
        const int q = threadIdx.x + b * kNT;
        if (SH::FULL || q < SH::NB) {
            int seq, j;
            V::template map<R>(q, seq, j);
            mul(seq, j, v[b]);
            dft<R, true>(v[b]);
        }
    }
    cbar();
    stage_write<V, R, 1>(sm, v);
    cbar();
}

// ---- in-place row stages (pass B) ----------------------------------------------------
// Pass B as an in-place Cooley-Tukey sequence: the forward transform is decimation in
// frequency (natural order in, digit-reversed spectrum out), the spectrum product uses a
// lam table stored in that digit-reversed order, and the inverse is decimation in time
// (digit-reversed in, natural order out) -- no permutation anywhere.  Every stage reads
// and writes the SAME slots, so a thread finishes its butterflies (load, DFT, store) with no
// barrier between the reads and the writes: one barrier per stage instead of the two of a
// Stockham stage (pass B: 4 barriers instead of 7).
// Butterfly (seq, b, q) of a stage with radix R and span M owns the row elements
// e = b R M + q + k M, k < R.  DIF: DFT_R, then output k times w_{RM}^{q k}; DIT: input k
// times w_{RM}^{-q k}, then IDFT_R.
template <class V, int R, int M>
struct Ip {
    static constexpr int PR = V::L / R;  // butterflies per row
    static constexpr int NB = V::S * PR;
    __device__ static __forceinline__ void map(int u, int& seq, int& e0, int& q) {
        seq = u / PR;
        const int w = u - seq * PR;
        q = w % M;
        e0 = (w / M) * (R * M) + q;
    }
};

template <class V, int R, int M, bool INV>
__device__ __forceinline__ void ip_stage(double2* sm, const double2* __restrict__ tw) {
    using IP = Ip<V, R, M>;
    constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
    for (int it = 0; it < BPT; ++it) {
        const int u = threadIdx.x + it * kNT;
        if (IP::NB % kNT != 0 && u >= IP::NB) break;
        int seq, e0, q;
        IP::map(u, seq, e0, q);
        double2 v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = sm[V::addr(seq, e0 + k * M)];
        double2 w = make_double2(1.0, 0.0);
        if (M > 1) {
            w = __ldg(tw + q * (V::L / (R * M)));  // w_{RM}^q = w_L^{q L / (R M)}
            if (INV) w.y = -w.y;
        }
        if (INV && M > 1) twiddle_pow<R>(v, w);
        dft<R, INV>(v);
        if (!INV && M > 1) twiddle_pow<R>(v, w);
#pragma unroll
        for (int k = 0; k < R; ++k) sm[V::addr(seq, e0 + k * M)] = v[k];
    }
    cbar();
}

template <class V, bool INV, int M, class List>
struct IpMids;
template <class V, bool INV, int M>
struct IpMids<V, INV, M, RL<>> {
    static constexpr int Mout = M;
    __device__ static __forceinline__ void run(double2*, const double2*) {}
};
// forward (DIF): spans shrink, M -> M / R; inverse (DIT): spans grow, M -> M R
template <class V, int M, int R, int... Rest>
struct IpMids<V, false, M, RL<R, Rest...>> {
    static constexpr int Mout = IpMids<V, false, M / R, RL<Rest...>>::Mout;
    __device__ static __forceinline__ void run(double2* sm, const double2* tw) {
        ip_stage<V, R, M / R, false>(sm, tw);
        IpMids<V, false, M / R, RL<Rest...>>::run(sm, tw);
    }
};
template <class V, int M, int R, int... Rest>
struct IpMids<V, true, M, RL<R, Rest...>> {
    static constexpr int Mout = IpMids<V, true, M * R, RL<Rest...>>::Mout;
    __device__ static __forceinline__ void run(double2* sm, const double2* tw) {
        ip_stage<V, R, M, true>(sm, tw);
        IpMids<V, true, M * R, RL<Rest...>>::run(sm, tw);
    }
};

// ---- plans ---------------------------------------------------------------------------
// N1: contiguous length (pass B, S rows per item), radices B0, BM..., BL (BMr = BM reversed).
// N2: strided length (passes A / C, TC columns per item), radices A0, AM..., AL.
// Columns (N2) take two register stages (one SMEM exchange per pass A / C); rows (N1) three.
struct PlanE6 {  // n = 1e6 (C4): 250 = 10 x 25, 4000 = 20 x 20 x 10
    static constexpr int N1 = 4000, N2 = 250, TC = 16, S = 1;
    static constexpr int A0 = 10, AL = 25, B0 = 20, BL = 10;
    using AM = RL<>;
    using AMr = RL<>;
    using BM = RL<20>;
    using BMr = RL<20>;
};
struct PlanE6c3 {  // n = 1e6, three column stages (10 x 5 x 5): the round-1 plan (variant 1)
    static constexpr int N1 = 4000, N2 = 250, TC = 16, S = 1;
    static constexpr int A0 = 10, AL = 5, B0 = 20, BL = 10;
    using AM = RL<5>;
    using AMr = RL<5>;
    using BM = RL<20>;
    using BMr = RL<20>;
};
struct Plan2E6 {  // n = 2e6 (C5): 500 = 20 x 25, 4000 = 20 x 20 x 10
    static constexpr int N1 = 4000, N2 = 500, TC = 8, S = 1;
    static constexpr int A0 = 20, AL = 25, B0 = 20, BL = 10;
    using AM = RL<>;
    using AMr = RL<>;
    using BM = RL<20>;
    using BMr = RL<20>;
};
struct PlanE5 {  // n = 1e5 (C3): 250 = 10 x 25, 400 = 20 x 20
    static constexpr int N1 = 400, N2 = 250, TC = 16, S = 10;
    static constexpr int A0 = 10, AL = 25, B0 = 20, BL = 20;
    using AM = RL<>;
    using AMr = RL<>;
    using BM = RL<>;
    using BMr = RL<>;
};
struct PlanE4 {  // n = 1e4 (parity tests; partial stages)
    static constexpr int N1 = 400, N2 = 25, TC = 16, S = 5;
    static constexpr int A0 = 5, AL = 5, B0 = 20, BL = 20;
    using AM = RL<>;
    using AMr = RL<>;
    using BM = RL<>;
    using BMr = RL<>;
};

struct Job {
    const double* V;
    int64_t ldv;
    double* out;
    int64_t ldo;
    const double* add;
    int64_t ldadd;
    unsigned* status;
    const int2* pairs;
    int np, per, G, ngroups;
    const double* lamB;  // lamT[k1 + N1 k2] = lam[k2 + N2 k1] / N
    const double* lamQ;
    double2* Y;          // kSlots x G x N
    const double2* tw1;  // w_N1^e
    const double2* tw2;  // w_N2^e
    const double2* tlo;  // w_N^{p & 1023}
    const double2* thi;  // w_N^{(p >> 10) 1024}
    unsigned* ctr;       // [0] ticket, [1 + 3 g + phase] completed items of group g
    int l2hint;          // evict_last policy on Y + discard after pass C (WC4DVAR_FFT_L2HINT)
    int phase_mask;      // profiling aid (WC4DVAR_FFT_PHASES, default 7): passes whose items run
    int sub;             // tiles per ticket (WC4DVAR_FFT_SUB)
    int acq;             // acquire loads on the dependency counters (WC4DVAR_FFT_ACQ, default 1)
    int slots;           // Y slots (WC4DVAR_FFT_SLOTS, default kSlots; >= 3)
    int ipb;             // pass B in place (DIF / DIT, digit-reversed lam); 0 = Stockham
    int prefetch;        // L2 prefetch of the next pass-A tile (WC4DVAR_FFT_PREFETCH, default 0)
    double2* Z;          // spectral modes: np x N spectra in pass B's digit-reversed row order
};

__device__ __forceinline__ double2 wN(const Job& jb, int64_t p) {  // w_N^p, 0 <= p < N
    return cmul(__ldg(jb.thi + (p >> 10)), __ldg(jb.tlo + (p & 1023)));
}

// window column c of the (Nsw+1)m view
__device__ __forceinline__ int64_t vcol(int c, int per, int64_t ld, int64_t n) {
    return (int64_t)(c / per) * ld + (int64_t)(c % per) * n;
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* a) {
    asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(a));
}
// Y traffic stays in L2: stores / in-place loads with an evict_last policy, and pass C
// discards each Y line after its last read (no write-back of dead data)
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_y(const double2* a, uint64_t pol) {
    if (!pol) return __ldcg(a);
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_y(double2* a, double2 v, uint64_t pol) {
    // no memory clobber: the compiler may keep interleaving the SMEM reads of later
    // butterflies with these stores; the volatile cbar() that ends the item orders them
    if (!pol) {
        __stcg(a, v);
        return;
    }
    asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol));
}
__device__ __forceinline__ void discard_l2(const void* a) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}
__device__ __forceinline__ void red_release(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// `af()` runs on every thread right after the first stage (its barrier passed, the stage's
// global loads consumed): the deferred completion release and the next item's L2 prefetch
template <class P, class AF>
__device__ __forceinline__ void item_a(const Job& jb, double2* sm, int p, int tile, AF af) {
    using VA = ColView<P::N2, P::TC>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    const int2 cp = jb.pairs[p];
    const double* x1 = jb.V + vcol(cp.x, jb.per, jb.ldv, N);
    const double* x2 = cp.y >= 0 ? jb.V + vcol(cp.y, jb.per, jb.ldv, N) : nullptr;
    double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int j10 = tile * P::TC;
    const uint64_t pol = jb.l2hint ? policy_evict_last() : 0;
    if (x2) {
        stage_first<VA, P::A0, false>(sm, [&](int seq, int i) {
            const int64_t g = j10 + seq + (int64_t)P::N1 * i;
            return make_double2(__ldcs(x1 + g), __ldcs(x2 + g));
        });
    } else {
        stage_first<VA, P::A0, false>(sm, [&](int seq, int i) {
            return make_double2(__ldcs(x1 + j10 + seq + (int64_t)P::N1 * i), 0.0);
        });
    }
    af();
    Mids<VA, false, P::A0, typename P::AM>::run(sm, jb.tw2);
    constexpr int LR = P::N2 / P::AL;
    stage_last<VA, P::AL, false>(sm, jb.tw2, [&](int seq, int j, double2(&v)[P::AL]) {
        const int64_t j1 = j10 + seq;
        double2 w = wN(jb, j1 * j);
        const double2 ws = wN(jb, j1 * LR);
#pragma unroll
        for (int r = 0; r < P::AL; ++r) {
            st_y(Yp + j1 + (int64_t)P::N1 * (j + r * LR), cmul(v[r], w), pol);
            if (r + 1 < P::AL) w = cmul(w, ws);
        }
    });
}

template <class P, class AF>
__device__ __forceinline__ void item_b(const Job& jb, double2* sm, int p, int rowblk, AF af) {
    using VB = RowView<P::N1, P::S>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    const int2 cp = jb.pairs[p];
    const double* lam = (cp.x % jb.per == 0) ? jb.lamB : jb.lamQ;
    double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int k20 = rowblk * P::S;
    const uint64_t pol = jb.l2hint ? policy_evict_last() : 0;
    stage_first<VB, P::B0, false>(sm, [&](int seq, int i) {
        return ld_y(Yp + (int64_t)P::N1 * (k20 + seq) + i, pol);
    });
    af();
    Mids<VB, false, P::B0, typename P::BM>::run(sm, jb.tw1);
    constexpr int LRt = P::N1 / P::BL;
    stage_turn<VB, P::BL>(sm, jb.tw1, [&](int seq, int j, double2(&v)[P::BL]) {
        const double* lr = lam + (int64_t)P::N1 * (k20 + seq) + j;
#pragma unroll
        for (int r = 0; r < P::BL; ++r) {
            const double l = __ldg(lr + r * LRt);
            v[r] = make_double2(l * v[r].x, l * v[r].y);
        }
    });
    Mids<VB, true, P::BL, typename P::BMr>::run(sm, jb.tw1);
    constexpr int LR = P::N1 / P::B0;
    stage_last<VB, P::B0, true>(sm, jb.tw1, [&](int seq, int j, double2(&v)[P::B0]) {
        const int64_t k2 = k20 + seq;
        double2 w = conj2(wN(jb, j * k2));
        const double2 ws = conj2(wN(jb, LR * k2));
        double2* yr = Yp + (int64_t)P::N1 * k2 + j;
#pragma unroll
        for (int r = 0; r < P::B0; ++r) {
            st_y(yr + r * LR, cmul(v[r], w), pol);
            if (r + 1 < P::B0) w = cmul(w, ws);
        }
    });
}

// pass B, in-place form (see ip_stage); lam is the digit-reversed table (lam_rev_kernel)
template <class P, class AF>
__device__ __forceinline__ void item_b_ip(const Job& jb, double2* sm, int p, int rowblk, AF af) {
    using VB = RowView<P::N1, P::S>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    constexpr int L = P::N1;
    const int2 cp = jb.pairs[p];
    const double* lam = (cp.x % jb.per == 0) ? jb.lamB : jb.lamQ;
    double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int k20 = rowblk * P::S;
    const uint64_t pol = jb.l2hint ? policy_evict_last() : 0;
    // DIF stage 1 (radix B0, span M1 = L / B0): natural-order loads from Y
    {
        constexpr int R = P::B0, M = L / P::B0;
        using IP = Ip<VB, R, M>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            const double2* yr = Yp + (int64_t)P::N1 * (k20 + seq) + e0;
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = ld_y(yr + k * M, pol);
            dft<R, false>(v);
            twiddle_pow<R>(v, __ldg(jb.tw1 + q));  // w_L^{q k}
#pragma unroll
            for (int k = 0; k < R; ++k) sm[VB::addr(seq, e0 + k * M)] = v[k];
        }
        cbar();
    }
    af();
    using FM = IpMids<VB, false, L / P::B0, typename P::BM>;
    FM::run(sm, jb.tw1);
    static_assert(FM::Mout == P::BL, "pass B radices must multiply to N1");
    // last DIF stage (radix BL, span 1) + spectrum product + first DIT stage, in registers
    {
        constexpr int R = P::BL;
        using IP = Ip<VB, R, 1>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = sm[VB::addr(seq, e0 + k)];
            dft<R, false>(v);
            const double* lr = lam + (int64_t)P::N1 * (k20 + seq) + e0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const double l = __ldg(lr + k);
                v[k] = make_double2(l * v[k].x, l * v[k].y);
            }
            dft<R, true>(v);
#pragma unroll
            for (int k = 0; k < R; ++k) sm[VB::addr(seq, e0 + k)] = v[k];
        }
        cbar();
    }
    using IM = IpMids<VB, true, P::BL, typename P::BMr>;
    IM::run(sm, jb.tw1);
    static_assert(IM::Mout == L / P::B0, "pass B radices must multiply to N1");
    // last DIT stage (radix B0, span L / B0): conjugate four-step twiddle, natural-order store
    {
        constexpr int R = P::B0, M = L / P::B0;
        using IP = Ip<VB, R, M>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = sm[VB::addr(seq, e0 + k * M)];
            twiddle_pow<R>(v, conj2(__ldg(jb.tw1 + q)));
            dft<R, true>(v);
            const int64_t k2 = k20 + seq;
            double2 w = conj2(wN(jb, e0 * k2));
            const double2 ws = conj2(wN(jb, M * k2));
            double2* yr = Yp + (int64_t)P::N1 * k2 + e0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                st_y(yr + k * M, cmul(v[k], w), pol);
                if (k + 1 < R) w = cmul(w, ws);
            }
        }
    }
}

// ---- spectral modes (forward-only / inverse-only transforms) -----------------------------
// MODE 1 (forward): passes A and B', where B' is the DIF half of pass B and leaves the
// UNSCALED spectrum of pair p in Z[p N + e + N1 k2] (frequency k2 + N2 f(e), f the digit
// reversal of the row radices).  MODE 2 (inverse): B'' reads such a spectrum, runs the DIT
// half of pass B into the Y slot, pass C finishes.  The window recurrence between the two
// runs on the spectra (spectral.cu).
template <class P, class AF>
__device__ __forceinline__ void item_b_fwd(const Job& jb, double2* sm, int p, int rowblk, AF af) {
    using VB = RowView<P::N1, P::S>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    constexpr int L = P::N1;
    double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int k20 = rowblk * P::S;
    const uint64_t pol = jb.l2hint ? policy_evict_last() : 0;
    {
        constexpr int R = P::B0, M = L / P::B0;
        using IP = Ip<VB, R, M>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            const double2* yr = Yp + (int64_t)P::N1 * (k20 + seq) + e0;
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = ld_y(yr + k * M, pol);
            dft<R, false>(v);
            twiddle_pow<R>(v, __ldg(jb.tw1 + q));
#pragma unroll
            for (int k = 0; k < R; ++k) sm[VB::addr(seq, e0 + k * M)] = v[k];
        }
        cbar();
    }
    af();
    if (jb.l2hint) {  // these Y rows are dead: drop them from L2 without a write-back
        static_assert((P::N1 * 16) % 128 == 0, "rows must cover whole 128-byte lines");
        constexpr int lpr = P::N1 * 16 / 128;
        const char* base = reinterpret_cast<const char*>(Yp + (int64_t)P::N1 * k20);
        for (int e = threadIdx.x; e < P::S * lpr; e += kNT) discard_l2(base + (int64_t)e * 128);
    }
    using FM = IpMids<VB, false, L / P::B0, typename P::BM>;
    FM::run(sm, jb.tw1);
    {
        constexpr int R = P::BL;
        using IP = Ip<VB, R, 1>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
        double2* zp = jb.Z + (int64_t)p * N;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = sm[VB::addr(seq, e0 + k)];
            dft<R, false>(v);
            double2* zr = zp + (int64_t)P::N1 * (k20 + seq) + e0;
#pragma unroll
            for (int k = 0; k < R; ++k) zr[k] = v[k];
        }
    }
}

template <class P, class AF>
__device__ __forceinline__ void item_b_inv(const Job& jb, double2* sm, int p, int rowblk, AF af) {
    using VB = RowView<P::N1, P::S>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    constexpr int L = P::N1;
    double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int k20 = rowblk * P::S;
    const uint64_t pol = jb.l2hint ? policy_evict_last() : 0;
    {
        constexpr int R = P::BL;
        using IP = Ip<VB, R, 1>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
        const double2* zp = jb.Z + (int64_t)p * N;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            const double2* zr = zp + (int64_t)P::N1 * (k20 + seq) + e0;
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = __ldg(zr + k);
            dft<R, true>(v);
#pragma unroll
            for (int k = 0; k < R; ++k) sm[VB::addr(seq, e0 + k)] = v[k];
        }
        cbar();
    }
    af();
    using IM = IpMids<VB, true, P::BL, typename P::BMr>;
    IM::run(sm, jb.tw1);
    {
        constexpr int R = P::B0, M = L / P::B0;
        using IP = Ip<VB, R, M>;
        constexpr int BPT = (IP::NB + kNT - 1) / kNT;
#pragma unroll
        for (int it = 0; it < BPT; ++it) {
            const int u = threadIdx.x + it * kNT;
            if (IP::NB % kNT != 0 && u >= IP::NB) break;
            int seq, e0, q;
            IP::map(u, seq, e0, q);
            double2 v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = sm[VB::addr(seq, e0 + k * M)];
            twiddle_pow<R>(v, conj2(__ldg(jb.tw1 + q)));
            dft<R, true>(v);
            const int64_t k2 = k20 + seq;
            double2 w = conj2(wN(jb, e0 * k2));
            const double2 ws = conj2(wN(jb, M * k2));
            double2* yr = Yp + (int64_t)P::N1 * k2 + e0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                st_y(yr + k * M, cmul(v[k], w), pol);
                if (k + 1 < R) w = cmul(w, ws);
            }
        }
    }
}

template <class P, bool ADD, class AF>
__device__ __forceinline__ void item_c(const Job& jb, double2* sm, int p, int tile, AF af) {
    using VA = ColView<P::N2, P::TC>;
    constexpr int64_t N = (int64_t)P::N1 * P::N2;
    const int2 cp = jb.pairs[p];
    const double2* Yp = jb.Y + ((int64_t)((p / jb.G) % jb.slots) * jb.G + p % jb.G) * N;
    const int j10 = tile * P::TC;
    stage_first<VA, P::AL, true>(sm, [&](int seq, int i) {
        return __ldcg(Yp + j10 + seq + (int64_t)P::N1 * i);
    });
    af();
    if (jb.l2hint) {  // this tile's Y lines are dead: drop them from L2 without a write-back
        static_assert((P::TC * 16) % 128 == 0, "column tile must cover whole 128-byte lines");
        constexpr int lpr = P::TC * 16 / 128;
        const char* base = reinterpret_cast<const char*>(Yp + j10);
        for (int e = threadIdx.x; e < P::N2 * lpr; e += kNT)
                discard_l2(base + (int64_t)(e / lpr) * P::N1 * 16 + (e % lpr) * 128);
    }
    Mids<VA, true, P::AL, typename P::AMr>::run(sm, jb.tw2);
    double* o1 = jb.out + vcol(cp.x, jb.per, jb.ldo, N) + j10;
    double* o2 = cp.y >= 0 ? jb.out + vcol(cp.y, jb.per, jb.ldo, N) + j10 : nullptr;
    const double* d1 = ADD ? jb.add + vcol(cp.x, jb.per, jb.ldadd, N) + j10 : nullptr;
    const double* d2 = (ADD && cp.y >= 0) ? jb.add + vcol(cp.y, jb.per, jb.ldadd, N) + j10 : nullptr;
    constexpr int LR = P::N2 / P::A0;
    bool bad = false;
    stage_last<VA, P::A0, true>(sm, jb.tw2, [&](int seq, int j, double2(&v)[P::A0]) {
        // add-term loads issued in chunks of CH ahead of the chunk's stores (out may alias
        // add, so the compiler cannot hoist them across the stores itself; CH <= 10 bounds the
        // registers they hold)
        constexpr int CH = P::A0 <= 10 ? P::A0 : (P::A0 % 10 == 0 ? 10 : 5);
#pragma unroll
        for (int r0 = 0; r0 < P::A0; r0 += CH) {
            double a1[CH], a2[CH];
            if (ADD) {
#pragma unroll
                for (int r = 0; r < CH; ++r) {
                    const int64_t g = seq + (int64_t)P::N1 * (j + (r0 + r) * LR);
                    a1[r] = __ldcs(d1 + g);
                    a2[r] = d2 ? __ldcs(d2 + g) : 0.0;
                }
            }
#pragma unroll
            for (int r = 0; r < CH; ++r) {
                const int64_t g = seq + (int64_t)P::N1 * (j + (r0 + r) * LR);
                double y1 = v[r0 + r].x, y2 = v[r0 + r].y;
                if (ADD) {  // out = v + D^{1/2} s (operators.cpp:141)
                    y1 = a1[r] + y1;
                    bad |= !isfinite(y1);
                }
                __stcs(o1 + g, y1);
                if (o2) {
                    if (ADD && d2) {
                        y2 = a2[r] + y2;
                        bad |= !isfinite(y2);
                    }
                    __stcs(o2 + g, y2);
                }
            }
        }
    });
    if (ADD && jb.status && bad) atomicOr(jb.status, ST_OUT_NONFINITE);
}

// MODE 0: the full convolution (A, B, C).  MODE 1: forward transform (A, B'); MODE 2: inverse
// transform (B'', C) -- the phase a mode lacks has no tickets.
template <class P, int CPS, bool ADD, bool IPB, int MODE>
__global__ void __launch_bounds__(kThreads, CPS) fftconv_kernel(const Job jb) {
    extern __shared__ double2 sm[];
    __shared__ unsigned s_ticket, s_next;
    // a ticket covers `sub` consecutive tiles (A / C) or row blocks (B) of one pair: fewer
    // tickets, so the per-ticket cost (ticket atomic, dependency read, two barriers, the
    // completion release) is paid once per `sub` tiles
    constexpr int tA = P::N1 / P::TC, tB = P::N2 / P::S;  // tiles / row blocks per pair
    const int nA1 = (tA + jb.sub - 1) / jb.sub, nB1 = (tB + jb.sub - 1) / jb.sub;  // tickets per pair
    const int nA = MODE == 2 ? 0 : jb.G * nA1, nB = jb.G * nB1, nC = MODE == 1 ? 0 : jb.G * nA1;
    const unsigned stepN = (unsigned)(nA + nB + nC);
    const unsigned total = stepN * (unsigned)(jb.ngroups + 2);
    // decode ticket t into (phase, group, item): step s = {A(s), B(s - 1), C(s - 2)}
    auto decode = [&](unsigned t, int& phase, int& g, int& r) {
        const int s = (int)(t / stepN);
        r = (int)(t - (unsigned)s * stepN);
        if (r < nA) {
            phase = 0;
            g = s;
        } else if (r < nA + nB) {
            phase = 1;
            g = s - 1;
            r -= nA;
        } else {
            phase = 2;
            g = s - 2;
            r -= nA + nB;
        }
    };
    // counter item t waits for: A(g) reuses the Y slot of C(g - kSlots); B(g) needs A(g);
    // C(g) needs B(g).  Every awaited item holds a smaller ticket, and a CTA holds at most
    // one unstarted (prefetched) ticket while it runs a smaller one, so the smallest
    // unfinished ticket always progresses: no deadlock (the deferred release below is
    // flushed before any wait that is not already satisfied).
    auto dependency = [&](unsigned t, const unsigned*& dep, unsigned& need) {
        dep = nullptr;
        need = 0;
        if (t >= total) return;
        int phase, g, r;
        decode(t, phase, g, r);
        if (g < 0 || g >= jb.ngroups) return;
        if (phase == 0 && g >= jb.slots) {  // slot reuse: its last reader is C (B' when forward-only)
            dep = jb.ctr + 1 + 3 * (g - jb.slots) + (MODE == 1 ? 1 : 2);
            need = (unsigned)(MODE == 1 ? nB : nC);
        } else if (phase == 1 && MODE == 2) {
            if (g >= jb.slots) {
                dep = jb.ctr + 1 + 3 * (g - jb.slots) + 2;
                need = (unsigned)nC;
            }
        } else if (phase == 1) {
            dep = jb.ctr + 1 + 3 * g + 0;
            need = (unsigned)nA;
        } else if (phase == 2) {
            dep = jb.ctr + 1 + 3 * g + 1;
            need = (unsigned)nB;
        }
    };
    // thread 0 owns the schedule: `next` is fetched one item ahead and its dependency
    // counter is read (acquire) at the end of the current item, so both round trips overlap
    // work.  The completion release of an item is DEFERRED to just after the first stage of
    // the following item: its MEMBAR then finds no outstanding global traffic of this warp
    // instead of draining the item's last-stage stores while the whole CTA waits.
    unsigned next = 0, seen = 0, need = 0;
    const unsigned* dep = nullptr;
    unsigned* pend = nullptr;
    if (threadIdx.x == 0) {
        next = atomicAdd(jb.ctr, 1u);
        dependency(next, dep, need);
        if (dep) seen = jb.acq ? ld_acquire(dep) : ld_relaxed(dep);
    }
    auto flush = [&]() {
        if (threadIdx.x == 0 && pend) {
            red_release(pend);
            pend = nullptr;
        }
    };
    auto after_first = [&]() {
        flush();
        if (!jb.prefetch) return;
        // L2 prefetch of the next item's HBM input (pass A reads V; B / C read L2-resident Y)
        int ph, g, r;
        const unsigned nt = s_next;
        if (nt >= total) return;
        decode(nt, ph, g, r);
        if (ph != 0 || g < 0 || g >= jb.ngroups) return;
        const int p = g * jb.G + r / nA1;
        if (p >= jb.np) return;
        const int2 cp = jb.pairs[p];
        constexpr int64_t N = (int64_t)P::N1 * P::N2;
        const int j10 = (r % nA1) * jb.sub * P::TC;
        const int lines = P::TC * 8 / 128 * jb.sub;  // 128-byte lines per row of the tile(s)
        for (int e = threadIdx.x; e < P::N2 * lines * 2; e += kNT) {
            const int col = e & 1, row = (e >> 1) / lines, l = (e >> 1) % lines;
            const int c = col ? cp.y : cp.x;
            if (c >= 0) prefetch_l2(jb.V + vcol(c, jb.per, jb.ldv, N) + j10 + (int64_t)P::N1 * row + l * 16);
        }
    };
    for (;;) {
        if (threadIdx.x == 0) {
            if (dep && seen < need) {
                if (pend) {  // never wait while holding an unreleased item
                    red_release(pend);
                    pend = nullptr;
                }
                do {
                    __nanosleep(64);
                    seen = jb.acq ? ld_acquire(dep) : ld_relaxed(dep);
                } while (seen < need);
            }
            s_ticket = next;
        }
        // Y is written with st.cg, published by red.release and read with ld.cg (L2) only
        // after thread 0's acquire load observed the counter and this barrier
        __syncthreads();
        const unsigned t = s_ticket;
        if (t >= total) break;
        if (threadIdx.x == 0) {
            next = atomicAdd(jb.ctr, 1u);
            s_next = next;  // read by after_first() behind the first stage's barrier
        }
        int phase, g, r;
        decode(t, phase, g, r);
        const bool valid = g >= 0 && g < jb.ngroups;
        bool ran = false;
        if (valid) {
            // pair index and the item inside it; groups are G consecutive pairs
            const int per_pair = phase == 1 ? nB1 : nA1;
            const int p = g * jb.G + r / per_pair, idx = r % per_pair;
            if (p < jb.np && ((jb.phase_mask >> phase) & 1)) {  // the last group may be partial
                const int u0 = idx * jb.sub, u1 = min(u0 + jb.sub, phase == 1 ? tB : tA);
                ran = true;
                for (int u = u0; u < u1; ++u) {
                    if (u > u0) __syncthreads();  // the previous tile's last stage read SMEM
                    if (phase == 0) {
                        item_a<P>(jb, sm, p, u, after_first);
                    } else if (phase == 1) {
                        if (MODE == 1) item_b_fwd<P>(jb, sm, p, u, after_first);
                        else if (MODE == 2) item_b_inv<P>(jb, sm, p, u, after_first);
                        else if (IPB) item_b_ip<P>(jb, sm, p, u, after_first);
                        else item_b<P>(jb, sm, p, u, after_first);
                    } else {
                        item_c<P, ADD>(jb, sm, p, u, after_first);
                    }
                }
            }
        }
        if (!ran) flush();  // no first stage ran: release the deferred item now
        if (threadIdx.x == 0) {
            dependency(next, dep, need);
            if (dep) seen = jb.acq ? ld_acquire(dep) : ld_relaxed(dep);
        }
        __syncthreads();  // every store of the item issued; s_ticket read; SMEM free
        if (threadIdx.x == 0 && valid) pend = jb.ctr + 1 + 3 * g + phase;
    }
    if (threadIdx.x == 0 && pend) red_release(pend);
}

// lamT[k1 + N1 k2] = Re spec[min(k, N - k)] / N, k = k2 + N2 k1 (real even spectrum)
__global__ void build_lam_kernel(int64_t N, int N1, int N2, const double2* __restrict__ spec, double* __restrict__ lamT) {
    const double inv_n = 1.0 / (double)N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k1 = e % N1, k2 = e / N1;
        const int64_t k = k2 + (int64_t)N2 * k1;
        lamT[e] = spec[k <= N - k ? k : N - k].x * inv_n;
    }
}

// in-place pass B: lamR[e + N1 k2] = lam at row frequency f(e), the digit reversal of the
// DIF radix sequence rad[0..nr) (rad[0] first): e = sum d_i M_i (M_i = span of stage i),
// f = sum d_i P_i (P_i = rad[0] ... rad[i-1])
struct Radices {
    int r[4];
    int n;
};
__global__ void build_lam_rev_kernel(int64_t N, int N1, int N2, Radices rd, const double2* __restrict__ spec,
                                     double* __restrict__ lamR) {
    const double inv_n = 1.0 / (double)N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(t % N1);
        const int64_t k2 = t / N1;
        int span = N1, pw = 1, f = 0;
        for (int i = 0; i < rd.n; ++i) {
            span /= rd.r[i];
            f += ((e / span) % rd.r[i]) * pw;
            pw *= rd.r[i];
        }
        const int64_t k = k2 + (int64_t)N2 * f;
        lamR[t] = spec[k <= N - k ? k : N - k].x * inv_n;
    }
}

template <class P>
constexpr size_t smem_bytes() {
    return sizeof(double2) * (size_t)std::max(ColView<P::N2, P::TC>::SMEM, RowView<P::N1, P::S>::SMEM);
}

template <class P, int CPS, bool ADD, bool IPB, int MODE>
void launch_cps(const Job& jb, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<P>();
    static_assert(sm <= 227 * 1024 / 2, "fftconv tile exceeds the per-CTA SMEM budget");
    static bool attr = false;
    if (!attr) {
        W4_CUDA(cudaFuncSetAttribute(fftconv_kernel<P, CPS, ADD, IPB, MODE>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
    }
    int dev = 0, nsm = kSMs, occ = 0;
    W4_CUDA(cudaGetDevice(&dev));
    W4_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    W4_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fftconv_kernel<P, CPS, ADD, IPB, MODE>, kThreads, sm));
    const int64_t items = (int64_t)(jb.ngroups + 2) * jb.G *
                          (2 * ((P::N1 / P::TC + jb.sub - 1) / jb.sub) + (P::N2 / P::S + jb.sub - 1) / jb.sub);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)nsm * std::max(occ, 1)));
    fftconv_kernel<P, CPS, ADD, IPB, MODE><<<grid, kThreads, sm, st>>>(jb);
    W4_LAUNCH();
}

// Two CTAs per SM (128 registers).  Measured and dropped: one CTA per SM (~250 registers,
// no spills: 19.7-20.6 vs 13.7 ms per C4 m = 64 D^{1/2}) and three (~104 registers, heavy
// spills: 23.7 vs 13.0 ms).
template <class P>
void launch(const Job& jb, cudaStream_t st) {
    if (jb.ipb) return jb.add ? launch_cps<P, 2, true, true, 0>(jb, st) : launch_cps<P, 2, false, true, 0>(jb, st);
    return jb.add ? launch_cps<P, 2, true, false, 0>(jb, st) : launch_cps<P, 2, false, false, 0>(jb, st);
}
template <class P>
void launch_fwd(const Job& jb, cudaStream_t st) {
    launch_cps<P, 2, false, true, 1>(jb, st);
}
template <class P>
void launch_inv(const Job& jb, cudaStream_t st) {
    return jb.add ? launch_cps<P, 2, true, true, 2>(jb, st) : launch_cps<P, 2, false, true, 2>(jb, st);
}

struct PlanInfo {
    int variant;  // WC4DVAR_FFT_VARIANT selects among plans of the same length (0 = default)
    Radices brad; // pass-B (row) DIF radices, first stage first
    int64_t N1, N2;
    size_t smem;
    void (*run)(const Job&, cudaStream_t);
    void (*run_fwd)(const Job&, cudaStream_t);  // spectral modes
    void (*run_inv)(const Job&, cudaStream_t);
};
#define W4_PLAN(P) P::N1, P::N2, smem_bytes<P>(), launch<P>, launch_fwd<P>, launch_inv<P>
const PlanInfo kPlans[] = {
    {0, {{20, 20, 10, 0}, 3}, W4_PLAN(PlanE6)},
    {1, {{20, 20, 10, 0}, 3}, W4_PLAN(PlanE6c3)},
    {0, {{20, 20, 10, 0}, 3}, W4_PLAN(Plan2E6)},
    {0, {{20, 20, 0, 0}, 2}, W4_PLAN(PlanE5)},
    {0, {{20, 20, 0, 0}, 2}, W4_PLAN(PlanE4)},
};
#undef W4_PLAN

}  // namespace

Fft4::~Fft4() {
    if (tables_) cudaFree(tables_);
    for (double*& l : lam_)
        if (l) cudaFree(l);
}

bool Fft4::init(int64_t N, const double2* const spec_half[4], cudaStream_t st) {
    int plan = -1;
    static const int variant = [] {
        const char* e = std::getenv("WC4DVAR_FFT_VARIANT");
        return e ? std::atoi(e) : 0;
    }();
    for (int i = 0; i < (int)(sizeof(kPlans) / sizeof(kPlans[0])); ++i)
        if (kPlans[i].N1 * kPlans[i].N2 == N && (plan < 0 || kPlans[i].variant == variant)) plan = i;
    if (plan < 0) return false;
    const int64_t N1 = kPlans[plan].N1, N2 = kPlans[plan].N2;
    const long double two_pi = 6.283185307179586476925286766559L;
    // in-register DFT twiddles (constant bank), once per process
    static bool cw = false;
    if (!cw) {
        double2 w[400];
        for (int e = 0; e < 400; ++e) {
            const long double a = -two_pi * (long double)e / 400.0L;
            w[e] = make_double2((double)cosl(a), (double)sinl(a));
        }
        W4_CUDA(cudaMemcpyToSymbol(c_w400, w, sizeof(w)));
        cw = true;
    }
    std::vector<double2> tab;
    auto push_len = [&](int64_t L) {
        const int64_t off = (int64_t)tab.size();
        for (int64_t e = 0; e < L; ++e) {
            const long double a = -two_pi * (long double)e / (long double)L;
            tab.push_back(make_double2((double)cosl(a), (double)sinl(a)));
        }
        return off;
    };
    const int64_t o1 = push_len(N1), o2 = push_len(N2);
    const int64_t olo = (int64_t)tab.size();
    for (int q = 0; q < 1024; ++q) {
        const long double a = -two_pi * (long double)(q % N) / (long double)N;
        tab.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
    const int64_t ohi = (int64_t)tab.size();
    for (int64_t h = 0; h <= N / 1024; ++h) {
        const long double a = -two_pi * (long double)((h * 1024) % N) / (long double)N;
        tab.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
    W4_CUDA(cudaMalloc(&tables_, sizeof(double2) * tab.size()));
    W4_CUDA(cudaMemcpyAsync(tables_, tab.data(), sizeof(double2) * tab.size(), cudaMemcpyHostToDevice, st));
    tw1_ = tables_ + o1;
    tw2_ = tables_ + o2;
    tlo_ = tables_ + olo;
    thi_ = tables_ + ohi;
    // pass B in place (default) or as Stockham stages (WC4DVAR_FFT_IPB=0): the lam layout follows
    static const int ipb_env = [] {
        const char* e = std::getenv("WC4DVAR_FFT_IPB");
        return e ? std::atoi(e) : 1;
    }();
    ipb_ = ipb_env;
    for (int i = 0; i < 4; ++i) {
        if (!spec_half[i]) continue;
        W4_CUDA(cudaMalloc(&lam_[i], sizeof(double) * N));
        const unsigned g = (unsigned)std::min<int64_t>(cdiv(N, 256), 4096);
        if (ipb_)
            build_lam_rev_kernel<<<g, 256, 0, st>>>(N, (int)N1, (int)N2, kPlans[plan].brad, spec_half[i], lam_[i]);
        else
            build_lam_kernel<<<g, 256, 0, st>>>(N, (int)N1, (int)N2, spec_half[i], lam_[i]);
        W4_LAUNCH();
    }
    W4_CUDA(cudaStreamSynchronize(st));  // tab is freed on return
    N_ = N;
    N1_ = N1;
    N2_ = N2;
    plan_ = plan;
    return true;
}

void Fft4::apply(bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
                 const double* add, int64_t ldadd, unsigned* status, DevBuf& ybuf, DevBuf& pairbuf,
                 cudaStream_t st, int only) {
    run(0, inv, Nsw, V, ldv, m, out, ldo, add, ldadd, status, nullptr, ybuf, pairbuf, st, only);
}

void Fft4::forward(int Nsw, const double* V, int64_t ldv, int64_t m, double2* Z, DevBuf& ybuf, cudaStream_t st,
                   bool pack_blocks) {
    run(pack_blocks ? 3 : 1, false, Nsw, V, ldv, m, nullptr, 0, nullptr, 0, nullptr, Z, ybuf, spair_, st, -1);
}

void Fft4::inverse(int Nsw, const double2* Z, int64_t m, double* out, int64_t ldo, const double* add,
                   int64_t ldadd, unsigned* status, DevBuf& ybuf, cudaStream_t st, bool pack_blocks) {
    run(pack_blocks ? 4 : 2, false, Nsw, nullptr, 0, m, out, ldo, add, ldadd, status, const_cast<double2*>(Z), ybuf,
        spair_, st, -1);
}

// mode 0: convolution; 1 / 2: forward / inverse transform, sketch columns packed in pairs;
// 3 / 4: forward / inverse transform of ONE column, window blocks packed in pairs
void Fft4::run(int mode, bool inv, int Nsw, const double* V, int64_t ldv, int64_t m, double* out, int64_t ldo,
               const double* add, int64_t ldadd, unsigned* status, double2* Z, DevBuf& ybuf, DevBuf& pairbuf,
               cudaStream_t st, int only) {
    // only = 0 / 1: every column uses the B / Q factor (callers pass Nsw = 0)
    const double* lamB = lam_[inv ? (only == 1 ? 3 : 2) : (only == 1 ? 1 : 0)];
    const double* lamQ = lam_[inv ? 3 : 1];
    require(mode != 0 || (lamB && lamQ), "apply_D_half_inv: inverse factors were not provided");
    require(mode == 0 || ipb_, "spectral transforms need the in-place pass B");
    const int per = Nsw + 1;
    const int64_t ncols = (int64_t)per * m;
    require(ncols < (int64_t)1 << 30, "circulant apply: too many columns");
    std::vector<int2> pairs;
    if (mode == 0) {
        // pair window columns that use the same factor: the i = 0 blocks (B) and the rest (Q)
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
    } else if (mode >= 3) {
        // one column: pair a packs its window blocks 2a (real part) and 2a + 1 (imaginary part);
        // the window kernel separates them by Hermitian symmetry (spectral.cu)
        require(m == 1, "block-packed transforms take one column");
        for (int a = 0; 2 * a < per; ++a) pairs.push_back(make_int2(2 * a, 2 * a + 1 < per ? 2 * a + 1 : -1));
    } else {
        // spectral modes: pair p = jj per + i packs window block i of sketch columns 2 jj and
        // 2 jj + 1, so the window recurrence runs on the packed spectra (it is complex-linear)
        for (int64_t jj = 0; jj < (m + 1) / 2; ++jj)
            for (int i = 0; i < per; ++i)
                pairs.push_back(make_int2((int)(2 * jj * per + i), 2 * jj + 1 < m ? (int)((2 * jj + 1) * per + i) : -1));
    }
    const int np = (int)pairs.size();
    // the pair table depends only on (m, Nsw, pairing): upload once per shape (the caller holds
    // the operator lock, so the cache is not shared between concurrent applies)
    const int pkind = mode == 0 ? 0 : (mode >= 3 ? 2 : 1);  // each pairing keeps its own table and cache
    int2* dpairs = (pkind == 2 ? hpair_ : (pkind ? spair_ : pairbuf)).get<int2>((size_t)np);
    if (pairs_m_[pkind] != m || pairs_per_[pkind] != per || pairs_ptr_[pkind] != dpairs) {
        W4_CUDA(cudaMemcpyAsync(dpairs, pairs.data(), sizeof(int2) * np, cudaMemcpyHostToDevice, st));
        W4_CUDA(cudaStreamSynchronize(st));  // pairs (pageable) is consumed before it goes away
        pairs_m_[pkind] = m;
        pairs_per_[pkind] = per;
        pairs_ptr_[pkind] = dpairs;
    }
    // G pairs per group: the Y slots (kSlots G 16 N bytes) stay within ~64 MB of L2
    static const int g_env = [] {
        const char* e = std::getenv("WC4DVAR_FFT_G");
        return e ? std::atoi(e) : 0;
    }();
    static const int slots = [] {
        const char* e = std::getenv("WC4DVAR_FFT_SLOTS");
        return e ? std::max(3, std::atoi(e)) : kSlots;
    }();
    int G = g_env > 0 ? g_env : (int)std::max<int64_t>(1, (64ll << 20) / (slots * 16 * N_));
    G = std::min(G, np);
    const int ngroups = (np + G - 1) / G;
    double2* Y = ybuf.get<double2>((size_t)slots * G * N_);
    unsigned* ctr = ctr_.get<unsigned>((size_t)1 + 3 * ngroups);
    W4_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * (1 + 3 * (size_t)ngroups), st));
    static const int l2hint = [] {
        const char* e = std::getenv("WC4DVAR_FFT_L2HINT");
        return e ? std::atoi(e) : 1;
    }();
    static const int phase_mask = [] {
        const char* e = std::getenv("WC4DVAR_FFT_PHASES");
        return e ? std::atoi(e) : 7;
    }();
    static const int sub = [] {
        const char* e = std::getenv("WC4DVAR_FFT_SUB");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    static const int acq = [] {
        const char* e = std::getenv("WC4DVAR_FFT_ACQ");
        return e ? std::atoi(e) : 1;
    }();
    static const int prefetch = [] {
        const char* e = std::getenv("WC4DVAR_FFT_PREFETCH");
        return e ? std::atoi(e) : 0;  // measured: 13.7 ms without vs 14.0 ms with (C4 m = 64)
    }();
    Job jb{V, ldv, out, ldo, add, ldadd, add ? status : nullptr, dpairs, np, per, G, ngroups,
           lamB, lamQ, Y, tw1_, tw2_, tlo_, thi_, ctr, l2hint, phase_mask, sub, acq, slots, ipb_, prefetch, Z};
    if (mode == 0) kPlans[plan_].run(jb, st);
    else if (mode == 1 || mode == 3) kPlans[plan_].run_fwd(jb, st);
    else kPlans[plan_].run_inv(jb, st);
}

// ---- spectral window support (spectral.cu) -------------------------------------------------
namespace {
// mhat[e + N1 k2] = (lft w^k + mid + rgt w^-k)^s, w = exp(-2 pi i / N), k = k2 + N2 f(e): the
// Fourier symbol of s sub-steps of the periodic 3-point TL step y_j = lft x_{j-1} + mid x_j +
// rgt x_{j+1} (models.cpp:27-45), in the row order pass B' leaves the spectra in
__global__ void build_symbol_kernel(int64_t N, int N1, int N2, Radices rd, double lft, double mid, double rgt,
                                    int s, double2* __restrict__ mhat) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(t % N1);
        const int64_t k2 = t / N1;
        int span = N1, pw = 1, f = 0;
        for (int i = 0; i < rd.n; ++i) {
            span /= rd.r[i];
            f += ((e / span) % rd.r[i]) * pw;
            pw *= rd.r[i];
        }
        const int64_t k = k2 + (int64_t)N2 * f;
        double sn, cs;
        sincospi(2.0 * (double)k / (double)N, &sn, &cs);  // w^k = cs - i sn
        const double2 one = make_double2(fma(lft + rgt, cs, mid), (rgt - lft) * sn);
        double2 acc = one;
        for (int i = 1; i < s; ++i) acc = cmul(acc, one);
        mhat[t] = acc;
    }
}
}  // namespace

void Fft4::row_radices(int (&r)[4], int& n) const {
    const Radices& rd = kPlans[plan_].brad;
    for (int i = 0; i < 4; ++i) r[i] = rd.r[i];
    n = rd.n;
}

int Fft4::last_radix() const {
    const Radices& r = kPlans[plan_].brad;
    return r.r[r.n - 1];
}

void Fft4::build_symbol(double lft, double mid, double rgt, int s, double2* mhat, cudaStream_t st) const {
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(N_, 256), 4096);
    build_symbol_kernel<<<g, 256, 0, st>>>(N_, (int)N1_, (int)N2_, kPlans[plan_].brad, lft, mid, rgt, s, mhat);
    W4_LAUNCH();
}

}  // namespace w4
