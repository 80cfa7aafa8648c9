// Compact-WY spectral LMP and fused PCG row passes (see lmp_pcg.cuh).
#include "lmp_pcg.cuh"

namespace w4 {
namespace {

constexpr int kBlock = 256;

enum { M_UTV = 0, M_APPLY = 1, M_APPLY_T = 2, M_P1 = 3, M_P2 = 4, M_P3 = 5 };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct PassArgs {
    const double* v;   // UTV / APPLY input
    const double* a;   // UTV dot operands (optional)
    const double* b;
    const double* gin; // APPLY coefficient vector (k)
    double* out;       // UTV result (k+1) / APPLY output vector
    double* x;
    double* r;
    double* p;
    const double* w;
};

template <int MODE>
__global__ void __launch_bounds__(kBlock)
    rowpass_kernel(const RowPassCtx c, const PassArgs A, int RB) {
    extern __shared__ double sm[];
    const int k = c.k;
    const int ks = RB + 1;
    double* Us = sm;                        // k x (RB+1)
    double* es = Us + (size_t)k * ks;       // RB
    double* ys = es + RB;                   // k
    __shared__ double wred[kBlock / 32];
    __shared__ int is_last;

    const int tid = threadIdx.x;
    const int64_t row0 = (int64_t)blockIdx.x * RB;
    const int64_t rem_rows = c.n - row0;
    const int rows = (int)(rem_rows < RB ? rem_rows : RB);

    // Stage this CTA's U rows once (coalesced per column) with cp.async: every copy of the
    // thread is in flight at once instead of one L2 round trip per element.
    for (int e = tid; e < k * RB; e += kBlock) {
        const int i = e / RB, rr = e % RB;
        if (rr < rows) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(Us + i * ks + rr));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d),
                         "l"(c.U + row0 + rr + (int64_t)i * c.ldu));
        } else {
            Us[i * ks + rr] = 0.0;
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // Coefficients for the U-apply: APPLY uses op(T) gin, P2 uses T^T g, P3 uses T h.
    if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P2 || MODE == M_P3) {
        const double* gv = (MODE == M_APPLY || MODE == M_APPLY_T) ? A.gin
                           : (MODE == M_P2)                     ? c.g
                                                                : c.h;
        const bool trans = (MODE == M_APPLY_T || MODE == M_P2);
        // one warp per coefficient, lanes stride j (independent L2 loads, fixed-order tree)
        const int warp = tid >> 5, lane = tid & 31;
        for (int i = warp; i < k; i += kBlock / 32) {
            double s = 0.0;
            if (trans) {  // (T^T g)_i = sum_{j<=i} T[j,i] g_j
                for (int j = lane; j <= i; j += 32) s += c.T[j + (int64_t)i * k] * gv[j];
            } else {      // (T h)_i = sum_{j>=i} T[i,j] h_j
                for (int j = i + lane; j < k; j += 32) s += c.T[i + (int64_t)j * k] * gv[j];
            }
            s = warp_sum(s);
            if (lane == 0) ys[i] = s;
        }
    }
    __syncthreads();

    double dotc = 0.0;
    if (tid < RB) {
        const int rr = tid;
        const int64_t row = row0 + rr;
        const bool live = rr < rows;
        double e = 0.0;
        if (MODE == M_UTV) {
            if (live) {
                e = A.v[row];
                if (A.a) dotc = A.a[row] * A.b[row];
            }
        } else if (MODE == M_APPLY || MODE == M_APPLY_T) {
            if (live) {
                double s = 0.0;
                for (int i = 0; i < k; ++i) s += Us[i * ks + rr] * ys[i];
                A.out[row] = A.v[row] - s;
            }
        } else if (MODE == M_P1) {
            if (live) {
                e = A.w[row];
                dotc = A.p[row] * e;
            }
        } else if (MODE == M_P2) {
            if (live) {
                const double alpha = c.scal[SC_ALPHA];
                double s = 0.0;
                for (int i = 0; i < k; ++i) s += Us[i * ks + rr] * ys[i];
                const double ctw = A.w[row] - s;          // C^T w
                A.x[row] = A.x[row] + alpha * A.p[row];   // x += alpha p
                const double rn = A.r[row] - alpha * ctw; // r -= alpha C^T w
                A.r[row] = rn;
                e = rn;
                dotc = rn * rn;
            }
        } else if (MODE == M_P3) {
            if (live) {
                const double beta = c.scal[SC_BETA];
                double s = 0.0;
                for (int i = 0; i < k; ++i) s += Us[i * ks + rr] * ys[i];
                A.p[row] = (A.r[row] - s) + beta * A.p[row];  // p = C r + beta p
            }
        }
        es[rr] = e;
    }
    if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P3) return;

    // Reduction: column i of U against es (fixed order), plus the block dot.
    double d = warp_sum(dotc);
    if ((tid & 31) == 0) wred[tid >> 5] = d;
    __syncthreads();
    double* part = c.partial + (int64_t)blockIdx.x * (k + 1);
    // one warp per U column: lanes stride the CTA's rows, then a shuffle tree (fixed order)
    for (int i = tid >> 5; i < k; i += kBlock / 32) {
        double s = 0.0;
        const double* col = Us + i * ks;
        for (int rr = tid & 31; rr < rows; rr += 32) s += col[rr] * es[rr];
        s = warp_sum(s);
        if ((tid & 31) == 0) part[i] = s;
    }
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) s += wred[w];
        part[k] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(c.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double* res = (MODE == M_UTV) ? A.out : (MODE == M_P1 ? c.g : c.h);
    // final sums over the CTAs' partials: one warp per entry, lanes stride the CTAs (the
    // loads of a lane are independent, so they pipeline instead of forming one long chain)
    // (each lane issues its up-to-8 loads per 256-CTA chunk before summing them in order)
    for (int i = tid >> 5; i <= k; i += kBlock / 32) {
        double s = 0.0;
        for (unsigned b0 = tid & 31; b0 < gridDim.x; b0 += 256) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const unsigned b = b0 + 32 * u;
                v[u] = b < gridDim.x ? __ldcg(c.partial + (int64_t)b * (k + 1) + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        s = warp_sum(s);
        if ((tid & 31) == 0) res[i] = s;
    }
    __syncthreads();
    if (tid == 0) {
        *c.counter = 0u;
        if (MODE == M_P1) {
            const double curv = res[k];
            c.scal[SC_CURV] = curv;
            c.scal[SC_ALPHA] = c.scal[SC_RHO] / curv;
        } else if (MODE == M_P2) {
            const double rn = res[k];
            c.scal[SC_RHO_NEXT] = rn;
            c.scal[SC_BETA] = rn / c.scal[SC_RHO];
            c.scal[SC_RHO] = rn;
        }
    }
}

int pick_rb(int k) {
    if (k <= 0) return kBlock;
    int rb = (int)((160 * 1024 / 8) / k) - 1;
    if (rb > kBlock) rb = kBlock;
    rb = (rb / 32) * 32;
    if (rb < 32) rb = 32;
    return rb;
}

template <int MODE>
void launch_pass(const RowPassCtx& c, const PassArgs& a, cudaStream_t st) {
    if (c.n == 0) return;
    const int RB = pick_rb(c.k);
    const size_t smem = sizeof(double) * ((size_t)c.k * (RB + 1) + RB + c.k);
    auto kern = rowpass_kernel<MODE>;
    if (smem + 1024 > 48 * 1024)  // + the kernel's static reduction scratch
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = cdiv(c.n, RB);
    kern<<<(unsigned)grid, kBlock, smem, st>>>(c, a, RB);
    W4_LAUNCH();
}

__global__ void build_T_kernel(int k, const double* __restrict__ S, const double* __restrict__ th,
                               double* __restrict__ T) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < k * k; e += nt) T[e] = 0.0;
    __syncthreads();
    for (int i = 0; i < k; ++i) {
        const double ci = 1.0 - 1.0 / sqrt(th[i]);
        for (int j = tid; j < i; j += nt) {
            double s = 0.0;
            for (int l = j; l < i; ++l) s += T[j + l * k] * S[l + i * k];
            T[j + i * k] = -ci * s;
        }
        if (tid == 0) T[i + i * k] = ci;
        __syncthreads();
    }
}

__global__ void sqdist_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                              double* out, double* partial, unsigned* counter) {
    __shared__ double wred[kBlock / 32];
    __shared__ int is_last;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kBlock) {
        const double d = b ? a[i] - b[i] : a[i];
        s += d * d;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) wred[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) t += wred[w];
        partial[blockIdx.x] = t;
        __threadfence();
        is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last && threadIdx.x < 32) {  // warp 0: lanes stride the partials, fixed-order tree
        __threadfence();
        double t = 0.0;
        for (unsigned b2 = threadIdx.x; b2 < gridDim.x; b2 += 32) t += __ldcg(partial + b2);
        t = warp_sum(t);
        if (threadIdx.x == 0) {
            *out = t;
            *counter = 0u;
        }
    }
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             const double* __restrict__ y, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a * x[i] + (y ? b * y[i] : 0.0);
}

__global__ void defect_kernel(int k, const double* __restrict__ S, double* out) {
    __shared__ double red[1024];
    double m = 0.0;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int i = e % k, j = e / k;
        const double v = fabs(S[e] - (i == j ? 1.0 : 0.0));
        m = (v > m || v != v) ? v : m;
    }
    red[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (unsigned i = 0; i < blockDim.x; ++i) t = (red[i] > t || red[i] != red[i]) ? red[i] : t;
        *out = t;
    }
}

}  // namespace

void lmp_build_T(int k, const double* S, const double* theta, double* T, cudaStream_t st) {
    if (k == 0) return;
    build_T_kernel<<<1, 256, 0, st>>>(k, S, theta, T);
    W4_LAUNCH();
}

void rowpass_utv(const RowPassCtx& c, const double* v, const double* a, const double* b,
                 double* out, cudaStream_t st) {
    PassArgs p{};
    p.v = v;
    p.a = a;
    p.b = b;
    p.out = out;
    launch_pass<M_UTV>(c, p, st);
}

void rowpass_apply(const RowPassCtx& c, bool transpose, const double* v, const double* g,
                   double* out, cudaStream_t st) {
    PassArgs p{};
    p.v = v;
    p.gin = g;
    p.out = out;
    if (transpose) launch_pass<M_APPLY_T>(c, p, st);
    else launch_pass<M_APPLY>(c, p, st);
}

void pcg_pass1(const RowPassCtx& c, const double* p, const double* w, cudaStream_t st) {
    PassArgs a{};
    a.p = const_cast<double*>(p);
    a.w = w;
    launch_pass<M_P1>(c, a, st);
}

void pcg_pass2(const RowPassCtx& c, double* x, double* r, const double* p, const double* w,
               cudaStream_t st) {
    PassArgs a{};
    a.x = x;
    a.r = r;
    a.p = const_cast<double*>(p);
    a.w = w;
    launch_pass<M_P2>(c, a, st);
}

void pcg_pass3(const RowPassCtx& c, const double* r, double* p, cudaStream_t st) {
    PassArgs a{};
    a.r = const_cast<double*>(r);
    a.p = p;
    launch_pass<M_P3>(c, a, st);
}

void sqdist(int64_t n, const double* a, const double* b, double* out, double* partial,
            unsigned* counter, cudaStream_t st) {
    int64_t grid = cdiv(n, kBlock);
    if (grid > 2 * kSMs) grid = 2 * kSMs;
    if (grid < 1) grid = 1;
    sqdist_kernel<<<(unsigned)grid, kBlock, 0, st>>>(n, a, b, out, partial, counter);
    W4_LAUNCH();
}

void axpby(int64_t n, double a, const double* x, double b, const double* y, double* out,
           cudaStream_t st) {
    if (n == 0) return;
    int64_t grid = cdiv(n, 256);
    if (grid > 8 * kSMs) grid = 8 * kSMs;
    axpby_kernel<<<(unsigned)grid, 256, 0, st>>>(n, a, x, b, y, out);
    W4_LAUNCH();
}

void defect_max(int k, const double* S, double* out, cudaStream_t st) {
    defect_kernel<<<1, 1024, 0, st>>>(k, S, out);
    W4_LAUNCH();
}

}  // namespace w4
