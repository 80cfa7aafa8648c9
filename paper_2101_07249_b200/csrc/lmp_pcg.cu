// Compact-WY spectral LMP and fused PCG row passes (see lmp_pcg.cuh).
#include "lmp_pcg.cuh"

#include <algorithm>
#include <cstdlib>

#include "bulk.cuh"

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

// Persistent row-pass kernel: a fixed grid (one CTA per SM) walks the row tiles; each
// tile's U rows (k column segments of RB contiguous doubles) and its vector segments land in
// shared memory by cp.async.bulk on an mbarrier, double-buffered, so the next tile streams
// from HBM while this one computes.  Column dots accumulate in registers across every tile
// a CTA owns (lane-strided rows, fixed order), so the cross-CTA reduction is over gridDim
// partials only.  Tiles that are partial or misaligned load with plain cooperative loads.
constexpr int kRP = 256;
constexpr int kStageDoubles = 12 * 1024;  // 96 KB per stage (U tile + vector segments)

__host__ __device__ constexpr int nvec_of(int mode) {
    return mode == M_UTV ? 3 : (mode == M_APPLY || mode == M_APPLY_T) ? 1 : mode == M_P1 ? 2 : mode == M_P2 ? 4 : 2;
}

// CPS: CTAs per SM.  1 when the stages hold U tiles (2 x 96 KB); without an LMP (k = 0) a tile
// is only RB rows of 2-4 vectors, and four co-resident CTAs keep enough bytes in flight.
template <int MODE, int NACC, int CPS = 1>
__global__ void __launch_bounds__(kRP, CPS)
    rowpass_kernel(const RowPassCtx c, const PassArgs A, int RB, int nparts, int bulk) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ double wred[kRP / 32];
    __shared__ int is_last;
    constexpr int NV = nvec_of(MODE);
    const int k = c.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = c.n;
    const int64_t ntiles = (n + RB - 1) / RB;
    const int stage_d = k * RB + NV * RB;
    double* stg[2] = {sm, sm + stage_d};
    double* ys = sm + 2 * stage_d;          // k (coefficients of the row dots)
    double* es = ys + ((k + 1) & ~1);       // RB (per-row values of the column dots)
    double* rp = es + RB;                   // nparts x RB (row-dot partials)
    const double* vsrc[4];
    if (MODE == M_UTV) { vsrc[0] = A.v; vsrc[1] = A.a; vsrc[2] = A.b; vsrc[3] = nullptr; }
    else if (MODE == M_APPLY || MODE == M_APPLY_T) { vsrc[0] = A.v; vsrc[1] = vsrc[2] = vsrc[3] = nullptr; }
    else if (MODE == M_P1) { vsrc[0] = A.w; vsrc[1] = A.p; vsrc[2] = vsrc[3] = nullptr; }
    else if (MODE == M_P2) { vsrc[0] = A.w; vsrc[1] = A.x; vsrc[2] = A.p; vsrc[3] = A.r; }
    else { vsrc[0] = A.r; vsrc[1] = A.p; vsrc[2] = vsrc[3] = nullptr; }

    auto tile_rows = [&](int64_t t) { return (int)min((int64_t)RB, n - t * RB); };
    auto is_bulk = [&](int64_t t) { return bulk && tile_rows(t) == RB; };
    // warp 0: arm the stage's barrier and issue the tile's bulk copies
    auto issue = [&](int64_t t, int s) {
        if (t >= ntiles || !is_bulk(t)) return;
        const int64_t row0 = t * RB;
        int nv = 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) nv += vsrc[v] != nullptr;
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bars[s], (unsigned)(sizeof(double) * RB * (k + nv)));
        }
        __syncwarp();
        if (c.blk_rb) {  // the whole tile is one contiguous k x RB block
            if (lane == 0 && k > 0)
                bulk_g2s(stg[s], c.U + t * (int64_t)k * RB, (unsigned)(sizeof(double) * RB * k), &bars[s]);
        } else {
            for (int i = lane; i < k; i += 32)
                bulk_g2s(stg[s] + (size_t)i * RB, c.U + row0 + (int64_t)i * c.ldu, sizeof(double) * RB, &bars[s]);
        }
        if (lane < NV && vsrc[lane])
            bulk_g2s(stg[s] + (size_t)(k + lane) * RB, vsrc[lane] + row0, sizeof(double) * RB, &bars[s]);
    };

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    // Coefficients for the U-apply: APPLY uses op(T) gin, P2 uses T^T g, P3 uses T h.
    if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P2 || MODE == M_P3) {
        const double* gv = (MODE == M_APPLY || MODE == M_APPLY_T) ? A.gin : (MODE == M_P2) ? c.g : c.h;
        const bool trans = (MODE == M_APPLY_T || MODE == M_P2);
        for (int i = warp; i < k; i += kRP / 32) {
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
    if (warp == 0) {
        issue(blockIdx.x, 0);
        issue((int64_t)blockIdx.x + gridDim.x, 1);
    }
    double alpha = 0.0, beta = 0.0;
    if (MODE == M_P2) alpha = c.scal[SC_ALPHA];
    if (MODE == M_P3) beta = c.scal[SC_BETA];

    double acc[NACC > 0 ? NACC : 1];
#pragma unroll
    for (int j = 0; j < (NACC > 0 ? NACC : 1); ++j) acc[j] = 0.0;
    double dotc = 0.0;
    unsigned phase[2] = {0u, 0u};
    const int part = tid / RB, prow = tid - part * RB;

    for (int64_t it = 0;; ++it) {
        const int64_t t = blockIdx.x + it * (int64_t)gridDim.x;
        if (t >= ntiles) break;
        const int s = (int)(it & 1);
        const int64_t row0 = t * RB;
        const int rows = tile_rows(t);
        double* Us = stg[s];
        double* Vs = Us + (size_t)k * RB;
        if (is_bulk(t)) {
            mbar_wait(&bars[s], phase[s]);
            phase[s] ^= 1u;
        } else {
            for (int e = tid; e < k * RB; e += kRP) {
                const int i = e / RB, r = e - i * RB;
                Us[e] = c.blk_rb ? c.U[t * (int64_t)k * RB + e]
                                 : (r < rows ? c.U[row0 + r + (int64_t)i * c.ldu] : 0.0);
            }
            for (int e = tid; e < NV * RB; e += kRP) {
                const int v = e / RB, r = e - v * RB;
                Vs[e] = (r < rows && vsrc[v]) ? vsrc[v][row0 + r] : 0.0;
            }
            __syncthreads();
        }
        // ---- row dots s_r = sum_i U[r, i] ys[i] (nparts column ranges, fixed-order combine)
        if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P2 || MODE == M_P3) {
            if (part < nparts && prow < rows) {
                const int i0 = part * k / nparts, i1 = (part + 1) * k / nparts;
                double sacc = 0.0;
                for (int i = i0; i < i1; ++i) sacc += Us[(size_t)i * RB + prow] * ys[i];
                rp[part * RB + prow] = sacc;
            }
            __syncthreads();
        }
        if (tid < rows) {
            const int r = tid;
            const int64_t row = row0 + r;
            double sr = 0.0;
            if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P2 || MODE == M_P3)
                for (int p = 0; p < nparts; ++p) sr += rp[p * RB + r];
            double e = 0.0;
            if (MODE == M_UTV) {
                e = Vs[r];
                if (vsrc[1]) dotc += Vs[RB + r] * Vs[2 * RB + r];
            } else if (MODE == M_APPLY || MODE == M_APPLY_T) {
                A.out[row] = Vs[r] - sr;
            } else if (MODE == M_P1) {
                e = Vs[r];                    // w
                dotc += Vs[RB + r] * e;       // p . w
            } else if (MODE == M_P2) {
                const double ctw = Vs[r] - sr;                   // C^T w
                A.x[row] = Vs[RB + r] + alpha * Vs[2 * RB + r];  // x += alpha p
                const double rn = Vs[3 * RB + r] - alpha * ctw;  // r -= alpha C^T w
                A.r[row] = rn;
                e = rn;
                dotc += rn * rn;
            } else {
                A.p[row] = (Vs[r] - sr) + beta * Vs[RB + r];  // p = C r + beta p
            }
            if (MODE == M_UTV || MODE == M_P1 || MODE == M_P2) es[r] = e;
        }
        if (MODE == M_UTV || MODE == M_P1 || MODE == M_P2) {
            __syncthreads();
            // column dots: warp w owns columns w + 8 j, lanes stride the tile's rows
            for (int r = lane; r < rows; r += 32) {
                const double er = es[r];
                const double* ur = Us + (size_t)warp * RB + r;
#pragma unroll
                for (int j = 0; j < NACC; ++j)
                    if (warp + 8 * j < k) acc[j] += ur[(size_t)8 * j * RB] * er;
            }
        }
        __syncthreads();  // stage s and es / rp are free
        if (warp == 0) issue(t + 2 * (int64_t)gridDim.x, s);
    }
    if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P3) return;

    // per-CTA partials: column dots (fixed shuffle tree) and the row dot
    double* partial = c.partial + (int64_t)blockIdx.x * (k + 1);
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
        const int i = warp + 8 * j;
        const double s = warp_sum(acc[j]);
        if (i < k && lane == 0) partial[i] = s;
    }
    const double d = warp_sum(dotc);
    if (lane == 0) wred[warp] = d;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kRP / 32; ++w) s += wred[w];
        partial[k] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(c.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double* res = (MODE == M_UTV) ? A.out : (MODE == M_P1 ? c.g : c.h);
    for (int i = warp; i <= k; i += kRP / 32) {
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(c.partial + (int64_t)b * (k + 1) + i);
        s = warp_sum(s);
        if (lane == 0) res[i] = s;
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

// Plain vector passes of the unpreconditioned PCG (k = 0, krylov.cpp:55-95 with C = I).  Same
// grid, row ownership (thread tid owns row tid of tiles blockIdx.x + it gridDim.x) and
// reduction order as rowpass_kernel<MODE, 0, 4>, so the results are bitwise the same; the
// vectors are read straight from global memory with UN tiles of every stream in flight per
// thread and no per-tile barrier (a 256-row tile of 2-4 vectors is too small for the
// bulk-copy ring: one or two tiles in flight per CTA left the pass latency-bound).
template <int MODE>
__global__ void __launch_bounds__(kRP, 4) vecpass_kernel(const RowPassCtx c, const PassArgs A) {
    __shared__ double wred[kRP / 32];
    __shared__ int is_last;
    constexpr int UN = (MODE == M_P2) ? 4 : 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = c.n;
    const int64_t stride = (int64_t)gridDim.x * kRP;
    double alpha = 0.0, beta = 0.0;
    if (MODE == M_P2) alpha = c.scal[SC_ALPHA];
    if (MODE == M_P3) beta = c.scal[SC_BETA];
    double dotc = 0.0;
    for (int64_t base = (int64_t)blockIdx.x * kRP + tid; base < n; base += UN * stride) {
        double v0[UN], v1[UN], v2[UN], v3[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int64_t row = base + u * stride;
            const bool ok = row < n;
            if (MODE == M_P1) {
                v0[u] = ok ? __ldcs(A.w + row) : 0.0;
                v1[u] = ok ? __ldcs(A.p + row) : 0.0;
            } else if (MODE == M_P2) {
                v0[u] = ok ? __ldcs(A.w + row) : 0.0;
                v1[u] = ok ? __ldcs(A.x + row) : 0.0;
                v2[u] = ok ? __ldcs(A.p + row) : 0.0;
                v3[u] = ok ? __ldcs(A.r + row) : 0.0;
            } else {
                v0[u] = ok ? __ldcs(A.r + row) : 0.0;
                v1[u] = ok ? __ldcs(A.p + row) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int64_t row = base + u * stride;
            if (row >= n) continue;
            if (MODE == M_P1) {
                const double e = v0[u];   // w
                dotc += v1[u] * e;        // p . w
            } else if (MODE == M_P2) {
                const double ctw = v0[u] - 0.0;           // C^T w with C = I
                A.x[row] = v1[u] + alpha * v2[u];         // x += alpha p
                const double rn = v3[u] - alpha * ctw;    // r -= alpha w
                A.r[row] = rn;
                dotc += rn * rn;
            } else {
                A.p[row] = (v0[u] - 0.0) + beta * v1[u];  // p = r + beta p
            }
        }
    }
    if (MODE == M_P3) return;
    double* partial = c.partial + (int64_t)blockIdx.x;
    const double d = warp_sum(dotc);
    if (lane == 0) wred[warp] = d;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kRP / 32; ++w) s += wred[w];
        partial[0] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(c.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double* res = (MODE == M_P1) ? c.g : c.h;
    if (warp == 0) {
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(c.partial + b);
        s = warp_sum(s);
        if (lane == 0) res[0] = s;
    }
    __syncthreads();
    if (tid == 0) {
        *c.counter = 0u;
        if (MODE == M_P1) {
            const double curv = res[0];
            c.scal[SC_CURV] = curv;
            c.scal[SC_ALPHA] = c.scal[SC_RHO] / curv;
        } else {
            const double rn = res[0];
            c.scal[SC_RHO_NEXT] = rn;
            c.scal[SC_BETA] = rn / c.scal[SC_RHO];
            c.scal[SC_RHO] = rn;
        }
    }
}

int pick_rb(int k) {
    int rb = kStageDoubles / (k + 4);
    rb = (rb / 16) * 16;
    if (rb > kRP) rb = kRP;
    if (rb < 16) rb = 16;
    return rb;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int MODE, int NACC>
void launch_pass_n(const RowPassCtx& c, const PassArgs& a, cudaStream_t st) {
    const int RB = c.blk_rb ? c.blk_rb : pick_rb(c.k);
    const int nparts = std::max(1, std::min(c.k > 0 ? c.k : 1, kRP / RB));
    constexpr int NV = nvec_of(MODE);
    const size_t smem =
        sizeof(double) * (2 * ((size_t)c.k * RB + (size_t)NV * RB) + ((c.k + 1) & ~1) + RB + (size_t)nparts * RB);
    auto kern = rowpass_kernel<MODE, NACC>;
    static int configured = 0;
    if (smem > 48 * 1024 && (size_t)configured < smem) {
        W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = (int)smem;
    }
    const double* vs[4] = {a.v, a.a, a.b, nullptr};
    if (MODE == M_P1) { vs[0] = a.w; vs[1] = a.p; vs[2] = nullptr; }
    if (MODE == M_P2) { vs[0] = a.w; vs[1] = a.x; vs[2] = a.p; vs[3] = a.r; }
    if (MODE == M_P3) { vs[0] = a.r; vs[1] = a.p; vs[2] = nullptr; }
    if (MODE == M_APPLY || MODE == M_APPLY_T) { vs[1] = vs[2] = nullptr; }
    bool bulk = (RB % 2 == 0) && (c.k == 0 || ((c.blk_rb || c.ldu % 2 == 0) && aligned16(c.U)));
    for (const double* v : vs) bulk = bulk && (v == nullptr || aligned16(v));
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        W4_CUDA(cudaGetDevice(&dev));
        W4_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t ntiles = cdiv(c.n, RB);
    if (NACC == 0 && c.k == 0) {  // plain vector passes: four CTAs per SM (partials: <= 2048 CTAs)
        const int64_t grid4 = std::max<int64_t>(1, std::min<int64_t>({ntiles, (int64_t)4 * nsm, (int64_t)2048}));
        if constexpr (MODE == M_P1 || MODE == M_P2 || MODE == M_P3) if (RB == kRP) {
            const char* e = getenv("WC4DVAR_PCG_VECPASS");  // 0: the bulk-copy ring kernel
            if (!(e && e[0] == '0')) {
                vecpass_kernel<MODE><<<(unsigned)grid4, kRP, 0, st>>>(c, a);
                W4_LAUNCH();
                return;
            }
        }
        rowpass_kernel<MODE, 0, 4><<<(unsigned)grid4, kRP, smem, st>>>(c, a, RB, nparts, bulk ? 1 : 0);
        W4_LAUNCH();
        return;
    }
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>({ntiles, (int64_t)nsm, cdiv(c.n, 32) + 1}));
    kern<<<(unsigned)grid, kRP, smem, st>>>(c, a, RB, nparts, bulk ? 1 : 0);
    W4_LAUNCH();
}

template <int MODE>
void launch_pass(const RowPassCtx& c, const PassArgs& a, cudaStream_t st) {
    if (c.n == 0) return;
    if (MODE == M_APPLY || MODE == M_APPLY_T || MODE == M_P3) return launch_pass_n<MODE, 0>(c, a, st);
    const int need = (c.k + 7) / 8;
    if (need <= 0) return launch_pass_n<MODE, 0>(c, a, st);
    if (need <= 1) return launch_pass_n<MODE, 1>(c, a, st);
    if (need <= 2) return launch_pass_n<MODE, 2>(c, a, st);
    if (need <= 4) return launch_pass_n<MODE, 4>(c, a, st);
    if (need <= 8) return launch_pass_n<MODE, 8>(c, a, st);
    if (need <= 16) return launch_pass_n<MODE, 16>(c, a, st);
    if (need <= 32) return launch_pass_n<MODE, 32>(c, a, st);
    return launch_pass_n<MODE, 64>(c, a, st);
}

__global__ void block_U_kernel(int64_t n, int k, int rb, const double* __restrict__ U, int64_t ldu,
                               double* __restrict__ B, int64_t total, int to_blocked) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = e / ((int64_t)k * rb);
        const int64_t w = e - tile * (int64_t)k * rb;
        const int64_t i = w / rb, r = w - i * rb;
        const int64_t row = tile * rb + r;
        if (to_blocked) B[e] = row < n ? U[row + i * ldu] : 0.0;
        else if (row < n) const_cast<double*>(U)[row + i * ldu] = B[e];
    }
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

int lmp_tile_rows(int k) { return pick_rb(k); }

int64_t lmp_blocked_size(int64_t n, int k) {
    const int rb = pick_rb(k);
    return cdiv(n, rb) * rb * (int64_t)k;
}

void lmp_block_U(int64_t n, int k, const double* U, int64_t ldu, double* Ublk, cudaStream_t st) {
    const int64_t total = lmp_blocked_size(n, k);
    if (!total) return;
    block_U_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 8 * kSMs), 256, 0, st>>>(n, k, pick_rb(k), U, ldu,
                                                                                             Ublk, total, 1);
    W4_LAUNCH();
}

void lmp_unblock_U(int64_t n, int k, const double* Ublk, double* U, int64_t ldu, cudaStream_t st) {
    const int64_t total = lmp_blocked_size(n, k);
    if (!total) return;
    block_U_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 8 * kSMs), 256, 0, st>>>(
        n, k, pick_rb(k), U, ldu, const_cast<double*>(Ublk), total, 0);
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
