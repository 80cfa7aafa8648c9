// Tiled window sweeps for large n and for Lorenz-96 (any n).
//
// One CTA owns a tile of T grid points of one sketch column and advances K window
// intervals per launch on a shared-memory region [t0 - HL, t0 + T + HR) whose halos
// (HL = K s rl, HR = K s rr for a stencil of radius (rl, rr) per sub-step) are recomputed
// redundantly, so tiles never communicate inside a launch; the valid region shrinks by
// (rl, rr) per sub-step and the tile centre stays valid.  State crossing a launch boundary
// goes through a ping-pong buffer.  When the whole periodic domain fits (n <= T) the tile
// is the domain itself ("resident" mode: indices wrap, nothing shrinks, one launch).
//
// Models: identity / upwind advection / advection-diffusion (1 stencil phase per
// sub-step) and the exact TL / adjoint of the RK4 Lorenz-96 step with stored stages
// (4 stencil phases per sub-step, models.cpp:92-148).
#include "sweep.cuh"

#include <algorithm>
#include <cstdlib>

namespace w4 {
namespace {

constexpr int kThreads = 512;

struct TileGeom {
    int T;        // tile centre size
    int HL, HR;   // halos (tiled mode)
    int R;        // region size in SMEM
    bool resident;
    int64_t ntiles;
};

// Stencil radius (left, right) of one TL sub-step (adjoint mirrors it).
__host__ __device__ inline void model_radius(int kind, int& rl, int& rr) {
    if (kind == WC4DVAR_MODEL_LORENZ96) {
        rl = 8;
        rr = 4;
    } else if (kind == WC4DVAR_MODEL_IDENTITY) {
        rl = 0;
        rr = 0;
    } else {
        rl = 1;
        rr = 1;
    }
}

struct Region {
    int R;
    bool resident;
    int origin;  // global grid index of region element 0 (|origin| < n)
    int n;       // grid points (n < 2^31)
    __device__ __forceinline__ int nb(int e, int d) const {  // neighbour index in SMEM
        if (!resident) return e + d;
        int x = e + d;
        if (x < 0) x += R;
        else if (x >= R) x -= R;
        return x;
    }
    // division-free periodic wrap of a grid index in (-n, 2n)
    __device__ __forceinline__ int wrap(int g) const { return g < 0 ? g + n : (g >= n ? g - n : g); }
    __device__ __forceinline__ int gidx(int e) const { return wrap(origin + e); }
};

// ---------------------------------------------------------------- single-phase stencils
template <int KIND, bool ADJ>
__device__ __forceinline__ double stencil1(const double* __restrict__ u, const Region& rg, int e,
                                           double c, double d) {
    if (KIND == WC4DVAR_MODEL_IDENTITY) return u[e];
    const double um = u[rg.nb(e, -1)], uc = u[e], up = u[rg.nb(e, 1)];
    if (!ADJ) {
        if (KIND == WC4DVAR_MODEL_ADVECTION) return uc - c * (uc - um);          // models.cpp:32
        return uc - c * (uc - um) + d * (up - 2.0 * uc + um);
    }
    if (KIND == WC4DVAR_MODEL_ADVECTION) return (1.0 - c) * uc + c * up;        // models.cpp:42
    return uc - c * (uc - up) + d * (um - 2.0 * uc + up);
}

// Lorenz-96 Jacobian (models.cpp:92-102) and its transpose (models.cpp:105-116) at e,
// with the stage vector staged in SMEM over the region.
__device__ __forceinline__ double l96_jac_s(const double* __restrict__ x, const double* __restrict__ v,
                                            const Region& rg, int e) {
    const int em2 = rg.nb(e, -2), em1 = rg.nb(e, -1), ep1 = rg.nb(e, 1);
    return -v[em2] * x[em1] - x[em2] * v[em1] + v[em1] * x[ep1] + x[em1] * v[ep1] - v[e];
}
__device__ __forceinline__ double l96_jac_t_s(const double* __restrict__ x, const double* __restrict__ l,
                                              const Region& rg, int e, double scale) {
    const int em2 = rg.nb(e, -2), em1 = rg.nb(e, -1), ep1 = rg.nb(e, 1), ep2 = rg.nb(e, 2);
    const double lp2 = scale * l[ep2], lp1 = scale * l[ep1], lm1 = scale * l[em1], lc = scale * l[e];
    return -x[ep1] * lp2 + (x[ep2] - x[em1]) * lp1 + x[em2] * lm1 - lc;
}

// Region slice of one stage vector -> SMEM with 8-byte cp.async (overlaps the current phase).
__device__ __forceinline__ void stage_load(double* dst, const double* __restrict__ src, const Region& rg,
                                           int R, int tid, int nt) {
    for (int e = tid - 2; e < R + 2; e += nt) {  // region plus the 2-element guards
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + e));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + rg.gidx(e)));
    }
    asm volatile("cp.async.commit_group;\n");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
#define stage_sync(idx)          \
    do {                         \
        cp_async_wait_all();     \
        __syncthreads();         \
        (idx) ^= 1;              \
    } while (0)

struct TiledArgs {
    ModelDev md;
    NetDev net;
    SweepArgs a;
    TileGeom geo;
    int i0, i1;             // forward: intervals [i0, i1); adjoint: from state s_{i1} down to s_{i0}
    const double* bin;      // boundary state in (n x m, ld n) or null (start of window)
    double* bout;           // boundary state out
    StencilTaps tp{};       // fused S-step stencil of this direction (blocked stencil kernels)
};

// ---------------------------------------------------------------- forward
template <int KIND>
__global__ void __launch_bounds__(kThreads) tiled_fwd_kernel(const TiledArgs ta, unsigned* status) {
    extern __shared__ double sm[];
    const ModelDev& md = ta.md;
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int R = geo.R;
    double* cur = sm;
    double* nxt = sm + R;
    double* t1 = sm + 2 * R;  // L96 temporaries
    double* t2 = sm + 3 * R;
    double* acc = sm + 4 * R;
    const int64_t n = md.n;
    const int64_t col = blockIdx.x;
    const int64_t tile = blockIdx.y;
    const int64_t t0 = tile * geo.T;
    const int tid = threadIdx.x, nt = blockDim.x;
    Region rg{R, geo.resident, geo.resident ? 0 : (int)(t0 - geo.HL), (int)n};
    const int c_lo = geo.resident ? 0 : geo.HL;                   // tile centre in SMEM
    const int c_hi = geo.resident ? R : geo.HL + (int)(n - t0 < (int64_t)geo.T ? n - t0 : (int64_t)geo.T);
    int rl, rr;
    model_radius(md.kind, rl, rr);
    const int s = md.s;
    const double* X = a.X + col * a.ldx;
    double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
    const int np = net.n_points;
    bool bad = false;

    // state x_{i0} on the region
    const double* src = ta.bin ? ta.bin + col * n : X;  // x_0 = X_0
    for (int e = tid; e < R; e += nt) {
        const int g = rg.gidx(e);
        cur[e] = src[g];
    }
    if (ta.i0 == 0) {  // x_0 is part of the trajectory (finite check, traj, obs at t_0)
        const int sl = net.slot[0];
        for (int e = c_lo + tid; e < c_hi; e += nt) {
            const int g = rg.gidx(e);
            const double x = cur[e];
            bad |= !isfinite(x);
            if (tr) tr[g] = x;
            if (a.fwd_obs && sl >= 0) {
                const int bb = net.pmap[g];
                if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
            }
        }
    }
    __syncthreads();
    // L96 stage double buffer, each with a 2-element guard per side (the adjoint Jacobian
    // reads the stage one point further left than the state)
    double* sbuf[2] = {sm + 5 * R + 2, sm + 6 * R + 6};
    int sbi = 0;
    if (KIND == WC4DVAR_MODEL_LORENZ96 && ta.i1 > ta.i0) {  // x1 of the first sub-step
        stage_load(sbuf[0], md.stages + (int64_t)ta.i0 * s * 4 * n, rg, R, tid, nt);
        cp_async_wait_all();
        __syncthreads();
    }
    int lo = 0, hi = R;  // valid region
    for (int i = ta.i0; i < ta.i1; ++i) {
        for (int k = 0; k < s; ++k) {
            if (!geo.resident) {
                lo += rl;
                hi -= rr;
            }
            const bool last = (k + 1 == s);
            if (KIND != WC4DVAR_MODEL_LORENZ96) {
                for (int e = lo + tid; e < hi; e += nt) nxt[e] = stencil1<KIND, false>(cur, rg, e, md.c, md.d);
            } else {
                // RK4 TL step (models.cpp:120-128), stages of sub-step i*s+k.  Stage x_p is
                // staged in SMEM (sb[cur]) while x_{p+1} streams into sb[nxt] by cp.async.
                const double* st = md.stages + ((int64_t)i * s + k) * 4 * n;
                const double dt = md.dt;
                const int l1 = geo.resident ? 0 : lo - 6, h1 = geo.resident ? R : hi + 3;
                stage_load(sbuf[sbi ^ 1], st + n, rg, R, tid, nt);
                for (int e = max(l1, 0) + tid; e < min(h1, R); e += nt) {
                    const double a1 = l96_jac_s(sbuf[sbi], cur, rg, e);
                    acc[e] = a1;
                    t1[e] = cur[e] + 0.5 * dt * a1;
                }
                stage_sync(sbi);
                const int l2 = geo.resident ? 0 : lo - 4, h2 = geo.resident ? R : hi + 2;
                stage_load(sbuf[sbi ^ 1], st + 2 * n, rg, R, tid, nt);
                for (int e = max(l2, 0) + tid; e < min(h2, R); e += nt) {
                    const double a2 = l96_jac_s(sbuf[sbi], t1, rg, e);
                    acc[e] = acc[e] + 2.0 * a2;
                    t2[e] = cur[e] + 0.5 * dt * a2;
                }
                stage_sync(sbi);
                const int l3 = geo.resident ? 0 : lo - 2, h3 = geo.resident ? R : hi + 1;
                stage_load(sbuf[sbi ^ 1], st + 3 * n, rg, R, tid, nt);
                for (int e = max(l3, 0) + tid; e < min(h3, R); e += nt) {
                    const double a3 = l96_jac_s(sbuf[sbi], t2, rg, e);
                    acc[e] = acc[e] + 2.0 * a3;
                    t1[e] = cur[e] + dt * a3;
                }
                stage_sync(sbi);
                {  // prefetch x1 of the next sub-step of this launch
                    const bool more = (k + 1 < s) || (i + 1 < ta.i1);
                    if (more) stage_load(sbuf[sbi ^ 1], st + 4 * n, rg, R, tid, nt);
                }
                for (int e = lo + tid; e < hi; e += nt) {
                    const double a4 = l96_jac_s(sbuf[sbi], t1, rg, e);
                    nxt[e] = cur[e] + (dt / 6.0) * (acc[e] + a4);
                }
                cp_async_wait_all();
                sbi ^= 1;
            }
            if (last) {
                // x_{i+1} = M_i x_i + X_{i+1}  (operators.cpp:88)
                const double* Xn = X + (int64_t)(i + 1) * n;
                const int sl = net.slot[i + 1];
                double* trn = tr ? tr + (int64_t)(i + 1) * n : nullptr;
                for (int e = lo + tid; e < hi; e += nt) {
                    const int g = rg.gidx(e);
                    const double x = nxt[e] + Xn[g];
                    nxt[e] = x;
                    if (e >= c_lo && e < c_hi) {
                        bad |= !isfinite(x);
                        if (trn) trn[g] = x;
                        if (a.fwd_obs && sl >= 0) {
                            const int bb = net.pmap[g];
                            if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                        }
                    }
                }
            }
            __syncthreads();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    if (ta.bout)
        for (int e = c_lo + tid; e < c_hi; e += nt) ta.bout[col * n + rg.gidx(e)] = cur[e];
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_FWD_NONFINITE);
}

// ---------------------------------------------------------------- adjoint
template <int KIND>
__global__ void __launch_bounds__(kThreads) tiled_adj_kernel(const TiledArgs ta, unsigned* status) {
    extern __shared__ double sm[];
    const ModelDev& md = ta.md;
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int R = geo.R;
    double* cur = sm;
    double* nxt = sm + R;
    double* t1 = sm + 2 * R;
    double* t2 = sm + 3 * R;
    double* acc = sm + 4 * R;
    const int64_t n = md.n;
    const int64_t col = blockIdx.x;
    const int64_t tile = blockIdx.y;
    const int64_t t0 = tile * geo.T;
    const int tid = threadIdx.x, nt = blockDim.x;
    // adjoint radius mirrors the TL one: (rr, rl)
    int rl, rr;
    model_radius(md.kind, rr, rl);
    const int HL = geo.resident ? 0 : geo.HR, HRr = geo.resident ? 0 : geo.HL;
    (void)HRr;
    Region rg{R, geo.resident, geo.resident ? 0 : (int)(t0 - HL), (int)n};
    const int c_lo = geo.resident ? 0 : HL;
    const int c_hi = geo.resident ? R : HL + (int)(n - t0 < (int64_t)geo.T ? n - t0 : (int64_t)geo.T);
    const int s = md.s;
    const double* V = a.V ? a.V + col * a.ldv : nullptr;
    const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* Sv = a.S + col * a.lds;
    const int np = net.n_points;
    bool bad = false;

    auto addend = [&](int i, int g) -> double {
        double x = V ? V[(int64_t)i * n + g] : 0.0;
        if (a.adj_obs) {
            const int sl = net.slot[i];
            if (sl >= 0) {
                int bb;
                if (net.sx) {
                    const int q = g / net.sx;
                    bb = q * net.sx == g ? q : -1;
                } else {
                    bb = net.pmap[g];
                }
                if (bb >= 0) x = V ? x + Yc[(int64_t)sl * np + bb] : Yc[(int64_t)sl * np + bb];
            }
        }
        return x;
    };

    // state s_{i1}
    if (ta.bin) {
        for (int e = tid; e < R; e += nt) cur[e] = ta.bin[col * n + rg.gidx(e)];
    } else {  // s_N = v_N + H_N^T y
        for (int e = tid; e < R; e += nt) {
            const int g = rg.gidx(e);
            const double x = addend(ta.i1, g);
            cur[e] = x;
            if (e >= c_lo && e < c_hi) {
                Sv[(int64_t)ta.i1 * n + g] = x;
                bad |= !isfinite(x);
            }
        }
    }
    __syncthreads();
    double* sbuf[2] = {sm + 5 * R + 2, sm + 6 * R + 6};  // guarded stage buffers (see fwd)
    int sbi = 0;
    if (KIND == WC4DVAR_MODEL_LORENZ96 && ta.i1 > ta.i0) {  // x4 of the last sub-step
        stage_load(sbuf[0], md.stages + (((int64_t)ta.i1 * s - 1) * 4 + 3) * n, rg, R, tid, nt);
        cp_async_wait_all();
        __syncthreads();
    }
    int lo = 0, hi = R;
    for (int i = ta.i1 - 1; i >= ta.i0; --i) {
        for (int kk = 0; kk < s; ++kk) {
            const int k = s - 1 - kk;  // sub-steps in reverse
            if (!geo.resident) {
                lo += rl;
                hi -= rr;
            }
            const bool last = (kk + 1 == s);
            if (KIND != WC4DVAR_MODEL_LORENZ96) {
                for (int e = lo + tid; e < hi; e += nt) nxt[e] = stencil1<KIND, true>(cur, rg, e, md.c, md.d);
            } else {
                // RK4 adjoint step (models.cpp:130-148)
                const double* st = md.stages + ((int64_t)i * s + k) * 4 * n;
                const double dt = md.dt, ee = dt / 6.0;
                const int l1 = geo.resident ? 0 : lo - 3, h1 = geo.resident ? R : hi + 6;
                stage_load(sbuf[sbi ^ 1], st + 2 * n, rg, R, tid, nt);
                for (int e = max(l1, 0) + tid; e < min(h1, R); e += nt) {
                    const double w = l96_jac_t_s(sbuf[sbi], cur, rg, e, ee);  // stage x4
                    acc[e] = cur[e] + w;
                    t1[e] = 2.0 * ee * cur[e] + dt * w;
                }
                stage_sync(sbi);
                const int l2 = geo.resident ? 0 : lo - 2, h2 = geo.resident ? R : hi + 4;
                stage_load(sbuf[sbi ^ 1], st + n, rg, R, tid, nt);
                for (int e = max(l2, 0) + tid; e < min(h2, R); e += nt) {
                    const double w = l96_jac_t_s(sbuf[sbi], t1, rg, e, 1.0);  // x3
                    acc[e] = acc[e] + w;
                    t2[e] = 2.0 * ee * cur[e] + 0.5 * dt * w;
                }
                stage_sync(sbi);
                const int l3 = geo.resident ? 0 : lo - 1, h3 = geo.resident ? R : hi + 2;
                stage_load(sbuf[sbi ^ 1], st, rg, R, tid, nt);
                for (int e = max(l3, 0) + tid; e < min(h3, R); e += nt) {
                    const double w = l96_jac_t_s(sbuf[sbi], t2, rg, e, 1.0);  // x2
                    acc[e] = acc[e] + w;
                    t1[e] = ee * cur[e] + 0.5 * dt * w;
                }
                stage_sync(sbi);
                {  // prefetch x4 of the previous sub-step (next in adjoint order)
                    const bool more = (k > 0) || (i > ta.i0);
                    if (more) stage_load(sbuf[sbi ^ 1], st - 4 * n + 3 * n, rg, R, tid, nt);
                }
                for (int e = lo + tid; e < hi; e += nt) {
                    const double w = l96_jac_t_s(sbuf[sbi], t1, rg, e, 1.0);  // x1
                    nxt[e] = acc[e] + w;
                }
                cp_async_wait_all();
                sbi ^= 1;
            }
            if (last) {
                // s_i = v_i + H_i^T y + M_i^T s_{i+1}  (operators.cpp:99)
                for (int e = lo + tid; e < hi; e += nt) {
                    const int g = rg.gidx(e);
                    const double x = addend(i, g) + nxt[e];
                    nxt[e] = x;
                    if (e >= c_lo && e < c_hi) {
                        Sv[(int64_t)i * n + g] = x;
                        bad |= !isfinite(x);
                    }
                }
            }
            __syncthreads();
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    if (ta.bout)
        for (int e = c_lo + tid; e < c_hi; e += nt) ta.bout[col * n + rg.gidx(e)] = cur[e];
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_ADJ_NONFINITE);
}

// ---------------------------------------------------------------- register-blocked tiles
// Radius-1 models with S sub-steps per interval: each thread owns P consecutive region
// points, gathers them with an S-point halo from SMEM once per interval and applies the
// S sub-steps in registers as one fused stencil (one barrier per interval instead of per
// sub-step).  Region R = nt * P = T + 2 K S; the valid region shrinks by S per side per
// interval.
//
// Gather P + 2S region values and apply the fused S-step stencil; results in v[S .. S+P).
// Rows carry GO >= ceil(S / P) guard slots on each side (`cur` points at the first region
// slot), so EVERY thread gathers with one base register and immediate offsets: no clamped
// edge path, whose two divergent warps per CTA used to hold every interval barrier (C4
// sweeps 7.4 -> 5.9 ms at m = 64).  Guard slots hold whatever was there; they only feed
// points outside the valid region, which are never emitted.
template <int S, int P>
__device__ __forceinline__ void blk_conv(const double* __restrict__ cur, int b, int ns, const StencilTaps& tp,
                                           double (&v)[P + 2 * S]) {
    constexpr int L = P + 2 * S;
    const double* base = cur + b / P;
#pragma unroll
    for (int u = 0; u < L; ++u) {
        const int d = u - S;
        const int dm = ((d % P) + P) % P, dq = (d - dm) / P;
        v[u] = base[dm * ns + dq];
    }
    double o[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        double acc = tp.t[0] * v[p];
#pragma unroll
        for (int k = 1; k <= 2 * S; ++k) acc = fma(tp.t[k], v[p + k], acc);
        o[p] = acc;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) v[S + p] = o[p];
}

// SMEM rows of the blocked tiles are point-major with a padded stride ns = nt + 2: region
// point e lives at (e % P) * ns + e / P.  Per-thread gathers (blk_conv) and the owner's
// P results then hit 32 consecutive slots per warp (conflict-free), and the coalesced
// row passes (loads, trajectory / state emits) see at most 2-way conflicts.
__device__ __forceinline__ void cp8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

// Row loads of the blocked tiles: element e = tid + k nt (k < P) of a region row goes to
// slot(e).  With nt % P == 0 and a region that does not cross the periodic boundary (every
// tile but the first and last of a column), the slot is s0 + k nt / P and the grid index
// origin + tid + k nt, so the loop is cp.async with immediate offsets on both sides.
template <int P, int NT>
struct RowPlan {
    int s0;    // slot of element tid
    int g0;    // grid index of element tid
    bool fast;
    __device__ void init(const Region& rg, int R, int tid, int nt, int ns, int go) {
        fast = nt % P == 0 && R == nt * P && rg.origin >= 0 && rg.origin + R <= rg.n;
        s0 = (tid % P) * ns + tid / P + go;
        g0 = rg.origin + tid;
    }
    template <class Slot>
    __device__ __forceinline__ void load(double* dst, const double* row, const Region& rg, int R, int tid, int nt,
                                         Slot slot) const {
        if (fast) {
            const int w = NT ? NT : nt;
            const double* src = row + g0;
            double* d = dst + s0;
#pragma unroll
            for (int k = 0; k < P; ++k) cp8(d + k * (w / P), src + k * w);
        } else {
            for (int e = tid; e < R; e += nt) cp8(dst + slot(e), row + rg.gidx(e));
        }
        asm volatile("cp.async.commit_group;\n");
    }
};

// Each CTA runs intervals i0..i1 of one tile of one column.  Per interval: one barrier,
// then (a) a coalesced pass that emits the previous state's tile centre (finite check,
// trajectory, observations -- stores coalesced instead of stride-P per thread), (b) the
// next interval's forcing row issued by cp.async into a double buffer (lands while the S
// sub-steps compute), (c) the register-blocked advance.  Every thread advances all its P
// points every interval: points that left the valid region (S per side per interval) only
// ever feed other invalid points and are never emitted, so no per-point validity test is
// needed.  NT = threads per CTA as a compile-time constant (0: blockDim.x).
template <int KIND, int S, int P, int NT>
__global__ void __launch_bounds__(NT ? NT : 512, NT == 256 ? 2 : 1) tiled_blk_fwd_kernel(const TiledArgs ta, unsigned* status) {
    extern __shared__ double sm[];
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int R = geo.R;
    const int tid = threadIdx.x, nt = NT ? NT : blockDim.x;
    constexpr int GO = (S + P - 1) / P;  // guard slots per row side
    const int ns = nt + 2 + 2 * GO, RS = P * ns;
    double* cur = sm;
    double* nxt = sm + RS;
    double* const fx0 = sm + 2 * RS;  // forcing X_{i+1}, prefetched (double buffer)
    double* const fx1 = sm + 3 * RS;
    const int n = (int)ta.md.n;
    const int64_t col = blockIdx.x;
    const int64_t t0 = (int64_t)blockIdx.y * geo.T;
    const Region rg{R, false, (int)(t0 - geo.HL), n};
    const int c_lo = geo.HL;
    const int c_hi = geo.HL + (int)((int64_t)n - t0 < geo.T ? (int64_t)n - t0 : geo.T);
    const double* X = a.X + col * a.ldx;
    double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
    const int np = net.n_points;
    const int b = tid * P;
    bool bad = false;
    double v[P + 2 * S];
    auto slot = [&](int e) { return (e % P) * ns + e / P + GO; };
    RowPlan<P, NT> rp;
    rp.init(rg, R, tid, nt, ns, GO);
    // regular network: observed points g = bb sx of the tile centre [g0, g1), bb from bb0
    const int sx = net.sx;
    const int g0 = (int)t0, g1 = (int)(t0 + (c_hi - c_lo));
    const int bb0 = sx ? (g0 + sx - 1) / sx : 0;

    if (ta.i1 > ta.i0) rp.load(fx0, X + (int64_t)(ta.i0 + 1) * n, rg, R, tid, nt, slot);
    const double* src = ta.bin ? ta.bin + col * n : X;  // x_0 = X_0
    for (int e = tid; e < R; e += nt) cur[slot(e)] = src[rg.gidx(e)];
    for (int i = ta.i0;; ++i) {
        cp_async_wait_all();
        __syncthreads();
        // emit x_i on the tile centre (x_{i0} only at the window start: otherwise the
        // previous launch emitted it).  Non-finite values cannot vanish along a linear sweep
        // (NaN / Inf propagate through every tap), so the finite check runs on the launch's
        // last state only; with a regular network only the observed points are visited.
        if (i > ta.i0 || ta.i0 == 0) {
            const int sl = net.slot[i];
            double* tri = tr ? tr + (int64_t)i * n : nullptr;
            const bool last = i == ta.i1;
            if (tri || last || (a.fwd_obs && sl >= 0 && !sx)) {
                for (int e = c_lo + tid; e < c_hi; e += nt) {
                    const int g = rg.gidx(e);
                    const double x = cur[slot(e)];
                    if (last) bad |= !isfinite(x);
                    if (tri) tri[g] = x;
                    if (a.fwd_obs && sl >= 0 && !sx) {
                        const int bb = net.pmap[g];
                        if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * x;
                    }
                }
            }
            if (a.fwd_obs && sl >= 0 && sx) {
                double* ys = Yc + (int64_t)sl * np;
                for (int bb = bb0 + tid; bb * sx < g1; bb += nt) ys[bb] = a.scale_fwd * cur[slot(bb * sx - g0 + c_lo)];
            }
        }
        if (i == ta.i1) break;
        const int k = i - ta.i0;
        if (i + 2 <= ta.i1) rp.load((k & 1) ? fx0 : fx1, X + (int64_t)(i + 2) * n, rg, R, tid, nt, slot);
        blk_conv<S, P>(cur + GO, b, ns, ta.tp, v);  // M_i = the S-step TL as one stencil
        const double* f = (k & 1) ? fx1 : fx0;
#pragma unroll
        for (int p = 0; p < P; ++p)  // x_{i+1} = M_i x_i + X_{i+1}  (operators.cpp:88)
            nxt[p * ns + tid + GO] = v[S + p] + f[p * ns + tid + GO];
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (ta.bout)
        for (int e = c_lo + tid; e < c_hi; e += nt) ta.bout[col * n + rg.gidx(e)] = cur[slot(e)];
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_FWD_NONFINITE);
}

template <int KIND, int S, int P, int NT>
__global__ void __launch_bounds__(NT ? NT : 512, NT == 256 ? 2 : 1) tiled_blk_adj_kernel(const TiledArgs ta, unsigned* status) {
    extern __shared__ double sm[];
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int R = geo.R;
    const int tid = threadIdx.x, nt = NT ? NT : blockDim.x;
    constexpr int GO = (S + P - 1) / P;  // guard slots per row side
    const int ns = nt + 2 + 2 * GO, RS = P * ns;
    double* cur = sm;
    double* nxt = sm + RS;
    double* const vb0 = sm + 2 * RS;  // v_{i-1} rows, prefetched (double buffer)
    double* const vb1 = sm + 3 * RS;
    const int n = (int)ta.md.n;
    const int64_t col = blockIdx.x;
    const int64_t t0 = (int64_t)blockIdx.y * geo.T;
    const Region rg{R, false, (int)(t0 - geo.HR), n};
    const int c_lo = geo.HR;
    const int c_hi = geo.HR + (int)((int64_t)n - t0 < geo.T ? (int64_t)n - t0 : geo.T);
    const double* V = a.V ? a.V + col * a.ldv : nullptr;
    const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* Sv = a.S + col * a.lds;
    const int np = net.n_points;
    const int b = tid * P;
    bool bad = false;
    double v[P + 2 * S];
    auto slot = [&](int e) { return (e % P) * ns + e / P + GO; };
    RowPlan<P, NT> rp;
    if (V) rp.init(rg, R, tid, nt, ns, GO);
    // H_i^T y part of the addend (sparse: observed points of observed times)
    auto obs_add = [&](int i, int g, double x) -> double {
        if (a.adj_obs) {
            const int sl = net.slot[i];
            if (sl >= 0) {
                int bb;
                if (net.sx) {
                    const int q = g / net.sx;
                    bb = (q * net.sx == g) ? q : -1;
                } else {
                    bb = net.pmap[g];
                }
                if (bb >= 0) x = V ? x + Yc[(int64_t)sl * np + bb] : Yc[(int64_t)sl * np + bb];
            }
        }
        return x;
    };
    // regular network: the thread's first point g_b = q_b sx + r_b (interval-invariant)
    const int sx = net.sx;
    const int g_b = rg.gidx(b < R ? b : R - 1);
    const int q_b = sx ? g_b / sx : 0, r_b = sx ? g_b - q_b * sx : 0;
    // H^T y fast path (no addend v, regular network with sx >= P / 2, region not wrapping):
    // the thread's observed points are op and op + sx (< P), y indices qf, qf + 1.  The
    // stencil result is stored first and y added in place by the owner thread: y + M^T s
    // either way (addition commutes), without per-point selects.
    const bool fobs_ok = !V && sx >= P / 2 && rg.origin >= 0 && rg.origin + R <= n;
    const int op = sx ? (sx - r_b) % sx : P;
    const int qf = q_b + (r_b ? 1 : 0);
    // tile centre rows are contiguous in the grid (no wrap): g = t0 + (e - c_lo)
    const bool inc = nt % P == 0;

    if (V && ta.i1 > ta.i0) rp.load(vb0, V + (int64_t)(ta.i1 - 1) * n, rg, R, tid, nt, slot);
    if (ta.bin) {
        for (int e = tid; e < R; e += nt) cur[slot(e)] = ta.bin[col * n + rg.gidx(e)];
    } else {  // s_N = v_N + H_N^T y
        for (int e = tid; e < R; e += nt) {
            const int g = rg.gidx(e);
            cur[slot(e)] = obs_add(ta.i1, g, V ? V[(int64_t)ta.i1 * n + g] : 0.0);
        }
    }
    for (int i = ta.i1;; --i) {  // cur = s_i
        cp_async_wait_all();
        __syncthreads();
        if (i < ta.i1 || !ta.bin) {  // emit s_i on the tile centre (finite check: last state)
            const bool last = i == ta.i0;
            double* Si = Sv + (int64_t)i * n;
            if (inc) {
                int s = slot(c_lo + tid);
                for (int e = c_lo + tid; e < c_hi; e += nt, s += nt / P) {
                    const double x = cur[s];
                    Si[t0 + (e - c_lo)] = x;
                    if (last) bad |= !isfinite(x);
                }
            } else {
                for (int e = c_lo + tid; e < c_hi; e += nt) {
                    const double x = cur[slot(e)];
                    Si[rg.gidx(e)] = x;
                    if (last) bad |= !isfinite(x);
                }
            }
        }
        if (i == ta.i0) break;
        const int k = ta.i1 - i;
        if (V && i - 2 >= ta.i0) rp.load((k & 1) ? vb0 : vb1, V + (int64_t)(i - 2) * n, rg, R, tid, nt, slot);
        // H^T y of the thread's P points first: all y loads in flight before the stencil
        // (the loads' latency then hides under the FMA chains)
        const int sl = a.adj_obs ? net.slot[i - 1] : -1;
        const bool fobs = fobs_ok && sl >= 0;
        double y0 = 0.0, y1 = 0.0;
        double yv[P];
        bool has[P];
        if (fobs) {
            const double* ys = Yc + (int64_t)sl * np;
            if (op < P) y0 = ys[qf];
            if (op + sx < P) y1 = ys[qf + 1];
#pragma unroll
            for (int p = 0; p < P; ++p) has[p] = false, yv[p] = 0.0;
        } else if (sl >= 0) {
            const double* ys = Yc + (int64_t)sl * np;
            if (sx) {  // regular network: observed iff g % sx == 0, bb = g / sx
                int g = g_b, q = q_b, r = r_b;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    has[p] = r == 0;
                    yv[p] = has[p] ? ys[q] : 0.0;
                    if (++g == n) g = q = r = 0;  // periodic wrap
                    else if (++r == sx) r = 0, ++q;
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const int bb = net.pmap[rg.gidx(min(b + p, R - 1))];
                    has[p] = bb >= 0;
                    yv[p] = has[p] ? ys[bb] : 0.0;
                }
            }
        } else {
#pragma unroll
            for (int p = 0; p < P; ++p) has[p] = false, yv[p] = 0.0;
        }
        blk_conv<S, P>(cur + GO, b, ns, ta.tp, v);  // M_i^T as one stencil
        const double* vr = (k & 1) ? vb1 : vb0;
        if (fobs) {
#pragma unroll
            for (int p = 0; p < P; ++p) nxt[p * ns + tid + GO] = v[S + p];
            if (op < P) nxt[op * ns + tid + GO] += y0;
            if (op + sx < P) nxt[(op + sx) * ns + tid + GO] += y1;
        } else {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                // s_{i-1} = v_{i-1} + H^T y + M^T s_i  (operators.cpp:99; obs_add order)
                double ad = V ? vr[p * ns + tid + GO] : 0.0;
                if (has[p]) ad = V ? ad + yv[p] : yv[p];
                nxt[p * ns + tid + GO] = ad + v[S + p];
            }
        }
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (ta.bout)
        for (int e = c_lo + tid; e < c_hi; e += nt) ta.bout[col * n + rg.gidx(e)] = cur[slot(e)];
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_ADJ_NONFINITE);
}

// Register-blocked tiled launch (radius-1 models, S in {1,5,10}, one fused S-step stencil
// per interval); false if not applicable.
template <int KIND, int S>
bool launch_tiled_blk(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                      cudaStream_t st, DevBuf& ws, int tile_override) {
    constexpr int P = 8;
    // WC4DVAR_TILED_NT: threads per CTA (256 default: two CTAs per SM, whose interval
    // barriers interleave -- C4 m = 64 sweeps 8.6 vs 9.3 ms with one 512-thread CTA); both
    // widths have compile-time instantiations.  WC4DVAR_TILED_KDIV: halo budget R / KDIV for
    // the intervals per launch (4 default)
    static const int nt_env = [] {
        const char* e = std::getenv("WC4DVAR_TILED_NT");
        return e ? std::atoi(e) : 256;
    }();
    static const int kdiv = [] {
        const char* e = std::getenv("WC4DVAR_TILED_KDIV");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    int nt = nt_env;
    int K = md.N;
    int R = nt * P;
    while (K > 1 && 2 * K * S > R / kdiv) --K;
    int T = R - 2 * K * S;
    if (tile_override > 0) {
        T = tile_override;
        K = std::max(1, std::min(md.N, std::max(T / (8 * S), 1)));
        R = T + 2 * K * S;
        nt = (int)cdiv(R, P);
        R = nt * P;
        T = R - 2 * K * S;
    }
    if (nt > 512 || T <= 0 || R > md.n) return false;
    TileGeom geo{T, K * S, K * S, R, false, cdiv(md.n, T)};
    const size_t smem = sizeof(double) * 4 * (size_t)P * (nt + 2 + 2 * ((S + P - 1) / P));  // cur, nxt, 2 prefetch rows
    auto fk = nt == 512 ? tiled_blk_fwd_kernel<KIND, S, P, 512>
              : nt == 256 ? tiled_blk_fwd_kernel<KIND, S, P, 256> : tiled_blk_fwd_kernel<KIND, S, P, 0>;
    auto ak = nt == 512 ? tiled_blk_adj_kernel<KIND, S, P, 512>
              : nt == 256 ? tiled_blk_adj_kernel<KIND, S, P, 256> : tiled_blk_adj_kernel<KIND, S, P, 0>;
    W4_CUDA(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    W4_CUDA(cudaFuncSetAttribute(ak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nl = (int)cdiv(md.N, K);
    double* bbuf = nl > 1 ? ws.get<double>((size_t)2 * md.n * a.m) : nullptr;
    const dim3 grid((unsigned)a.m, (unsigned)geo.ntiles);
    TiledArgs ta{md, net, a, geo, 0, 0, nullptr, nullptr};
    if (a.do_fwd)
        for (int l = 0; l < nl; ++l) {
            ta.i0 = l * K;
            ta.i1 = std::min(md.N, (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            ta.tp = stencil_power(KIND, md.c, md.d, S, false);
            fk<<<grid, nt, smem, st>>>(ta, status);
            W4_LAUNCH();
        }
    if (a.do_adj)
        for (int l = 0; l < nl; ++l) {
            ta.i1 = md.N - l * K;
            ta.i0 = std::max(0, md.N - (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            ta.tp = stencil_power(KIND, md.c, md.d, S, true);
            ak<<<grid, nt, smem, st>>>(ta, status);
            W4_LAUNCH();
        }
    return true;
}

// ---------------------------------------------------------------- Lorenz-96, register-blocked
// CB sketch columns share one CTA and one SMEM copy of each RK4 stage slice; each thread
// keeps P consecutive region points of one column in registers.  One phase = one Jacobian
// product (models.cpp:92-116): the thread publishes its P values to an SMEM exchange row,
// one barrier, then reads its 2+1 (TL) / 1+2 (adjoint) halo values and the stage slice
// around its points (LDS.128).  Exchange rows and stage buffers are double-buffered, so a
// phase costs a single barrier while the next stage streams in by cp.async.  Arithmetic is
// written in the same order as the SMEM kernels above (and the oracle).
constexpr int kL96P = 8;
constexpr int kL96G = 0;  // (rows carry their guards inside the interleaved layout)

// SMEM rows use an interleaved layout so every per-thread access is a conflict-free LDS.128
// / STS.128 across the warp: point pair (2k, 2k+1) of thread j lives at double2 slot
// k (NTC + 2) + j + 1; slots j = -1 and j = NTC are the left / right guards.
template <int CB, int NTC_>
struct L96Lay {
    static constexpr int NTC = NTC_;              // threads per column
    static constexpr int NT = CB * NTC;           // threads per CTA
    static constexpr int R = NTC * kL96P;         // region points
    // row size in doubles, padded so consecutive exchange rows start 8 / CB bank groups
    // apart -- with column-fast lanes (lane = j CB + column) a quarter warp's 8 STS / LDS.128
    // then hit 8 distinct 16-byte bank groups
    static constexpr int LD = kL96P * (NTC + 2) + 2 * (8 / (CB < 8 ? CB : 8));
    // 4 stage ring buffers + 2 x CB exchange rows
    static constexpr size_t smem_bytes = sizeof(double) * (4 * LD + 2 * CB * LD);
};
template <int NTC>
__device__ __forceinline__ int l96_slot(int k, int j) { return k * (NTC + 2) + j + 1; }

// Region slice [-2, R+2) of one stage vector -> interleaved SMEM row (8-byte cp.async).
template <int P, int NTC>
__device__ __forceinline__ void stage_load_il(double* dst, const double* __restrict__ src, const Region& rg,
                                              int R, int tid, int nt) {
    // consecutive threads take consecutive point pairs, so the global reads coalesce
    for (int pi = tid; pi < R / 2 + 2; pi += nt) {
        const int e = 2 * pi - 2;
        const int jj = (e + P) / P - 1;  // floor(e / P) for e >= -P
        const int k = (e - jj * P) >> 1;
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + 2 * l96_slot<NTC>(k, jj)));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + rg.gidx(e)));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 8), "l"(src + rg.gidx(e + 1)));
    }
    asm volatile("cp.async.commit_group;\n");
}

template <int P, int NTC>
__device__ __forceinline__ void l96_publish(double* exr, int b, const double (&v)[P]) {
    double2* r2 = reinterpret_cast<double2*>(exr);
    const int j = b / P;
    // neighbours read only the first and the last point pair of a thread (the TL / adjoint
    // halos are 2 + 1 points), so only those two pairs are published
    r2[l96_slot<NTC>(0, j)] = make_double2(v[0], v[1]);
    r2[l96_slot<NTC>(P / 2 - 1, j)] = make_double2(v[P - 2], v[P - 1]);
}

template <int P, int NTC>
__device__ __forceinline__ void l96_stage_regs(const double* xs, int j, double (&xv)[P + 4]) {
    const double2* r2 = reinterpret_cast<const double2*>(xs);
    const double2 lft = r2[l96_slot<NTC>(P / 2 - 1, j - 1)], rgt = r2[l96_slot<NTC>(0, j + 1)];
    xv[0] = lft.x;  // x[b-2 .. b+P+1]
    xv[1] = lft.y;
#pragma unroll
    for (int k = 0; k < P / 2; ++k) {
        const double2 q = r2[l96_slot<NTC>(k, j)];
        xv[2 + 2 * k] = q.x;
        xv[3 + 2 * k] = q.y;
    }
    xv[P + 2] = rgt.x;
    xv[P + 3] = rgt.y;
}

// a = J(x) v on the thread's points (l96_jac_s order)
template <int P, int NTC>
__device__ __forceinline__ void l96_tl_phase(const double* xs, const double* exr, int b, const double (&v)[P],
                                             double (&out)[P]) {
    const int j = b / P;
    double xv[P + 4];
    l96_stage_regs<P, NTC>(xs, j, xv);
    const double2* e2 = reinterpret_cast<const double2*>(exr);
    double w[P + 3];  // v[b-2 .. b+P]
    const double2 h = e2[l96_slot<NTC>(P / 2 - 1, j - 1)];
    w[0] = h.x;
    w[1] = h.y;
#pragma unroll
    for (int p = 0; p < P; ++p) w[p + 2] = v[p];
    w[P + 2] = e2[l96_slot<NTC>(0, j + 1)].x;
#pragma unroll
    for (int p = 0; p < P; ++p)
        out[p] = -w[p] * xv[p + 1] - xv[p] * w[p + 1] + w[p + 1] * xv[p + 3] + xv[p + 1] * w[p + 3] - w[p + 2];
}

// w = J(x)^T (scale l) on the thread's points (l96_jac_t_s order)
template <int P, int NTC>
__device__ __forceinline__ void l96_adj_phase(const double* xs, const double* exr, int b, const double (&l)[P],
                                              double scale, double (&out)[P]) {
    const int j = b / P;
    double xv[P + 4];
    l96_stage_regs<P, NTC>(xs, j, xv);
    const double2* e2 = reinterpret_cast<const double2*>(exr);
    double w[P + 3];  // l[b-1 .. b+P+1]
    w[0] = e2[l96_slot<NTC>(P / 2 - 1, j - 1)].y;
#pragma unroll
    for (int p = 0; p < P; ++p) w[p + 1] = l[p];
    const double2 h = e2[l96_slot<NTC>(0, j + 1)];
    w[P + 1] = h.x;
    w[P + 2] = h.y;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const double lp2 = scale * w[p + 3], lp1 = scale * w[p + 2], lm1 = scale * w[p], lc = scale * w[p + 1];
        out[p] = -xv[p + 3] * lp2 + (xv[p + 4] - xv[p + 1]) * lp1 + xv[p] * lm1 - lc;
    }
}

// Stage sg (global RK4 stage index (interval * s + sub-step) * 4 + stage; one per phase)
// -> ring buffer sg & 3.  Each phase issues exactly one commit group (empty outside
// [lo, hi)) so that the phase barrier's wait_group 2 leaves the next two stages in flight.
template <int P, int NTC>
__device__ __forceinline__ void l96_prefetch(double* sx, int LD, const double* __restrict__ stages, int64_t sg,
                                             int64_t lo, int64_t hi, int n, const Region& rg, int R, int tid,
                                             int nt) {
    if (sg >= lo && sg < hi)
        stage_load_il<P, NTC>(sx + (int)(sg & 3) * LD, stages + sg * n, rg, R, tid, nt);
    else
        asm volatile("cp.async.commit_group;\n");
}

// barrier of one phase: this thread's copies of the current stage land (two newer stages
// may stay in flight), everyone's exchange row and stage copies are visible
#define L96_PHASE_SYNC()                                          \
    do {                                                          \
        asm volatile("cp.async.wait_group 2;\n" ::: "memory"); \
        __syncthreads();                                          \
    } while (0)
#define L96_PREFETCH() \
    l96_prefetch<P, Lay::NTC>(sx, LD, md.stages, sg + 3 * kDir, sg_lo, sg_hi, n, rg, R, tid, nt)

template <int CB, int NTC>
__global__ void __launch_bounds__(CB * NTC, 65536 / (CB * NTC * 128)) l96_blk_fwd_kernel(const TiledArgs ta, unsigned* status) {
    using Lay = L96Lay<CB, NTC>;
    constexpr int P = kL96P, R = Lay::R, LD = Lay::LD, G = kL96G;
    extern __shared__ __align__(16) double l96sm[];
    double* sx = l96sm;           // [2][LD] stage slices
    double* ex = l96sm + 4 * LD;  // [2][CB][LD] exchange rows
    const ModelDev& md = ta.md;
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int n = (int)md.n;
    const int tid = threadIdx.x, nt = blockDim.x;
    // column-fast lanes: the CB threads that own the same points of different columns are
    // adjacent, so their stage-slice loads (same addresses) are served as SMEM broadcasts
    const int cg = tid % CB, b = (tid / CB) * P;
    const int64_t col = (int64_t)blockIdx.x * CB + cg;
    const bool live = col < a.m;
    const int64_t t0 = (int64_t)blockIdx.y * geo.T;
    const Region rg{R, false, (int)(t0 - geo.HL), n};
    const int c_lo = geo.HL;
    const int c_hi = geo.HL + (int)((int64_t)n - t0 < geo.T ? (int64_t)n - t0 : geo.T);
    const int s = md.s;
    const double dt = md.dt;
    const double* X = a.X + (live ? col : 0) * a.ldx;
    double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* tr = a.traj ? a.traj + col * a.ldtraj : nullptr;
    const int np = net.n_points;
    bool bad = false;

    for (int r = tid; r < 2 * CB * P; r += nt) {  // exchange-row guard slots: finite, never written
        const int row = r / P, k = (r % P) >> 1, side = r & 1;
        reinterpret_cast<double2*>(ex + row * LD)[l96_slot<Lay::NTC>(k, side ? Lay::NTC : -1)] =
            make_double2(0.0, 0.0);
    }
    constexpr int kDir = 1;  // stages consumed in increasing order
    const int64_t sg_lo = (int64_t)ta.i0 * s * 4, sg_hi = (int64_t)ta.i1 * s * 4;
    int64_t sg = sg_lo;
    for (int u = 0; u < 3; ++u) l96_prefetch<P, Lay::NTC>(sx, LD, md.stages, sg + u, sg_lo, sg_hi, n, rg, R, tid, nt);

    double cur[P], t[P], acc[P], av[P];
    {
        const double* src = ta.bin ? ta.bin + col * n : X;
#pragma unroll
        for (int p = 0; p < P; ++p) cur[p] = live ? src[rg.gidx(b + p)] : 0.0;
    }
    if (ta.i0 == 0 && live) {
        const int sl = net.slot[0];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int e = b + p;
            if (e >= c_lo && e < c_hi) {
                const int g = rg.gidx(e);
                bad |= !isfinite(cur[p]);
                if (tr) tr[g] = cur[p];
                if (a.fwd_obs && sl >= 0) {
                    const int bb = net.pmap[g];
                    if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * cur[p];
                }
            }
        }
    }
    int pb = 0;
    for (int i = ta.i0; i < ta.i1; ++i) {
        // forcing X_{i+1} of this interval's end, loaded now so its latency hides under the
        // s RK4 steps
        double xf[P];
        if (live) {
            const double* Xn = X + (int64_t)(i + 1) * n;
#pragma unroll
            for (int p = 0; p < P; ++p) xf[p] = Xn[rg.gidx(b + p)];
        }
        for (int k = 0; k < s; ++k) {
            // RK4 TL step (models.cpp:120-128)
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, cur);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_tl_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, cur, av);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = av[p];
                t[p] = cur[p] + 0.5 * dt * av[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_tl_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, av);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = acc[p] + 2.0 * av[p];
                t[p] = cur[p] + 0.5 * dt * av[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_tl_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, av);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = acc[p] + 2.0 * av[p];
                t[p] = cur[p] + dt * av[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_tl_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, av);
#pragma unroll
            for (int p = 0; p < P; ++p) cur[p] = cur[p] + (dt / 6.0) * (acc[p] + av[p]);
            sg += kDir;
            pb ^= 1;
        }
        // x_{i+1} = M_i x_i + X_{i+1}  (operators.cpp:88)
        if (live) {
            const int sl = net.slot[i + 1];
            double* trn = tr ? tr + (int64_t)(i + 1) * n : nullptr;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const int e = b + p;
                const int g = rg.gidx(e);
                cur[p] = cur[p] + xf[p];
                if (e >= c_lo && e < c_hi) {
                    bad |= !isfinite(cur[p]);
                    if (trn) trn[g] = cur[p];
                    if (a.fwd_obs && sl >= 0) {
                        int bb;
                        if (net.sx) {
                            const int q = g / net.sx;
                            bb = q * net.sx == g ? q : -1;
                        } else {
                            bb = net.pmap[g];
                        }
                        if (bb >= 0) Yc[(int64_t)sl * np + bb] = a.scale_fwd * cur[p];
                    }
                }
            }
        }
    }
    if (ta.bout && live) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int e = b + p;
            if (e >= c_lo && e < c_hi) ta.bout[col * n + rg.gidx(e)] = cur[p];
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_FWD_NONFINITE);
}

template <int CB, int NTC>
__global__ void __launch_bounds__(CB * NTC, 65536 / (CB * NTC * 128)) l96_blk_adj_kernel(const TiledArgs ta, unsigned* status) {
    using Lay = L96Lay<CB, NTC>;
    constexpr int P = kL96P, R = Lay::R, LD = Lay::LD, G = kL96G;
    extern __shared__ __align__(16) double l96sm[];
    double* sx = l96sm;
    double* ex = l96sm + 4 * LD;
    const ModelDev& md = ta.md;
    const NetDev& net = ta.net;
    const SweepArgs& a = ta.a;
    const TileGeom& geo = ta.geo;
    const int n = (int)md.n;
    const int tid = threadIdx.x, nt = blockDim.x;
    // column-fast lanes: the CB threads that own the same points of different columns are
    // adjacent, so their stage-slice loads (same addresses) are served as SMEM broadcasts
    const int cg = tid % CB, b = (tid / CB) * P;
    const int64_t col = (int64_t)blockIdx.x * CB + cg;
    const bool live = col < a.m;
    const int64_t t0 = (int64_t)blockIdx.y * geo.T;
    const Region rg{R, false, (int)(t0 - geo.HR), n};  // adjoint: mirrored halos
    const int c_lo = geo.HR;
    const int c_hi = geo.HR + (int)((int64_t)n - t0 < geo.T ? (int64_t)n - t0 : geo.T);
    const int s = md.s;
    const double dt = md.dt, ee = dt / 6.0;
    const double* V = a.V ? a.V + col * a.ldv : nullptr;
    const double* Yc = a.Y ? a.Y + col * net.q : nullptr;
    double* Sv = a.S + col * a.lds;
    const int np = net.n_points;
    bool bad = false;
    auto addend = [&](int i, int g) -> double {
        double x = V ? V[(int64_t)i * n + g] : 0.0;
        if (a.adj_obs) {
            const int sl = net.slot[i];
            if (sl >= 0) {
                const int bb = net.pmap[g];
                if (bb >= 0) x = V ? x + Yc[(int64_t)sl * np + bb] : Yc[(int64_t)sl * np + bb];
            }
        }
        return x;
    };

    for (int r = tid; r < 2 * CB * P; r += nt) {
        const int row = r / P, k = (r % P) >> 1, side = r & 1;
        reinterpret_cast<double2*>(ex + row * LD)[l96_slot<Lay::NTC>(k, side ? Lay::NTC : -1)] =
            make_double2(0.0, 0.0);
    }
    constexpr int kDir = -1;  // stages consumed in decreasing order (x4 of the last sub-step first)
    const int64_t sg_lo = (int64_t)ta.i0 * s * 4, sg_hi = (int64_t)ta.i1 * s * 4;
    int64_t sg = sg_hi - 1;
    for (int u = 0; u < 3; ++u) l96_prefetch<P, Lay::NTC>(sx, LD, md.stages, sg - u, sg_lo, sg_hi, n, rg, R, tid, nt);

    double cur[P], t[P], acc[P], w[P];
    if (!live) {
#pragma unroll
        for (int p = 0; p < P; ++p) cur[p] = 0.0;
    } else if (ta.bin) {
#pragma unroll
        for (int p = 0; p < P; ++p) cur[p] = ta.bin[col * n + rg.gidx(b + p)];
    } else {  // s_N = v_N + H_N^T y
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int e = b + p;
            const int g = rg.gidx(e);
            cur[p] = addend(ta.i1, g);
            if (e >= c_lo && e < c_hi) {
                Sv[(int64_t)ta.i1 * n + g] = cur[p];
                bad |= !isfinite(cur[p]);
            }
        }
    }
    int pb = 0;
    for (int i = ta.i1 - 1; i >= ta.i0; --i) {
        // v_i + H_i^T y of this interval's end, loaded now (latency hidden by the s steps)
        double adv[P];
        if (live) {
#pragma unroll
            for (int p = 0; p < P; ++p) adv[p] = addend(i, rg.gidx(b + p));
        }
        for (int kk = 0; kk < s; ++kk) {
            // RK4 adjoint step (models.cpp:130-148)
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, cur);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_adj_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, cur, ee, w);  // x4
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = cur[p] + w[p];
                t[p] = 2.0 * ee * cur[p] + dt * w[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_adj_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, 1.0, w);  // x3
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = acc[p] + w[p];
                t[p] = 2.0 * ee * cur[p] + 0.5 * dt * w[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_adj_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, 1.0, w);  // x2
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = acc[p] + w[p];
                t[p] = ee * cur[p] + 0.5 * dt * w[p];
            }
            sg += kDir;
            pb ^= 1;
            l96_publish<P, Lay::NTC>(ex + (pb * CB + cg) * LD + G, b, t);
            L96_PHASE_SYNC();
            L96_PREFETCH();
            l96_adj_phase<P, Lay::NTC>(sx + (int)(sg & 3) * LD, ex + (pb * CB + cg) * LD + G, b, t, 1.0, w);  // x1
#pragma unroll
            for (int p = 0; p < P; ++p) cur[p] = acc[p] + w[p];
            sg += kDir;
            pb ^= 1;
        }
        // s_i = v_i + H_i^T y + M_i^T s_{i+1}  (operators.cpp:99)
        if (live) {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const int e = b + p;
                const int g = rg.gidx(e);
                cur[p] = adv[p] + cur[p];
                if (e >= c_lo && e < c_hi) {
                    Sv[(int64_t)i * n + g] = cur[p];
                    bad |= !isfinite(cur[p]);
                }
            }
        }
    }
    if (ta.bout && live) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int e = b + p;
            if (e >= c_lo && e < c_hi) ta.bout[col * n + rg.gidx(e)] = cur[p];
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status, ST_ADJ_NONFINITE);
}

// Register-blocked Lorenz-96 launch; false if the region does not fit the domain.
template <int CB, int NTC>
bool launch_l96_blk(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                    cudaStream_t st, DevBuf& ws) {
    using Lay = L96Lay<CB, NTC>;
    const int per = md.s * 12;  // (8 + 4) halo points per sub-step
    int K = 1;                  // intervals per launch: redundant halo work 12 s K / R
    while (K < md.N && (K + 1) * per <= Lay::R / 16) ++K;
    const int T = Lay::R - K * per;
    if (T < Lay::R / 2 || Lay::R > md.n) return false;
    TileGeom geo{T, K * md.s * 8, K * md.s * 4, Lay::R, false, cdiv(md.n, T)};
    if (geo.ntiles > 65535) return false;
    auto fk = l96_blk_fwd_kernel<CB, NTC>;
    auto ak = l96_blk_adj_kernel<CB, NTC>;
    W4_CUDA(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::smem_bytes));
    W4_CUDA(cudaFuncSetAttribute(ak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::smem_bytes));
    const int nl = (int)cdiv(md.N, K);
    double* bbuf = nl > 1 ? ws.get<double>((size_t)2 * md.n * a.m) : nullptr;
    const dim3 grid((unsigned)cdiv(a.m, CB), (unsigned)geo.ntiles);
    TiledArgs ta{md, net, a, geo, 0, 0, nullptr, nullptr};
    if (a.do_fwd)
        for (int l = 0; l < nl; ++l) {
            ta.i0 = l * K;
            ta.i1 = std::min(md.N, (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            fk<<<grid, Lay::NT, Lay::smem_bytes, st>>>(ta, status);
            W4_LAUNCH();
        }
    if (a.do_adj)
        for (int l = 0; l < nl; ++l) {
            ta.i1 = md.N - l * K;
            ta.i0 = std::max(0, md.N - (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            ak<<<grid, Lay::NT, Lay::smem_bytes, st>>>(ta, status);
            W4_LAUNCH();
        }
    return true;
}

// WC4DVAR_L96_BLK: 0 = SMEM phase kernels only, 1 = register-blocked whenever the region
// fits the domain (tests), unset = register-blocked for the tiled (large-n) regime.
// WC4DVAR_L96_CB: CTA shape of the register-blocked kernel as columns x threads per column
// (1: 2x256, 2: 4x128, 4: 4x64 (default, 2 CTAs per SM), 8: 8x64, 16: 16x32).
bool try_l96_blk(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status, cudaStream_t st,
                 DevBuf& ws, bool tiled_regime) {
    static const int mode = [] {
        const char* e = std::getenv("WC4DVAR_L96_BLK");
        return e ? std::atoi(e) : -1;
    }();
    static const int cb = [] {
        const char* e = std::getenv("WC4DVAR_L96_CB");
        return e ? std::atoi(e) : 4;
    }();
    if (mode == 0 || (mode < 0 && !tiled_regime)) return false;
    // a single column (PCG, Lanczos) on the 4-column shape would leave 3 / 4 of every CTA
    // idle: one column per CTA, 256 threads
    if (a.m == 1 && !std::getenv("WC4DVAR_L96_CB") && launch_l96_blk<1, 256>(md, net, a, status, st, ws))
        return true;
    switch (cb) {
        case 1: return launch_l96_blk<2, 256>(md, net, a, status, st, ws);
        case 2: return launch_l96_blk<4, 128>(md, net, a, status, st, ws);
        case 4: return launch_l96_blk<4, 64>(md, net, a, status, st, ws);
        case 16: return launch_l96_blk<16, 32>(md, net, a, status, st, ws);
        default: return launch_l96_blk<8, 64>(md, net, a, status, st, ws);
    }
}

template <int KIND>
void launch_tiled(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                  cudaStream_t st, DevBuf& ws, int tile_override) {
    int rl, rr;
    model_radius(md.kind, rl, rr);
    const int nbuf = (KIND == WC4DVAR_MODEL_LORENZ96) ? 7 : 2;
    const int64_t smem_cap = 200 * 1024 / (8 * nbuf);  // region doubles per buffer
    if (KIND == WC4DVAR_MODEL_LORENZ96 && tile_override <= 0 &&
        try_l96_blk(md, net, a, status, st, ws, md.n > smem_cap))
        return;
    TileGeom geo{};
    int K = md.N;  // intervals per launch
    if (md.n <= smem_cap && (tile_override <= 0 || tile_override >= md.n)) {
        geo.resident = true;
        geo.T = (int)md.n;
        geo.R = (int)md.n;
        geo.HL = geo.HR = 0;
        geo.ntiles = 1;
    } else {
        if (KIND != WC4DVAR_MODEL_LORENZ96) {
            bool done = false;
            switch (md.s) {
                case 1: done = launch_tiled_blk<KIND, 1>(md, net, a, status, st, ws, tile_override); break;
                case 5: done = launch_tiled_blk<KIND, 5>(md, net, a, status, st, ws, tile_override); break;
                case 10: done = launch_tiled_blk<KIND, 10>(md, net, a, status, st, ws, tile_override); break;
                default: break;
            }
            if (done) return;
        }
        geo.resident = false;
        // tile: 4096 points (L96) / 8192 (stencils) when it fits, halo <= T/4
        int T = (int)std::min<int64_t>(smem_cap * 3 / 4, KIND == WC4DVAR_MODEL_LORENZ96 ? 4096 : 8192);
        if (tile_override > 0) T = tile_override;
        const int per = md.s * (rl + rr);
        K = std::max(1, std::min<int>(md.N, (int)((smem_cap - T) / std::max(per, 1))));
        while (K > 1 && per * K > std::max(T / 4, per)) --K;
        geo.T = T;
        geo.HL = K * md.s * rl;
        geo.HR = K * md.s * rr;
        geo.R = T + geo.HL + geo.HR;
        require(geo.R <= smem_cap, "tiled sweep: halo does not fit shared memory");
        require(geo.R <= md.n, "tiled sweep: tile plus halo exceeds the periodic domain");
        geo.ntiles = cdiv(md.n, T);
    }
    const size_t smem = sizeof(double) * ((size_t)nbuf * geo.R + 8);
    auto fk = tiled_fwd_kernel<KIND>;
    auto ak = tiled_adj_kernel<KIND>;
    W4_CUDA(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    W4_CUDA(cudaFuncSetAttribute(ak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nl = geo.resident ? 1 : (int)cdiv(md.N, K);
    double* bbuf = nullptr;
    if (nl > 1) bbuf = ws.get<double>((size_t)2 * md.n * a.m);
    const dim3 grid((unsigned)a.m, (unsigned)geo.ntiles);
    TiledArgs ta{md, net, a, geo, 0, 0, nullptr, nullptr};
    if (a.do_fwd) {
        for (int l = 0; l < nl; ++l) {
            ta.i0 = l * K;
            ta.i1 = std::min(md.N, (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            fk<<<grid, kThreads, smem, st>>>(ta, status);
            W4_LAUNCH();
        }
    }
    if (a.do_adj) {  // mirrored radius: same region size, origin shifted (see kernel)
        for (int l = 0; l < nl; ++l) {
            ta.i1 = md.N - l * K;
            ta.i0 = std::max(0, md.N - (l + 1) * K);
            ta.bin = l == 0 ? nullptr : bbuf + (size_t)((l + 1) % 2) * md.n * a.m;
            ta.bout = l + 1 < nl ? bbuf + (size_t)(l % 2) * md.n * a.m : nullptr;
            ak<<<grid, kThreads, smem, st>>>(ta, status);
            W4_LAUNCH();
        }
    }
}

}  // namespace

void sweep_tiled(const ModelDev& md, const NetDev& net, const SweepArgs& a, unsigned* status,
                 cudaStream_t st, DevBuf& ws, int tov) {
    if (a.m == 0) return;
    switch (md.kind) {
        case WC4DVAR_MODEL_IDENTITY: launch_tiled<WC4DVAR_MODEL_IDENTITY>(md, net, a, status, st, ws, tov); break;
        case WC4DVAR_MODEL_ADVECTION: launch_tiled<WC4DVAR_MODEL_ADVECTION>(md, net, a, status, st, ws, tov); break;
        case WC4DVAR_MODEL_ADVDIFF: launch_tiled<WC4DVAR_MODEL_ADVDIFF>(md, net, a, status, st, ws, tov); break;
        case WC4DVAR_MODEL_LORENZ96: launch_tiled<WC4DVAR_MODEL_LORENZ96>(md, net, a, status, st, ws, tov); break;
        default: throw InvalidArgument("sweep: unknown model kind");
    }
}

}  // namespace w4
