// fp64 DMMA GEMM kernels (see gemm.cuh).
#include "gemm.cuh"

#include <cstdlib>
#include <map>
#include <mutex>

namespace w4 {
namespace {

constexpr int BK = 16;
// [col][k] tiles read with LDS.128 under the permuted k order (see gemm_sym_kernel):
// stride 24 doubles keeps 16-byte fragment loads bank-conflict free.
constexpr int KS = BK + 8;
// Every DMMA kernel feeds the MMA's logical k = t0 with physical k = 2 t0 and logical
// k = t0 + 4 with physical 2 t0 + 1, so all kernels accumulate each output element in the
// same order (block apply == column-wise apply bitwise, whichever tile shape runs).

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma16x8x4(double (&d)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// One k8 step of a warp tile as two m16n8k4 sweeps (physical k = 2 t0, then 2 t0 + 1):
// consecutive MMAs are independent, so no DMMA waits on the one just issued, and every
// element accumulates in the same order as the m16n8k8 form.
template <int MI, int NI>
__device__ __forceinline__ void mma_k8(double (&acc)[MI][NI][4], const double (&af)[MI][4],
                                       const double (&bf)[NI][2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma16x8x4(acc[i][j], af[i][2 * h], af[i][2 * h + 1], bf[j][h]);
}

template <int VEC>
__device__ __forceinline__ void cp_async_vec(void* smem, const double* gmem, int valid,
                                             const double* safe) {
    const double* src = valid > 0 ? gmem : safe;
    if (VEC == 2)
        cp_async16(smem, src, valid * 8);
    else
        cp_async8(smem, src, valid * 8);
}

// cudaFuncSetAttribute is per device: remember which devices are configured.
void configure_smem(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, bool> done;
    int dev = 0;
    W4_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(kern, dev);
    if (done.count(key)) return;
    W4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done[key] = true;
}

// The stream-K scratch comes from the device's default stream-ordered pool; keep what the
// pool has reserved across synchronisations (default threshold 0 returns it to the driver
// at every sync, turning each call's cudaMallocAsync into a fresh mapping).
void keep_pool_reserved() {
    static std::mutex mu;
    static std::map<int, bool> done;
    int dev = 0;
    W4_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(dev)) return;
    cudaMemPool_t pool;
    W4_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = 64ull << 20;  // the scratch is ~19 MB per concurrent GEMM
    W4_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    done[dev] = true;
}

struct PassTable {
    GemmPass p[2];
    int64_t tiles_m[2];
    int64_t tile_start[3];
};

// ---------------------------------------------------------------------------
// NN kernel: A tile stored [k][m] (stride BM+4), B tile stored [n][k] (stride BK+4).
// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES, int VEC>
__global__ void __launch_bounds__(WM * WN * 32)
    gemm_nn_kernel(const PassTable tab, unsigned* __restrict__ status) {
    constexpr int NT = WM * WN * 32;
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MI = WTM / 16, NI = WTN / 8;
    constexpr int APAD = BM + 2;  // rows 2t0 apart by 2*APAD == 4 (mod 16): conflict-free
    constexpr int A_ELEMS = BK * APAD, B_ELEMS = BN * KS;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_ELEMS;

    int64_t tile = blockIdx.x;
    const int pi = tile >= tab.tile_start[1] ? 1 : 0;
    const GemmPass& P = tab.p[pi];
    tile -= tab.tile_start[pi];
    const int64_t tm = tile % tab.tiles_m[pi];
    const int64_t tn = tile / tab.tiles_m[pi];
    const int64_t m0 = tm * BM, n0 = tn * BN;
    const int64_t M = P.M, K = P.K, ncols = P.ncols;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t0 = lane & 3;

    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    const int64_t kend = P.upper_tri ? (n0 + BN < K ? n0 + BN : K) : K;
    const int64_t ktiles = (kend + BK - 1) / BK;

    auto load_stage = [&](int stage, int64_t kt) {
        const int64_t k0 = kt * BK;
        double* as = As + stage * A_ELEMS;
        double* bs = Bs + stage * B_ELEMS;
        constexpr int ACH = BK * BM / VEC;
#pragma unroll
        for (int ch = tid; ch < ACH; ch += NT) {
            const int kk = ch / (BM / VEC);
            const int rr = (ch % (BM / VEC)) * VEC;
            const int64_t row = m0 + rr, kcol = k0 + kk;
            int valid = 0;
            if (kcol < K) {
                const int64_t rem = M - row;
                valid = rem >= VEC ? VEC : (rem > 0 ? (int)rem : 0);
            }
            cp_async_vec<VEC>(as + kk * APAD + rr, P.A + kcol * P.lda + row, valid, P.A);
        }
        constexpr int BCH = BN * BK / VEC;
#pragma unroll
        for (int ch = tid; ch < BCH; ch += NT) {
            const int nn = ch / (BK / VEC);
            const int kk = (ch % (BK / VEC)) * VEC;
            const int64_t c = n0 + nn, kr = k0 + kk;
            int valid = 0;
            const double* src = P.A;
            if (c < ncols) {
                const int64_t rem = K - kr;
                valid = rem >= VEC ? VEC : (rem > 0 ? (int)rem : 0);
                src = P.in.col(c) + kr;
            }
            cp_async_vec<VEC>(bs + nn * KS + kk, src, valid, P.A);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_commit();
    }

    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage((int)(nk % STAGES), nk);
            cp_commit();
        }
        const double* as = As + (kt % STAGES) * A_ELEMS;
        const double* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
        for (int k8 = 0; k8 < BK; k8 += 8) {
            double af[MI][4], bf[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int r = wm * WTM + i * 16 + g;
                af[i][0] = as[(k8 + 2 * t0) * APAD + r];
                af[i][1] = as[(k8 + 2 * t0) * APAD + r + 8];
                af[i][2] = as[(k8 + 2 * t0 + 1) * APAD + r];
                af[i][3] = as[(k8 + 2 * t0 + 1) * APAD + r + 8];
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int c = wn * WTN + j * 8 + g;
                const double2 bb = *reinterpret_cast<const double2*>(bs + c * KS + k8 + 2 * t0);
                bf[j][0] = bb.x;
                bf[j][1] = bb.y;
            }
            mma_k8(acc, af, bf);
        }
    }
    cp_wait<0>();

    bool bad = false;
    const double alpha = P.alpha;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = n0 + wn * WTN + j * 8 + 2 * t0 + h;
            if (c >= ncols) continue;
            double* outc = const_cast<double*>(P.out.col(c));
            const double* addc = P.add.base ? P.add.col(c) : nullptr;
#pragma unroll
            for (int i = 0; i < MI; ++i) {
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int64_t r = m0 + wm * WTM + i * 16 + g + 8 * v;
                    if (r >= M) continue;
                    double val = alpha * acc[i][j][2 * v + h];
                    if (addc) val = addc[r] + val;
                    bad |= !isfinite(val);
                    outc[r] = val;
                }
            }
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_OUT_NONFINITE);
}

template <int BM, int BN, int WM, int WN, int STAGES, int VEC>
void launch_nn(const PassTable& tab, int64_t ntiles, unsigned* status, cudaStream_t stream) {
    constexpr int APAD = BM + 2;
    const size_t smem = sizeof(double) * STAGES * (BK * APAD + BN * KS);
    auto kern = gemm_nn_kernel<BM, BN, WM, WN, STAGES, VEC>;
    configure_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<(unsigned)ntiles, WM * WN * 32, smem, stream>>>(tab, status);
    W4_LAUNCH();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------------------
// Symmetric-A kernel (the D^{1/2} factors): because A = A^T, the A tile can be loaded as
// [m][k] rows straight from A's columns, so BOTH operands sit k-contiguous in SMEM.  The
// MMA's logical k index is permuted (logical t0 <-> physical 2 t0, logical t0+4 <->
// physical 2 t0 + 1) so each thread's (a0,a2), (a1,a3) and (b0,b1) fragment pairs are
// adjacent doubles: one LDS.128 each.  Row stride 24 doubles keeps the 16-byte loads
// bank-conflict free.  Warp tile 64 x 32 (16 MMAs per k8 per warp).
// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(WM * WN * 32, 1)
    gemm_sym_kernel(const PassTable tab, unsigned* __restrict__ status) {
    constexpr int NT = WM * WN * 32;
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MI = WTM / 16, NI = WTN / 8;
    constexpr int A_ELEMS = BM * KS, B_ELEMS = BN * KS;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_ELEMS;

    int64_t tile = blockIdx.x;
    const int pi = tile >= tab.tile_start[1] ? 1 : 0;
    const GemmPass& P = tab.p[pi];
    tile -= tab.tile_start[pi];
    const int64_t tm = tile % tab.tiles_m[pi];
    const int64_t tn = tile / tab.tiles_m[pi];
    const int64_t m0 = tm * BM, n0 = tn * BN;
    const int64_t M = P.M, K = P.K, ncols = P.ncols;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t0 = lane & 3;

    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    const int64_t ktiles = (K + BK - 1) / BK;
    auto load_stage = [&](int stage, int64_t kt) {
        const int64_t k0 = kt * BK;
        double* as = As + stage * A_ELEMS;
        double* bs = Bs + stage * B_ELEMS;
        constexpr int ACH = BM * BK / 2;
#pragma unroll
        for (int ch = tid; ch < ACH; ch += NT) {
            const int mm = ch / (BK / 2);
            const int kk = (ch % (BK / 2)) * 2;
            const int64_t row = m0 + mm, kr = k0 + kk;
            int valid = 0;
            const double* src = P.A;
            if (row < M) {
                const int64_t rem = K - kr;
                valid = rem >= 2 ? 2 : (rem > 0 ? (int)rem : 0);
                src = P.A + row * P.lda + kr;  // column `row` of A == row `row` (symmetric)
            }
            cp_async_vec<2>(as + mm * KS + kk, src, valid, P.A);
        }
        constexpr int BCH = BN * BK / 2;
#pragma unroll
        for (int ch = tid; ch < BCH; ch += NT) {
            const int nn = ch / (BK / 2);
            const int kk = (ch % (BK / 2)) * 2;
            const int64_t c = n0 + nn, kr = k0 + kk;
            int valid = 0;
            const double* src = P.A;
            if (c < ncols) {
                const int64_t rem = K - kr;
                valid = rem >= 2 ? 2 : (rem > 0 ? (int)rem : 0);
                src = P.in.col(c) + kr;
            }
            cp_async_vec<2>(bs + nn * KS + kk, src, valid, P.A);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_commit();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage((int)(nk % STAGES), nk);
            cp_commit();
        }
        const double* as = As + (kt % STAGES) * A_ELEMS;
        const double* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
        for (int k8 = 0; k8 < BK; k8 += 8) {
            double af[MI][4], bf[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int r = wm * WTM + i * 16 + g;
                const double2 lo = *reinterpret_cast<const double2*>(as + r * KS + k8 + 2 * t0);
                const double2 hi = *reinterpret_cast<const double2*>(as + (r + 8) * KS + k8 + 2 * t0);
                af[i][0] = lo.x;
                af[i][2] = lo.y;
                af[i][1] = hi.x;
                af[i][3] = hi.y;
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int c = wn * WTN + j * 8 + g;
                const double2 bb = *reinterpret_cast<const double2*>(bs + c * KS + k8 + 2 * t0);
                bf[j][0] = bb.x;
                bf[j][1] = bb.y;
            }
            mma_k8(acc, af, bf);
        }
    }
    cp_wait<0>();

    bool bad = false;
    const double alpha = P.alpha;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = n0 + wn * WTN + j * 8 + 2 * t0 + h;
            if (c >= ncols) continue;
            double* outc = const_cast<double*>(P.out.col(c));
            const double* addc = P.add.base ? P.add.col(c) : nullptr;
#pragma unroll
            for (int i = 0; i < MI; ++i) {
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int64_t r = m0 + wm * WTM + i * 16 + g + 8 * v;
                    if (r >= M) continue;
                    double val = alpha * acc[i][j][2 * v + h];
                    if (addc) val = addc[r] + val;
                    bad |= !isfinite(val);
                    outc[r] = val;
                }
            }
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_OUT_NONFINITE);
}

template <int BM, int BN, int WM, int WN, int STAGES>
void launch_sym(const PassTable& tab, int64_t ntiles, unsigned* status, cudaStream_t stream) {
    const size_t smem = sizeof(double) * STAGES * (BM * KS + BN * KS);
    auto kern = gemm_sym_kernel<BM, BN, WM, WN, STAGES>;
    configure_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<(unsigned)ntiles, WM * WN * 32, smem, stream>>>(tab, status);
    W4_LAUNCH();
}

// ---------------------------------------------------------------------------
// Warp-specialised symmetric-A kernel: one producer warp streams the A / B tiles with
// cp.async into a STAGES-deep ring and signals per-stage "full" mbarriers
// (cp.async.mbarrier.arrive.noinc); 16 consumer warps wait on "full", run the DMMA k-steps
// and release the stage through "empty" mbarriers.  No block-wide barrier in the main
// loop, so the tensor pipe is not drained every k-tile.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

// Stream-K schedule that keeps every output element's accumulation order identical to the
// one-CTA-per-tile kernel (so block apply == column apply stays bitwise): the T tiles x KT
// k-tiles are cut into G equal contiguous ranges, one per CTA.  With T >= G every range
// spans >= KT k-tiles, so each tile is split in at most two pieces: a "start" piece
// (k-tiles [0, c)) at the end of range b and an "end" piece ([c, KT)) at the beginning of
// range b+1.  CTA b runs its start piece FIRST and publishes the raw DMMA accumulators,
// then its full tiles, then its end piece, which resumes from CTA b-1's published
// accumulators -- by then CTA b-1 has long finished its own first piece (no waits when
// the range is >= KT).  With G = T this is the plain one-tile-per-CTA grid.
struct SkSched {
    int64_t s, e, KT, full0, full1;
    bool has_start, has_end;
    __device__ SkSched(int64_t b, int64_t G, int64_t T, int64_t kt) : KT(kt) {
        const int64_t I = T * KT;
        s = b * I / G;
        e = (b + 1) * I / G;
        has_start = (e % KT) != 0;
        has_end = (s % KT) != 0;
        full0 = (s + KT - 1) / KT;
        full1 = e / KT;
    }
    __device__ int64_t count() const { return (int64_t)has_start + (full1 - full0) + (int64_t)has_end; }
    // kind: 0 full tile, 1 start piece (publish), 2 end piece (resume)
    __device__ void get(int64_t i, int64_t& tile, int64_t& kb, int64_t& ke, int& kind) const {
        if (has_start) {
            if (i == 0) {
                tile = e / KT;
                kb = 0;
                ke = e - tile * KT;
                kind = 1;
                return;
            }
            --i;
        }
        if (i < full1 - full0) {
            tile = full0 + i;
            kb = 0;
            ke = KT;
            kind = 0;
            return;
        }
        tile = s / KT;
        kb = s - tile * KT;
        ke = KT;
        kind = 2;
    }
};

struct TileXY {
    int pi;
    int64_t m0, n0;
};
template <int BM, int BN>
__device__ __forceinline__ TileXY tile_xy(const PassTable& tab, int64_t tile) {
    const int pi = tile >= tab.tile_start[1] ? 1 : 0;
    tile -= tab.tile_start[pi];
    return TileXY{pi, (tile % tab.tiles_m[pi]) * BM, (tile / tab.tiles_m[pi]) * BN};
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

constexpr int kSkMaxPieces = 64;  // pieces per CTA (host falls back to one tile per CTA beyond)

struct SkArgs {
    int64_t KT;        // k-tiles per tile (all passes share K)
    double* partial;   // [G][32 * NC] published accumulators (null: plain grid)
    int* flags;        // [G], zeroed before the launch
};

// SMEM row stride RS: KS (= BK + 8, padded, conflict-free by padding) or BK (unpadded, the
// 16-byte chunk index XOR-swizzled with bit 2 by the row parity: the two rows a quarter-warp
// reads with LDS.128 then land in disjoint bank groups, and the producer's lane-rotated
// chunk order stays conflict-free).  Unpadded stages are 2/3 the size, so 6 fit in SMEM.
template <int RS>
__device__ __forceinline__ int swz(int row, int chunk) {
    return RS == BK ? (chunk ^ ((row & 1) << 2)) : chunk;
}

template <int BM, int BN, int WM, int WN, int STAGES, int RS, int NPW>
__global__ void __launch_bounds__(WM * WN * 32 + 32 * NPW, 1)
    gemm_sym_ws_kernel(const PassTable tab, unsigned* __restrict__ status, const SkArgs sk) {
    constexpr int NC = WM * WN * 32;  // consumer threads
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MI = WTM / 16, NI = WTN / 8;
    constexpr int A_ELEMS = BM * RS, B_ELEMS = BN * RS;
    static_assert(BM % 32 == 0 && BN % 32 == 0, "tile");
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_ELEMS;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * B_ELEMS);
    uint64_t* empty = full + STAGES;

    // pass table and this CTA's piece list in SMEM (dynamic indexing without local copies)
    __shared__ PassTable s_tab;
    __shared__ int4 s_piece[kSkMaxPieces];  // {tile, kb, ke, kind}
    __shared__ int s_np;

    const int tid = threadIdx.x;
    if (tid == 0) {
        s_tab = tab;
        const SkSched sched(blockIdx.x, gridDim.x, tab.tile_start[2], sk.KT);
        const int np = (int)sched.count();
        for (int i = 0; i < np; ++i) {
            int64_t tl, kb, ke;
            int kind;
            sched.get(i, tl, kb, ke, kind);
            s_piece[i] = make_int4((int)tl, (int)kb, (int)ke, kind);
        }
        s_np = np;
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 32 * NPW);
            mbar_init(&empty[s], WM * WN);
        }
    }
    __syncthreads();

    if (warp >= WM * WN) {
        // ===== producer warp(s) =====  (NPW = 2: warp 0 streams A, warp 1 streams B)
        const int pw = warp - WM * WN;
        const bool doA = NPW == 1 || pw == 0, doB = NPW == 1 || pw == 1;
        // Lane l owns A rows l + 32u and B columns l + 32u (pointers computed once per
        // tile).  It copies the 8 16-byte chunks of each row in the lane-rotated order
        // (ch + l) & 7: with the 192-byte row stride the 8 lanes of a quarter-warp then hit
        // 8 distinct 4-bank groups, so the SMEM writes are conflict-free.
        constexpr int AU = BM / 32, BU = BN / 32;
        unsigned it = 0;  // ring position, continuous across pieces
        const int npieces = s_np;
        for (int pc = 0; pc < npieces; ++pc) {
            const int4 pe = s_piece[pc];
            const int64_t tile = pe.x, kb = pe.y, ke = pe.z;
            const TileXY xy = tile_xy<BM, BN>(s_tab, tile);
            const GemmPass& P = s_tab.p[xy.pi];
            const int64_t K = P.K;
            const double* const safe = P.A;  // register copy: cp.async asm would force reloads
            const double* arow[AU];
            bool aok[AU];
            const double* bcol[BU];
            bool bok[BU];
#pragma unroll
            for (int u = 0; u < AU; ++u) {
                const int64_t row = xy.m0 + lane + 32 * u;
                aok[u] = row < P.M;
                arow[u] = P.A + (aok[u] ? row : 0) * P.lda;  // column `row` of A == row (symmetric)
            }
#pragma unroll
            for (int u = 0; u < BU; ++u) {
                const int64_t c = xy.n0 + lane + 32 * u;
                bok[u] = c < P.ncols;
                bcol[u] = bok[u] ? P.in.col(c) : P.A;
            }
            for (int kt = (int)kb; kt < (int)ke; ++kt, ++it) {
                const int s = (int)(it % STAGES);
                const unsigned ph = (it / STAGES) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                const int64_t k0 = kt * BK;
                double* as = As + s * A_ELEMS + lane * RS;
                double* bs = Bs + s * B_ELEMS + lane * RS;
                if (k0 + BK <= K) {
                    // interior k-tile: no tail predicates (out-of-range rows / columns point at
                    // valid memory and zero-fill through the src-size operand)
#pragma unroll
                    for (int cc = 0; cc < BK / 2; ++cc) {
                        const int ch = (cc + lane) & 7;
                        const int sc = 2 * swz<RS>(lane, ch);
                        if (doA)
#pragma unroll
                            for (int u = 0; u < AU; ++u)
                                cp_async16(as + u * 32 * RS + sc, arow[u] + k0 + 2 * ch, aok[u] ? 16 : 0);
                        if (doB)
#pragma unroll
                            for (int u = 0; u < BU; ++u)
                                cp_async16(bs + u * 32 * RS + sc, bcol[u] + k0 + 2 * ch, bok[u] ? 16 : 0);
                    }
                    mbar_arrive_cp_async(&full[s]);
                    continue;
                }
#pragma unroll
                for (int cc = 0; cc < BK / 2; ++cc) {
                    const int ch = (cc + lane) & 7;
                    const int sc = 2 * swz<RS>(lane, ch);  // rows lane + 32 u share the parity
                    const int64_t kr = k0 + 2 * ch;
                    const int64_t rem = K - kr;
                    const int kval = rem >= 2 ? 2 : (rem > 0 ? (int)rem : 0);
                    if (doA)
#pragma unroll
                        for (int u = 0; u < AU; ++u)
                            cp_async_vec<2>(as + u * 32 * RS + sc, arow[u] + kr, aok[u] ? kval : 0, safe);
                    if (doB)
#pragma unroll
                        for (int u = 0; u < BU; ++u)
                            cp_async_vec<2>(bs + u * 32 * RS + sc, bcol[u] + kr, bok[u] ? kval : 0, safe);
                }
                mbar_arrive_cp_async(&full[s]);
            }
        }
        cp_wait<0>();
        return;
    }

    // ===== consumer warps =====
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t0 = lane & 3;
    bool bad = false;
    unsigned it = 0;
    const int npieces = s_np;
    for (int pc = 0; pc < npieces; ++pc) {
    const int4 pe = s_piece[pc];
    const int kb = pe.y, ke = pe.z, kind = pe.w;
    double acc[MI][NI][4];
    if (kind == 2) {  // resume CTA b-1's accumulators (published by its first piece)
        if (tid == 0)
            while (ld_acquire(sk.flags + blockIdx.x - 1) == 0) __nanosleep(64);
        asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
        const double* src = sk.partial + (size_t)(blockIdx.x - 1) * (MI * NI * 4) * NC + tid;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][j][v] = __ldcg(src + ((i * NI + j) * 4 + v) * NC);
    } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
    }

    for (int kt = (int)kb; kt < (int)ke; ++kt, ++it) {
        const int s = (int)(it % STAGES);
        const unsigned ph = (it / STAGES) & 1u;
        mbar_wait(&full[s], ph);
        const double* as = As + s * A_ELEMS;
        const double* bs = Bs + s * B_ELEMS;
#pragma unroll
        for (int k8 = 0; k8 < BK; k8 += 8) {
            double af[MI][4], bf[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int r = wm * WTM + i * 16 + g;
                const int sc = 2 * swz<RS>(r, k8 / 2 + t0);  // rows r and r + 8 share the parity
                const double2 lo = *reinterpret_cast<const double2*>(as + r * RS + sc);
                const double2 hi = *reinterpret_cast<const double2*>(as + (r + 8) * RS + sc);
                af[i][0] = lo.x;
                af[i][2] = lo.y;
                af[i][1] = hi.x;
                af[i][3] = hi.y;
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int c = wn * WTN + j * 8 + g;
                const double2 bb = *reinterpret_cast<const double2*>(bs + c * RS + 2 * swz<RS>(c, k8 / 2 + t0));
                bf[j][0] = bb.x;
                bf[j][1] = bb.y;
            }
            mma_k8(acc, af, bf);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    if (kind == 1) {  // publish the raw accumulators of this tile's first k-tiles
        double* dst = sk.partial + (size_t)blockIdx.x * (MI * NI * 4) * NC + tid;
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) __stcg(dst + ((i * NI + j) * 4 + v) * NC, acc[i][j][v]);
        __threadfence();
        asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
        if (tid == 0) st_release(sk.flags + blockIdx.x, 1);
        continue;
    }
    const TileXY xy = tile_xy<BM, BN>(s_tab, s_piece[pc].x);
    // stores go through st.global (__stcg): a generic-pointer store could alias SMEM and
    // would force a reload of the s_tab fields after each one
    const ColMap& omap = s_tab.p[xy.pi].out;
    const ColMap& amap = s_tab.p[xy.pi].add;
    const int64_t Mrows = s_tab.p[xy.pi].M, ncols = s_tab.p[xy.pi].ncols;
    const double alpha = s_tab.p[xy.pi].alpha;
    if (!amap.base) {  // plain D^{1/2} v
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t c = xy.n0 + wn * WTN + j * 8 + 2 * t0 + h;
                if (c >= ncols) continue;
                double* oc = const_cast<double*>(omap.col(c));
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int64_t r = xy.m0 + wm * WTM + i * 16 + g + 8 * v;
                        if (r >= Mrows) continue;
                        const double val = alpha * acc[i][j][2 * v + h];
                        bad |= !isfinite(val);
                        __stcg(oc + r, val);
                    }
            }
        continue;
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) {
        // the add term (v of out = v + D^{1/2}s) through the read-only path, all of this
        // column block's loads issued before its stores (else each load waits on HBM in turn)
        const double* addc[2];
        double* outc[2];
        double addv[2][MI][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = xy.n0 + wn * WTN + j * 8 + 2 * t0 + h;
            const bool ok = c < ncols;
            outc[h] = ok ? const_cast<double*>(omap.col(c)) : nullptr;
            addc[h] = (ok && amap.base) ? amap.col(c) : nullptr;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int64_t r = xy.m0 + wm * WTM + i * 16 + g + 8 * v;
                    addv[h][i][v] = (addc[h] && r < Mrows) ? __ldg(addc[h] + r) : 0.0;
                }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!outc[h]) continue;
#pragma unroll
            for (int i = 0; i < MI; ++i) {
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int64_t r = xy.m0 + wm * WTM + i * 16 + g + 8 * v;
                    if (r >= Mrows) continue;
                    double val = alpha * acc[i][j][2 * v + h];
                    if (addc[h]) val = addv[h][i][v] + val;
                    bad |= !isfinite(val);
                    __stcg(outc[h] + r, val);
                }
            }
        }
    }
    }  // pieces
    if (status && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_OUT_NONFINITE);
}

// Grid: one CTA per SM in stream-K mode when the tile count is not a multiple of the SM
// count (WC4DVAR_GEMM_SK=0 forces one CTA per tile).  Partials / flags come from the
// stream-ordered pool, so concurrent GEMMs on different streams never share them.
template <int BM, int BN, int WM, int WN, int STAGES, int RS = KS, int NPW = 1>
void launch_sym_ws(const PassTable& tab, int64_t ntiles, unsigned* status, cudaStream_t stream) {
    constexpr int NC = WM * WN * 32;
    const size_t smem = sizeof(double) * STAGES * (BM * RS + BN * RS) + 2 * STAGES * sizeof(uint64_t);
    auto kern = gemm_sym_ws_kernel<BM, BN, WM, WN, STAGES, RS, NPW>;
    configure_smem(reinterpret_cast<const void*>(kern), smem);
    static const int sk_mode = [] {
        const char* e = std::getenv("WC4DVAR_GEMM_SK");
        return e ? std::atoi(e) : 1;
    }();
    const int first = tab.tile_start[1] > 0 ? 0 : 1;
    SkArgs sk{cdiv(tab.p[first].K, BK), nullptr, nullptr};
    bool same_k = true;
    for (int i = 0; i < 2; ++i)
        if (tab.tile_start[i + 1] > tab.tile_start[i]) same_k = same_k && tab.p[i].K == tab.p[first].K;
    int64_t grid = ntiles;
    if (sk_mode && same_k && ntiles > kSMs && ntiles % kSMs != 0 && ntiles / kSMs + 3 <= kSkMaxPieces &&
        ntiles < (int64_t)1 << 31 && sk.KT < (int64_t)1 << 31)
        grid = kSMs;
    if (grid != ntiles) {
        keep_pool_reserved();
        const size_t pbytes = sizeof(double) * (size_t)grid * NC * (BM * BN / NC);
        char* buf = nullptr;
        W4_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), pbytes + sizeof(int) * grid, stream));
        sk.partial = reinterpret_cast<double*>(buf);
        sk.flags = reinterpret_cast<int*>(buf + pbytes);
        W4_CUDA(cudaMemsetAsync(sk.flags, 0, sizeof(int) * grid, stream));
        kern<<<(unsigned)grid, NC + 32 * NPW, smem, stream>>>(tab, status, sk);
        W4_LAUNCH();
        W4_CUDA(cudaFreeAsync(buf, stream));
        return;
    }
    kern<<<(unsigned)grid, NC + 32 * NPW, smem, stream>>>(tab, status, sk);
    W4_LAUNCH();
}

// ---------------------------------------------------------------------------
// Few-column symmetric GEMM: one warp per 16 x 8 output tile ("unit"), fragments loaded
// straight from global/L2 into a D-deep register ring (no SMEM, no barriers).  With the
// bitwise-order constraint every output element is one sequential chain over K, so the
// only parallelism is across tiles; one warp per tile maximises it (PCG: n/16 x (N+1)/8
// warps) and the prefetch ring keeps each chain fed.  Same fragment k-permutation and the
// same two-phase m16n8k4 order as mma_k8.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) gemm_chain_kernel(const PassTable tab, unsigned* __restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int64_t unit = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (unit >= tab.tile_start[2]) return;
    const int pi = unit >= tab.tile_start[1] ? 1 : 0;
    const GemmPass& P = tab.p[pi];
    const int64_t u = unit - tab.tile_start[pi];
    const int64_t m0 = (u % tab.tiles_m[pi]) * 16, n0 = (u / tab.tiles_m[pi]) * 8;
    const int64_t M = P.M, K = P.K, ncols = P.ncols;
    const int g = lane >> 2, t0 = lane & 3;
    const int64_t r_lo = m0 + g, r_hi = m0 + g + 8, cb = n0 + g;
    const bool ok_lo = r_lo < M, ok_hi = r_hi < M, ok_b = cb < ncols;
    // symmetric A: row r of A is column r (contiguous in k)
    const double* a_lo = P.A + (ok_lo ? r_lo : 0) * P.lda + 2 * t0;
    const double* a_hi = P.A + (ok_hi ? r_hi : 0) * P.lda + 2 * t0;
    const double* bp = (ok_b ? P.in.col(cb) : P.A) + 2 * t0;
    const int KB = (int)(K / 8);  // full k8 blocks; a K tail is handled after the loop
    // main loop: unconditional loads from clamped rows / columns, invalid lanes zeroed by
    // a select (branch-free, so the ring of D loads really is in flight)
    // running pointers advanced once per D-chunk; ring loads use constant offsets
    const double2* pl = reinterpret_cast<const double2*>(a_lo);
    const double2* ph = reinterpret_cast<const double2*>(a_hi);
    const double2* pb = reinterpret_cast<const double2*>(bp);
    auto load = [&](int kb, double2& al, double2& ah, double2& b) {  // kb relative to the pointers
        al = __ldg(pl + 4 * kb);
        ah = __ldg(ph + 4 * kb);
        b = __ldg(pb + 4 * kb);
    };
    auto fix = [&](double2& al, double2& ah, double2& b) {
        if (!ok_lo) al = make_double2(0.0, 0.0);
        if (!ok_hi) ah = make_double2(0.0, 0.0);
        if (!ok_b) b = make_double2(0.0, 0.0);
    };
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double2 ra[D], rh[D], rb[D];
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < KB) load(d, ra[d], rh[d], rb[d]);
    int kb = 0;
    for (; kb + D <= KB; kb += D) {
        const bool more = kb + 2 * D <= KB;  // whole next chunk in range: unpredicated loads
#pragma unroll
        for (int d = 0; d < D; ++d) {
            double2 al = ra[d], ah = rh[d], b = rb[d];
            if (more || kb + d + D < KB) load(d + D, ra[d], rh[d], rb[d]);
            fix(al, ah, b);
            dmma16x8x4(acc, al.x, ah.x, b.x);  // physical k = 2 t0
            dmma16x8x4(acc, al.y, ah.y, b.y);  // physical k = 2 t0 + 1
        }
        pl += 4 * D;
        ph += 4 * D;
        pb += 4 * D;
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {  // remaining (< D) full blocks, already loaded
        if (kb + d < KB) {
            double2 al = ra[d], ah = rh[d], b = rb[d];
            fix(al, ah, b);
            dmma16x8x4(acc, al.x, ah.x, b.x);
            dmma16x8x4(acc, al.y, ah.y, b.y);
        }
    }
    if ((int64_t)KB * 8 < K) {  // K tail: zero-fill like the cp.async kernels
        const int64_t k = (int64_t)KB * 8;
        const bool v0 = k + 2 * t0 < K, v1 = k + 2 * t0 + 1 < K;
        const double2 al = make_double2(ok_lo && v0 ? a_lo[k] : 0.0, ok_lo && v1 ? a_lo[k + 1] : 0.0);
        const double2 ah = make_double2(ok_hi && v0 ? a_hi[k] : 0.0, ok_hi && v1 ? a_hi[k + 1] : 0.0);
        const double2 b = make_double2(ok_b && v0 ? bp[k] : 0.0, ok_b && v1 ? bp[k + 1] : 0.0);
        dmma16x8x4(acc, al.x, ah.x, b.x);
        dmma16x8x4(acc, al.y, ah.y, b.y);
    }
    bool bad = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + 2 * t0 + h;
        if (c >= ncols) continue;
        double* outc = const_cast<double*>(P.out.col(c));
        const double* addc = P.add.base ? P.add.col(c) : nullptr;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int64_t r = m0 + g + 8 * v;
            if (r >= M) continue;
            double val = P.alpha * acc[2 * v + h];
            if (addc) val = addc[r] + val;
            bad |= !isfinite(val);
            outc[r] = val;
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_OUT_NONFINITE);
}

// ---------------------------------------------------------------------------
// TN split kernel: both tiles stored [col][k] (stride KPAD).
// Partial (split s) of C tile -> work[s][m2][m1] col-major m1 x m2.
// ---------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int STAGES, int VEC>
__global__ void __launch_bounds__(WM * WN * 32)
    gemm_tn_kernel(int64_t R, int64_t m1, int64_t m2, const double* __restrict__ A, int64_t lda,
                   const double* __restrict__ B, int64_t ldb, int64_t rows_per_split,
                   int64_t tiles_m, int64_t tiles_n, double* __restrict__ work, bool sym) {
    constexpr int NT = WM * WN * 32;
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MI = WTM / 16, NI = WTN / 8;
    constexpr int A_ELEMS = BM * KS, B_ELEMS = BN * KS;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * A_ELEMS;

    // tile t of a split: plain (tm, tn) grid, or with sym the upper-triangle tiles
    // (tm <= tn) of a square grid enumerated column by column
    const int64_t t = blockIdx.x;
    int64_t tm, tn, split;
    if (sym) {
        const int64_t ntri = tiles_m * (tiles_m + 1) / 2;
        split = t / ntri;
        int64_t u = t - split * ntri;
        tn = 0;
        while (u > tn) {
            u -= tn + 1;
            ++tn;
        }
        tm = u;
    } else {
        tm = t % tiles_m;
        tn = (t / tiles_m) % tiles_n;
        split = t / (tiles_m * tiles_n);
    }
    const int64_t i0 = tm * BM, j0 = tn * BN;
    const int64_t r_begin = split * rows_per_split;
    const int64_t r_end = min(R, r_begin + rows_per_split);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t0 = lane & 3;

    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    const int64_t ktiles = r_end > r_begin ? (r_end - r_begin + BK - 1) / BK : 0;

    auto load_stage = [&](int stage, int64_t kt) {
        const int64_t k0 = r_begin + kt * BK;
        double* as = As + stage * A_ELEMS;
        double* bs = Bs + stage * B_ELEMS;
        constexpr int ACH = BM * BK / VEC;
#pragma unroll
        for (int ch = tid; ch < ACH; ch += NT) {
            const int ii = ch / (BK / VEC);
            const int kk = (ch % (BK / VEC)) * VEC;
            const int64_t c = i0 + ii, kr = k0 + kk;
            int valid = 0;
            const double* src = A;
            if (c < m1) {
                const int64_t rem = r_end - kr;
                valid = rem >= VEC ? VEC : (rem > 0 ? (int)rem : 0);
                src = A + c * lda + kr;
            }
            cp_async_vec<VEC>(as + ii * KS + kk, src, valid, A);
        }
        constexpr int BCH = BN * BK / VEC;
#pragma unroll
        for (int ch = tid; ch < BCH; ch += NT) {
            const int jj = ch / (BK / VEC);
            const int kk = (ch % (BK / VEC)) * VEC;
            const int64_t c = j0 + jj, kr = k0 + kk;
            int valid = 0;
            const double* src = B;
            if (c < m2) {
                const int64_t rem = r_end - kr;
                valid = rem >= VEC ? VEC : (rem > 0 ? (int)rem : 0);
                src = B + c * ldb + kr;
            }
            cp_async_vec<VEC>(bs + jj * KS + kk, src, valid, B);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_commit();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage((int)(nk % STAGES), nk);
            cp_commit();
        }
        const double* as = As + (kt % STAGES) * A_ELEMS;
        const double* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
        for (int k8 = 0; k8 < BK; k8 += 8) {
            double af[MI][4], bf[NI][2];
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                const int r = wm * WTM + i * 16 + g;
                const double2 lo = *reinterpret_cast<const double2*>(as + r * KS + k8 + 2 * t0);
                const double2 hi = *reinterpret_cast<const double2*>(as + (r + 8) * KS + k8 + 2 * t0);
                af[i][0] = lo.x;
                af[i][2] = lo.y;
                af[i][1] = hi.x;
                af[i][3] = hi.y;
            }
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const int c = wn * WTN + j * 8 + g;
                const double2 bb = *reinterpret_cast<const double2*>(bs + c * KS + k8 + 2 * t0);
                bf[j][0] = bb.x;
                bf[j][1] = bb.y;
            }
            mma_k8(acc, af, bf);
        }
    }
    cp_wait<0>();

    double* P = work + split * m1 * m2;
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t c = j0 + wn * WTN + j * 8 + 2 * t0 + h;
            if (c >= m2) continue;
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int64_t r = i0 + wm * WTM + i * 16 + g + 8 * v;
                    if (r < m1) P[c * m1 + r] = acc[i][j][2 * v + h];
                }
        }
}

__global__ void reduce_splits_kernel(int64_t m1, int64_t m2, int64_t nsplit,
                                     const double* __restrict__ work, double alpha,
                                     double* __restrict__ C, int64_t ldc, int sym_bm) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m1 * m2) return;
    const int64_t r0 = e % m1, c0 = e / m1;
    const int64_t out = r0 + c0 * ldc;
    // Gram: the partials of a tile below the diagonal were never computed; read the mirror
    if (sym_bm && r0 / sym_bm > c0 / sym_bm) e = c0 + r0 * m1;
    double s = 0.0;
    for (int64_t k = 0; k < nsplit; ++k) s += work[k * m1 * m2 + e];  // fixed order
    C[out] = alpha * s;
}

template <int BM, int BN, int WM, int WN, int STAGES, int VEC>
void launch_tn(int64_t R, int64_t m1, int64_t m2, const double* A, int64_t lda, const double* B,
               int64_t ldb, double* work, int64_t rows_per_split, int64_t nsplit,
               cudaStream_t stream, bool sym = false) {
    const size_t smem = sizeof(double) * STAGES * (BM * KS + BN * KS);
    auto kern = gemm_tn_kernel<BM, BN, WM, WN, STAGES, VEC>;
    configure_smem(reinterpret_cast<const void*>(kern), smem);
    const int64_t tm = cdiv(m1, BM), tn = cdiv(m2, BN);
    const int64_t tiles = sym ? tm * (tm + 1) / 2 : tm * tn;
    kern<<<(unsigned)(tiles * nsplit), WM * WN * 32, smem, stream>>>(
        R, m1, m2, A, lda, B, ldb, rows_per_split, tm, tn, work, sym);
    W4_LAUNCH();
}

}  // namespace

void gemm_nn(const GemmPass* passes, int npass, unsigned* status, cudaStream_t stream) {
    PassTable tab{};
    int64_t total_cols = 0, maxM = 0;
    bool vec2 = true;
    for (int i = 0; i < npass; ++i) {
        tab.p[i] = passes[i];
        total_cols += passes[i].ncols;
        maxM = passes[i].M > maxM ? passes[i].M : maxM;
        const GemmPass& p = passes[i];
        vec2 = vec2 && aligned16(p.A) && (p.lda % 2 == 0) && aligned16(p.in.base) &&
               (p.in.ld_outer % 2 == 0) && (p.in.stride % 2 == 0);
    }
    for (int i = npass; i < 2; ++i) tab.p[i] = GemmPass{};
    bool sym = vec2;
    for (int i = 0; i < npass; ++i) sym = sym && passes[i].symA && passes[i].M == passes[i].K;
    int64_t ws_tiles = 0;  // 128 x 128 tiles of the warp-specialised kernel, per pass
    for (int i = 0; i < npass; ++i) ws_tiles += cdiv(passes[i].M, 128) * cdiv(passes[i].ncols, 128);
    if (sym && 2 * ws_tiles >= kSMs) {
        int64_t start = 0;
        for (int i = 0; i < 2; ++i) {
            tab.tile_start[i] = start;
            if (i < npass && passes[i].ncols > 0 && passes[i].M > 0) {
                tab.tiles_m[i] = cdiv(passes[i].M, 128);
                start += tab.tiles_m[i] * cdiv(passes[i].ncols, 128);
            } else {
                tab.tiles_m[i] = 1;
            }
        }
        tab.tile_start[2] = start;
        static const int ws_mode = [] {
            const char* e = std::getenv("WC4DVAR_GEMM_WS");
            return e ? std::atoi(e) : 4;
        }();
        if (start > 0) {
            // WC4DVAR_GEMM_WS: 4 (default) = 16 consumer warps of 32x32 + 2 producer warps (A, B),
            // 1 = one producer warp, 2 = 8 consumer warps of 64x32
            // 3: unpadded swizzled stages, 6-deep ring
            if (ws_mode == 3) launch_sym_ws<128, 128, 4, 4, 6, BK>(tab, start, status, stream);
            else if (ws_mode == 4) launch_sym_ws<128, 128, 4, 4, 4, KS, 2>(tab, start, status, stream);
            else if (ws_mode == 2) launch_sym_ws<128, 128, 2, 4, 4>(tab, start, status, stream);
            else if (ws_mode) launch_sym_ws<128, 128, 4, 4, 4>(tab, start, status, stream);
            else launch_sym<128, 128, 4, 4, 3>(tab, start, status, stream);
        }
        return;
    }
    // Few columns (the single-vector applies of PCG: n x (N+1) columns): 64 x 32 tiles would
    // leave most SMs idle, so run one warp per 16 x 8 output tile with register-prefetched
    // fragments (gemm_chain_kernel).  Every shape accumulates each element in the same DMMA
    // order, so the choice never changes a bit of the result.
    static const int chain_mode = [] {
        const char* e = std::getenv("WC4DVAR_GEMM_CHAIN");
        return e ? std::atoi(e) : 1;
    }();
    if (sym && chain_mode > 0 && cdiv(maxM, 64) * cdiv(total_cols, 32) < kSMs) {
        int64_t units = 0;
        for (int i = 0; i < 2; ++i) {
            tab.tile_start[i] = units;
            if (i < npass && passes[i].ncols > 0 && passes[i].M > 0) {
                tab.tiles_m[i] = cdiv(passes[i].M, 16);
                units += tab.tiles_m[i] * cdiv(passes[i].ncols, 8);
            } else {
                tab.tiles_m[i] = 1;
            }
        }
        tab.tile_start[2] = units;
        if (units == 0) return;
        const unsigned grid = (unsigned)cdiv(units, 4);
        switch (chain_mode) {  // prefetch depth in k8 steps
            case 4: gemm_chain_kernel<4><<<grid, 128, 0, stream>>>(tab, status); break;
            case 6: gemm_chain_kernel<6><<<grid, 128, 0, stream>>>(tab, status); break;
            case 8: gemm_chain_kernel<8><<<grid, 128, 0, stream>>>(tab, status); break;
            default: gemm_chain_kernel<10><<<grid, 128, 0, stream>>>(tab, status); break;
        }
        W4_LAUNCH();
        return;
    }
    // Tile shape: big tiles when there are enough of them to fill the chip twice; 128 x 128
    // tiles with 16 warps for the tall x (>= 128 wide) products of the sketches (Y R^{-1},
    // Z W at k + l = 256: WC4DVAR_GEMM_NN = 1 forces the 128 x 64 shape, 2 the 128 x 128 one)
    static const int nn_env = [] {
        const char* e = std::getenv("WC4DVAR_GEMM_NN");
        return e ? std::atoi(e) : 0;
    }();
    const bool big = cdiv(maxM, 128) * cdiv(total_cols, 64) >= 2 * kSMs;
    const bool huge = vec2 && big && (nn_env == 2 || (nn_env == 0 && total_cols >= 128 &&
                                                        cdiv(maxM, 128) * cdiv(total_cols, 128) >= 2 * kSMs));
    const int BMv = big ? 128 : 64, BNv = huge ? 128 : (big ? 64 : 32);
    int64_t start = 0;
    for (int i = 0; i < 2; ++i) {
        tab.tile_start[i] = start;
        if (i < npass && passes[i].ncols > 0 && passes[i].M > 0) {
            tab.tiles_m[i] = cdiv(passes[i].M, BMv);
            start += tab.tiles_m[i] * cdiv(passes[i].ncols, BNv);
        } else {
            tab.tiles_m[i] = 1;
        }
    }
    tab.tile_start[2] = start;
    if (start == 0) return;
    if (huge) {
        launch_nn<128, 128, 4, 4, 3, 2>(tab, start, status, stream);
    } else if (big) {
        if (vec2) launch_nn<128, 64, 4, 2, 3, 2>(tab, start, status, stream);
        else launch_nn<128, 64, 4, 2, 3, 1>(tab, start, status, stream);
    } else {
        if (vec2) launch_nn<64, 32, 2, 2, 4, 2>(tab, start, status, stream);
        else launch_nn<64, 32, 2, 2, 4, 1>(tab, start, status, stream);
    }
}

void gemm_tn(int64_t R, int64_t m1, int64_t m2, const double* A, int64_t lda, const double* B,
             int64_t ldb, double alpha, double* C, int64_t ldc, DevBuf& work,
             cudaStream_t stream, bool sym_result) {
    if (m1 == 0 || m2 == 0) return;
    // tile variant (WC4DVAR_GEMM_TN, default 0 = by shape): 1: 64x64 / 4 warps / 4 stages,
    // 2: 64x64 / 8 warps, 3: 128x64 / 8 warps / 3 stages, 4: 128x128 / 16 warps / 3 stages
    static const int var_env = [] {
        const char* e = std::getenv("WC4DVAR_GEMM_TN");
        return e ? std::atoi(e) : 0;
    }();
    int var = var_env;
    // measured (C4 n = 1.7e7, m = 256): 128x128 / 16 warps 28.2 TF/s vs 64x64 / 4 warps ~17;
    // at m = 64 (C3) the 64x64 tiles win (25 vs 7 TF/s: a 128-wide tile is half empty)
    // symmetric results (Grams, Y^T A Y): only the upper-triangle tiles run, and 64 x 64 tiles cut
    // more of the square (10 of 16 at m = 256) than 128 x 128 ones (3 of 4): measured 143 vs 169 ms
    // of tall GEMMs per C4 k + l = 256 REVD
    const bool sym_shape = (A == B || sym_result) && m1 == m2 && lda == ldb;
    if (var == 0) var = (m1 >= 128 && m2 >= 128) ? (sym_shape ? 1 : 4) : (m1 >= 128 ? 3 : 1);
    const int BM = (var >= 3) ? 128 : 64, BN = (var == 4) ? 128 : 64;
    const int ctas_per_sm = (var == 4) ? 1 : 2;
    // Gram (A^T A): upper-triangle tiles only (square tiles; WC4DVAR_GEMM_SYRK=0 disables)
    static const bool syrk_env = [] {
        const char* e = std::getenv("WC4DVAR_GEMM_SYRK");
        return !(e && std::atoi(e) == 0);
    }();
    const bool vec2 = aligned16(A) && aligned16(B) && lda % 2 == 0 && ldb % 2 == 0;
    const bool sym = syrk_env && (A == B || sym_result) && m1 == m2 && lda == ldb && BM == BN && vec2 && var != 2 &&
                     cdiv(m1, BM) > 1;
    const int64_t tiles = sym ? cdiv(m1, BM) * (cdiv(m1, BM) + 1) / 2 : cdiv(m1, BM) * cdiv(m2, BN);
    // (sym: whole waves -- floor -- so no split lands in a one-CTA tail wave)
    int64_t nsplit = sym ? std::max<int64_t>(1, (int64_t)ctas_per_sm * kSMs / tiles)
                         : cdiv((int64_t)ctas_per_sm * kSMs, tiles);
    const int64_t min_rows = 256;
    if (nsplit * min_rows > R) nsplit = cdiv(R, min_rows);
    if (nsplit < 1) nsplit = 1;
    int64_t rows_per_split = cdiv(R, nsplit);
    rows_per_split = cdiv(rows_per_split, BK) * BK;
    nsplit = R > 0 ? cdiv(R, rows_per_split) : 1;
    double* w = work.get<double>((size_t)(nsplit * m1 * m2));
    if (R == 0) {
        W4_CUDA(cudaMemsetAsync(w, 0, sizeof(double) * m1 * m2, stream));
    } else if (!vec2) {
        launch_tn<64, 64, 2, 2, 4, 1>(R, m1, m2, A, lda, B, ldb, w, rows_per_split, nsplit, stream);
    } else if (var == 2) {
        launch_tn<64, 64, 2, 4, 4, 2>(R, m1, m2, A, lda, B, ldb, w, rows_per_split, nsplit, stream);
    } else if (var == 3) {
        launch_tn<128, 64, 4, 2, 3, 2>(R, m1, m2, A, lda, B, ldb, w, rows_per_split, nsplit, stream);
    } else if (var == 4) {
        launch_tn<128, 128, 4, 4, 3, 2>(R, m1, m2, A, lda, B, ldb, w, rows_per_split, nsplit, stream, sym);
    } else {
        launch_tn<64, 64, 2, 2, 4, 2>(R, m1, m2, A, lda, B, ldb, w, rows_per_split, nsplit, stream, sym);
    }
    const int64_t e = m1 * m2;
    reduce_splits_kernel<<<(unsigned)cdiv(e, 256), 256, 0, stream>>>(m1, m2, nsplit, w, alpha, C,
                                                                        ldc, (sym && R > 0) ? BM : 0);
    W4_LAUNCH();
}

}  // namespace w4
