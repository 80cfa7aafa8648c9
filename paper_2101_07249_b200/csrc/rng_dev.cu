// Device NormalStream (random.hpp:14-42) for the Gaussian sketch gaussian_matrix
// (randevd.cpp:16-21): std::mt19937_64 + the reference's Box-Muller, column-major fill,
// generated on the GPU with MT19937-64 jump-ahead so every column (or row shard) of the
// reference's single serial stream starts at its own offset.
//
//   * The 19937-degree characteristic polynomial p of the MT19937-64 transition is found
//     once per process by Berlekamp-Massey on the engine's own bit sequence.
//   * A jump by D raw draws is g(A) with g = x^D mod p (square-and-multiply in GF(2)[x]),
//     applied as  state_{+D} = XOR over the set coefficients i of g of window_{+i}:
//     the state at offset k is the window of 312 recurrence words x_k .. x_{k+311}
//     (x_k's low 31 bits are don't-care), so g(A) s only needs the next L words of the
//     sequence from s.
//   * Column j of an n_total-row Gaussian matrix starts at raw draw 2 (n_total j + row0):
//     one host jump to the first column, then a one-CTA device chain of column jumps,
//     then one CTA per column runs the engine (two-phase twist in shared memory) and the
//     Box-Muller transform.
// Raw 64-bit outputs are bit-exact with libstdc++; the normals use the device log / cos /
// sqrt (a few ulp from glibc's), pinned by tests/test_gpu_rng.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace w4 {
void set_last_error(const std::string& msg);
namespace {

constexpr int MT_NW = 312;                // state words
constexpr int MT_MID = 156;
constexpr int MT_L = 19937;               // degree of the characteristic polynomial
constexpr int PW = (MT_L + 64) / 64;      // 312 words hold degrees 0 .. L (bit L included)
constexpr uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;

__host__ __device__ inline uint64_t mt_next_word(uint64_t xk, uint64_t xk1, uint64_t xkm) {
    const uint64_t y = (xk & UPPER) | (xk1 & LOWER);
    return xkm ^ (y >> 1) ^ ((y & 1ULL) ? MATRIX_A : 0ULL);
}

__host__ __device__ inline uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// std::mersenne_twister_engine seeding ([rand.eng.mers], f = 6364136223846793005).
void mt_seed(uint64_t seed, uint64_t* st) {
    st[0] = seed;
    for (int i = 1; i < MT_NW; ++i) st[i] = 6364136223846793005ULL * (st[i - 1] ^ (st[i - 1] >> 62)) + (uint64_t)i;
}

// x_{k+312} = x_{k+156} ^ twist(x_k, x_{k+1}) extended from the window seq[0..311].
void mt_extend(std::vector<uint64_t>& seq, size_t total) {
    const size_t have = seq.size();
    seq.resize(total);
    for (size_t k = have; k < total; ++k)
        seq[k] = mt_next_word(seq[k - MT_NW], seq[k - MT_NW + 1], seq[k - MT_MID]);
}

// ----------------------------------------------------------------------- GF(2)[x]

// this ^= src << shift (bit arrays, this large enough).
void xor_shifted(std::vector<uint64_t>& dst, const std::vector<uint64_t>& src, size_t shift) {
    const size_t ws = shift >> 6, bs = shift & 63;
    const size_t n = src.size();
    if (bs == 0) {
        for (size_t i = 0; i < n && i + ws < dst.size(); ++i) dst[i + ws] ^= src[i];
        return;
    }
    for (size_t i = 0; i < n; ++i) {
        if (i + ws < dst.size()) dst[i + ws] ^= src[i] << bs;
        if (i + ws + 1 < dst.size()) dst[i + ws + 1] ^= src[i] >> (64 - bs);
    }
}

// Characteristic polynomial p (degree L, bit i = coefficient of x^i) of the MT19937-64
// state transition, by Berlekamp-Massey on the top bit of the recurrence words.
std::vector<uint64_t> compute_charpoly() {
    const size_t nbits = 2 * (size_t)MT_L + 256;
    std::vector<uint64_t> seq(MT_NW);
    mt_seed(5489ULL, seq.data());
    mt_extend(seq, nbits);
    const size_t cw = (MT_L + 1 + 63) / 64 + 2;
    std::vector<uint64_t> C(cw, 0), B(cw, 0), T(cw, 0), R(cw, 0);
    C[0] = B[0] = 1;
    size_t L = 0, m = 1;
    for (size_t n = 0; n < nbits; ++n) {
        // R bit i = s_{n-i}
        for (size_t i = cw - 1; i > 0; --i) R[i] = (R[i] << 1) | (R[i - 1] >> 63);
        R[0] = (R[0] << 1) | (seq[n] >> 63);
        uint64_t acc = 0;
        for (size_t i = 0; i < cw; ++i) acc ^= C[i] & R[i];
        const int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
        } else if (2 * L <= n) {
            T = C;
            xor_shifted(C, B, m);
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            xor_shifted(C, B, m);
            ++m;
        }
    }
    if (L != (size_t)MT_L) throw DeviceError("mt19937_64 jump-ahead: unexpected linear complexity");
    // p(x) = x^L C(1/x)
    std::vector<uint64_t> p(PW, 0);
    for (size_t i = 0; i <= L; ++i)
        if ((C[i >> 6] >> (i & 63)) & 1ULL) p[(L - i) >> 6] |= 1ULL << ((L - i) & 63);
    return p;
}

struct JumpTables {
    std::vector<uint64_t> p;                     // degree L
    std::vector<std::vector<uint64_t>> pshift;   // p << s, s = 0..63 (PW + 1 words)
    std::map<uint64_t, std::vector<int32_t>> terms;
    std::mutex mu;
};

JumpTables& tables() {
    static JumpTables* t = [] {
        auto* j = new JumpTables;
        j->p = compute_charpoly();
        j->pshift.resize(64);
        for (int s = 0; s < 64; ++s) {
            std::vector<uint64_t> v(PW + 1, 0);
            xor_shifted(v, j->p, s);
            j->pshift[s] = v;
        }
        return j;
    }();
    return *t;
}

inline uint64_t spread32(uint32_t x) {
    uint64_t v = x;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFULL;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFULL;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0FULL;
    v = (v | (v << 2)) & 0x3333333333333333ULL;
    v = (v | (v << 1)) & 0x5555555555555555ULL;
    return v;
}

// t (degree < 2L) mod p -> degree < L, in place.
void reduce(std::vector<uint64_t>& t, const JumpTables& J) {
    for (int64_t i = 2 * (int64_t)MT_L; i >= MT_L; --i) {
        if (!((t[i >> 6] >> (i & 63)) & 1ULL)) continue;
        const int64_t sh = i - MT_L;
        const std::vector<uint64_t>& ps = J.pshift[sh & 63];
        const size_t ws = (size_t)(sh >> 6);
        for (size_t k = 0; k < ps.size() && k + ws < t.size(); ++k) t[k + ws] ^= ps[k];
    }
}

// Set coefficients of x^D mod p (sorted).
std::vector<int32_t> jump_terms(uint64_t D) {
    JumpTables& J = tables();
    {
        std::lock_guard<std::mutex> lk(J.mu);
        auto it = J.terms.find(D);
        if (it != J.terms.end()) return it->second;
    }
    std::vector<int32_t> out;
    if (D < (uint64_t)MT_L) {
        out.push_back((int32_t)D);
    } else {
        const size_t tw = 2 * PW + 2;
        std::vector<uint64_t> r(tw, 0), sq(tw, 0);
        r[0] = 1;  // r = 1
        int top = 63;
        while (!((D >> top) & 1ULL)) --top;
        for (int b = top; b >= 0; --b) {
            // r = r^2 mod p
            std::fill(sq.begin(), sq.end(), 0);
            for (size_t k = 0; k < (size_t)PW; ++k) {
                sq[2 * k] = spread32((uint32_t)r[k]);
                sq[2 * k + 1] = spread32((uint32_t)(r[k] >> 32));
            }
            reduce(sq, J);
            std::swap(r, sq);
            if ((D >> b) & 1ULL) {  // r = r x mod p
                for (size_t k = tw - 1; k > 0; --k) r[k] = (r[k] << 1) | (r[k - 1] >> 63);
                r[0] <<= 1;
                if ((r[MT_L >> 6] >> (MT_L & 63)) & 1ULL)
                    for (size_t k = 0; k < (size_t)PW; ++k) r[k] ^= J.p[k];
            }
        }
        for (int32_t i = 0; i < MT_L; ++i)
            if ((r[i >> 6] >> (i & 63)) & 1ULL) out.push_back(i);
    }
    std::lock_guard<std::mutex> lk(J.mu);
    J.terms[D] = out;
    return out;
}

// Host jump of a state window by the polynomial with coefficients `terms`.
void host_jump(const uint64_t* st, const std::vector<int32_t>& terms, uint64_t* out) {
    std::vector<uint64_t> seq(st, st + MT_NW);
    const int32_t top = terms.empty() ? 0 : terms.back();
    mt_extend(seq, (size_t)top + MT_NW);
    std::vector<uint64_t> acc(MT_NW, 0);
    for (int32_t i : terms)
        for (int t = 0; t < MT_NW; ++t) acc[t] ^= seq[(size_t)i + t];
    std::memcpy(out, acc.data(), sizeof(uint64_t) * MT_NW);
}

// ----------------------------------------------------------------------- kernels
constexpr int CHAIN_THREADS = 320;
constexpr int CHAIN_SEQ = MT_L + MT_NW + 32;  // words of the extended sequence

// states[c] = jump^c (state0), c = 0 .. count-1 (one CTA; the jump polynomial's set
// coefficients in `terms`).  Shared memory: the extended sequence (~162 KB).
__global__ void __launch_bounds__(CHAIN_THREADS) mt_jump_chain_kernel(
    const uint64_t* __restrict__ state0, const int32_t* __restrict__ terms, int nterms, int seq_len,
    int64_t count, uint64_t* __restrict__ states) {
    extern __shared__ uint64_t seq[];
    const int t = threadIdx.x;
    for (int i = t; i < MT_NW; i += blockDim.x) {
        seq[i] = state0[i];
        states[i] = state0[i];
    }
    __syncthreads();
    for (int64_t c = 1; c < count; ++c) {
        for (int base = MT_NW; base < seq_len; base += MT_NW) {
            // phase 1: k = base - 312 + i, i < 156 reads only the previous block
            if (t < MT_MID) {
                const int k = base - MT_NW + t;
                if (k + MT_NW < seq_len) seq[k + MT_NW] = mt_next_word(seq[k], seq[k + 1], seq[k + MT_MID]);
            }
            __syncthreads();
            if (t < MT_NW - MT_MID) {
                const int k = base - MT_NW + MT_MID + t;
                if (k + MT_NW < seq_len) seq[k + MT_NW] = mt_next_word(seq[k], seq[k + 1], seq[k + MT_MID]);
            }
            __syncthreads();
        }
        uint64_t acc = 0;
        if (t < MT_NW)
            for (int j = 0; j < nterms; ++j) acc ^= seq[__ldg(terms + j) + t];
        __syncthreads();
        if (t < MT_NW) {
            seq[t] = acc;
            states[c * MT_NW + t] = acc;
        }
        __syncthreads();
    }
}

constexpr int GEN_THREADS = MT_MID;  // one word per phase and one normal per thread per twist

// Column j: out[j*ldo + i], i < rows = the normals of the stream whose state window is
// states[j] (raw outputs = temper of the words after the window).  raw != 0 writes the
// raw 64-bit outputs instead (2 per "row") for the bit-exact engine test.
__global__ void __launch_bounds__(GEN_THREADS) mt_normal_kernel(const uint64_t* __restrict__ states,
                                                               int64_t rows, double* __restrict__ out,
                                                               int64_t ldo, int raw) {
    __shared__ uint64_t ring[2][MT_NW];
    const int t = threadIdx.x;
    const int64_t col = blockIdx.x;
    const uint64_t* st = states + col * MT_NW;
    ring[0][t] = st[t];
    ring[0][t + MT_MID] = st[t + MT_MID];
    __syncthreads();
    double* dst = out + col * ldo;
    constexpr double two_pi = 6.283185307179586476925286766559;
    int cur = 0;
    for (int64_t r0 = 0; r0 < rows; r0 += MT_MID) {
        const int nx = cur ^ 1;
        // x_{k+312}: phase 1 (i < 156) from the old block, phase 2 also from phase-1 words
        const uint64_t* o = ring[cur];
        uint64_t* w = ring[nx];
        w[t] = mt_next_word(o[t], o[t + 1], o[t + MT_MID]);
        __syncthreads();
        {
            const int i = t + MT_MID;
            const uint64_t xk1 = (i + 1 < MT_NW) ? o[i + 1] : w[0];
            w[i] = mt_next_word(o[i], xk1, w[i - MT_MID]);
        }
        __syncthreads();
        const int64_t r = r0 + t;
        if (r < rows) {
            const uint64_t a = mt_temper(w[2 * t]);
            const uint64_t b = mt_temper(w[2 * t + 1]);
            if (raw) {
                reinterpret_cast<uint64_t*>(dst)[2 * r] = a;
                reinterpret_cast<uint64_t*>(dst)[2 * r + 1] = b;
            } else {
                // random.hpp:21-24
                const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
                const double u2 = (double)(b >> 11) * 0x1.0p-53;
                dst[r] = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(two_pi, u2)));
            }
        }
        cur = nx;
    }
}

}  // namespace

void mt_seed_public(uint64_t seed, uint64_t* st) { mt_seed(seed, st); }
void mt_extend_public(std::vector<uint64_t>& seq, size_t total) { mt_extend(seq, total); }
uint64_t mt_temper_public(uint64_t y) { return mt_temper(y); }
void host_jump_public(const uint64_t* st, uint64_t D, uint64_t* out) {
    if (D == 0) {
        std::memcpy(out, st, sizeof(uint64_t) * MT_NW);
        return;
    }
    host_jump(st, jump_terms(D), out);
}

// out (rows x cols, ldo) = rows [row0, row0 + rows) x columns [col0, col0 + cols) of
// gaussian_matrix(n_total, *, seed).  Device pointer on the current device.
void gaussian_block_dev(int64_t n_total, int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                        uint64_t seed, double* out, int64_t ldo, bool raw, cudaStream_t st) {
    require(n_total >= 0 && row0 >= 0 && rows >= 0 && col0 >= 0 && cols >= 0 && row0 + rows <= n_total,
            "gaussian_matrix: block outside the matrix");
    require(ldo >= (raw ? 2 * rows : rows), "gaussian_matrix: ldo too small");
    if (rows == 0 || cols == 0) return;
    uint64_t s0[MT_NW], s1[MT_NW];
    mt_seed(seed, s0);
    const uint64_t D0 = 2ULL * ((uint64_t)n_total * (uint64_t)col0 + (uint64_t)row0);
    if (D0) {
        host_jump(s0, jump_terms(D0), s1);
    } else {
        std::memcpy(s1, s0, sizeof(s0));
    }
    uint64_t* d_states = nullptr;
    int32_t* d_terms = nullptr;
    W4_CUDA(cudaMallocAsync(&d_states, sizeof(uint64_t) * MT_NW * cols, st));
    W4_CUDA(cudaMemcpyAsync(d_states, s1, sizeof(s1), cudaMemcpyHostToDevice, st));
    std::vector<int32_t> terms;
    if (cols > 1) {
        terms = jump_terms(2ULL * (uint64_t)n_total);
        const int seq_len = terms.back() + MT_NW;
        W4_CUDA(cudaMallocAsync(&d_terms, sizeof(int32_t) * terms.size(), st));
        W4_CUDA(cudaMemcpyAsync(d_terms, terms.data(), sizeof(int32_t) * terms.size(), cudaMemcpyHostToDevice, st));
        const size_t smem = sizeof(uint64_t) * (size_t)(seq_len + MT_NW);
        W4_CUDA(cudaFuncSetAttribute(mt_jump_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        mt_jump_chain_kernel<<<1, CHAIN_THREADS, smem, st>>>(d_states, d_terms, (int)terms.size(), seq_len, cols,
                                                             d_states);
        W4_LAUNCH();
    }
    mt_normal_kernel<<<(unsigned)cols, GEN_THREADS, 0, st>>>(d_states, rows, out, ldo, raw ? 1 : 0);
    W4_LAUNCH();
    if (d_terms) W4_CUDA(cudaFreeAsync(d_terms, st));
    W4_CUDA(cudaFreeAsync(d_states, st));
    if (!terms.empty()) W4_CUDA(cudaStreamSynchronize(st));  // host vector lifetime
}

}  // namespace w4

namespace {
int api_status(const std::exception& e) {
    w4::set_last_error(e.what());
    if (dynamic_cast<const w4::InvalidArgument*>(&e)) return WC4DVAR_INVALID_ARGUMENT;
    if (dynamic_cast<const w4::NumericalError*>(&e)) return WC4DVAR_NUMERICAL;
    return WC4DVAR_DEVICE;
}
}  // namespace

extern "C" int wc4dvar_gpu_gaussian_block_dev(int64_t n_total, int64_t row0, int64_t rows, int64_t col0,
                                              int64_t cols, uint64_t seed, double* out, int64_t ldo,
                                              int device, void* stream) {
    try {
        w4::require(out != nullptr || rows * cols == 0, "gaussian_matrix: null output");
        w4::DeviceGuard g(device);
        w4::gaussian_block_dev(n_total, row0, rows, col0, cols, seed, out, ldo, false,
                               static_cast<cudaStream_t>(stream));
        return WC4DVAR_OK;
    } catch (const std::exception& e) {
        return api_status(e);
    }
}

extern "C" int wc4dvar_gpu_mt19937_raw_dev(uint64_t seed, uint64_t offset, int64_t count, uint64_t* out,
                                           int device, void* stream) {
    try {
        w4::require(offset % 2 == 0 && count % 2 == 0 && count >= 0, "mt19937_raw: offset and count must be even");
        w4::require(out != nullptr || count == 0, "mt19937_raw: null output");
        w4::DeviceGuard g(device);
        // a one-column "matrix" of count/2 rows starting at raw draw `offset`
        const int64_t rows = count / 2;
        w4::gaussian_block_dev((int64_t)(offset / 2) + rows, (int64_t)(offset / 2), rows, 0, 1, seed,
                               reinterpret_cast<double*>(out), 2 * rows, true, static_cast<cudaStream_t>(stream));
        return WC4DVAR_OK;
    } catch (const std::exception& e) {
        return api_status(e);
    }
}

// Host twin of the device jump (same polynomial, same window XOR): `count` raw outputs of
// std::mt19937_64(seed) from draw `offset`.  Lets the CPU test suite pin the jump-ahead
// arithmetic against libstdc++ golden vectors without a GPU.
extern "C" int wc4dvar_gpu_mt19937_raw_host(uint64_t seed, uint64_t offset, int64_t count, uint64_t* out) {
    try {
        w4::require(count >= 0 && (out != nullptr || count == 0), "mt19937_raw: bad arguments");
        uint64_t s0[312], s1[312];
        w4::mt_seed_public(seed, s0);
        w4::host_jump_public(s0, offset, s1);
        std::vector<uint64_t> seq(s1, s1 + 312);
        w4::mt_extend_public(seq, (size_t)count + 312);
        for (int64_t i = 0; i < count; ++i) out[i] = w4::mt_temper_public(seq[312 + (size_t)i]);
        return WC4DVAR_OK;
    } catch (const std::exception& e) {
        return api_status(e);
    }
}
