// Shared host/device helpers for the wc4dvar B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/wc4dvar_gpu.h"

namespace w4 {

// Error types carried to the C-ABI status codes (types.hpp:14-30 of the reference).
struct InvalidArgument : std::runtime_error {
    explicit InvalidArgument(const std::string& w) : std::runtime_error(w) {}
};
struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

inline void require(bool cond, const std::string& what) {
    if (!cond) throw InvalidArgument(what);
}

#define W4_CUDA(expr)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw ::w4::DeviceError(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Kernel launches issued by this library (wc4dvar_gpu_launch_count): every launch site
// is followed by W4_LAUNCH().
extern std::atomic<long long> g_launch_count;

#define W4_LAUNCH()                                                                      \
    do {                                                                                 \
        ::w4::g_launch_count.fetch_add(1, std::memory_order_relaxed);                    \
        cudaError_t _e = cudaGetLastError();                                             \
        if (_e != cudaSuccess)                                                           \
            throw ::w4::DeviceError(std::string("kernel launch (") + __FILE__ + ":" +       \
                                    std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
    } while (0)

// Status bits written by kernels into a device word (finite checks of
// HessianOperator::apply, operators.cpp:133-143).
enum : unsigned {
    ST_FWD_NONFINITE = 1u,
    ST_ADJ_NONFINITE = 2u,
    ST_OUT_NONFINITE = 4u,
};

constexpr int kSMs = 148;  // B200

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* get(size_t count) {
        const size_t need = count * sizeof(T);
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            W4_CUDA(cudaMalloc(&p, need));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
};

// Grow-only pinned host buffer.
struct PinBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
    template <class T>
    T* get(size_t count) {
        const size_t need = count * sizeof(T);
        if (need > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            W4_CUDA(cudaMallocHost(&p, need));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        W4_CUDA(cudaGetDevice(&prev));
        if (prev != dev) W4_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace w4
