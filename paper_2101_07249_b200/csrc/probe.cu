// fp64 tensor-core (DMMA) peak probe: every SM runs warps of independent
// mma.sync.m16n8k8.f64 chains; the sustained rate is the roofline denominator for the
// D^{1/2} GEMM (MEASURED_PEAKS.json only carries bf16 and HBM).
#include "common.cuh"

namespace w4 {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* sink) {
    double a[4], b[2], d[kChains][4];
    const int t = threadIdx.x;
    for (int i = 0; i < 4; ++i) a[i] = 1.0 + 1e-3 * (t + i);
    b[0] = 0.5;
    b[1] = 0.25;
    for (int c = 0; c < kChains; ++c)
        for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
    double s = 0;
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345.678) sink[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace

double probe_dmma_tflops() {
    double* sink = nullptr;
    W4_CUDA(cudaMalloc(&sink, sizeof(double) * 4096));
    cudaEvent_t e0, e1;
    W4_CUDA(cudaEventCreate(&e0));
    W4_CUDA(cudaEventCreate(&e1));
    const int blocks = kSMs * 4, threads = 256, iters = 4096;
    dmma_peak_kernel<<<blocks, threads>>>(256, sink);  // warm-up
    W4_LAUNCH();
    W4_CUDA(cudaEventRecord(e0));
    dmma_peak_kernel<<<blocks, threads>>>(iters, sink);
    W4_CUDA(cudaEventRecord(e1));
    W4_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    W4_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    const double warps = (double)blocks * threads / 32;
    const double flops = warps * iters * kChains * 2.0 * 16 * 8 * 8;
    return flops / (ms * 1e-3) / 1e12;
}

}  // namespace w4
