// FP64 dependent-issue latency and per-scheduler throughput on the device, for the analysis of
// the FFT butterfly kernels:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_latency_probe.cu -o /tmp/fp64lat && /tmp/fp64lat
// For ILP chains per thread in {1, 2, 4, 8} and warps per CTA in {1, 4, 8, 16} (one CTA per SM)
// it prints cycles per DFMA per warp and the SM-wide DFMA rate per clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void probe(double* out, long long* cyc, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(int warps) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * nsm * warps * 32);
    cudaMalloc(&cyc, sizeof(long long) * nsm);
    const int iters = 2000;
    probe<ILP><<<nsm, warps * 32>>>(out, cyc, iters, 0.999999, 1e-9);
    probe<ILP><<<nsm, warps * 32>>>(out, cyc, iters, 0.999999, 1e-9);
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double per_warp_instr = (double)iters * 8 * ILP;
    printf("ILP %d warps/SM %2d: %.2f cycles per DFMA per warp, %.1f DFMA lanes per clock per SM\n", ILP, warps,
           h / per_warp_instr, per_warp_instr * warps * 32 / h);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 8, 14, 16, 32}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
    }
    return 0;
}
