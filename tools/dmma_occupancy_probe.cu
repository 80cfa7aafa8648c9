// DMMA throughput vs resident warps per SM and independent accumulators per warp:
// what occupancy / ILP does the fp64 tensor pipe need to saturate on B200?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_occupancy_probe.cu -o /tmp/dprobe
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(int iters, double* sink) {
    double a0 = 1.0 + threadIdx.x * 1e-3, a1 = 0.5, b0 = 0.25, d[CH][4];
    for (int c = 0; c < CH; ++c)
        for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                         : "d"(a0), "d"(a1), "d"(b0));
    }
    double s = 0;
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 1.2345) sink[0] = s;
}

template <int CH>
void run(int warps_per_sm) {
    double* sink;
    cudaMalloc(&sink, 8);
    const int threads = 32 * warps_per_sm;  // one block per SM
    const int iters = 4096;
    k<CH><<<148, threads>>>(64, sink);
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("warps/SM %2d chains %2d : launch failed\n", warps_per_sm, CH);
        cudaFree(sink);
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<CH><<<148, threads>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    // a launch that does not fit (registers x threads) fails without running: report it
    // instead of dividing the flop count by a zero-length interval
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("warps/SM %2d chains %2d : launch failed (%s)\n", warps_per_sm, CH, cudaGetErrorString(err));
        cudaFree(sink);
        return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps_per_sm * iters * CH * 2.0 * 16 * 8 * 4;
    printf("warps/SM %2d chains %2d : %6.2f TF/s\n", warps_per_sm, CH, flops / ms / 1e9);
    cudaFree(sink);
}

int main() {
    for (int w : {4, 8, 16, 32}) {
        run<4>(w);
        run<8>(w);
        run<16>(w);
    }
    return 0;
}
