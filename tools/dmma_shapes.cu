// Throughput of the fp64 mma.sync shapes on this GPU (all SMs, 16 warps / SM, 8 independent
// accumulator chains per warp): m8n8k4 vs m16n8k4 vs m16n8k8.
#include <cstdio>

template <int SHAPE>
__global__ void __launch_bounds__(512) k(int iters, double* sink) {
    double acc[8][4];
    for (int c = 0; c < 8; ++c)
        for (int v = 0; v < 4; ++v) acc[c][v] = threadIdx.x * 1e-9 + c;
    double a0 = 1.0 + threadIdx.x * 1e-12, a1 = 0.5, a2 = 0.25, a3 = 0.125, b0 = 0.999, b1 = 1.001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (SHAPE == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a0), "d"(b0));
            else if (SHAPE == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3]) : "d"(a0), "d"(a1), "d"(b0));
            else
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                             : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
        }
    }
    double s = 0;
    for (int c = 0; c < 8; ++c)
        for (int v = 0; v < 4; ++v) s += acc[c][v];
    if (s == 12345.0) sink[0] = s;
}

template <int SHAPE>
void run(const char* name, double fma_per_instr) {
    double* sink;
    cudaMalloc(&sink, 8);
    const int iters = 2000;
    k<SHAPE><<<148, 512>>>(16, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<SHAPE><<<148, 512>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    const double instr = 148.0 * 16 * iters * 8;
    printf("%-8s %s: %.3f ms, %.2f TF/s\n", name, err == cudaSuccess ? "ok" : cudaGetErrorString(err), ms,
           2.0 * fma_per_instr * instr / ms / 1e9);
    cudaFree(sink);
}

int main() {
    run<0>("m8n8k4", 8 * 8 * 4);
    run<1>("m16n8k4", 16 * 8 * 4);
    run<2>("m16n8k8", 16 * 8 * 8);
    return 0;
}
