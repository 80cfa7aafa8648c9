// Microbenchmark: fp64 throughput of DMMA (tensor pipe), DFMA (fp64 pipe) and both mixed,
// to decide whether a hybrid DMMA+DFMA GEMM can exceed the DMMA roofline on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu -o /tmp/fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0 DMMA, 1 DFMA, 2 mixed (warp-interleaved)
__global__ void __launch_bounds__(256) k(int iters, double* sink) {
    double a[4], b[2], d[8][4], f[16];
    const int t = threadIdx.x;
    for (int i = 0; i < 4; ++i) a[i] = 1.0 + 1e-3 * (t + i);
    b[0] = 0.5;
    b[1] = 0.25;
    for (int c = 0; c < 8; ++c)
        for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
    for (int i = 0; i < 16; ++i) f[i] = 1e-3 * i;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
                    "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                    : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                    : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
        }
        if (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int r = 0; r < (MODE == 1 ? 16 : 4); ++r)
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a[i & 3], b[i & 1]);
        }
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    for (int i = 0; i < 16; ++i) s += f[i];
    if (s == 12345.678) sink[blockIdx.x] = s;
}

template <int MODE>
void run(const char* name) {
    double* sink;
    cudaMalloc(&sink, 8 * 4096);
    const int blocks = 148 * 4, threads = 256, iters = 2048;
    k<MODE><<<blocks, threads>>>(64, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = blocks * threads / 32.0;
    double mma_flops = (MODE == 0 || MODE == 2) ? warps * iters * 8 * 2.0 * 16 * 8 * 8 : 0;
    double fma_flops = (MODE == 1) ? blocks * threads * (double)iters * 16 * 16 * 2
                       : (MODE == 2) ? blocks * threads * (double)iters * 4 * 16 * 2 : 0;
    printf("%-6s %8.3f ms  dmma %7.2f TF/s  dfma %7.2f TF/s  total %7.2f TF/s\n", name, ms,
           mma_flops / ms / 1e9, fma_flops / ms / 1e9, (mma_flops + fma_flops) / ms / 1e9);
    cudaFree(sink);
}

int main() {
    run<0>("dmma");
    run<1>("dfma");
    run<2>("mixed");
    return 0;
}
