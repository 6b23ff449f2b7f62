// Microbenchmark: does the FP64 tensor-core path (DMMA m8n8k4) run next to the FP64 FMA pipe on this GPU?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o benchmarks/_dmma_probe benchmarks/dmma_probe.cu && benchmarks/_dmma_probe
// Three kernels with the same launch shape: DFMA chains only, DMMA chains only, both interleaved 8 DFMA : 1 DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double x) {
    double f[8], c[8];
    for (int i = 0; i < 8; ++i) { f[i] = x + i + threadIdx.x; c[i] = x - i; }
    const double a = x * 1.0000001, b = x * 0.9999999;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);       // 32 DFMA
        }
        if (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);   // 4 DMMA = 32 DFMA-equivalents of work per lane
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += f[i] + c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
float run(double* out, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    probe<MODE><<<148 * 8, 256>>>(out, 16, 1.0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    probe<MODE><<<148 * 8, 256>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    const int iters = 20000;
    const double lanes = 148.0 * 8 * 256 * iters;
    float t0 = run<0>(out, iters), t1 = run<1>(out, iters), t2 = run<2>(out, iters);
    printf("DFMA only : %8.3f ms  %6.2f TFLOP/s\n", t0, lanes * 32 * 2 / t0 / 1e9);
    printf("DMMA only : %8.3f ms  %6.2f TFLOP/s (4 x m8n8k4 per lane-iter = 4*512 flop per warp)\n", t1, 148.0 * 8 * 8 * iters * 4 * 512 / t1 / 1e9);
    printf("both      : %8.3f ms  (sum of the two alone: %.3f ms; max: %.3f ms)\n", t2, t0 + t1, t0 > t1 ? t0 : t1);
    return 0;
}
