// Does a warp-wide DFMA (16 fp64 lanes per SM sub-partition: two pipe cycles)
// also hold the sub-partition's ISSUE port for two cycles?  Each thread runs
// 8 independent DFMA chains with K independent full-rate fp32 FFMAs per DFMA.  If issue continues during the
// DFMA's second cycle, time stays flat up to K = 1; if it is blocked, time
// grows by one cycle per extra instruction from K = 1 on.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_issue fp64_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void __launch_bounds__(256) k(double* out, float* iout, int iters, double a, double b, float m, float c) {
    double x[8];
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = threadIdx.x * 1e-3 + i;
        y[i] = threadIdx.x * 1e-3f + i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            x[i] = fma(x[i], a, b);
#pragma unroll
            for (int j = 0; j < K; ++j) y[(i + j) & 7] = fmaf(y[(i + j) & 7], m, c);
        }
    }
    double s = 0;
    float t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        s += x[i];
        t += y[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    iout[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int K>
void run(double* d, float* di, int sms) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<K><<<sms * 8, 256>>>(d, di, 64, 1.0000001, 1e-9, 1.0001f, 1e-7f);
    cudaEventRecord(e0);
    k<K><<<sms * 8, 256>>>(d, di, iters, 1.0000001, 1e-9, 1.0001f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // warp-DFMAs per sub-partition: 8 CTAs x 8 warps / 4 SMSPs per SM
    const double dfma_per_smsp = 16.0 * iters * 8;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("K=%d  %.3f ms  cycles per DFMA per sub-partition (at %d MHz nominal): %.3f\n", K, ms,
           clk / 1000, ms * 1e-3 * clk * 1e3 / dfma_per_smsp);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    float* di;
    cudaMalloc(&d, sms * 8 * 256 * sizeof(double));
    cudaMalloc(&di, sms * 8 * 256 * sizeof(float));
    run<0>(d, di, sms);
    run<1>(d, di, sms);
    run<2>(d, di, sms);
    run<3>(d, di, sms);
    run<4>(d, di, sms);
    return 0;
}
