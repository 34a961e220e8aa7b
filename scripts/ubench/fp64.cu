// fp64.cu -- fp64 throughput on B200: DFMA (CUDA cores) and DMMA (mma.sync m8n8k4 f64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64 fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += a[i];
    if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; i++) acc[i][0] = acc[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 4; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int threads : {128, 256, 512}) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            dfma_kernel<<<sms * 4, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)sms * 4 * threads;
        printf("DFMA threads=%d  %.2f TFLOP/s\n", threads, flops / (ms * 1e-3) / 1e12);
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            dmma_kernel<<<sms * 4, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        // per warp-level mma: 8x8x4 MACs = 256 MAC = 512 flop; 4 per iter per warp
        flops = 512.0 * 4 * iters * (double)sms * 4 * threads / 32;
        printf("DMMA threads=%d  %.2f TFLOP/s\n", threads, flops / (ms * 1e-3) / 1e12);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
