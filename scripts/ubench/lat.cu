// Latency microbenchmarks on sm_100a (single warp): SHFL chain, FFMA chain, FMNMX+FFMA chain,
// mbarrier arrive->try_wait round trip, LDS chain.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__global__ void k_shfl(float *out, long long *cyc, int n) {
    float x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) x = __shfl_sync(0xffffffffu, x, (i & 7)) + 1.0f;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl_nodiv(float *out, long long *cyc, int n) {
    float x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; i++) asm volatile("shfl.sync.idx.b32 %0, %0, 3, 0x1f, 0xffffffff;" : "+f"(x));
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void k_ffma(float *out, long long *cyc, int n, float a) {
    float x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; i++) x = fmaf(x, a, 0.5f);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
__global__ void k_mnmx_ffma(float *out, long long *cyc, int n, float a) {
    float x = threadIdx.x, y = 0.1f;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; i++) { x = fmaxf(x, -y); x = fmaf(x, a, 0.5f); }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
}
__global__ void k_lds(float *out, long long *cyc, int n) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) & 1023;
    __syncwarp();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) p = s[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
}
int main() {
    float *out; long long *cyc, h[8] = {};
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64); cudaMemset(cyc, 0, 64);
    const int n = 4096;
    for (int rep = 0; rep < 2; rep++) {
        k_shfl<<<1, 32>>>(out, cyc, n);
        k_shfl_nodiv<<<1, 32>>>(out, cyc, n);
        k_ffma<<<1, 32>>>(out, cyc, n, 0.999f);
        k_mnmx_ffma<<<1, 32>>>(out, cyc, n, 0.999f);
        k_lds<<<1, 32>>>(out, cyc, n);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
    printf("cycles per op: shfl(+fadd, dyn lane) %.1f | shfl.sync const %.1f | ffma %.1f | fmnmx+ffma %.1f | lds chain %.1f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
    return 0;
}
