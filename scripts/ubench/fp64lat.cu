// fp64lat.cu -- latency (one warp, dependent chain) and throughput (many warps, independent
// chains) of DFMA, F2F.F64.F32, F2F.F32.F64, SHFL, VOTE on this GPU (clock64 cycles).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64lat fp64lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat_kernel(double *out, float *outf, int iters, long long *cyc) {
    double d = threadIdx.x * 1e-3 + 1.0, e = 1.0000001;
    float f = threadIdx.x * 1e-3f + 1.f;
    unsigned u = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            if (OP == 0) d = fma(d, e, 1e-9);                       // DFMA chain
            if (OP == 1) { d = (double)f; f = (float)(d * 1.0000001); }   // F2F.F64.F32 + DMUL + F2F.F32.F64
            if (OP == 2) f = __shfl_sync(0xffffffffu, f, (threadIdx.x + 1) & 31);
            if (OP == 3) u = __ballot_sync(0xffffffffu, (u & 1) != 0) + threadIdx.x;
            if (OP == 4) f = fmaf(f, 1.0000001f, 1e-9f);            // FFMA chain
            if (OP == 5) d = d + (double)f;                         // F2F + DADD chain via d
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = d + u;
    outf[blockIdx.x * blockDim.x + threadIdx.x] = f;
}

template <int OP>
__global__ void tput_kernel(double *out, int iters, long long *cyc) {
    double d[8];
    float f[8];
    for (int j = 0; j < 8; j++) { d[j] = threadIdx.x + j; f[j] = threadIdx.x * 0.5f + j; }
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (OP == 0) d[j] = fma(d[j], 1.0000001, 1e-9);
            if (OP == 1) d[j] = d[j] + (double)f[j];                 // F2F.F64.F32 + DADD
            if (OP == 4) f[j] = fmaf(f[j], 1.0000001f, 1e-9f);
        }
        if (OP == 1) for (int j = 0; j < 8; j++) f[j] += 1.0f;
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < 8; j++) s += d[j] + f[j];
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double *out; float *outf; long long *cyc, h[1024];
    cudaMalloc(&out, 1 << 24); cudaMalloc(&outf, 1 << 24); cudaMalloc(&cyc, 8192);
    const int iters = 1000;
    const char *names[] = {"DFMA", "F2F64+DMUL+F2F32", "SHFL", "VOTE+IADD", "FFMA", "F2F64+DADD"};
    void (*lk[])(double *, float *, int, long long *) = {lat_kernel<0>, lat_kernel<1>, lat_kernel<2>, lat_kernel<3>, lat_kernel<4>, lat_kernel<5>};
    for (int op = 0; op < 6; op++) {
        lk[op]<<<1, 32>>>(out, outf, 10, cyc);
        lk[op]<<<1, 32>>>(out, outf, iters, cyc);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("latency %-20s %.1f cyc per op\n", names[op], (double)h[0] / (iters * 16));
    }
    void (*tk[])(double *, int, long long *) = {tput_kernel<0>, tput_kernel<1>, tput_kernel<4>};
    const char *tn[] = {"DFMA", "F2F64+DADD", "FFMA"};
    for (int o = 0; o < 3; o++)
        for (int warps = 4; warps <= 32; warps *= 2) {
            tk[o]<<<1, warps * 32>>>(out, 10, cyc);
            tk[o]<<<1, warps * 32>>>(out, iters, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)iters * 8 * warps;   // warp-instructions (of the main op)
            printf("throughput %-12s %2d warps: %.2f warp-ops per cycle per SM\n", tn[o], warps, ops / h[0]);
        }
    return 0;
}
