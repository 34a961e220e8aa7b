// Residual-GS solver chain micro-benchmark: one warp runs the row-to-row recurrence of
// rgs_kernel's solver loop (ballot -> lowest lane -> broadcast dv + diagonal-tile load -> FMA ->
// projected update -> compare) on synthetic data; optional background warps load shared memory
// and do F2F + DFMA like the stream warps.  Prints cycles per change.
#include <cstdio>
#include <cuda_runtime.h>

template <int BG, int NPV = 7>
__global__ void chain(int iters, float *out, unsigned long long *cyc, int skip0) {
    __shared__ float diag[32 * 32];
    __shared__ float panel[8][224];
    __shared__ float4 ring[8][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) diag[i] = 1e-3f * (i % 7);
    for (int i = threadIdx.x; i < 8 * 224; i += blockDim.x) (&panel[0][0])[i] = 1e-4f * (i % 5);
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&ring[0][0])[i] = make_float4(1, 2, 3, 4);
    __syncthreads();
    if (wid == 0) {
        float xo = 1.0f + lane, w = 0.5f, invd = 0.9f, acc[7] = {0, 0, 0, 0, 0, 0, 0}, pvp[7] = {0, 0, 0, 0, 0, 0, 0}, dvp = 0.f;
        int pos_r = 0;
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            const float xn = xo + fmaxf(w, -xo);
            const float dl = xn - xo;
            const unsigned m = __ballot_sync(0xffffffffu, lane >= pos_r && xn != xo);
            const int t = __ffs(m) - 1;
#pragma unroll
            for (int d = 0; d < NPV; d++) acc[d] = fmaf(pvp[d], dvp, acc[d]);
            if (m == 0u) { pos_r = 0; continue; }
            const float dv = __shfl_sync(0xffffffffu, dl, t);
            const float a0 = diag[32 * t + lane];
            if (lane == t) xo = xn;
            w = fmaf(-invd * dv, a0, w) + 1e-3f;   // keeps every row changing
            const float *pr = panel[t & 7] + lane;
            dvp = dv;
#pragma unroll
            for (int d = 0; d < NPV; d++) pvp[d] = pr[32 * d];
            pos_r = (t + 1) & 31;
        }
        const unsigned long long t1 = clock64();
        if (lane == 0) cyc[0] = t1 - t0;
        float sacc = 0;
        for (int d = 0; d < 7; d++) sacc += acc[d];
        out[lane] = xo + w + sacc;
    } else if (BG && !(skip0 && (wid & 3) == 0)) {
        // background: stream-like fp64 updates from shared memory (BG 1), shared loads only (BG 2),
        // F2F + DFMA on registers only (BG 3), nn bit-placement widening from shared memory (BG 4)
        double r[8];
        for (int e = 0; e < 8; e++) r[e] = 0.0;
        float4 q0 = make_float4(lane, 1, 2, 3), q1 = q0;
        for (int it = 0; it < iters / 2; it++) {
            const double dx = 1e-7 * (it & 3);
#pragma unroll 4
            for (int j = 0; j < 4; j++) {
                float4 v0, v1;
                if (BG == 3) { v0 = q0; v1 = q1; q0.x += 1.f; q1.y += 1.f; }
                else { v0 = ring[j][lane]; v1 = ring[j + 4][(lane + 32) & 255]; }
                if (BG == 2) {
                    r[0] += v0.x + v1.x; r[1] += v0.y + v1.y; r[2] += v0.z + v1.z; r[3] += v0.w + v1.w;
                } else if (BG == 4) {
                    auto nn = [](float f) { const unsigned u = __float_as_uint(f); return __hiloint2double((int)(u >> 3), (int)(u << 29)); };
                    r[0] = fma(nn(v0.x), dx, r[0]); r[1] = fma(nn(v0.y), dx, r[1]);
                    r[2] = fma(nn(v0.z), dx, r[2]); r[3] = fma(nn(v0.w), dx, r[3]);
                    r[4] = fma(nn(v1.x), dx, r[4]); r[5] = fma(nn(v1.y), dx, r[5]);
                    r[6] = fma(nn(v1.z), dx, r[6]); r[7] = fma(nn(v1.w), dx, r[7]);
                } else {
                    r[0] = fma((double)v0.x, dx, r[0]); r[1] = fma((double)v0.y, dx, r[1]);
                    r[2] = fma((double)v0.z, dx, r[2]); r[3] = fma((double)v0.w, dx, r[3]);
                    r[4] = fma((double)v1.x, dx, r[4]); r[5] = fma((double)v1.y, dx, r[5]);
                    r[6] = fma((double)v1.z, dx, r[6]); r[7] = fma((double)v1.w, dx, r[7]);
                }
            }
        }
        double s = 0;
        for (int e = 0; e < 8; e++) s += r[e];
        out[32 * wid + lane] = (float)s;
    }
}

int main() {
    float *out;
    unsigned long long *cyc, h;
    cudaMalloc(&out, 4096 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 100000;
    for (int mode = 0; mode <= 3; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            switch (mode) {
                case 0: chain<0, 7><<<1, 32>>>(iters, out, cyc, 0); break;
                case 1: chain<0, 1><<<1, 32>>>(iters, out, cyc, 0); break;
                case 2: chain<1, 7><<<1, 32 * 6>>>(iters, out, cyc, 0); break;
                case 3: chain<1, 1><<<1, 32 * 6>>>(iters, out, cyc, 0); break;
            }
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("mode %d (0: alone 7 panel loads, 1: alone 1 load, 2: 5 stream warps 7 loads, 3: 5 stream warps 1 load): %.1f cycles per change\n", mode, (double)h / iters);
    }
    return 0;
}
