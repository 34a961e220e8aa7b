// k_psf.cu -- S5 PSF matrix on the compressed grid (+ S6 restriction of b).
//
// Eq. 9-12 restricted by Eq. 23, reading R1:
//   A~_ij = |e_i^H e_j|^2 / M^2  over the kept nodes i, j.
// Real-GEMM decomposition of the complex Gram G = E~^H E~ with X = Re E~, Y = Im E~:
//   Re G = X^T X + Y^T Y,   Im G = X^T Y - Y^T X,   A = (Re G^2 + Im G^2) / M^2.
// G is Hermitian, so A is symmetric: only tile pairs I <= J are computed and mirrored.
//
// steer_kept_kernel: kept steering planes in fp32 (phases from fp64 k*d and fp64 sincos,
// rounded once), and b~ = b[keep] (S6).
// gram_kernel (v1): SIMT fp32 tiles 64x64, K = m in chunks of 16 staged in shared memory.
#include <math.h>

#include "dwc_internal.cuh"

namespace dwc {

__global__ void steer_kept_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
                                  const double *__restrict__ freq, const BinLayout *__restrict__ lay,
                                  const int32_t *__restrict__ keep_idx, const double *__restrict__ b,
                                  float *__restrict__ xplanes, float *__restrict__ bt) {
    const int bin = blockIdx.y;
    const BinLayout L = lay[bin];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L.sp) return;
    const int M = g.m;
    float *X = xplanes + L.v_off * 2 * M;
    if (i < L.nk) {
        const int s = keep_idx[(size_t)bin * g.S + i];
        const double k = kTwoPi * freq[bin] / g.c0;
        for (int m = 0; m < M; m++) {
            const double d = dist[(size_t)m * g.S + s], a = amp[(size_t)m * g.S + s];
            double sn, cs;
            sincos(k * d, &sn, &cs);
            X[(size_t)m * L.sp + i] = (float)(a * cs);
            X[(size_t)(M + m) * L.sp + i] = (float)(-(a * sn));
        }
        if (b) bt[L.v_off + i] = (float)b[(size_t)bin * g.S + s];
    } else {
        for (int m = 0; m < 2 * M; m++) X[(size_t)m * L.sp + i] = 0.f;
        if (b) bt[L.v_off + i] = 0.f;
    }
}

int launch_steer_kept(const Geo &g, const double *dist, const double *amp, int n_bins,
                      const double *freq, const BinLayout *lay, const int32_t *keep_idx,
                      const double *b, float *xplanes, float *bt, int max_sp, cudaStream_t st) {
    dim3 grid((max_sp + 127) / 128, n_bins);
    steer_kept_kernel<<<grid, 128, 0, st>>>(g, dist, amp, freq, lay, keep_idx, b, xplanes, bt);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------------------------
constexpr int kGT = 64;   // output tile
constexpr int kGK = 16;   // K chunk

__global__ void __launch_bounds__(256)
gram_kernel(int M, const int4 *__restrict__ tiles, const BinLayout *__restrict__ lay,
            const float *__restrict__ xplanes, float *__restrict__ A) {
    __shared__ float sXi[kGK][kGT], sYi[kGK][kGT], sXj[kGK][kGT], sYj[kGK][kGT];
    const int4 t = tiles[blockIdx.x];  // (bin, I, J, -)
    const BinLayout L = lay[t.x];
    const int i0 = t.y * kGT, j0 = t.z * kGT;
    const float *X = xplanes + L.v_off * 2 * M;
    const float *Y = X + (size_t)M * L.sp;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
    float re[4][4], im[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) re[a][c] = im[a][c] = 0.f;
    for (int m0 = 0; m0 < M; m0 += kGK) {
        for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
            const int kk = e / kGT, col = e % kGT;
            const int m = m0 + kk;
            const bool okm = m < M;
            const int ci = i0 + col, cj = j0 + col;
            sXi[kk][col] = (okm && ci < L.sp) ? X[(size_t)m * L.sp + ci] : 0.f;
            sYi[kk][col] = (okm && ci < L.sp) ? Y[(size_t)m * L.sp + ci] : 0.f;
            sXj[kk][col] = (okm && cj < L.sp) ? X[(size_t)m * L.sp + cj] : 0.f;
            sYj[kk][col] = (okm && cj < L.sp) ? Y[(size_t)m * L.sp + cj] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; kk++) {
            float xi[4], yi[4], xj[4], yj[4];
#pragma unroll
            for (int a = 0; a < 4; a++) {
                xi[a] = sXi[kk][ty * 4 + a];
                yi[a] = sYi[kk][ty * 4 + a];
                xj[a] = sXj[kk][tx * 4 + a];
                yj[a] = sYj[kk][tx * 4 + a];
            }
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    re[a][c] = fmaf(xi[a], xj[c], re[a][c]);
                    re[a][c] = fmaf(yi[a], yj[c], re[a][c]);
                    im[a][c] = fmaf(xi[a], yj[c], im[a][c]);
                    im[a][c] = fmaf(-yi[a], xj[c], im[a][c]);
                }
        }
        __syncthreads();
    }
    const float inv_m2 = 1.0f / ((float)M * (float)M);
    float *Ab = A + L.a_off;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int i = i0 + ty * 4 + a, j = j0 + tx * 4 + c;
            if (i < L.sp && j < L.sp) {
                const float v = (re[a][c] * re[a][c] + im[a][c] * im[a][c]) * inv_m2;
                Ab[(size_t)i * L.sp + j] = v;
                if (t.y != t.z) Ab[(size_t)j * L.sp + i] = v;
            }
        }
}

int launch_gram(int m, int n_tiles, const int4 *tiles, const BinLayout *lay_dev,
                const float *xplanes, float *A, cudaStream_t st) {
    if (n_tiles <= 0) return 0;
    gram_kernel<<<n_tiles, 256, 0, st>>>(m, tiles, lay_dev, xplanes, A);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
