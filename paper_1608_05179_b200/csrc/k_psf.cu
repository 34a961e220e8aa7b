// k_psf.cu -- S5 PSF matrix on the compressed grid (+ S6 restriction of b).
//
// Eq. 9-12 restricted by Eq. 23, reading R1:
//   A~_ij = |e_i^H e_j|^2 / M^2  over the kept nodes i, j.
// Real-GEMM decomposition of the complex Gram G = E~^H E~ with X = Re E~, Y = Im E~:
//   Re G = X^T X + Y^T Y,   Im G = X^T Y - Y^T X,   A = (Re G^2 + Im G^2) / M^2.
// G is Hermitian, so A is symmetric: only tile pairs I <= J are computed and mirrored.
//
// steer_kept_kernel: kept steering planes (fp64 phases and sincos), and b~ = b[keep] (S6,
// kept in fp64: rounding b~ to fp32 perturbs the system the sweeps converge to).
// gram_kernel: fp64 accumulation, 64x64 tiles, K = m in chunks of 16 staged in shared
// memory; the |G|^2/M^2 epilogue rounds once to fp32 and stores the tiled layout the GS
// kernel streams (dwc_internal.cuh tiled_index).  Measured on the configs, an fp32
// accumulated Gram leaves |A - A_oracle| ~ 2e-7 (rel. L2), which GS amplifies ~10^3-10^4x
// in ill-conditioned low-frequency bins (map error > 1e-3); fp64 accumulation gives the
// correctly rounded fp32 A (~1e-8).  Only I <= J tiles are computed and entries with
// j >= i are written together with their mirror, so A is exactly symmetric.
#include <math.h>

#include "dwc_internal.cuh"

namespace dwc {

__global__ void steer_kept_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
                                  const double *__restrict__ freq, const BinLayout *__restrict__ lay,
                                  const int32_t *__restrict__ keep_idx, const double *__restrict__ b,
                                  double *__restrict__ xplanes, double *__restrict__ bt) {
    const int bin = blockIdx.y;
    const BinLayout L = lay[bin];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L.sp) return;
    const int M = g.m;
    double *X = xplanes + L.v_off * 2 * M;
    if (i < L.nk) {
        const int s = keep_idx[(size_t)bin * g.S + i];
        const double k = kTwoPi * freq[bin] / g.c0;
        for (int m = 0; m < M; m++) {
            const double d = dist[(size_t)m * g.S + s], a = amp[(size_t)m * g.S + s];
            double sn, cs;
            sincos(k * d, &sn, &cs);
            X[(size_t)m * L.sp + i] = a * cs;
            X[(size_t)(M + m) * L.sp + i] = -(a * sn);
        }
        if (b) bt[L.v_off + i] = b[(size_t)bin * g.S + s];
    } else {
        for (int m = 0; m < 2 * M; m++) X[(size_t)m * L.sp + i] = 0.0;
        if (b) bt[L.v_off + i] = 0.0;
    }
}

int launch_steer_kept(const Geo &g, const double *dist, const double *amp, int n_bins,
                      const double *freq, const BinLayout *lay, const int32_t *keep_idx,
                      const double *b, double *xplanes, double *bt, int max_sp, cudaStream_t st) {
    dim3 grid((max_sp + 127) / 128, n_bins);
    steer_kept_kernel<<<grid, 128, 0, st>>>(g, dist, amp, freq, lay, keep_idx, b, xplanes, bt);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------------------------
constexpr int kGT = 64;   // output tile
constexpr int kGK = 16;   // K chunk

__global__ void __launch_bounds__(256)
gram_kernel(int M, const int4 *__restrict__ tiles, const BinLayout *__restrict__ lay,
            const double *__restrict__ xplanes, float *__restrict__ A) {
    __shared__ double sXi[kGK][kGT], sYi[kGK][kGT], sXj[kGK][kGT], sYj[kGK][kGT];
    const int4 t = tiles[blockIdx.x];  // (bin, I, J, -)
    const BinLayout L = lay[t.x];
    const int i0 = t.y * kGT, j0 = t.z * kGT;
    const double *X = xplanes + L.v_off * 2 * M;
    const double *Y = X + (size_t)M * L.sp;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
    double re[4][4], im[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) re[a][c] = im[a][c] = 0.0;
    for (int m0 = 0; m0 < M; m0 += kGK) {
        for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
            const int kk = e / kGT, col = e % kGT;
            const int m = m0 + kk;
            const bool okm = m < M;
            const int ci = i0 + col, cj = j0 + col;
            sXi[kk][col] = (okm && ci < L.sp) ? X[(size_t)m * L.sp + ci] : 0.0;
            sYi[kk][col] = (okm && ci < L.sp) ? Y[(size_t)m * L.sp + ci] : 0.0;
            sXj[kk][col] = (okm && cj < L.sp) ? X[(size_t)m * L.sp + cj] : 0.0;
            sYj[kk][col] = (okm && cj < L.sp) ? Y[(size_t)m * L.sp + cj] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; kk++) {
            double xi[4], yi[4], xj[4], yj[4];
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
                    re[a][c] = fma(xi[a], xj[c], re[a][c]);
                    re[a][c] = fma(yi[a], yj[c], re[a][c]);
                    im[a][c] = fma(xi[a], yj[c], im[a][c]);
                    im[a][c] = fma(-yi[a], xj[c], im[a][c]);
                }
        }
        __syncthreads();
    }
    const double m2 = (double)M * (double)M;
    float *Ab = A + L.a_off;
    const int T = L.sp >> 5;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int i = i0 + ty * 4 + a, j = j0 + tx * 4 + c;
            if (i < L.sp && j < L.sp && j >= i) {
                const float v = (float)((re[a][c] * re[a][c] + im[a][c] * im[a][c]) / m2);
                Ab[tiled_index(T, i, j)] = v;
                if (j != i) Ab[tiled_index(T, j, i)] = v;
            }
        }
}

int launch_gram(int m, int n_tiles, const int4 *tiles, const BinLayout *lay_dev,
                const double *xplanes, float *A, cudaStream_t st) {
    if (n_tiles <= 0) return 0;
    gram_kernel<<<n_tiles, 256, 0, st>>>(m, tiles, lay_dev, xplanes, A);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
