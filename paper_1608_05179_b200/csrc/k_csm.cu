// k_csm.cu -- the step before the path: the cross-spectral matrix of
// every bin from its snapshot spectra, Eq. 1,
//   C = (1/I) sum_i p_i p_i^H,   P = [p_1 .. p_I] in C^{M x I},
// in fp64 (the DAS map and the bit-exact threshold downstream need fp64 C).
//
// One CTA per 64 x 64 output tile of one bin: 256 threads, thread (ty, tx) accumulates the
// 4 x 4 outputs (ty + 16a, tx + 16b) in registers; the K dimension (snapshots) is staged 16 at a
// time through shared memory (row stride 17 complex: conflict-free column reads).  Output
// either the full C (stage entry point) or, for the path, directly the half-Hermitian padded
// Ch the DAS kernel consumes (upper triangle, halved real diagonal, zeros elsewhere).
#include "dwc_internal.cuh"

namespace dwc {

constexpr int kCsmT = 64;    // output tile
constexpr int kCsmK = 16;    // snapshots per stage
constexpr int kCsmLd = kCsmK + 1;

__global__ void __launch_bounds__(256)
csm_kernel(int M, int Mp, int I, const double2 *__restrict__ snap, double2 *__restrict__ out, int half, int dr) {
    __shared__ double2 As[kCsmT * kCsmLd], Bs[kCsmT * kCsmLd];
    const int bin = blockIdx.z, mt = blockIdx.y, nt = blockIdx.x;
    const int Mo = half ? Mp : M;   // output leading dimension
    if (mt * kCsmT >= Mo || nt * kCsmT >= Mo) return;
    const double2 *P = snap + (size_t)bin * M * I;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double2 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = make_double2(0.0, 0.0);
    const bool upper_only = half && nt < mt;   // Ch is zero below the diagonal tiles
    for (int i0 = 0; i0 < I && !upper_only; i0 += kCsmK) {
        // stage P rows of both tiles, snapshots i0..i0+15 (256 threads x 4 elements each)
        for (int e = threadIdx.x; e < kCsmT * kCsmK; e += 256) {
            const int r = e / kCsmK, k = e % kCsmK, i = i0 + k;
            const int ma = mt * kCsmT + r, nb = nt * kCsmT + r;
            As[r * kCsmLd + k] = (ma < M && i < I) ? P[(size_t)ma * I + i] : make_double2(0.0, 0.0);
            Bs[r * kCsmLd + k] = (nb < M && i < I) ? P[(size_t)nb * I + i] : make_double2(0.0, 0.0);
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < kCsmK; k++) {
            double2 av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) av[a] = As[(ty + 16 * a) * kCsmLd + k];
#pragma unroll
            for (int b = 0; b < 4; b++) bv[b] = Bs[(tx + 16 * b) * kCsmLd + k];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) {   // acc += p_m conj(p_n)
                    acc[a][b].x = fma(av[a].x, bv[b].x, acc[a][b].x);
                    acc[a][b].x = fma(av[a].y, bv[b].y, acc[a][b].x);
                    acc[a][b].y = fma(av[a].y, bv[b].x, acc[a][b].y);
                    acc[a][b].y = fma(-av[a].x, bv[b].y, acc[a][b].y);
                }
        }
        __syncthreads();
    }
    const double inv = 1.0 / (double)I;
    double2 *O = out + (size_t)bin * Mo * Mo;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int m = mt * kCsmT + ty + 16 * a, n = nt * kCsmT + tx + 16 * b;
            if (m >= Mo || n >= Mo) continue;
            double2 v = make_double2(acc[a][b].x * inv, acc[a][b].y * inv);
            if (half) {
                if (m >= M || n >= M || n < m) v = make_double2(0.0, 0.0);
                else if (n == m) v = dr ? make_double2(0.0, 0.0) : make_double2(v.x * 0.5, 0.0);
            }
            O[(size_t)m * Mo + n] = v;
        }
}

int launch_csm(int M, int n_bins, int I, const double *snap, double *out, int half, int dr, cudaStream_t st) {
    const int Mo = half ? das_mpad(M) : M;
    const int t = (Mo + kCsmT - 1) / kCsmT;
    dim3 grid(t, t, n_bins);
    csm_kernel<<<grid, 256, 0, st>>>(M, das_mpad(M), I, (const double2 *)snap, (double2 *)out, half, dr);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
