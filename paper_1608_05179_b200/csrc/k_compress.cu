// k_compress.cu -- S3/S4: wavelet detail, threshold and order-preserving compaction.
//
// Algorithm 1, Eq. 15 (:189-194), Eq. 20-22 (:219-233); readings R5-R10.
// Alg. 1 predicts every level from the values of b itself (reading R8), so the levels are
// independent and the whole transform is ONE pass over the grid: node (r,c) belongs to
// level l = J - min(v2(r), v2(c), J) (v2 = 2-adic valuation, v2(0) = inf); its detail is
// b - interp(b on G^(l-1)) with the linear stencil of reading R7 (interior midpoint, right
// edge linear extrapolation, else constant) or the 4-point cubic stencil of reading R19
// (DWC_CUBIC; Lagrange through the 4 nearest coarse nodes, linear fallback).  All arithmetic is fp64 with explicit
// round-to-nearest intrinsics (no FMA contraction) in exactly the order of the oracle's
// definition, so the same b gives the same keep set bit for bit.
//
// One CTA (1024 threads) per bin: block max|b| -> eps_eff -> 1024-node tiles in ascending
// order, ballot + warp-prefix + block scan -> ascending keep list (reading R9).  HBM-bound:
// b is read twice (max, then detail taps that hit L1/L2), keep list written once.
#include <math.h>

#include "dwc_internal.cuh"

namespace dwc {

constexpr int kCmpThreads = 1024;

__device__ __forceinline__ int max_level_of(int n) {
    int J = 0;
    while ((2 << J) <= n) J++;
    return J;
}

// 1-D taps at fine stride h (reading R7).
__device__ __forceinline__ int taps1d(int i, int h, int n, int *pos, double *w) {
    const int H = 2 * h;
    if (i % H == 0) { pos[0] = i; w[0] = 1.0; return 1; }
    if (i + h <= n - 1) { pos[0] = i - h; w[0] = 0.5; pos[1] = i + h; w[1] = 0.5; return 2; }
    if (i - 3 * h >= 0) { pos[0] = i - h; w[0] = 1.5; pos[1] = i - 3 * h; w[1] = -0.5; return 2; }
    pos[0] = i - h; w[0] = 1.0;
    return 1;
}

// 1-D taps of the 4-point predictor (reading R19), ascending positions; weights k/16 exact.
__device__ __forceinline__ int taps1d_cubic(int i, int h, int n, int *pos, double *w) {
    const int H = 2 * h;
    if (i % H == 0) { pos[0] = i; w[0] = 1.0; return 1; }
    int o0, o1, o2, o3;
    double w0, w1, w2, w3;
    if (i - 3 * h >= 0 && i + 3 * h <= n - 1) {
        o0 = -3; o1 = -1; o2 = 1; o3 = 3; w0 = -1.0; w1 = 9.0; w2 = 9.0; w3 = -1.0;
    } else if (i - 3 * h < 0 && i + 5 * h <= n - 1) {
        o0 = -1; o1 = 1; o2 = 3; o3 = 5; w0 = 5.0; w1 = 15.0; w2 = -5.0; w3 = 1.0;
    } else if (i + h <= n - 1 && i + 3 * h > n - 1 && i - 5 * h >= 0) {
        o0 = -5; o1 = -3; o2 = -1; o3 = 1; w0 = 1.0; w1 = -5.0; w2 = 15.0; w3 = 5.0;
    } else if (i + h > n - 1 && i - 7 * h >= 0) {
        o0 = -7; o1 = -5; o2 = -3; o3 = -1; w0 = -5.0; w1 = 21.0; w2 = -35.0; w3 = 35.0;
    } else {
        return taps1d(i, h, n, pos, w);
    }
    pos[0] = i + o0 * h; pos[1] = i + o1 * h; pos[2] = i + o2 * h; pos[3] = i + o3 * h;
    w[0] = w0 / 16.0; w[1] = w1 / 16.0; w[2] = w2 / 16.0; w[3] = w3 / 16.0;
    return 4;
}

__device__ __forceinline__ int level_of(int r, int c, int J) {
    const int vr = r == 0 ? J : min(__ffs(r) - 1, J);
    const int vc = c == 0 ? J : min(__ffs(c) - 1, J);
    return J - min(vr, vc);
}

// detail d = b - pred at a level >= 1 node; t_a = sum_q w_q * b[r_a][c_q], pred = sum_a w_a t_a,
// both sums left to right, every product and sum rounded (the oracle's order)
template <int kOrder>
__device__ __forceinline__ double detail_at(const double *__restrict__ b, int n, int r, int c,
                                            int lev, int J) {
    const int h = 1 << (J - lev);
    int rp[4], cp[4];
    double rw[4], cw[4];
    const int nr = kOrder == 3 ? taps1d_cubic(r, h, n, rp, rw) : taps1d(r, h, n, rp, rw);
    const int nc = kOrder == 3 ? taps1d_cubic(c, h, n, cp, cw) : taps1d(c, h, n, cp, cw);
    double pred = 0.0;
    for (int a = 0; a < nr; a++) {
        double t = __dmul_rn(cw[0], b[(size_t)rp[a] * n + cp[0]]);
        for (int q = 1; q < nc; q++) t = __dadd_rn(t, __dmul_rn(cw[q], b[(size_t)rp[a] * n + cp[q]]));
        const double v = __dmul_rn(rw[a], t);
        pred = (a == 0) ? v : __dadd_rn(pred, v);
    }
    return __dsub_rn(b[(size_t)r * n + c], pred);
}

template <int kOrder>
__global__ void __launch_bounds__(kCmpThreads)
compress_kernel(int n, const double *__restrict__ bmaps, double eps, int eps_mode, int full_grid,
                int32_t *__restrict__ n_keep, int32_t *__restrict__ keep_idx,
                uint8_t *__restrict__ level, int *__restrict__ flag) {
    __shared__ double red[32];
    __shared__ int wcount[32];
    __shared__ int woff[32];
    __shared__ int total_s;
    const int S = n * n;
    const int bin = blockIdx.x;
    const double *b = bmaps + (size_t)bin * S;
    int32_t *keep = keep_idx + (size_t)bin * S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // max |b| (exact in any order)
    double mx = 0.0;
    bool bad = false;
    for (int s = tid; s < S; s += kCmpThreads) {
        const double a = fabs(b[s]);
        bad |= !isfinite(a);
        mx = fmax(mx, a);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    if (__syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
    if (warp == 0) {
        double v = red[lane];
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    const double maxabs = red[0];
    const double eps_eff = (eps_mode == 0) ? __dmul_rn(eps, maxabs) : eps;
    const bool degenerate = (eps_mode == 0 && maxabs == 0.0);
    const int J = max_level_of(n);

    int running = 0;
    for (int base = 0; base < S; base += kCmpThreads) {
        const int s = base + tid;
        bool kp = false;
        if (s < S) {
            const int r = s / n, c = s - (s / n) * n;
            const int lev = level_of(r, c, J);
            if (level) level[(size_t)bin * S + s] = (uint8_t)lev;
            if (full_grid || lev == 0) kp = true;
            else if (!degenerate) kp = fabs(detail_at<kOrder>(b, n, r, c, lev, J)) >= eps_eff;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, kp);
        if (lane == 0) wcount[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            const int v = wcount[lane];
            int incl = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            woff[lane] = incl - v;
            if (lane == 31) total_s = incl;
        }
        __syncthreads();
        if (kp) keep[running + woff[warp] + __popc(bal & ((1u << lane) - 1u))] = s;
        running += total_s;
        __syncthreads();
    }
    for (int s = running + tid; s < S; s += kCmpThreads) keep[s] = -1;
    if (tid == 0) n_keep[bin] = running;
}

int launch_compress(int n, int n_bins, const double *b, double eps, int eps_mode, int full_grid,
                    int order, int32_t *n_keep, int32_t *keep_idx, uint8_t *level, int *flag,
                    cudaStream_t st) {
    if (order == 3)
        compress_kernel<3><<<n_bins, kCmpThreads, 0, st>>>(n, b, eps, eps_mode, full_grid, n_keep, keep_idx, level,
                                                            flag);
    else
        compress_kernel<1><<<n_bins, kCmpThreads, 0, st>>>(n, b, eps, eps_mode, full_grid, n_keep, keep_idx, level,
                                                            flag);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
