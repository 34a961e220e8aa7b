// k_das.cu -- S1 steering tables and S2 DAS map kernels (sm_100a).
//
// S1 (Eq. 3-4, 7; reading R1): the normalised steering vector
//   e_ms = sqrt(M) * exp(-j k d_ms) / (d_ms * ||g_s||),  ||g_s||^2 = sum_m 1/d_ms^2,
// split into a frequency-independent amplitude table amp[m][s] = sqrt(M)/(d_ms ||g_s||)
// and distance table dist[m][s] (both fp64, s fastest -> coalesced), computed once per
// call, and the per-bin phase k*d_ms evaluated with fp64 sincos inside the consumers.
//
// S2 (Eq. 2): b_s = Re(e_s^H C e_s) / M^2 in fp64, never forming E^H C E.
// Hermitian form (reading R3): b = sum_m C_mm |e_m|^2 + 2 Re sum_{m<n} conj(e_m) C_mn e_n,
// half the flops of the full quadratic form.  One CTA = P scan points x TSUB threads per
// point (256 threads); the P steering columns live in shared memory ([m][p], conflict-free);
// each thread holds an 8-column chunk of e_n in registers and streams rows m of C through
// L1 as warp-uniform broadcast loads.  fp64 CUDA-core bound (B200 has no faster fp64 path).
#include <math.h>

#include "dwc_internal.cuh"

namespace dwc {

__global__ void geom_tables_kernel(Geo g, double *__restrict__ dist, double *__restrict__ amp,
                                   int *__restrict__ flag) {
    const double sqm = sqrt((double)g.m);
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < g.S; s += gridDim.x * blockDim.x) {
        const int r = s / g.n, c = s - (s / g.n) * g.n;
        const double px = node_x(g, c), py = node_y(g, r), pz = g.z0;
        double inv2 = 0.0;
        bool sing = false;
        for (int m = 0; m < g.m; m++) {
            const double dx = px - g.mic[3 * m], dy = py - g.mic[3 * m + 1], dz = pz - g.mic[3 * m + 2];
            const double d = sqrt(dx * dx + dy * dy + dz * dz);
            sing |= !(d > 0.0);
            dist[(size_t)m * g.S + s] = d;
            inv2 += 1.0 / (d * d);
        }
        const double nrm = sqrt(inv2);
        for (int m = 0; m < g.m; m++) {
            const double d = dist[(size_t)m * g.S + s];
            amp[(size_t)m * g.S + s] = sqm / (d * nrm);
        }
        if (sing) atomicOr(flag, 4);
    }
}

int launch_geom_tables(const Geo &g, double *dist, double *amp, int *flag, cudaStream_t st) {
    const int threads = 256;
    int blocks = (g.S + threads - 1) / threads;
    geom_tables_kernel<<<blocks, threads, 0, st>>>(g, dist, amp, flag);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

__device__ __forceinline__ double2 steer_elem(double d, double a, double k) {
    double sn, cs;
    sincos(k * d, &sn, &cs);
    return make_double2(a * cs, -(a * sn));
}

__global__ void steer_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
                             const double *__restrict__ freq, int n_pts,
                             const int32_t *__restrict__ idx, double2 *__restrict__ E) {
    const double k = kTwoPi * freq[0] / g.c0;
    const int total = n_pts * g.m;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int pt = t / g.m, m = t - (t / g.m) * g.m;
        const int s = idx[pt];
        E[t] = steer_elem(dist[(size_t)m * g.S + s], amp[(size_t)m * g.S + s], k);
    }
}

int launch_steer(const Geo &g, const double *dist, const double *amp, const double *freq,
                 int n_pts, const int32_t *idx, double *E, cudaStream_t st) {
    if (n_pts <= 0) return 0;
    const int threads = 256;
    long total = (long)n_pts * g.m;
    int blocks = (int)((total + threads - 1) / threads);
    steer_kernel<<<blocks, threads, 0, st>>>(g, dist, amp, freq, n_pts, idx, (double2 *)E);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// ------------------------------------------------------------------------------------
constexpr int kDasThreads = 256;
constexpr int kNch = 8;  // n-chunk held in registers

__device__ __forceinline__ void cmac(double2 &acc, double2 a, double2 b) {  // acc += a*b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cjmac(double2 &acc, double2 a, double2 b) {  // acc += conj(a)*b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

// One chunk c of 8 columns: returns 2*Re(sum_{m<n, n in chunk} conj(e_m) C_mn e_n)
// + sum_{n in chunk} C_nn |e_n|^2 for the thread's point.
__device__ __forceinline__ double das_chunk(const double2 *__restrict__ C, int M, int c,
                                            const double2 *__restrict__ Es, int P, int p) {
    const int n0 = c * kNch;
    double2 en[kNch];
#pragma unroll
    for (int j = 0; j < kNch; j++) en[j] = (n0 + j < M) ? Es[(n0 + j) * P + p] : make_double2(0.0, 0.0);
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    const bool full = (n0 + kNch <= M);
    // rows strictly above the chunk
#pragma unroll 2
    for (int m = 0; m < n0; m++) {
        const double2 em = Es[m * P + p];
        const double2 *row = C + (size_t)m * M + n0;
        double2 t0 = make_double2(0.0, 0.0), t1 = make_double2(0.0, 0.0);
        if (full) {
#pragma unroll
            for (int j = 0; j < kNch; j += 2) {
                cmac(t0, __ldg(row + j), en[j]);
                cmac(t1, __ldg(row + j + 1), en[j + 1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kNch; j++)
                if (n0 + j < M) cmac(t0, __ldg(row + j), en[j]);
        }
        t0.x += t1.x;
        t0.y += t1.y;
        if (m & 1) cjmac(acc1, em, t0); else cjmac(acc0, em, t0);
    }
    // pairs inside the chunk (a < b) and the diagonal
    double diag = 0.0;
#pragma unroll
    for (int a = 0; a < kNch; a++) {
        if (n0 + a < M) {
            const double2 *row = C + (size_t)(n0 + a) * M + n0;
            const double2 caa = __ldg(row + a);
            diag = fma(caa.x, en[a].x * en[a].x + en[a].y * en[a].y, diag);
            double2 t = make_double2(0.0, 0.0);
#pragma unroll
            for (int b = a + 1; b < kNch; b++)
                if (n0 + b < M) cmac(t, __ldg(row + b), en[b]);
            cjmac(acc0, en[a], t);
        }
    }
    return 2.0 * (acc0.x + acc1.x) + diag;
}

__global__ void __launch_bounds__(kDasThreads)
das_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
           const double *__restrict__ freq, const double2 *__restrict__ csm,
           double *__restrict__ b, int P) {
    extern __shared__ double2 Es[];  // [M][P]
    __shared__ double part[kDasThreads];
    const int M = g.m;
    const int bin = blockIdx.y;
    const int s0 = blockIdx.x * P;
    const double k = kTwoPi * freq[bin] / g.c0;
    for (int t = threadIdx.x; t < M * P; t += kDasThreads) {
        const int m = t / P, p = t - (t / P) * P;
        const int s = s0 + p;
        double2 e = make_double2(0.0, 0.0);
        if (s < g.S) e = steer_elem(dist[(size_t)m * g.S + s], amp[(size_t)m * g.S + s], k);
        Es[t] = e;
    }
    __syncthreads();
    const int p = threadIdx.x % P, sub = threadIdx.x / P, tsub = kDasThreads / P;
    const double2 *C = csm + (size_t)bin * M * M;
    const int NC = (M + kNch - 1) / kNch;
    double acc = 0.0;
    for (int q = sub; q < (NC + 1) / 2; q += tsub) {
        acc += das_chunk(C, M, q, Es, P, p);
        if (NC - 1 - q != q) acc += das_chunk(C, M, NC - 1 - q, Es, P, p);
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (sub == 0 && s0 + p < g.S) {
        double v = part[p];
        for (int j = 1; j < tsub; j++) v += part[j * P + p];
        b[(size_t)bin * g.S + s0 + p] = v / ((double)M * (double)M);
    }
}

// Hermitian part H = (C + C^H)/2 of every bin's CSM (reading R3).  For an exactly
// Hermitian input this is the identity bit for bit.
__global__ void hermitize_kernel(int M, long total, const double2 *__restrict__ C,
                                 double2 *__restrict__ H) {
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
        const long bin = t / ((long)M * M);
        const int r = (int)(t - bin * M * M);
        const int i = r / M, j = r - (r / M) * M;
        const double2 a = C[t];
        const double2 b = C[bin * M * M + (long)j * M + i];
        H[t] = make_double2((a.x + b.x) * 0.5, (a.y - b.y) * 0.5);
    }
}

int launch_hermitize(int M, int n_bins, const double *csm, double *H, cudaStream_t st) {
    long total = (long)n_bins * M * M;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    hermitize_kernel<<<blocks, 256, 0, st>>>(M, total, (const double2 *)csm, (double2 *)H);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int das_points_per_cta(int M) {
    int P = 128;
    while (P > 16 && P * M > 4096) P >>= 1;
    return P;
}

int launch_das(const Geo &g, const double *dist, const double *amp, int n_bins,
               const double *freq, const double *csm, double *b, cudaStream_t st) {
    const int P = das_points_per_cta(g.m);
    const size_t smem = (size_t)16 * g.m * P;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(das_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    dim3 grid((g.S + P - 1) / P, n_bins);
    das_kernel<<<grid, kDasThreads, smem, st>>>(g, dist, amp, freq, (const double2 *)csm, b, P);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
