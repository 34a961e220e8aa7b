// k_das.cu -- S1 steering tables and S2 DAS map kernels (sm_100a).
//
// S1 (Eq. 3-4, 7; reading R1): the normalised steering vector
//   e_ms = sqrt(M) * exp(-j k d_ms) / (d_ms * ||g_s||),  ||g_s||^2 = sum_m 1/d_ms^2,
// split into a frequency-independent amplitude table amp[m][s] = sqrt(M)/(d_ms ||g_s||)
// and distance table dist[m][s] (both fp64, s fastest -> coalesced), computed once per
// call, and the per-bin phase k*d_ms evaluated with fp64 sincospi inside the consumers.
//
// S2 (Eq. 2): b_s = Re(e_s^H C e_s) / M^2 in fp64, never forming E^H C E
// (das_kernel below: triangular register-blocked GEMM on the half-Hermitian CSM).
#include <math.h>

#include "dwc_internal.cuh"

namespace dwc {

// Paper-literal amplitudes (NEXT-4, Eq. 4 and :130 Eq. 7, distances to the array
// centre = the origin): ampv[m][s] = d_ms / |r_s| (the focus vector v) and ampg[m][s] = |r_s| / d_ms
// (the propagation vector g); written when the pointers are not NULL.
__global__ void geom_tables_kernel(Geo g, double *__restrict__ dist, double *__restrict__ amp,
                                   int *__restrict__ flag, double *__restrict__ ampv, double *__restrict__ ampg) {
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
        const double rn = sqrt(px * px + py * py + pz * pz);
        for (int m = 0; m < g.m; m++) {
            const double d = dist[(size_t)m * g.S + s];
            amp[(size_t)m * g.S + s] = sqm / (d * nrm);
            if (ampv) {
                ampv[(size_t)m * g.S + s] = d / rn;
                ampg[(size_t)m * g.S + s] = rn / d;
            }
        }
        if (sing) atomicOr(flag, 4);
    }
}

int launch_geom_tables(const Geo &g, double *dist, double *amp, int *flag, cudaStream_t st, double *ampv,
                       double *ampg) {
    const int threads = 256;
    int blocks = (g.S + threads - 1) / threads;
    geom_tables_kernel<<<blocks, threads, 0, st>>>(g, dist, amp, flag, ampv, ampg);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// e = a exp(-j k d) with the phase in half-turns, kpi = k / pi = 2 f / c0: sincospi reduces
// its argument exactly (subtract the nearest integer) -- cheaper than sincos' Cody-Waite
// reduction, same ~1e-16 relative accuracy of e.
__device__ __forceinline__ double2 steer_elem(double d, double a, double kpi) {
    double sn, cs;
    sincospi(kpi * d, &sn, &cs);
    return make_double2(a * cs, -(a * sn));
}

__global__ void steer_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
                             const double *__restrict__ freq, int n_pts,
                             const int32_t *__restrict__ idx, double2 *__restrict__ E) {
    const double k = 2.0 * freq[0] / g.c0;   // half-turns per metre
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
// S2 as a register-blocked triangular complex GEMM.  With the half-Hermitian matrix
//   Ch[m][n] = H[m][n] (n > m),  H[m][m] / 2 (n = m),  0 (n < m),   H = (C + C^H)/2,
// b_s = 2 Re(e_s^H Ch e_s) / M^2 -- the Hermitian form at half the flops.  A CTA = P scan points
// of one bin, 2 points per lane (P = 64; 4 warps when Mp <= 64, else 8 warps; the 1-point-per-
// lane form, P = 32 with 8 warps, remains behind DAS_BIG=0); their steering vectors Es[n][p] (Mp x P complex,
// Mp = M rounded up to 8, zero rows beyond M) in shared memory.  Warp w owns the row-group
// pairs (q, G-1-q), q = w, w+NW, ... (G = Mp/4 groups of 4 rows), paired so every warp has the
// same triangular work, and reads those 8 rows of Ch through L1 (DAS_DIRECT_C).  Lane l
// owns points l (+32).  Per n a thread reads 8 row entries (broadcast loads) and e_n of its
// points and does 8 or 16 complex MACs; W = Ch e stays in registers; the epilogue reduces
// Re(conj(e_m) W_m) over the rows and the warps in fixed order (deterministic).  fp64 CUDA
// cores (B200 DFMA and DMMA peak are the same, ~36 TFLOP/s measured).
constexpr int kDasThreads = 256;
#ifndef DAS_UNROLL
#define DAS_UNROLL 8
#endif
constexpr int kDasUnroll = DAS_UNROLL;
constexpr int kDasWarps = kDasThreads / 32;

__device__ __forceinline__ void cmac(double2 &acc, double2 a, double2 b) {  // acc += a*b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

int das_mpad(int M) { return (M + 7) / 8 * 8; }

template <int PPL, bool kBoth, int P = 32 * PPL>
__device__ __forceinline__ void das_rows(const double2 *__restrict__ ca, const double2 *__restrict__ cb,
                                         const double2 *__restrict__ Es, int Mp,
                                         int n0, int n1, int lane, double2 Wa[4][PPL], double2 Wb[4][PPL]) {
#pragma unroll kDasUnroll
    for (int n = n0; n < n1; n++) {
        double2 e[PPL];
#pragma unroll
        for (int j = 0; j < PPL; j++) e[j] = Es[n * P + ((lane + 32 * j) & (P - 1))];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const double2 c = ca[r * Mp + n];
#pragma unroll
            for (int j = 0; j < PPL; j++) cmac(Wa[r][j], c, e[j]);
        }
        if (kBoth) {
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const double2 c = cb[r * Mp + n];
#pragma unroll
                for (int j = 0; j < PPL; j++) cmac(Wb[r][j], c, e[j]);
            }
        }
    }
}

// DAS_DIRECT_C (default): the 8 Ch rows a warp works on are read as warp-broadcast read-only
// global loads (L1-resident) instead of being staged in a per-warp shared-memory slice: 64 KB
// of shared memory per CTA instead of 96 -> three CTAs per SM (register-limited at 168), cfg3
// DAS stage 3.18 -> 2.94 ms with DAS_UNROLL 8 (4: 2.98, 2: 3.10).  Only for the 2-points-per-
// lane forms: with one point per lane the broadcast loads per DFMA double and the direct form
// was slower (cfg5 DAS 196 -> 215 ms), so that form keeps the staging.
#ifndef DAS_DIRECT_C
#define DAS_DIRECT_C 1
#endif
// P: points per CTA (32 PPL; P = 16 for the largest arrays: 16 Mp P bytes of steering vectors
// must fit in shared memory, and at Mp = 512 only P = 16 does -- lanes 16..31 then repeat lanes
// 0..15 and their results are dropped)
template <int PPL, int NW, int P = 32 * PPL>
__global__ void __launch_bounds__(32 * NW, (DAS_DIRECT_C && PPL == 2) ? (NW == 4 ? 3 : 1) : 2)
das_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
           const double *__restrict__ freq, const double2 *__restrict__ Ch, int Mp, double *__restrict__ b, int dr) {
    constexpr bool kDirect = DAS_DIRECT_C && (PPL == 2 || P < 32);
    extern __shared__ double2 smem_d2[];
    double2 *Es = smem_d2;                       // [Mp][P]
    double2 *Cw = smem_d2 + (size_t)Mp * P;      // [warp][8 rows][Mp]
    __shared__ double part[NW][P];
    const int M = g.m;
    const int bin = blockIdx.y;
    const int s0 = blockIdx.x * P;
    const double k = 2.0 * freq[bin] / g.c0;   // half-turns per metre
    // steering vectors of the CTA's points: the (dist, amp) table entries of 8 elements per
    // thread are loaded before any is used, so their latency is paid once per 8 (not per element)
    constexpr int kEU = 8;
    for (int base = 0; base < Mp * P; base += (32 * NW) * kEU) {
        double dd[kEU], aa[kEU];
#pragma unroll
        for (int u = 0; u < kEU; u++) {
            const int t = base + u * (32 * NW) + threadIdx.x;
            const int m = t / P, s = s0 + t % P;
            const bool ok = t < Mp * P && m < M && s < g.S;
            dd[u] = ok ? __ldg(dist + (size_t)m * g.S + s) : 0.0;
            aa[u] = ok ? __ldg(amp + (size_t)m * g.S + s) : -1.0;   // -1: padding element
        }
#pragma unroll
        for (int u = 0; u < kEU; u++) {
            const int t = base + u * (32 * NW) + threadIdx.x;
            if (t < Mp * P) Es[t] = (aa[u] >= 0.0) ? steer_elem(dd[u], aa[u], k) : make_double2(0.0, 0.0);
        }
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = Mp / 4;
    const double2 *C = Ch + (size_t)bin * Mp * Mp;
    double2 *cw = Cw + (size_t)w * 8 * Mp;
    double acc[PPL];
#pragma unroll
    for (int j = 0; j < PPL; j++) acc[j] = 0.0;
    for (int qa = w; qa < G / 2; qa += NW) {
        const int qb = G - 1 - qa;
        const double2 *ca = kDirect ? C + (size_t)(4 * qa) * Mp : cw;
        const double2 *cb = kDirect ? C + (size_t)(4 * qb) * Mp : cw + 4 * Mp;
        if constexpr (!kDirect) {
            __syncwarp();
            for (int t = lane; t < 8 * Mp; t += 32) {   // rows 4qa..4qa+3, 4qb..4qb+3 of Ch (cp.async:
                const int r = t / Mp, n = t - (t / Mp) * Mp;   // all 16-byte copies in flight at once)
                const int m = (r < 4) ? 4 * qa + r : 4 * qb + r - 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(cw + t)),
                             "l"(C + (size_t)m * Mp + n)
                             : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();
        }
        double2 Wa[4][PPL], Wb[4][PPL];
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int j = 0; j < PPL; j++) Wa[r][j] = Wb[r][j] = make_double2(0.0, 0.0);
        das_rows<PPL, false, P>(ca, cb, Es, Mp, 4 * qa, 4 * qb, lane, Wa, Wb);   // only rows of qa reach n < 4 qb
        das_rows<PPL, true, P>(ca, cb, Es, Mp, 4 * qb, Mp, lane, Wa, Wb);
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int j = 0; j < PPL; j++) {
                const int pj = (lane + 32 * j) & (P - 1);
                const double2 ea = Es[(4 * qa + r) * P + pj], eb = Es[(4 * qb + r) * P + pj];
                acc[j] += ea.x * Wa[r][j].x + ea.y * Wa[r][j].y + eb.x * Wb[r][j].x + eb.y * Wb[r][j].y;
            }
    }
#pragma unroll
    for (int j = 0; j < PPL; j++)
        if (lane + 32 * j < P) part[w][lane + 32 * j] = acc[j];
    __syncthreads();
    if (threadIdx.x < P && s0 + (int)threadIdx.x < g.S) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < NW; q++) v += part[q][threadIdx.x];
        if (dr) {   // R20: normalised by M^2 - M, negative values clamped (the diagonal is already gone)
            const double bv = 2.0 * v / ((double)M * (double)M - (double)M);
            b[(size_t)bin * g.S + s0 + threadIdx.x] = bv > 0.0 ? bv : 0.0;
        } else {
            b[(size_t)bin * g.S + s0 + threadIdx.x] = 2.0 * v / ((double)M * (double)M);
        }
    }
}

// Half-Hermitian, zero-padded CSM Ch (Mp x Mp per bin) from the input C (reading R3: only the
// Hermitian part H = (C + C^H)/2 enters Re(e^H C e)).
__global__ void hermitize_kernel(int M, int Mp, long total, const double2 *__restrict__ C,
                                 double2 *__restrict__ Ch, int dr) {
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
        const long bin = t / ((long)Mp * Mp);
        const int r = (int)(t - bin * Mp * Mp);
        const int i = r / Mp, j = r - (r / Mp) * Mp;
        double2 v = make_double2(0.0, 0.0);
        if (i < M && j < M && j >= i) {
            const double2 a = C[bin * M * M + (long)i * M + j];
            const double2 c = C[bin * M * M + (long)j * M + i];
            v = make_double2((a.x + c.x) * 0.5, (a.y - c.y) * 0.5);
            if (j == i) v = dr ? make_double2(0.0, 0.0) : make_double2(v.x * 0.5, 0.0);   // R20: no diagonal
        }
        Ch[t] = v;
    }
}

int launch_hermitize(int M, int n_bins, const double *csm, double *H, int dr, cudaStream_t st) {
    const int Mp = das_mpad(M);
    long total = (long)n_bins * Mp * Mp;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    hermitize_kernel<<<blocks, 256, 0, st>>>(M, Mp, total, (const double2 *)csm, (double2 *)H, dr);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_das(const Geo &g, const double *dist, const double *amp, int n_bins,
               const double *freq, const double *csm_half, double *b, int dr, cudaStream_t st) {
    const int Mp = das_mpad(g.m);
#ifndef DAS_P64
#define DAS_P64 1
#endif
    // 32 points x 8 warps; DAS_P64: 64 points
    // (2 per lane) x 4 warps, twice the DFMAs per loaded Ch entry
#ifndef DAS_BIG
#define DAS_BIG 1
#endif
    // DAS_BIG (M > 64): 64 points (2 per lane) x 8 warps, Ch through L1, one CTA per SM (128 KB
    // of steering vectors, 252 registers): cfg5 DAS 192 -> 170 ms, cfg4 3.15 -> 2.80 ms against
    // 32 points x 8 warps with the Ch rows staged
    // the largest arrays (Mp > 208): 16 points per CTA, Ch through L1 (16 Mp 16 bytes of steering)
    const bool huge = Mp > 208;
    const bool big = !huge && DAS_BIG && DAS_DIRECT_C && Mp > 64 && DAS_P64;
    if (huge) {
        const size_t smem16 = (size_t)16 * Mp * 16;
        if (smem16 > 220 * 1024) return -1;
        if (raise_smem_limit(das_kernel<1, kDasWarps, 16>, smem16) !=
            cudaSuccess)
            return -1;
        dim3 grid16((g.S + 15) / 16, n_bins);
        das_kernel<1, kDasWarps, 16><<<grid16, kDasThreads, smem16, st>>>(g, dist, amp, freq, (const double2 *)csm_half, Mp,
                                                                          b, dr);
        return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
    }
    const int P = ((Mp <= 64 && DAS_P64) || big) ? 64 : 32;
    const int NWv = (P == 64 && !big) ? 4 : kDasWarps;
    const size_t smem = (size_t)16 * Mp * (P + ((DAS_DIRECT_C && P == 64) ? 0 : 8 * NWv));
    if (smem > 220 * 1024) return -1;
    // (per device and kernel: a process may drive several devices)
    const cudaError_t e = big ? raise_smem_limit(das_kernel<2, kDasWarps>, smem)
                        : (P == 64) ? raise_smem_limit(das_kernel<2, 4>, smem)
                                    : raise_smem_limit(das_kernel<1, kDasWarps>, smem);
    if (e != cudaSuccess) return -1;
    dim3 grid((g.S + P - 1) / P, n_bins);
    if (big)
        das_kernel<2, kDasWarps><<<grid, kDasThreads, smem, st>>>(g, dist, amp, freq, (const double2 *)csm_half, Mp, b, dr);
    else if (P == 64)
        das_kernel<2, 4><<<grid, 128, smem, st>>>(g, dist, amp, freq, (const double2 *)csm_half, Mp, b, dr);
    else
        das_kernel<1, kDasWarps><<<grid, kDasThreads, smem, st>>>(g, dist, amp, freq, (const double2 *)csm_half, Mp, b, dr);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
