// dwc_internal.cuh -- internal declarations of the B200 (sm_100a) implementation behind
// include/dwc.h.  Nothing here is visible through the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/dwc.h"

// Checked build (-DDWC_CHECKED, libdwc_checked.so, run by tests/test_gpu_checked.py): device-side
// invariants of the Gauss-Seidel kernels' rings, slots, parities and indices report and trap;
// mbarrier waits get a watchdog.  Compiled out of the production library.
#ifdef DWC_CHECKED
#define DWC_DCHECK(cond, what)                                                                          \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("[dwc checked] %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x, what);                                                             \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define DWC_DCHECK(cond, what) ((void)0)
#endif

namespace dwc {

// Raise a kernel's dynamic shared-memory limit (cudaFuncAttributeMaxDynamicSharedMemorySize) on
// the current device to at least `bytes` (dwc_api.cu).  The attribute belongs to the function and
// device, not to the context or stream: two host threads driving two contexts set it concurrently,
// and a plain set to each call's own need could lower it under the other thread's launch (which
// then fails with cudaErrorInvalidValue).  It is only ever raised, under a lock.
cudaError_t raise_smem_limit(const void *fn, size_t bytes);
template <typename F>
inline cudaError_t raise_smem_limit(F *fn, size_t bytes) {
    return raise_smem_limit((const void *)fn, bytes);
}

// Scan-grid + array geometry as the kernels see it (all fp64, device pointers).
struct Geo {
    int m;          // microphones
    int n;          // nodes per side
    int S;          // n*n
    double L, z0, cx, cy, dx, c0;
    const double *mic;  // dev m*3
};

__host__ __device__ inline double node_x(const Geo &g, int c) { return g.cx - g.L / 2.0 + (double)c * g.dx; }
__host__ __device__ inline double node_y(const Geo &g, int r) { return g.cy - g.L / 2.0 + (double)r * g.dx; }

constexpr double kTwoPi = 6.283185307179586476925286766559;

// ---- launchers (each returns the number of kernels it launched, or -1 on launch error)

// Frequency-independent steering tables: dist[m][s] = |r_s - r_m| and
// amp[m][s] = sqrt(M) / (dist * ||g_s||) with ||g_s||^2 = sum_m 1/dist^2 (reading R1).
// Sets *singular (dev int) to 1 when some distance is 0.
// ampv / ampg (nullable, M x S each): the paper-literal amplitudes d/|r| (Eq. 4) and |r|/d (Eq. 7).
int launch_geom_tables(const Geo &g, double *dist, double *amp, int *flag, cudaStream_t st, double *ampv = nullptr,
                       double *ampg = nullptr);

// S1 for a list of nodes: E[pt][m] complex128 interleaved.
int launch_steer(const Geo &g, const double *dist, const double *amp, const double *freq,
                 int n_pts, const int32_t *idx, double *E, cudaStream_t st);

// Half-Hermitian part of the CSMs (reading R3), zero padded to das_mpad(M): H (dev) holds
// n_bins * Mp * Mp complex128 (upper triangle of (C + C^H)/2, diagonal halved).
int das_mpad(int M);
// dr: diagonal removal (reading R20) -- the diagonal of Ch is zero.
int launch_hermitize(int M, int n_bins, const double *csm, double *H, int dr, cudaStream_t st);

// Eq. 1 (k_csm.cu): C_k = P_k P_k^H / I from snapshot spectra snap [n_bins][M][I] complex128.
// half = 0: full C [n_bins][M][M]; half = 1: the half-Hermitian padded Ch of launch_hermitize.
int launch_csm(int M, int n_bins, int I, const double *snap, double *out, int half, int dr, cudaStream_t st);

// S2: b[k][s] for n_bins bins; freq dev[n_bins]; csm_half = launch_hermitize's output.
int launch_das(const Geo &g, const double *dist, const double *amp, int n_bins,
               const double *freq, const double *csm_half, double *b, int dr, cudaStream_t st);

// S3+S4: compaction of kept nodes.  order 1: linear predictor (R7), 3: cubic (R19).
// flag (dev int): bit 1 set when b has a non-finite value.
int launch_compress(int n, int n_bins, const double *b, double eps, int eps_mode, int full_grid,
                    int order, int32_t *n_keep, int32_t *keep_idx, uint8_t *level, int *flag,
                    cudaStream_t st);

// Per-bin layout of the compressed systems, built on the host after n_keep is known.
struct BinLayout {
    int32_t nk;       // S~
    int32_t sp;       // padded size (multiple of 32)
    int64_t a_off;    // float offset of A~_k (sym_tiles(sp/32) tiles of 1024 floats)
    int64_t v_off;    // offset of per-bin vectors (sp entries)
    int32_t rp;       // S~ padded to the PSF tile rows (128)
    int32_t g;        // GS CTAs per bin (gs_group_size(nk)); fixes the tile order of A~_k
    int64_t r_off;    // row offset of the bin's PSF operand digits and row scales
    int64_t d_off;    // residual GS kernel: float offset of the dense row-major sp x sp A~_k
};

// The residual GS kernel's solver carries the contributions of each step's changes to the next
// kRgsWin row blocks itself (k_rgs.cu); it reads them from the dense row-major A~ only.
#ifndef RGS_WIN
#define RGS_WIN 3
#endif
// 3 measured best on B200 (cfg3 GS band -8 %, cfg4 -16 %, cfg5 -27 % against 7; 1, 2, 4, 5, 6,
// 9 and 11 slower): each change costs the solver W panel loads + FMAs and the panel producer W
// segments per changed row, while the stream warps keep W + 1 steps of slack.
constexpr int kRgsWin = RGS_WIN;

// S5 + S6 on the tensor cores (k_psf.cu): int8 digit operands of the kept steering vectors
// (opA: psf_opa_bytes, opB: psf_opb_bytes for sum rp rows; rsc: sum rp doubles), b~ = b[keep]
// into bt (fp64, zero padded to sp; skipped when b is NULL), then A~_k over the (bin, I, J)
// list of 128x32 output tiles touching the upper triangle, both triangles written.
// wt != NULL: diagonal removal (R20) -- the slice kernel writes |e_mr|^2 there (M doubles per
// padded row, layout wt[r_off*M + m*rp + r]) and the epilogue forms the DR PSF.
int psf_kp(int m);
size_t psf_opa_bytes(int m, int64_t rows);
size_t psf_opb_bytes(int m, int64_t rows);
int psf_tile_rows();
int psf_tile_cols();
// Adense != NULL: the residual GS layout -- A~_k dense row-major at Adense + d_off (row stride
// sp, zero padded), nothing at A; else the symmetric tile layout of the dense-stream kernel at
// A + a_off.
// ampb != NULL: the paper-literal PSF (NEXT-4): the A side (rows) from amp = d/|r| (Eq. 4 v), the
// B side (columns) from ampb = |r|/d (Eq. 7 g), rscb their column scales (sum rp doubles); the
// tile list then covers every tile and Adense receives the TRANSPOSE of the asymmetric A_P
// (Adense[j][i] = A_P[i][j], so the residual kernel reads column c of A_P as row c).
int launch_psf(const Geo &g, const double *dist, const double *amp, int n_bins, const double *freq,
               const BinLayout *lay, const int32_t *keep_idx, const double *b, int max_rp, int n_tiles,
               const int4 *tiles, int8_t *opA, int8_t *opB, double *rsc, double *bt, double *wt, float *A,
               float *Adense, cudaStream_t st, const double *ampb = nullptr, double *rscb = nullptr);

// S5 storage layout of A~_k (written by the PSF epilogue, streamed by the GS kernel).
// A~ is symmetric (reading R1), so only one triangle is stored.  32x32 fp32 tiles, column-major
// inside a tile (element (32I+r, 32J+c) at [c*32 + r]); T = sp/32 tile rows; g = CTAs the GS
// kernel gives the bin (gs_group_size); tile indices relative to the bin's base a_off/1024:
//   D_k  = A[k][k]             at k                        (T tiles)
//   L_k  = A[k][(k-1) mod T]   at T + k                    (T tiles; first sub-diagonal)
//   LL_k = A[k][(k-2) mod T]   at 2T + k                   (T tiles; second sub-diagonal)
//   U(I,J) = A[I][J], J > I    at 3T + row_base(I) + pos   (T(T-1)/2 tiles)
// Row I's U tiles are grouped by owner CTA o = own_of(g, J) and ascending in J inside a group,
// so the tiles a GS CTA streams from one row block are one contiguous run.  Ownership is a
// periodic pattern weighted by the CTAs' stream warps: the sub-group leader (owner 0) runs the
// solver, L and D warps and streams with 3 warps, the others with 5, so for g = 4 the leader
// owns 3 of every 18 column blocks (period 0123123 0123123 0123, 5 each for 1..3), for g = 2 3
// of every 8 (01101101).
// GS_PAT4 / GS_PAT2 (experiment): period of the g = 4 / g = 2 pattern, the leader owning
// period - 15 / period - 5 blocks of it (17, 18, 19 / 7, 8, 9); defaults 18 and 8.
#ifndef GS_PAT4
#define GS_PAT4 18
#endif
#ifndef GS_PAT2
#define GS_PAT2 8
#endif
__host__ __device__ inline int own_period(int g) { return g == 4 ? GS_PAT4 : (g == 2 ? GS_PAT2 : 1); }
__host__ __device__ inline int own_weight(int g, int o) {
    return g == 4 ? (o == 0 ? GS_PAT4 - 15 : 5) : (g == 2 ? (o == 0 ? GS_PAT2 - 5 : 5) : 1);
}
__host__ __device__ inline int own_of(int g, int J) {
#if GS_PAT4 == 17
    if (g == 4) return (int)((0x39e7939e4ull >> (2 * (J % 17))) & 3ull);   // 0123 1230 1231 2312 3
#elif GS_PAT4 == 19
    if (g == 4) return (int)((0x39e4e4e4e4ull >> (2 * (J % 19))) & 3ull);  // 0123 0123 0123 0123 123
#else
    if (g == 4) return (int)((0xE4E7939E4ull >> (2 * (J % 18))) & 3ull);   // 0,1,2,3,1,2,3,0,1,2,3,1,2,3,0,1,2,3
#endif
#if GS_PAT2 == 7
    if (g == 2) return (0x6Eu >> (J % 7)) & 1u;                                // 0,1,1,1,0,1,1
#elif GS_PAT2 == 9
    if (g == 2) return (0x1AAu >> (J % 9)) & 1u;                               // 0,1,0,1,0,1,0,1,1
#else
    if (g == 2) return (0xB6u >> (J % 8)) & 1u;                                // 0,1,1,0,1,1,0,1
#endif
    return 0;
}
// positions of owner o inside one period (bit r set: J = r mod period is owned by o)
__host__ __device__ inline uint32_t own_mask(int g, int o) {
#if GS_PAT4 == 17
    if (g == 4) return o == 0 ? 0x81u : (o == 1 ? 0x4912u : (o == 2 ? 0x9224u : 0x12448u));
#elif GS_PAT4 == 19
    if (g == 4) return o == 0 ? 0x1111u : (o == 1 ? 0x12222u : (o == 2 ? 0x24444u : 0x48888u));
#else
    if (g == 4) return o == 0 ? 0x4081u : (o == 1 ? 0x8912u : (o == 2 ? 0x11224u : 0x22448u));
#endif
#if GS_PAT2 == 7
    if (g == 2) return o == 0 ? 0x11u : 0x6Eu;
#elif GS_PAT2 == 9
    if (g == 2) return o == 0 ? 0x55u : 0x1AAu;
#else
    if (g == 2) return o == 0 ? 0x49u : 0xB6u;
#endif
    return 1u;
}
__host__ __device__ inline int popc32(uint32_t v) {
#ifdef __CUDA_ARCH__
    return __popc(v);
#else
    return __builtin_popcount(v);
#endif
}
// number of J in [0, x] owned by o (O(1): whole periods + popcount of the partial one)
__host__ __device__ inline int sym_cnt(int x, int o, int g) {
    if (x < 0) return 0;
    const int P = own_period(g), full = (x + 1) / P, rem = (x + 1) - full * P;
    return full * own_weight(g, o) + popc32(own_mask(g, o) & ((1u << rem) - 1u));
}
// the idx-th (0-based) J owned by o
__host__ __device__ inline int own_nth(int g, int o, int idx) {
    const int P = own_period(g), w = own_weight(g, o);
    int k = idx % w, J = (idx / w) * P;
    for (int r = 0;; r++)
        if (own_of(g, r) == o && k-- == 0) return J + r;
}
__host__ __device__ inline int sym_row_base(int T, int I) { return I * (T - 1) - I * (I - 1) / 2; }
__host__ __device__ inline int sym_run_len(int T, int g, int I, int o) {
    return sym_cnt(T - 1, o, g) - sym_cnt(I, o, g);
}
__host__ __device__ inline int sym_run_start(int T, int g, int I, int o) {
    int s = 0;
    for (int q = 0; q < o; q++) s += sym_run_len(T, g, I, q);
    return 3 * T + sym_row_base(T, I) + s;
}
__host__ __device__ inline int sym_u_tile(int T, int g, int I, int J) {
    const int o = own_of(g, J);
    return sym_run_start(T, g, I, o) + (sym_cnt(J - 1, o, g) - sym_cnt(I, o, g));
}
// stored tiles holding block (a, b) of A~ (up to three: U(0,T-1) is also L_0, U(0,T-2) also
// LL_0, ...; for T <= 2 the L / LL copies coincide with D or U)
__host__ __device__ inline int sym_targets(int T, int g, int a, int b, int t[3]) {
    int n = 0;
    if (a == b) t[n++] = a;
    else if (b > a) t[n++] = sym_u_tile(T, g, a, b);
    if (b == (a + T - 1) % T) t[n++] = T + a;
    if (b == (a + 2 * T - 2) % T) t[n++] = 2 * T + a;
    return n;
}
// The same with the sub-group size G a compile-time constant (the period divisions become
// multiplies); sym_targets_g dispatches on g.  For per-element hot paths (the PSF epilogue).
template <int G>
__host__ __device__ inline int sym_cnt_t(int x, int o) {
    constexpr int P = G == 4 ? GS_PAT4 : (G == 2 ? GS_PAT2 : 1);
    if (x < 0) return 0;
    const int full = (x + 1) / P, rem = (x + 1) - full * P;
    return full * own_weight(G, o) + popc32(own_mask(G, o) & ((1u << rem) - 1u));
}
template <int G>
__host__ __device__ inline int sym_u_tile_t(int T, int I, int J) {
    const int o = own_of(G, J);
    int s = 3 * T + sym_row_base(T, I);
    for (int q = 0; q < o; q++) s += sym_cnt_t<G>(T - 1, q) - sym_cnt_t<G>(I, q);
    return s + (sym_cnt_t<G>(J - 1, o) - sym_cnt_t<G>(I, o));
}
template <int G>
__host__ __device__ inline int sym_targets_t(int T, int a, int b, int t[3]) {
    int n = 0;
    if (a == b) t[n++] = a;
    else if (b > a) t[n++] = sym_u_tile_t<G>(T, a, b);
    int k1 = a + T - 1, k2 = a + 2 * T - 2;   // (a - 1) mod T, (a - 2) mod T
    while (k1 >= T) k1 -= T;
    while (k2 >= T) k2 -= T;
    if (b == k1) t[n++] = T + a;
    if (b == k2) t[n++] = 2 * T + a;
    return n;
}
__host__ __device__ inline int sym_u_tile_g(int T, int g, int I, int J) {
    return g == 4 ? sym_u_tile_t<4>(T, I, J) : (g == 2 ? sym_u_tile_t<2>(T, I, J) : sym_u_tile_t<1>(T, I, J));
}
__host__ __device__ inline int sym_targets_g(int T, int g, int a, int b, int t[3]) {
    return g == 4 ? sym_targets_t<4>(T, a, b, t) : (g == 2 ? sym_targets_t<2>(T, a, b, t) : sym_targets_t<1>(T, a, b, t));
}
__host__ __device__ inline int64_t sym_tiles(int T) { return (int64_t)T * (T - 1) / 2 + 3 * (int64_t)T; }

// dense row-major n x n <-> symmetric tile layout (zero padded to sp; g as above) for the
// stage entry points.  to_sym reads the upper triangle of src only.
int launch_tile_convert(int to_sym, int n, int sp, int g, const float *src, float *dst, cudaStream_t st);

// S7+S8: Gauss-Seidel sweeps, persistent cluster kernel over LPT-ordered work items
// (gs_item_ints() ints each: g, bin[4]); writes x_out (per bin at v_off, nullable) and
// scatters into x_map[k*S + keep[i]] (nullable).
size_t gs_smem_bytes(int max_sp, int ystride);
int gs_ystride(int nk);
int gs_cluster_size();
int gs_item_ints();
int gs_group_size(int nk);
// What a GS launch ran (dwc_stats gs_* fields).
struct GsLaunchInfo {
    int kernel = 0;      // DWC_GS_KERNEL_*
    int xtra_tiles = 0;  // extra ring tiles (the <true> instantiation) or 0
    int ctas = 0;        // CTAs of the grid
    int max_group = 0;   // largest CTAs-per-bin of the launch
};
// items_host / lay_host (nullable): host copies used to size the L2 prefetch window.
int launch_gs(int n_items, const int *items, const BinLayout *lay_dev, int max_sp, int ystride, int *counter,
              const float *A, const void *packets, int sweeps, float *x_out, float *x_map, const int32_t *keep_idx,
              int S, int num_sms, const int *items_host, const BinLayout *lay_host, cudaStream_t st,
              GsLaunchInfo *info);

// S7+S8 in residual-update form (k_rgs.cu): one CTA per bin, bins in the order order_dev
// (LPT); A~ as written by launch_psf with Adense; bt = b~ (fp64, zero padded to sp);
// n_updates (dev, nullable) += the number of row updates (x changes) over all sweeps.
size_t rgs_smem_bytes(int max_sp);
// largest padded system the automatic kernel choice gives the residual kernel (DWC_RGS_AUTO_MAX_SP overrides)
int rgs_auto_max_sp();
// CTAs per bin of the residual kernel for a system of sp padded points (1: r in one CTA's registers).
int rgs_cluster_size(int sp, bool wide);
// Launch class of a system of sp padded points (bins of one class share a residual-kernel launch).
int rgs_size_class(int sp, bool wide, int pair_max_sp = 0);
// Systems of at most this many padded points run two CTAs per SM (0: none).
int rgs_pair_max_sp(int band_max_sp, int n_bins, int num_sms, bool throughput);
int launch_rgs(int n_bins, const int *order_dev, const BinLayout *lay_dev, int max_sp, int *counter,
               const float *Adense, const double *bt, int sweeps, float *x_out, float *x_map,
               const int32_t *keep_idx, int S, int num_sms, unsigned long long *n_updates, cudaStream_t st,
               GsLaunchInfo *info, int alt = 0, int nonneg = 0, int wide_clusters = 1, int pair_max_sp = 0);
// dwc_gs: dense row-major n x n -> padded dense sp x sp (symmetric: from the upper triangle;
// general: transposed).
int launch_rgs_convert(int n, int sp, const float *src, float *dense, cudaStream_t st, int general = 0);
// n x n row-major out of a padded sp x sp dense matrix (transposed if transpose).
int launch_dense_extract(int n, int sp, const float *src, float *out, int transpose, cudaStream_t st);

// Per-block solver packets (1/A_ii, within-group scaled coefficients, b~ block) for the GS
// kernel: gs_packet_bytes() bytes per 32-row block, bin k's packets at v_off/32.
int gs_packet_bytes();
int launch_gs_prep(int n_bins, int max_sp, const BinLayout *lay_dev, const float *A, const double *bt,
                   void *packets, cudaStream_t st);

// S7 with alternating sweep directions (k_gs_alt.cu, reading R21): one CTA per bin on the same
// symmetric-packed A~ and b~ (bt, fp64, zero padded to sp).
int launch_gs_alt(int n_bins, const BinLayout *lay_dev, int max_sp, const float *A, const double *bt, int sweeps,
                  float *x_out, float *x_map, const int32_t *keep_idx, int S, cudaStream_t st);

// dwc_gs precondition: bit 2 of *flag set when some A_ii <= 0 or non-finite (k_keep.cu).
int launch_diag_check(int n, const float *A, int *flag, cudaStream_t st);

// Keep-set bitmasks (k_keep.cu): ceil(S/32) uint32 words per bin.
int launch_keep_mask(int n_bins, int S, const int32_t *n_keep, const int32_t *keep_idx, uint32_t *mask,
                     cudaStream_t st);
int launch_keep_unmask(int n_bins, int S, const uint32_t *mask, int32_t *n_keep, int32_t *keep_idx,
                       cudaStream_t st);

}  // namespace dwc
