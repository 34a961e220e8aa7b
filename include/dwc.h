/*
 * dwc.h -- C ABI of the B200-native DAMAS-on-wavelet-compressed-grid library.
 *
 * One data-parallel hot path (Ma & Liu, arXiv 1608.05179, /root/reference/PAPER.md):
 * for every frequency bin of a band
 *   S1 steering vectors            Eq. 3-4, 7
 *   S2 DAS map b = diag(E^H C E)/M^2   Eq. 2
 *   S3/S4 wavelet detail + threshold   Alg. 1, Eq. 15-22
 *   S5 PSF on the kept points A = |E^H E|^2/M^2   Eq. 9-12, 23
 *   S6 restrict b                  Eq. 23
 *   S7 non-negative Gauss-Seidel   Eq. 13-14
 *   S8 embed the solution on the full grid
 * Readings of ambiguous passages are listed in DESIGN.md ("Readings" R1..R18).
 *
 * Conventions (all entry points):
 *  - Every size is int32 and explicit; every struct is POD.
 *  - "dev" pointers are CUDA device pointers on the context's device (e.g. torch
 *    tensors); "host" pointers are ordinary host memory, read/written only during the
 *    call.  The caller owns every buffer passed in; the library never frees or retains a
 *    caller pointer after the call returns.
 *  - Work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default stream).
 *    Unless stated, calls return after enqueueing (results valid once the stream reaches
 *    that point).  dwc_solve_band performs exactly one internal device->host read (the
 *    kept-point counts, to size the PSF storage) and otherwise stays asynchronous.
 *  - Argument validation happens on the host before any launch.  On failure the call
 *    returns a negative dwc_status and dwc_last_error() describes it; no output is
 *    written in that case, with two exceptions detected after launches: DWC_ENUMERIC found on
 *    the device (outputs undefined), and a compressed band whose largest kept set S~ exceeds
 *    the on-chip capacity of the Gauss-Seidel kernels (S~ is only known after S4: DWC_EINVAL,
 *    b_map / n_keep / keep_idx then hold the S2-S4 results, x_map is not written; a full-grid
 *    band is checked before any launch).  No copy into a caller's host buffer outlives a failed
 *    call.
 *  - A context is used by one host thread at a time.  Different devices need different
 *    contexts.  Calls on one context may use different streams: each call's work is ordered
 *    after the previous call's (the context's workspace is shared).
 *  - Scan grid node s = row*n + col sits at x = cx - L/2 + col*dx, y = cy - L/2 + row*dx,
 *    z = z0, dx = L/(n-1) (reading R17).
 *  - A CSM is m*m complex128, row-major, C[i][j] at (i*m + j), interleaved (re, im)
 *    (Eq. 1).  Only its Hermitian part affects the map (reading R3).
 */
#ifndef DWC_H
#define DWC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DWC_API __attribute__((visibility("default")))
#else
#define DWC_API
#endif

typedef struct dwc_ctx dwc_ctx; /* opaque; one per CUDA device */

typedef enum {
    DWC_OK = 0,
    DWC_EINVAL = -1,     /* invalid argument (sizes, geometry, eps <= 0, sweeps < 1, NULL) */
    DWC_ESINGULAR = -2,  /* a scan-grid node coincides with a microphone */
    DWC_ENUMERIC = -3,   /* non-finite CSM/map value or A_ii <= 0 */
    DWC_ENOMEM = -4,     /* device or pinned-host allocation failed */
    DWC_ECUDA = -5,      /* CUDA runtime failure (message from the runtime) */
    DWC_ESTATE = -6      /* wrong device / unsupported device (needs sm_100) */
} dwc_status;

/* Microphone array (Fig. 1 origin at the array centre). */
typedef struct {
    int32_t m;              /* number of microphones M, 2 <= m <= DWC_MAX_MICS */
    const double *mic_xyz;  /* host, m*3 metres, (x, y, z) per microphone */
    double c0;              /* speed of sound (m/s), > 0 */
} dwc_array;

/* Scan plane parallel to the array at distance z0. */
typedef struct {
    int32_t n;        /* nodes per side N >= 2, S = n*n */
    double side_len;  /* L > 0 (m); dx = L/(n-1) */
    double z0;        /* plane distance (m), > 0 */
    double cx, cy;    /* plane centre (m) */
} dwc_grid;

/* Compression threshold and solver controls. */
typedef struct {
    double epsilon;   /* > 0; relative (eps * max|b|) or absolute */
    int32_t eps_mode; /* 0 = relative, 1 = absolute (reading R6) */
    int32_t sweeps;   /* Gauss-Seidel sweeps >= 1 from x0 = 0 */
    int32_t flags;    /* DWC_FULL_GRID: keep every node (the paper's "original grid"); DWC_CUBIC;
                         DWC_DIAG_REMOVAL; DWC_ALT_SWEEPS; DWC_GS_DENSE_STREAM / DWC_GS_RESIDUAL;
                         DWC_PAPER_PSF; DWC_THROUGHPUT (each documented below) */
} dwc_params;

#define DWC_FULL_GRID 1
/* DWC_CUBIC: 4-point (cubic, Deslauriers-Dubuc family) interpolating predictor in S3 instead
 * of the linear one (reading R19): Lagrange interpolation through
 * the 4 nearest coarse nodes, linear rule where fewer than 4 are in reach.  Changes only the
 * compressed index set (and so everything downstream). */
#define DWC_CUBIC 2
/* DWC_DIAG_REMOVAL: CSM diagonal removal (reading R20): the DAS map
 * leaves out the C_mm terms, is normalised by M^2 - M and clamped at 0; the PSF is the
 * matching A_ij = (|e_i^H e_j|^2 - sum_m |e_mi|^2 |e_mj|^2) / (M^2 - M), clamped at 0.
 * Uncorrelated microphone noise (a diagonal CSM term) then drops out of the map. */
#define DWC_DIAG_REMOVAL 4
/* DWC_ALT_SWEEPS: alternating sweep directions (original DAMAS practice; reading
 * R21): sweep 2p in ascending row order (Eq. 13-14), sweep 2p+1 descending.  Runs on the kernel
 * the choice below picks: the residual kernel walks the alternating visit sequence; in place of
 * the dense-stream kernel a simpler one-CTA-per-bin kernel runs (DWC_GS_KERNEL_ALT). */
#define DWC_ALT_SWEEPS 8
/* Gauss-Seidel kernel of the sweeps (both keep Eq. 13-14's row and sweep order exactly and differ
 * in summation order only):
 *  - residual-update kernel: the residual r = A x - b of the current iterate kept on chip in fp64,
 *    updated with the row of A~ of every x that changes (one CTA per bin; systems above 2560
 *    points split r over a cluster of up to 8 CTAs);
 *  - dense-stream cluster kernel: every row dot recomputed from the symmetric-packed A~ streamed
 *    through shared memory (up to 4 CTAs per bin).
 * Default: the residual kernel when the band's largest system has at most 20480 points (padded
 * to 32), else the dense-stream kernel.  DWC_GS_DENSE_STREAM / DWC_GS_RESIDUAL force one
 * (setting both is DWC_EINVAL).  dwc_stats.gs_kernel reports which ran, gs_max_group the
 * largest CTAs per bin. */
#define DWC_GS_DENSE_STREAM 16
#define DWC_GS_RESIDUAL 32
/* DWC_PAPER_PSF: the paper-literal beamformer and PSF (NEXT-4, fidelity study of reading R1): the
 * DAS map with Eq. 4's focus vector v_m = (d_m/|r|) e^{-jkd_m} and the PSF
 * A_P[i][j] = |v_i^H g_j|^2 / M^2 with Eq. 7's g_m = (|r|/d_m) e^{-jkd_m}, |r| the
 * distance to the array centre (the origin).  A_P is not symmetric: the PSF covers
 * every tile, the sweeps (Eq. 13-14, forward) run on the residual kernel with A_P stored
 * transposed.  Not with DWC_DIAG_REMOVAL or DWC_GS_DENSE_STREAM (DWC_EINVAL); with DWC_ALT_SWEEPS.
 * The sweeps' convergence is not guaranteed (A_P has an indefinite symmetric part). */
#define DWC_PAPER_PSF 64
/* DWC_THROUGHPUT: a hint that this band is one of several in flight (bands streamed in, on other
 * contexts / streams): the residual kernel then runs every system of up to 1280 points two CTAs
 * per SM (half the registers and shared memory each), so overlapping bands share
 * the SMs; without it only the systems of at most 2/3 of the band's largest size do, and only
 * when the band has more bins than SMs.  The iterates are bitwise identical either way (the
 * kernel's arithmetic and order do not depend on the class).  Measured on cfg3 (one B200): one
 * band alone 24.0 -> 28.6 ms, bands in flight 14.2 k -> 16.7 k bins/s.  Ignored by the
 * dense-stream kernel. */
#define DWC_THROUGHPUT 128
#define DWC_MAX_MICS 512

/* Create / destroy a context on CUDA device `device`.  The device must be sm_100
 * (B200).  dwc_destroy frees the context's workspace pool. */
DWC_API dwc_status dwc_create(int device, dwc_ctx **out);
DWC_API dwc_status dwc_destroy(dwc_ctx *ctx);

/* ---- the batched hot path (S0..S8) ------------------------------------------------
 * n_bins >= 1 frequency bins; freq_hz host[n_bins] (> 0).
 * csm      dev  n_bins*m*m complex128 (interleaved), bin k at k*m*m.
 * n_keep   dev  int32[n_bins]          (out) S~_k = number of kept nodes (>= |G^0|).
 * keep_idx dev  int32[n_bins*S]        (out) kept node indices of bin k, ascending, at k*S;
 *                                            entries n_keep[k]..S-1 are -1.
 * x_map    dev  float[n_bins*S]        (out) DAMAS source-power descriptors on the full
 *                                            grid after `sweeps` sweeps; 0 off the kept set.
 * b_map    dev  double[n_bins*S]       (out, nullable) the DAS map of every bin.
 * warn     host uint32[n_bins]         (out, nullable) bit0: dx/B > 0.2 at that bin
 *                                      (Eq. 24 beamwidth).
 * Errors: DWC_EINVAL, DWC_ESINGULAR, DWC_ENUMERIC, DWC_ENOMEM, DWC_ECUDA. */
DWC_API dwc_status dwc_solve_band(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid,
                          const dwc_params *p, int32_t n_bins, const double *freq_hz,
                          const double *csm, int32_t *n_keep, int32_t *keep_idx,
                          float *x_map, double *b_map, uint32_t *warn, void *cuda_stream);

/* Same computation with HOST buffers (csm, n_keep, keep_idx, x_map, b_map all host; b_map
 * nullable).  The host<->device copies are part of the call, which returns when the
 * outputs are in host memory.  Page-locked (pinned) host buffers make the copies
 * asynchronous DMA; pageable buffers work but are staged by the CUDA runtime.  With a pinned
 * keep_idx the keep set is read back on an internal copy stream as soon as it is final (after
 * S4), overlapping the PSF and the sweeps. */
DWC_API dwc_status dwc_solve_band_host(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid,
                               const dwc_params *p, int32_t n_bins, const double *freq_hz,
                               const double *csm, int32_t *n_keep, int32_t *keep_idx,
                               float *x_map, double *b_map, uint32_t *warn, void *cuda_stream);

/* The same path from the microphones' snapshot spectra: the CSM of each
 * bin is formed on the device by Eq. 1, C = (1/I) sum_i p_i p_i^H, in fp64,
 * and consumed by the DAS without leaving the GPU.  snap dev complex128
 * [n_bins][m][n_snap] (interleaved re,im; row = microphone, snapshots contiguous); the other
 * arguments as dwc_solve_band.  Errors as dwc_solve_band, DWC_EINVAL for n_snap < 1. */
DWC_API dwc_status dwc_solve_band_snapshots(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid,
                                    const dwc_params *p, int32_t n_bins, const double *freq_hz,
                                    int32_t n_snap, const double *snap, int32_t *n_keep, int32_t *keep_idx,
                                    float *x_map, double *b_map, uint32_t *warn, void *cuda_stream);

/* ---- stage entry points (parity tests feed identical inputs to GPU and oracle) ---- */

/* Eq. 1: CSMs from snapshot spectra.  snap as dwc_solve_band_snapshots; csm dev complex128
 * [n_bins][m][m] row-major (out), fp64.  Errors: DWC_EINVAL, DWC_ECUDA. */
DWC_API dwc_status dwc_csm(dwc_ctx *ctx, int32_t m, int32_t n_bins, int32_t n_snap, const double *snap,
                           double *csm, void *cuda_stream);

/* S1: normalised steering vectors e_s = sqrt(M) g_s/||g_s|| of n_pts nodes (reading R1;
 * PAPER.md:102-110 Eq. 3-4, :128-131 Eq. 7).
 * idx dev int32[n_pts]; E dev complex128 [n_pts][m] interleaved (out). */
DWC_API dwc_status dwc_steer(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, double freq_hz,
                     int32_t n_pts, const int32_t *idx, double *E, void *cuda_stream);

/* S2: DAS maps b_k(s) = Re(e_s^H C_k e_s)/M^2 in fp64 (Eq. 2; diagonal removal
 * PAPER.md:96).  csm dev as in dwc_solve_band;
 * flags: 0, DWC_DIAG_REMOVAL, or DWC_PAPER_PSF (Eq. 4's v instead of e);
 * b_map dev double[n_bins*S] (out). */
DWC_API dwc_status dwc_das(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, int32_t n_bins,
                   const double *freq_hz, const double *csm, int32_t flags, double *b_map, void *cuda_stream);

/* S3+S4: wavelet details in fp64 (no FMA contraction, reading R7 stencil) and threshold
 * (Alg. 1 and Eq. 15-22);
 * b_map dev double[n_bins*S]; n_keep/keep_idx as in dwc_solve_band (out);
 * level dev uint8[n_bins*S] (out, nullable): resolution level of each node (Eq. 15). */
DWC_API dwc_status dwc_compress(dwc_ctx *ctx, const dwc_grid *grid, const dwc_params *p,
                        int32_t n_bins, const double *b_map, int32_t *n_keep,
                        int32_t *keep_idx, uint8_t *level, void *cuda_stream);

/* S5: PSF matrix on n_keep nodes, A[i][j] = |e_i^H e_j|^2/M^2, fp32 accurate (Eq. 9-12,
 * PAPER.md:139-160, restricted to the kept nodes by Eq. 23).
 * keep_idx dev int32[n_keep]; flags: 0, DWC_DIAG_REMOVAL, or DWC_PAPER_PSF (the asymmetric
 * A_P[i][j] = |v_i^H g_j|^2/M^2, Eq. 4 x Eq. 7); A dev float[n_keep*n_keep]
 * row-major (out). */
DWC_API dwc_status dwc_psf(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, double freq_hz,
                   int32_t n_keep, const int32_t *keep_idx, int32_t flags, float *A, void *cuda_stream);

/* S7: `sweeps` forward projected Gauss-Seidel sweeps from x0 = 0 on one system (Eq. 13-14,
 * PAPER.md:167-180; alternating directions: SPEC.md:308, reading R21).
 * A dev float[n*n] row-major, symmetric (as A~ is, reading R1) with A_ii > 0: only the upper
 * triangle (j >= i) is read, the lower one is taken as its transpose -- unless flags has
 * DWC_PAPER_PSF: then A is a general matrix (the paper-literal PSF), read in full, sweeps on the
 * residual kernel.
 * flags: 0, DWC_ALT_SWEEPS, DWC_GS_DENSE_STREAM / DWC_GS_RESIDUAL (kernel choice), DWC_PAPER_PSF;
 * b dev double[n], x dev float[n] (out).
 * Errors: DWC_EINVAL (n < 1, sweeps < 1, NULL, unknown flags, n beyond the on-chip x capacity),
 * DWC_ENUMERIC (some A_ii <= 0 or non-finite: checked on the device and read back, so this
 * call synchronises `cuda_stream` once before the sweeps), DWC_ECUDA. */
DWC_API dwc_status dwc_gs(dwc_ctx *ctx, int32_t n, const float *A, const double *b, int32_t sweeps,
                  int32_t flags, float *x, void *cuda_stream);

/* ---- multi-GPU gather helpers --------------------------------------- */

/* Keep set -> bitmask (the multi-GPU gather of a band whose bins are solved independently,
 * PAPER.md:545-547): for each of n_bins bins, mask holds W = ceil(S/32) uint32 words; bit
 * (s % 32) of word s/32 is set iff node s is in the bin's keep list.  n_keep dev int32[n_bins],
 * keep_idx dev int32[n_bins*S] ascending (as dwc_solve_band writes it), mask dev
 * uint32[n_bins*W] (out).  The bitmask is what the ranks all-gather (S/8 bytes per bin
 * instead of 4 S).  Errors: DWC_EINVAL (S < 1, n_bins < 0, NULL), DWC_ECUDA. */
DWC_API dwc_status dwc_keep_mask(dwc_ctx *ctx, int32_t n_bins, int32_t S, const int32_t *n_keep,
                                 const int32_t *keep_idx, uint32_t *mask, void *cuda_stream);

/* Bitmask -> keep set: the inverse of dwc_keep_mask (ascending list, -1 padded to S; the keep
 * set of Alg. 1). */
DWC_API dwc_status dwc_keep_unmask(dwc_ctx *ctx, int32_t n_bins, int32_t S, const uint32_t *mask,
                                   int32_t *n_keep, int32_t *keep_idx, void *cuda_stream);

/* ---- diagnostics ------------------------------------------------------------------ */

/* Per-call statistics of the last dwc_solve_band / dwc_solve_band_host on this context.
 * Stage times are measured with CUDA events on the call's stream only when timing is
 * enabled (dwc_set_timing); reading them synchronises on those events. */
typedef struct {
    int32_t n_bins;
    int64_t sum_keep;         /* sum_k S~_k */
    double sum_keep_sq;       /* sum_k S~_k^2 */
    double gs_bytes;          /* sum_k sweeps * 2 S~_k (S~_k + 1): the symmetric-packed fp32 A~_k
                                 once per sweep (algorithmic bytes of the GS stream) */
    double psf_flops;         /* real flops of the PSF Gram (8*M*S~^2 per bin, full square) */
    double das_flops;         /* real flops of the DAS quadratic forms (8*M^2*S per bin) */
    int32_t launches;         /* kernels launched by the call */
    float ms_total;           /* event time of the whole call (timing on) */
    float ms_das, ms_compress, ms_psf, ms_gs; /* per-stage event times (timing on) */
    /* Which Gauss-Seidel kernel the last dwc_solve_band / dwc_gs launched (also set by dwc_gs):
     * DWC_GS_KERNEL_* below, the extra shared-memory ring tiles it was given, the CTAs of its
     * grid and the largest number of CTAs it gave one bin. */
    int32_t gs_kernel;
    int32_t gs_xtra_tiles;
    int32_t gs_ctas;
    int32_t gs_max_group;
    int64_t gs_updates;       /* residual kernel: row updates (x changes) over all bins and sweeps */
    double gs_row_bytes;      /* residual kernel: bytes of the rows of A~ those updates streamed
                                 (4 sp per update; the panels of predicted rows come on top) */
} dwc_stats;

#define DWC_GS_KERNEL_NONE 0
#define DWC_GS_KERNEL_CLUSTER 1       /* dense-stream cluster kernel, fixed shared-memory ring   */
#define DWC_GS_KERNEL_CLUSTER_XTRA 2  /* the same with extra ring tiles behind its tables        */
#define DWC_GS_KERNEL_ALT 3           /* one-CTA-per-bin alternating sweeps (ALT + DENSE_STREAM) */
#define DWC_GS_KERNEL_RESIDUAL 4      /* residual-update kernel (either sweep order)             */

DWC_API dwc_status dwc_set_timing(dwc_ctx *ctx, int enable);
DWC_API dwc_status dwc_get_stats(dwc_ctx *ctx, dwc_stats *out);

DWC_API const char *dwc_last_error(void);            /* thread-local; valid until the next call */
DWC_API size_t dwc_workspace_bytes(const dwc_ctx *ctx);
DWC_API const char *dwc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DWC_H */
