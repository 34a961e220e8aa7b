// dwc_internal.cuh -- internal declarations of the B200 (sm_100a) implementation behind
// include/dwc.h.  Nothing here is visible through the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dwc.h"

namespace dwc {

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
int launch_geom_tables(const Geo &g, double *dist, double *amp, int *flag, cudaStream_t st);

// S1 for a list of nodes: E[pt][m] complex128 interleaved.
int launch_steer(const Geo &g, const double *dist, const double *amp, const double *freq,
                 int n_pts, const int32_t *idx, double *E, cudaStream_t st);

// Hermitian part of the CSMs (reading R3), into H (dev, same layout).
int launch_hermitize(int M, int n_bins, const double *csm, double *H, cudaStream_t st);

// S2: b[k][s] for n_bins bins; freq dev[n_bins]; csm dev.
int launch_das(const Geo &g, const double *dist, const double *amp, int n_bins,
               const double *freq, const double *csm, double *b, cudaStream_t st);

// S3+S4: compaction of kept nodes.  flag (dev int): bit 1 set when b has a non-finite value.
int launch_compress(int n, int n_bins, const double *b, double eps, int eps_mode, int full_grid,
                    int32_t *n_keep, int32_t *keep_idx, uint8_t *level, int *flag,
                    cudaStream_t st);

// Per-bin layout of the compressed systems, built on the host after n_keep is known.
struct BinLayout {
    int32_t nk;       // S~
    int32_t sp;       // padded size (multiple of 32)
    int64_t a_off;    // float offset of A~_k (sp*sp dense row-major)
    int64_t v_off;    // offset of per-bin vectors (sp entries)
    int32_t rp;       // S~ padded to the PSF tile rows (128)
    int32_t pad_;
    int64_t r_off;    // row offset of the bin's PSF operand digits and row scales
};

// S5 + S6 on the tensor cores (k_psf.cu): int8 digit operands of the kept steering vectors
// (opA: psf_opa_bytes, opB: psf_opb_bytes for sum rp rows; rsc: sum rp doubles), b~ = b[keep]
// into bt (fp64, zero padded to sp; skipped when b is NULL), then A~_k over the (bin, I, J)
// list of 128x64 output tiles touching the upper triangle, both triangles written.
int psf_kp(int m);
size_t psf_opa_bytes(int m, int64_t rows);
size_t psf_opb_bytes(int m, int64_t rows);
int psf_tile_rows();
int psf_tile_cols();
int launch_psf(const Geo &g, const double *dist, const double *amp, int n_bins, const double *freq,
               const BinLayout *lay, const int32_t *keep_idx, const double *b, int max_rp, int n_tiles,
               const int4 *tiles, int8_t *opA, int8_t *opB, double *rsc, double *bt, float *A, cudaStream_t st);

// S5 storage layout of A~_k (shared by the Gram epilogue and the GS kernel): 32x32 fp32
// tiles, column-major inside a tile, row-block-major; T = sp/32; element (i, j) at
//   a_off + ((i/32)*T + j/32)*1024 + (j%32)*32 + (i%32).
__host__ __device__ inline size_t tiled_index(int T, int i, int j) {
    return ((size_t)(i >> 5) * T + (j >> 5)) * 1024 + (size_t)(j & 31) * 32 + (i & 31);
}

// dense row-major n x n <-> tiled sp x sp (zero padded) conversions (stage entry points).
int launch_tile_convert(int to_tiled, int n, int sp, const float *src, float *dst, cudaStream_t st);

// S7+S8: Gauss-Seidel sweeps, persistent cluster kernel over LPT-ordered work items
// (gs_item_ints() ints each: g, bin[4]); writes x_out (per bin at v_off, nullable) and
// scatters into x_map[k*S + keep[i]] (nullable).
size_t gs_smem_bytes(int max_sp);
int gs_cluster_size();
int gs_item_ints();
int gs_group_size(int nk);
int launch_gs(int n_items, const int *items, const BinLayout *lay_dev, int max_sp, int *counter, const float *A,
              const void *packets, int sweeps, float *x_out, float *x_map, const int32_t *keep_idx, int S,
              int num_sms, cudaStream_t st);

// Per-block solver packets (1/A_ii, within-group scaled coefficients, b~ block) for the GS
// kernel: gs_packet_bytes() bytes per 32-row block, bin k's packets at v_off/32.
int gs_packet_bytes();
int launch_gs_prep(int n_bins, int max_sp, const BinLayout *lay_dev, const float *A, const double *bt,
                   void *packets, cudaStream_t st);

}  // namespace dwc
