// k_gs_alt.cu -- S7 with alternating sweep directions (reading R21): the
// original DAMAS practice of forward / backward sweeps, on the same symmetric-packed
// A~ the main kernel streams (dwc_internal.cuh layout).  Sweep 2p runs the rows ascending (Eq.
// 13-14), sweep 2p+1 descending, same projected update.
//
// A variant for fidelity studies, not the bench path: one CTA per bin, 8 warps.  Per 32-row block
// k (in sweep order) the warps form P_k = sum_{J != k} A[I_k, I_J] x_J with the latest x --
// U(k, J) as a row tile for J > k, U(J, k)^T for J < k, read straight from global/L2 -- then one
// warp runs the in-block recurrence in the sweep's row order: lane l holds column l of the
// diagonal tile in registers and row l's scaled residual (step form, one shuffle per row; the
// block's starting residual is formed with b~ in fp64).
#include "dwc_internal.cuh"

namespace dwc {

constexpr int kAltThreads = 256;
constexpr int kAltWarps = kAltThreads / 32;

// row tile: acc[q] (rows 4rq+q, partial over columns c = cq + 4i) += tile[c][4rq+q] x[c]
__device__ __forceinline__ void alt_row_dot(const float *__restrict__ tile, const float *__restrict__ x, int rq,
                                            int cq, float acc[4]) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int c = cq + 4 * i;
        const float4 v = __ldg(reinterpret_cast<const float4 *>(tile + c * 32 + 4 * rq));
        const float xv = x[c];
        acc[0] = fmaf(v.x, xv, acc[0]);
        acc[1] = fmaf(v.y, xv, acc[1]);
        acc[2] = fmaf(v.z, xv, acc[2]);
        acc[3] = fmaf(v.w, xv, acc[3]);
    }
}
// transposed tile: lane o gets sum_r tile[o][r] x[r] (column o of the column-major tile)
__device__ __forceinline__ float alt_col_dot(const float *__restrict__ tile, const float *__restrict__ x, int lane) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int r0 = 4 * ((k + lane) & 7);
        const float4 v = __ldg(reinterpret_cast<const float4 *>(tile + lane * 32 + r0));
        t = fmaf(v.x, x[r0], t);
        t = fmaf(v.y, x[r0 + 1], t);
        t = fmaf(v.z, x[r0 + 2], t);
        t = fmaf(v.w, x[r0 + 3], t);
    }
    return t;
}

__device__ __forceinline__ void alt_prefetch_l2(const float *tiles, int n) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tiles), "r"(n * 4096) : "memory");
}

// In-block recurrence in "step form" (as the main kernel): lane l owns row l; with
// w_l = -r_l / A_ll the rows t in sweep order take delta_t = max(w_t, -x_t) (x_t + delta_t =
// max(x_t - r_t / A_tt, 0), Eq. 14), broadcast it, and every lane applies w_l -= (A_lt / A_ll)
// delta_t -- one shuffle per row instead of a warp reduction per row.  col[t] = D[t][l] = A_lt.
template <bool kBack>
__device__ __forceinline__ void alt_block_recurrence(const float col[32], double base, float &xl, float dll, int lane) {
    const float inv = dll > 0.f ? 1.f / dll : 0.f;   // padding rows never move (w = 0, x = 0)
    float part = 0.f;                                 // D x^old for row l: the in-block part of r_l
#pragma unroll
    for (int t = 0; t < 32; t++) part = fmaf(col[t], __shfl_sync(0xffffffffu, xl, t), part);
    float w = (float)(-(base + (double)part) * (double)inv);
    float sc[32];
#pragma unroll
    for (int t = 0; t < 32; t++) sc[t] = col[t] * inv;   // A_lt / A_ll
#pragma unroll
    for (int tt = 0; tt < 32; tt++) {
        const int t = kBack ? 31 - tt : tt;
        const float d = __shfl_sync(0xffffffffu, fmaxf(w, -xl), t);
        if (lane == t) xl += d;
        w = fmaf(-sc[t], d, w);
    }
}

__global__ void __launch_bounds__(kAltThreads)
gs_alt_kernel(const BinLayout *__restrict__ lay, const float *__restrict__ A, const double *__restrict__ bt,
              int sweeps, float *__restrict__ x_out, float *__restrict__ x_map, const int32_t *__restrict__ keep_idx,
              int S) {
    extern __shared__ float xs[];   // sp floats
    __shared__ float red[kAltWarps][32];
    const int bin = blockIdx.x;
    const BinLayout L = lay[bin];
    const int sp = L.sp, T = sp >> 5, g = L.g;
    const float *Ab = A + L.a_off;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int rq = lane & 7, cq = lane >> 3;
    for (int i = tid; i < sp; i += kAltThreads) xs[i] = 0.f;
    __syncthreads();
    for (int it = 0; it < sweeps; it++) {
        const bool back = it & 1;
        for (int kk = 0; kk < T; kk++) {
            const int k = back ? T - 1 - kk : kk;
            // the next step's tiles into L2 while this step runs (they do not depend on x): its row
            // runs (one contiguous run per owner group of the layout) and its column tiles
            if (lane == 0) {
                const bool last = kk + 1 == T;
                const int kn = last ? (back ? 0 : T - 1) : (back ? k - 1 : k + 1);
                if (w == 0)
                    for (int o = 0; o < g; o++) {
                        const int len = sym_run_len(T, g, kn, o);
                        if (len > 0) alt_prefetch_l2(Ab + (size_t)sym_run_start(T, g, kn, o) * 1024, len);
                    }
                for (int J = w; J < kn; J += kAltWarps) alt_prefetch_l2(Ab + (size_t)sym_u_tile_g(T, g, J, kn) * 1024, 1);
            }
            // P_k over the other column blocks, with the latest x
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            float acc_t = 0.f;
#pragma unroll 2
            for (int J = w; J < k; J += kAltWarps)
                acc_t += alt_col_dot(Ab + (size_t)sym_u_tile_g(T, g, J, k) * 1024, xs + 32 * J, lane);
            const int J1 = k + 1 + ((w - (k + 1)) % kAltWarps + kAltWarps) % kAltWarps;   // first J > k with J = w mod 8
#pragma unroll 2
            for (int J = J1; J < T; J += kAltWarps)
                alt_row_dot(Ab + (size_t)sym_u_tile_g(T, g, k, J) * 1024, xs + 32 * J, rq, cq, acc);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 8);
                acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 16);
                acc[q] += __shfl_sync(0xffffffffu, acc_t, 4 * rq + q);
            }
            if (cq == 0) {
#pragma unroll
                for (int q = 0; q < 4; q++) red[w][4 * rq + q] = acc[q];
            }
            __syncthreads();
            if (w == 0) {
                float p = 0.f;
#pragma unroll
                for (int q = 0; q < kAltWarps; q++) p += red[q][lane];
                const int row = 32 * k + lane;
                const float *D = Ab + (size_t)k * 1024;   // D_k, column-major: D[t][l] at [l*32 + t]
                float col[32];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(D + lane * 32 + 4 * q));
                    col[4 * q] = v.x; col[4 * q + 1] = v.y; col[4 * q + 2] = v.z; col[4 * q + 3] = v.w;
                }
                const float dll = (row < L.nk) ? col[lane] : 0.f;   // padding rows never move
                const double base = (double)p - bt[L.v_off + row];
                float xl = xs[row];
                if (back) alt_block_recurrence<true>(col, base, xl, dll, lane);
                else alt_block_recurrence<false>(col, base, xl, dll, lane);
                xs[row] = xl;
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < L.nk; i += kAltThreads) {
        const float v = xs[i];
        if (x_out) x_out[L.v_off + i] = v;
        if (x_map) x_map[(size_t)bin * S + keep_idx[(size_t)bin * S + i]] = v;
    }
}

int launch_gs_alt(int n_bins, const BinLayout *lay_dev, int max_sp, const float *A, const double *bt, int sweeps,
                  float *x_out, float *x_map, const int32_t *keep_idx, int S, cudaStream_t st) {
    const size_t smem = (size_t)max_sp * 4;
    if (smem > 48 * 1024 &&
        raise_smem_limit(gs_alt_kernel, smem) != cudaSuccess)
        return -1;
    gs_alt_kernel<<<n_bins, kAltThreads, smem, st>>>(lay_dev, A, bt, sweeps, x_out, x_map, keep_idx, S);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
