// k_gs.cu -- S7 DAMAS non-negative Gauss-Seidel sweeps (+ S8 embed), the time sink.
//
// Eq. 13-14, readings R4, R11, R12, R18:
//   r_i = sum_{j<i} A_ij x_j^(n+1) + sum_{j>=i} A_ij x_j^(n) - b_i,
//   x_i^(n+1) = max(x_i^(n) - r_i / A_ii, 0),  i ascending, x^0 = 0, fixed sweep count.
// The row order and sweep order are kept exactly; only the summation order of each row
// dot differs from the oracle (fp32 storage of A~, fp32 accumulation).
//
// Block formulation (B = 32 rows): rows of block k need x^(n+1) of blocks < k.  Split
//   r_{I_k} = P_k + A[I_k, I_{k-1}] x_{k-1}^new - b_{I_k}
// where P_k = A[I_k, all blocks except k-1] x (x current, in-block old values) is
// computed by 7 "stream" warps WHILE the solver warp solves block k-1; only the 32x32
// sub-diagonal product and the in-block triangular recurrence sit on the critical path.
// The triangular recurrence runs in one warp in "step form": w_l = -r_l / A_ll,
//   delta_t = max(w_t, -x_t)    (x_t + delta_t = max(x_t + w_t, 0), exact projection)
//   w_l   -= (A_lt / A_ll) delta_t  for all lanes l,   x_t += delta_t,
// i.e. a 3-instruction dependency chain (FMNMX -> SHFL -> FFMA) per row.
//
// Data: A~_k dense row-major fp32 (ld = sp, multiple of 32, zero padded), streamed once
// per sweep from HBM/L2 with coalesced 16-byte loads (each row block is one contiguous
// 128*sp-byte range); x and the two staged 32x32 tiles live in shared memory.
// Persistent CTAs pull bins from an LPT-ordered queue (largest S~ first).
#include "dwc_internal.cuh"

namespace dwc {

constexpr int kGsWarps = 8;
constexpr int kGsThreads = kGsWarps * 32;
constexpr int kTS = 33;  // padded stride of staged tiles (conflict-free transposed access)

struct GsShared {
    float Lt[2][32 * kTS];   // Lt[t][l] = A[row0+l][prev0+t]
    float Dt[2][32 * kTS];   // Dt[t][l] = A[row0+l][row0+t]
    float Pw[2][kGsWarps - 1][32];
    float bts[2][32];
    int item;
};

__device__ __forceinline__ float4 ldg_stream(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Stream warps: P for block kn (all column blocks except kx), stage tiles and b~.
__device__ __forceinline__ void gs_stage(GsShared &sh, const float *__restrict__ xs,
                                         const float *__restrict__ Ab, const float *__restrict__ btb,
                                         int sp, int kx, int kn, int nbuf, int wid, int lane) {
    const float *Arow = Ab + (size_t)(32 * kn) * sp;
    float acc[32];
#pragma unroll
    for (int r = 0; r < 32; r++) acc[r] = 0.f;
    for (int col = (wid - 1) * 128 + 4 * lane; col - 4 * lane < sp; col += (kGsWarps - 1) * 128) {
        const bool valid = col < sp;
        const int cb = col >> 5;
        float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid && cb != kx) xv = *reinterpret_cast<const float4 *>(xs + col);
        const bool stL = valid && cb == kx, stD = valid && cb == kn;
        const int tL = col - 32 * kx, tD = col - 32 * kn;
#pragma unroll
        for (int rg = 0; rg < 32; rg += 8) {
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; q++)
                v[q] = valid ? ldg_stream(Arow + (size_t)(rg + q) * sp + col) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int r = rg + q;
                float a = acc[r];
                a = fmaf(v[q].x, xv.x, a);
                a = fmaf(v[q].y, xv.y, a);
                a = fmaf(v[q].z, xv.z, a);
                a = fmaf(v[q].w, xv.w, a);
                acc[r] = a;
                if (stL) {
                    float *L = sh.Lt[nbuf];
                    L[(tL + 0) * kTS + r] = v[q].x;
                    L[(tL + 1) * kTS + r] = v[q].y;
                    L[(tL + 2) * kTS + r] = v[q].z;
                    L[(tL + 3) * kTS + r] = v[q].w;
                }
                if (stD) {
                    float *D = sh.Dt[nbuf];
                    D[(tD + 0) * kTS + r] = v[q].x;
                    D[(tD + 1) * kTS + r] = v[q].y;
                    D[(tD + 2) * kTS + r] = v[q].z;
                    D[(tD + 3) * kTS + r] = v[q].w;
                }
            }
        }
    }
    // transpose-reduce: after 5 butterfly stages lane l holds the warp's sum for row l
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; i++) {
            const float send = upper ? acc[i] : acc[i + s];
            const float keep = upper ? acc[i + s] : acc[i];
            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    sh.Pw[nbuf][wid - 1][lane] = acc[0];
    if (wid == 1) sh.bts[nbuf][lane] = btb[32 * kn + lane];
}

__global__ void __launch_bounds__(kGsThreads, 2)
gs_kernel(int n_bins, const BinLayout *__restrict__ lay, const int32_t *__restrict__ order,
          int *__restrict__ counter, const float *__restrict__ A, const float *__restrict__ bt,
          int sweeps, float *__restrict__ x_out, float *__restrict__ x_map,
          const int32_t *__restrict__ keep_idx, int S) {
    extern __shared__ __align__(16) float xs[];
    __shared__ GsShared sh;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (;;) {
        if (tid == 0) sh.item = atomicAdd(counter, 1);
        __syncthreads();
        const int item = sh.item;
        if (item >= n_bins) break;
        const int bin = order ? order[item] : item;
        const BinLayout L = lay[bin];
        const int sp = L.sp, nk = L.nk, T = sp >> 5;
        const float *Ab = A + L.a_off;
        const float *btb = bt + L.v_off;
        for (int i = tid; i < sp; i += kGsThreads) xs[i] = 0.f;
        __syncthreads();
        const int total = sweeps * T;
        // prologue: P_0 (x = 0) and tiles for block 0; "previous" block is T-1
        if (wid > 0) gs_stage(sh, xs, Ab, btb, sp, T - 1, 0, 0, wid, lane);
        float xprev = 0.f;
        __syncthreads();
        for (int g = 0; g < total; g++) {
            const int k = g % T;
            if (wid == 0) {
                const int buf = g & 1, row0 = 32 * k;
                float acc = 0.f;
#pragma unroll
                for (int w = 0; w < kGsWarps - 1; w++) acc += sh.Pw[buf][w][lane];
                const float *Lb = sh.Lt[buf];
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
                    a0 = fmaf(Lb[(t + 0) * kTS + lane], __shfl_sync(0xffffffffu, xprev, t + 0), a0);
                    a1 = fmaf(Lb[(t + 1) * kTS + lane], __shfl_sync(0xffffffffu, xprev, t + 1), a1);
                    a2 = fmaf(Lb[(t + 2) * kTS + lane], __shfl_sync(0xffffffffu, xprev, t + 2), a2);
                    a3 = fmaf(Lb[(t + 3) * kTS + lane], __shfl_sync(0xffffffffu, xprev, t + 3), a3);
                }
                acc += (a0 + a1) + (a2 + a3);
                const float r = acc - sh.bts[buf][lane];
                const float *Db = sh.Dt[buf];
                const float dii = Db[lane * kTS + lane];
                const float invd = (row0 + lane < nk) ? 1.0f / dii : 0.f;
                float w = -r * invd;
                float xo = xs[row0 + lane];
                float dp[32];
#pragma unroll
                for (int t = 0; t < 32; t++) dp[t] = Db[t * kTS + lane] * invd;
#pragma unroll
                for (int t = 0; t < 32; t++) {
                    const float cand = fmaxf(w, -xo);
                    const float d = __shfl_sync(0xffffffffu, cand, t);
                    w = fmaf(-dp[t], d, w);
                    xo = (lane == t) ? xo + d : xo;
                }
                xs[row0 + lane] = xo;
                xprev = xo;
            } else if (g + 1 < total) {
                gs_stage(sh, xs, Ab, btb, sp, k, (g + 1) % T, (g + 1) & 1, wid, lane);
            }
            __syncthreads();
        }
        for (int i = tid; i < nk; i += kGsThreads) {
            const float v = xs[i];
            if (x_out) x_out[L.v_off + i] = v;
            if (x_map) x_map[(size_t)bin * S + keep_idx[(size_t)bin * S + i]] = v;
        }
        __syncthreads();
    }
}

__global__ void f64_to_f32_kernel(const double *__restrict__ src, float *__restrict__ dst, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = (float)src[i];
}

int launch_f64_to_f32(const double *src, float *dst, int n, cudaStream_t st) {
    f64_to_f32_kernel<<<(n + 255) / 256, 256, 0, st>>>(src, dst, n);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int gs_smem_bytes(int max_sp) { return max_sp * 4; }

int launch_gs(int n_bins, const BinLayout *lay_dev, int max_sp, const int32_t *order,
              int *counter, const float *A, const float *bt, int sweeps, float *x_out,
              float *x_map, const int32_t *keep_idx, int S, int num_sms, cudaStream_t st) {
    const int smem = gs_smem_bytes(max_sp);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(gs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_kernel, kGsThreads, smem);
    if (per_sm < 1) per_sm = 1;
    int grid = num_sms * per_sm;
    if (grid > n_bins) grid = n_bins;
    gs_kernel<<<grid, kGsThreads, smem, st>>>(n_bins, lay_dev, order, counter, A, bt, sweeps,
                                              x_out, x_map, keep_idx, S);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
