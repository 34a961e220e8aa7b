// k_rgs.cu -- S7 DAMAS Gauss-Seidel sweeps (+ S8 embed) in residual-update form.
//
// Eq. 13-14, readings R4, R11, R12, R18: for n = 1..sweeps, i ascending,
//   r_i = sum_j A_ij x_j - b_i   (x_j of this sweep for j < i, of the previous one for j > i)
//   x_i <- max(x_i - r_i / A_ii, 0),   x^0 = 0.
// The row order and the sweep order are kept exactly.  Instead of recomputing every row dot
// from A (S~^2 multiply-adds per sweep), the kernel keeps the residual vector r = A x - b of
// the current iterate on chip, in fp64, and whenever x_c changes by dx_c adds dx_c * A[c, :]
// (row c = column c, A is symmetric, reading R1) to it.  In exact arithmetic this is the same
// sequence of iterates; r only ever receives products of A (fp32) and exact x differences, so
// it equals A x - b of the fp32 iterate to fp64 rounding -- more accurate than an fp32 row dot.
// The work per sweep is (number of rows whose x changes) x S~ instead of S~^2: DAMAS solutions
// are sparse (measured on cfg2-cfg5: 5-25 % of the kept nodes change per sweep, fewer as the
// sweeps converge), and a row whose x does not change costs no memory traffic at all.
//
// Block formulation (B = 32 rows, T = sp/32 blocks, global step s solves block k = s mod T):
//  * solver (warp 0, lane = row of the block): the residuals of the block are
//      ac_i = r_i (stored, fp64 -> fp32) + carry_i
//    where carry holds the contributions of the changes of the last nsub = min(kSub, T-1)
//    steps, accumulated by the solver itself from the staged sub-diagonal tiles
//    A[k+d, k] (d = 1..nsub).  Then, in row order, the next row whose x changes is found with
//    one ballot over the block (the rows in between keep their x exactly), its change is
//    broadcast, and every row's ac (D tile) and carry (sub-diagonal tiles) are updated; a
//    block with q changing rows takes q + 1 ballot rounds instead of a 32-row chain.
//  * stream (warps 2..7): after the solver publishes the changes of step s (a list of
//    (c, dx_c), dx in fp64), add dx_c * A[c, :] to the stored r of every block except the
//    nsub blocks the solver carries (those are added after the solver has read them, at the
//    stream step of that block), reading the rows of the dense row-major A~ from L2/HBM.
//    The solver of step s needs stream step s - nsub - 1 complete: nsub steps of slack.
//  * producer (warp 1): bulk copies of the tiles D_k, A[k+1, k] .. A[k+nsub, k] of each step
//    into a 3-deep staging ring.
// One CTA per bin (every bin of a band runs concurrently when the band fits the SMs); bins
// are taken in descending S~ order from a global counter.
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "dwc_internal.cuh"

namespace dwc {

namespace {

constexpr int kRThreads = 256;
constexpr int kNStream = 6;          // stream warps 2..7
constexpr int kRStg = 3;             // band-tile staging depth (steps)
constexpr int kNList = 8;            // change-list ring (steps)
constexpr int kTileF = 1024;         // floats per 32x32 tile

struct __align__(16) RgsEntry {
    double dx;   // x_new - x_old, exact in fp64
    int c;       // row (bin-relative)
    int pad;
};

struct __align__(128) RgsSmem {
    float tiles[kRStg][kRgsSub + 1][kTileF];   // D_k, A[k+1,k], ..., A[k+kSub,k] (column-major tiles)
    RgsEntry list[kNList][32];
    int cnt[kNList];
    unsigned long long stg_full[kRStg], stg_empty[kRStg];
    unsigned long long dready[kNList], sdone[kNList];
    int item;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "R_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra R_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ float4 ldg_stream(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

}  // namespace

// r (fp64, sp) and x (fp32, sp) follow RgsSmem in dynamic shared memory.
__global__ void __launch_bounds__(kRThreads, 2)
rgs_kernel(int n_items, const int *__restrict__ order, const BinLayout *__restrict__ lay, int *__restrict__ counter,
           const float *__restrict__ Aband, const float *__restrict__ Adense, const double *__restrict__ bt, int sweeps,
           float *__restrict__ x_out, float *__restrict__ x_map, const int32_t *__restrict__ keep_idx, int S,
           unsigned long long *__restrict__ n_updates) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    RgsSmem &sh = *reinterpret_cast<RgsSmem *>(smem_raw);
    double *rs = reinterpret_cast<double *>(smem_raw + sizeof(RgsSmem));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long my_updates = 0;

    for (;;) {
        if (tid == 0) sh.item = atomicAdd(counter, 1);
        __syncthreads();
        const int item = sh.item;
        if (item >= n_items) break;
        const int bin = order[item];
        const BinLayout L = lay[bin];
        const int sp = L.sp, nk = L.nk, T = sp >> 5;
        const int nsub = min(kRgsSub, T - 1);
        const int total = sweeps * T;
        float *xs = reinterpret_cast<float *>(rs + sp);
        for (int i = tid; i < sp; i += kRThreads) {
            rs[i] = -bt[L.v_off + i];   // r = A x0 - b with x0 = 0 (b~ zero padded)
            xs[i] = 0.f;
        }
        if (tid == 0) {
            for (int i = 0; i < kRStg; i++) {
                mbar_init(&sh.stg_full[i], 1);
                mbar_init(&sh.stg_empty[i], 1);
            }
            for (int i = 0; i < kNList; i++) {
                mbar_init(&sh.dready[i], 1);
                mbar_init(&sh.sdone[i], kNStream);
            }
            fence_mbar_init();
        }
        __syncthreads();
        const float *Ab = Aband + L.a_off;     // band tiles: tile d*T + k = A[k][(k - d) mod T]
        const float *Ad = Adense + L.d_off;    // dense row-major sp x sp

        if (wid == 1) {
            // ================= producer: the band tiles of every step
            if (lane == 0) {
                for (int s = 0, k = 0; s < total; s++, k = (k + 1 == T) ? 0 : k + 1) {
                    const int sl = s % kRStg;
                    mbar_wait(&sh.stg_empty[sl], ((s / kRStg) & 1) ^ 1);
                    mbar_expect_tx(&sh.stg_full[sl], (uint32_t)(nsub + 1) * kTileF * 4);
                    bulk_g2s(sh.tiles[sl][0], Ab + (size_t)k * kTileF, kTileF * 4, &sh.stg_full[sl]);
                    for (int d = 1; d <= nsub; d++) {
                        int kd = k + d;
                        if (kd >= T) kd -= T;   // A[k+d, k] = tile d*T + (k+d)
                        bulk_g2s(sh.tiles[sl][d], Ab + ((size_t)d * T + kd) * kTileF, kTileF * 4, &sh.stg_full[sl]);
                    }
                }
            }
        } else if (wid == 0) {
            // ================= solver: lane = row 32k + lane of the current block
            float carry[kRgsSub];
#pragma unroll
            for (int d = 0; d < kRgsSub; d++) carry[d] = 0.f;
            for (int s = 0, k = 0; s < total; s++, k = (k + 1 == T) ? 0 : k + 1) {
                const int sl = s % kRStg, li = s % kNList;
                mbar_wait(&sh.stg_full[sl], (s / kRStg) & 1);
                const float *Dt = sh.tiles[sl][0];
                const int row = 32 * k + lane;
                // 1/A_ii as the dense-stream kernel forms it; padding rows never change
                const float invd = (row < nk) ? __frcp_rn(Dt[lane * 33]) : 0.f;
                float xo = xs[row];
                const int sw = s - nsub - 1;   // the stream step the stored r of this block needs
                if (sw >= 0) mbar_wait(&sh.sdone[sw % kNList], (sw / kNList) & 1);
                float ac = (float)rs[row] + carry[0];
                float acc[kRgsSub];
#pragma unroll
                for (int d = 0; d < kRgsSub; d++) acc[d] = 0.f;
                RgsEntry *lst = sh.list[li];
                int pos = 0, q = 0;
                for (;;) {
                    const float w = -ac * invd;
                    const float xn = xo + fmaxf(w, -xo);   // = max(xo - ac/A_ii, 0)
                    const unsigned m = __ballot_sync(0xffffffffu, lane >= pos && xn != xo);
                    if (m == 0u) break;
                    const int t = __ffs(m) - 1;
                    const float dv = __shfl_sync(0xffffffffu, xn - xo, t);
                    if (lane == t) {
                        lst[q].dx = (double)xn - (double)xo;
                        lst[q].c = row;
                        xo = xn;
                    }
                    ac = fmaf(Dt[t * 32 + lane], dv, ac);
#pragma unroll
                    for (int d = 0; d < kRgsSub; d++)
                        if (d < nsub) acc[d] = fmaf(sh.tiles[sl][d + 1][t * 32 + lane], dv, acc[d]);
                    pos = t + 1;
                    q++;
                }
                xs[row] = xo;
                if (lane == 0) sh.cnt[li] = q;
                my_updates += (unsigned long long)q;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sh.dready[li]);
                    mbar_arrive(&sh.stg_empty[sl]);
                }
                // contributions destined for the next nsub steps (fixed summation order)
#pragma unroll
                for (int d = 0; d + 1 < kRgsSub; d++) carry[d] = carry[d + 1] + acc[d];
                carry[kRgsSub - 1] = acc[kRgsSub - 1];
            }
        } else {
            // ================= stream warps: r += dx_c A[c, :] for every change of every step
            // warp w owns the 128-column chunks q = w, w + 6, ...; lane l the 4 columns 128q + 4l..+3
            const int w = wid - 2;
            const int nq = (sp + 127) >> 7;
            const int sub = lane >> 3;   // 32-column block inside the chunk
            for (int s = 0, k = 0; s < total; s++, k = (k + 1 == T) ? 0 : k + 1) {
                const int li = s % kNList;
                mbar_wait(&sh.dready[li], (s / kNList) & 1);
                const int n = sh.cnt[li];
                const RgsEntry *lst = sh.list[li];
                // blocks the solver carries for this step's changes (applied at their own steps)
                int kd[kRgsSub];
#pragma unroll
                for (int d = 0; d < kRgsSub; d++) {
                    int b = k + 1 + d;
                    while (b >= T) b -= T;
                    kd[d] = (d < nsub) ? b : -1;
                }
                for (int q = w; q < nq; q += kNStream) {
                    const int col = 128 * q + 4 * lane;
                    const int blk = 4 * q + sub;
                    bool on = col < sp;
#pragma unroll
                    for (int d = 0; d < kRgsSub; d++) on = on && blk != kd[d];
                    if (!on || n == 0) continue;
                    double2 *rp = reinterpret_cast<double2 *>(rs + col);
                    double2 r01 = rp[0], r23 = rp[1];
                    for (int e0 = 0; e0 < n; e0 += 8) {
                        float4 v[8];
                        double dx[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            if (e0 + u < n) {
                                const RgsEntry E = lst[e0 + u];
                                v[u] = ldg_stream(Ad + (size_t)E.c * sp + col);
                                dx[u] = E.dx;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            if (e0 + u < n) {
                                r01.x = fma((double)v[u].x, dx[u], r01.x);
                                r01.y = fma((double)v[u].y, dx[u], r01.y);
                                r23.x = fma((double)v[u].z, dx[u], r23.x);
                                r23.y = fma((double)v[u].w, dx[u], r23.y);
                            }
                        }
                    }
                    rp[0] = r01;
                    rp[1] = r23;
                }
                // the carried contributions of steps s-1 .. s-nsub to block k, now that the
                // solver has read it (its owner warp, in step order: no other warp writes block k)
                if (((k >> 2) % kNStream) == w && sub == (k & 3)) {
                    const int col = 32 * k + 4 * (lane & 7);
                    double2 *rp = reinterpret_cast<double2 *>(rs + col);
                    double2 r01 = rp[0], r23 = rp[1];
                    for (int d = 1; d <= nsub; d++) {
                        if (s - d < 0) break;
                        const int lj = (s - d) % kNList;
                        const int nd = sh.cnt[lj];
                        for (int e = 0; e < nd; e++) {
                            const RgsEntry E = sh.list[lj][e];
                            const float4 v = ldg_stream(Ad + (size_t)E.c * sp + col);
                            r01.x = fma((double)v.x, E.dx, r01.x);
                            r01.y = fma((double)v.y, E.dx, r01.y);
                            r23.x = fma((double)v.z, E.dx, r23.x);
                            r23.y = fma((double)v.w, E.dx, r23.y);
                        }
                    }
                    rp[0] = r01;
                    rp[1] = r23;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.sdone[li]);
            }
        }
        __syncthreads();
        // ---- output: x~ and the embedded full-grid map (S8)
        for (int i = tid; i < nk; i += kRThreads) {
            const float v = xs[i];
            if (x_out) x_out[L.v_off + i] = v;
            if (x_map) x_map[(size_t)bin * S + keep_idx[(size_t)bin * S + i]] = v;
        }
        __syncthreads();
    }
    if (n_updates && wid == 0 && lane == 0 && my_updates) atomicAdd(n_updates, my_updates);
}

size_t rgs_smem_bytes(int max_sp) { return sizeof(RgsSmem) + (size_t)max_sp * (8 + 4); }

int rgs_band_tiles(int T) { return (std::min(kRgsSub, T - 1) + 1) * T; }

int launch_rgs(int n_bins, const int *order_dev, const BinLayout *lay_dev, int max_sp, int *counter,
               const float *Aband, const float *Adense, const double *bt, int sweeps, float *x_out, float *x_map,
               const int32_t *keep_idx, int S, int num_sms, unsigned long long *n_updates, cudaStream_t st,
               GsLaunchInfo *info) {
    const size_t smem = (rgs_smem_bytes(max_sp) + 127) / 128 * 128;
    if (smem > 227 * 1024) return -1;
    if (cudaFuncSetAttribute(rgs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rgs_kernel, kRThreads, smem) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    int grid = std::min(n_bins, num_sms * per_sm);
    static const int cta_env = getenv("DWC_RGS_CTAS") ? atoi(getenv("DWC_RGS_CTAS")) : 0;   // experiment
    if (cta_env > 0 && cta_env < grid) grid = cta_env;
    if (grid < 1) grid = 1;
    if (info) {
        info->kernel = DWC_GS_KERNEL_RESIDUAL;
        info->xtra_tiles = 0;
        info->ctas = grid;
        info->max_group = 1;
    }
    rgs_kernel<<<grid, kRThreads, smem, st>>>(n_bins, order_dev, lay_dev, counter, Aband, Adense, bt, sweeps, x_out,
                                              x_map, keep_idx, S, n_updates);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// dwc_gs input conversion: dense row-major n x n (upper triangle read, reading R1) -> the
// padded dense sp x sp matrix and the band tiles of the residual kernel.
__global__ void rgs_convert_kernel(int n, int sp, const float *__restrict__ src, float *__restrict__ dense,
                                   float *__restrict__ band) {
    const int T = sp >> 5, nsub = min(kRgsSub, T - 1);
    const long total = (long)sp * sp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / sp), j = (int)(e - (long)(e / sp) * sp);
        const int lo = min(i, j), hi = max(i, j);
        const float v = (hi < n) ? src[(size_t)lo * n + hi] : 0.f;
        dense[e] = v;
        int d = (i >> 5) - (j >> 5);
        if (d < 0) d += T;
        if (d <= nsub) band[((size_t)d * T + (i >> 5)) * kTileF + (j & 31) * 32 + (i & 31)] = v;
    }
}

int launch_rgs_convert(int n, int sp, const float *src, float *dense, float *band, cudaStream_t st) {
    const long total = (long)sp * sp;
    const int blocks = (int)std::min<long>((total + 255) / 256, 148L * 32);
    rgs_convert_kernel<<<blocks, 256, 0, st>>>(n, sp, src, dense, band);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
