// k_psf.cu -- S5 PSF matrix on the compressed grid (+ S6 restriction of b), on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Eq. 9-12 restricted by Eq. 23, reading R1:
//   A~_ij = |e_i^H e_j|^2 / M^2  over the kept nodes i, j.
// Real-GEMM form of the complex Gram G = E~^H E~: with the per-node real vectors
//   X_i = [Re e_i ; Im e_i]  and  Z_i = [-Im e_i ; Re e_i]   (length 2M),
//   Re G_ij = X_i . X_j,   Im G_ij = Z_i . X_j,   A = (Re G^2 + Im G^2) / M^2.
//
// Precision: GS amplifies errors of A~ 10^3-10^4x in ill-conditioned bins, so
// A~ must be fp32-accurate -- an fp32-accumulated Gram (|dA| ~ 2e-7) already fails the 1e-3 map
// tolerance, and so does 3-pass TF32 with fp32 accumulation.  The Gram therefore runs as an
// exact integer product: every row X_i (and Z_i) is scaled by a power of two 2^q_i and split
// into kSl = 4 signed int8 digits, v 2^q = sum_s a_s 128^-(s+1) + rho, |rho| <= 2^-29, computed
// exactly in fp64.  The digit products P_st = D_s^T D_t are exact int32 sums on the tensor
// cores; the pairs with s + t = w share accumulator w (w = 0..3, pairs with s + t > 3 are
// below the residual and dropped), so Re G and Im G take 4 accumulators each:
//   G_ij = 2^-(q_i + q_j + 35) * (acc_0 2^21 + acc_1 2^14 + acc_2 2^7 + acc_3)   (int64, exact)
// The epilogue squares in fp64 and rounds A once to fp32: |dA| <~ 1e-8, the accuracy of the
// correctly rounded fp64 A.  G is computed exactly (integer), so A_ij and A_ji are bitwise
// equal and only output tiles touching the upper triangle are computed (the rest mirrored).
//
// Kernels
//  psf_slice_kernel  one warp per kept node: fp64 steering (sincospi of k d / pi, amplitude table),
//                    power-of-two row scale, int8 digits of X and Z written directly in the
//                    tensor-core operand layout; b~ = b[keep] (S6, fp64).
//  psf_tc_kernel     one CTA per 128 x 32 output tile (bin, I, J), two CTAs per SM (256 TMEM
//                    columns and 110 KB of shared memory each) so one CTA's epilogue overlaps the
//                    other's loads and MMAs: warp 0 streams the K steps (32 bytes of K per step:
//                    32 KB of A digits, 4 KB of B digits, two bulk copies) into a 3-deep ring;
//                    one thread of warp 1 issues the 20 MMAs (128x32x32, int8 -> s32) per step
//                    into 8 TMEM accumulators; warps 2-5 read TMEM and write A~ in the GS tile
//                    layout (symmetric tile layout, dwc_internal.cuh), from (i, j) and the
//                    mirror (j, i); the target tiles of the warp's 32x32 block are resolved once.
//
// Operand layout (per bin; rp = nk rounded up to 128 rows, kp = 2M rounded up to 32 bytes):
//   A side (8 matrices mt = X_0..X_3, Z_0..Z_3), byte of (mt, row r, k):
//     (k/32)*(rp*256) + (r/8)*2048 + mt*256 + ((k/16)%2)*128 + (r%8)*16 + k%16
//   B side (4 matrices t = X_0..X_3):
//     (k/32)*(rp*128) + (r/8)*1024 + t*256 + ((k/16)%2)*128 + (r%8)*16 + k%16
// so a 128-row A tile (64-row B tile) of one K step is a single contiguous 32 KB (8 KB) block,
// and in shared memory each matrix is the canonical K-major no-swizzle UMMA layout with
// LBO = 128 B and SBO = 2048 B (A) / 1024 B (B).
#include <math.h>

#include "dwc_internal.cuh"
#include "sm100.cuh"

namespace dwc {

using namespace sm100;

constexpr int kSl = 4;                     // int8 digits per value
constexpr int kTM = 128;                   // output tile rows (MMA M)
constexpr int kTN = 32;                    // output tile cols (MMA N) = one 32-column block
constexpr int kAMat = 2 * kSl;             // X_s, Z_s
constexpr int kBMat = kSl;                 // X_t
constexpr int kABytes = kTM * 32 * kAMat;  // 32 KB per K step
constexpr int kBBytes = kTN * 32 * kBMat;  //  4 KB per K step
constexpr int kNS = 3;                     // ring depth
constexpr int kTmemCols = 2 * kSl * kTN;   // 8 accumulators x 32 columns = 256
constexpr int kPsfThreads = 192;

__host__ __device__ inline size_t opa_index(int rp, int mt, int r, int k) {
    return (size_t)(k >> 5) * ((size_t)rp * 256) + (size_t)(r >> 3) * 2048 + mt * 256 + ((k >> 4) & 1) * 128 +
           (r & 7) * 16 + (k & 15);
}
__host__ __device__ inline size_t opb_index(int rp, int t, int r, int k) {
    return (size_t)(k >> 5) * ((size_t)rp * 128) + (size_t)(r >> 3) * 1024 + t * 256 + ((k >> 4) & 1) * 128 +
           (r & 7) * 16 + (k & 15);
}

// exact int8 digits of v in [-127/128, 127/128]: v = sum_s a[s] 128^-(s+1) + rho
__device__ __forceinline__ void digits(double v, int a[kSl]) {
#pragma unroll
    for (int s = 0; s < kSl; s++) {
        v *= 128.0;                // exact
        const double d = rint(v);  // |d| <= 127 for s = 0, <= 64 after
        a[s] = (int)d;
        v -= d;                    // exact (fraction of a double)
    }
}

__global__ void __launch_bounds__(256)
psf_slice_kernel(Geo g, const double *__restrict__ dist, const double *__restrict__ amp,
                 const double *__restrict__ freq, const BinLayout *__restrict__ lay,
                 const int32_t *__restrict__ keep_idx, const double *__restrict__ b, int kp,
                 int8_t *__restrict__ opA, int8_t *__restrict__ opB, double *__restrict__ rsc,
                 double *__restrict__ bt, double *__restrict__ wt) {
    const int bin = blockIdx.y;
    const BinLayout L = lay[bin];
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= L.rp) return;
    const int M = g.m;
    int8_t *A = opA + (size_t)L.r_off * kp * kAMat;
    int8_t *B = opB + (size_t)L.r_off * kp * kBMat;
    if (r < L.nk) {
        const int s = keep_idx[(size_t)bin * g.S + r];
        // power-of-two row scale from the amplitude bound |Re e|, |Im e| <= amp
        double amax = 0.0;
        for (int m = lane; m < M; m += 32) amax = fmax(amax, amp[(size_t)m * g.S + s]);
#pragma unroll
        for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        int e;
        const double f = frexp(amax, &e);         // amax = f 2^e, f in [0.5, 1)
        const int q = (f > 127.0 / 128.0) ? -e - 1 : -e;  // |v| 2^q <= 127/128
        const double kpi = 2.0 * freq[bin] / g.c0;   // k / pi: phase in half-turns
        for (int m = lane; m < M; m += 32) {
            const double d = dist[(size_t)m * g.S + s], a = amp[(size_t)m * g.S + s];
            double sn, cs;
            sincospi(kpi * d, &sn, &cs);
            int dr[kSl], di[kSl];
            const double er = a * cs, ei = -(a * sn);
            digits(ldexp(er, q), dr);
            digits(ldexp(ei, q), di);
            if (wt) wt[(size_t)L.r_off * M + (size_t)m * L.rp + r] = er * er + ei * ei;   // |e_mr|^2 (R20)
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, m)] = (int8_t)dr[t];            // X_t = [Re; Im]
                A[opa_index(L.rp, t, r, M + m)] = (int8_t)di[t];
                A[opa_index(L.rp, kSl + t, r, m)] = (int8_t)(-di[t]);   // Z_t = [-Im; Re]
                A[opa_index(L.rp, kSl + t, r, M + m)] = (int8_t)dr[t];
                B[opb_index(L.rp, t, r, m)] = (int8_t)dr[t];
                B[opb_index(L.rp, t, r, M + m)] = (int8_t)di[t];
            }
        }
        for (int kk = 2 * M + lane; kk < kp; kk += 32) {
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, kk)] = 0;
                A[opa_index(L.rp, kSl + t, r, kk)] = 0;
                B[opb_index(L.rp, t, r, kk)] = 0;
            }
        }
        if (lane == 0) {
            rsc[L.r_off + r] = ldexp(1.0, -2 * q - 35);
            if (b) bt[L.v_off + r] = b[(size_t)bin * g.S + s];
        }
    } else {
        if (wt)
            for (int m = lane; m < M; m += 32) wt[(size_t)L.r_off * M + (size_t)m * L.rp + r] = 0.0;
        for (int kk = lane; kk < kp; kk += 32) {
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, kk)] = 0;
                A[opa_index(L.rp, kSl + t, r, kk)] = 0;
                B[opb_index(L.rp, t, r, kk)] = 0;
            }
        }
        if (lane == 0) {
            rsc[L.r_off + r] = 0.0;
            if (b && r < L.sp) bt[L.v_off + r] = 0.0;
        }
    }
}

struct __align__(1024) PsfSmem {
    int8_t a[kNS][kABytes];
    int8_t b[kNS][kBBytes];
    double rcol[kTN];                      // row scales of the tile's columns
    unsigned long long full[kNS], empty[kNS], tmem_full;
    uint32_t tmem_base;
};

template <bool kDR>
__global__ void __launch_bounds__(kPsfThreads, 2)
psf_tc_kernel(int M, int kp, const int4 *__restrict__ tiles, const BinLayout *__restrict__ lay,
              const int8_t *__restrict__ opA, const int8_t *__restrict__ opB, const double *__restrict__ rsc,
              const double *__restrict__ wt, float *__restrict__ Aout) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    PsfSmem &sm = *reinterpret_cast<PsfSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 tl = tiles[blockIdx.x];  // (bin, I: 128-row block, J: 64-col block)
    const BinLayout L = lay[tl.x];
    const int nkc = kp >> 5;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kNS; i++) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        mbar_init(&sm.tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        if (lane == 0) {  // producer: one K step = one 32 KB A block + one 8 KB B block
            const int8_t *ga = opA + (size_t)L.r_off * kp * kAMat + (size_t)tl.y * (kTM / 8) * 2048;
            const int8_t *gb = opB + (size_t)L.r_off * kp * kBMat + (size_t)tl.z * (kTN / 8) * 1024;
            for (int kc = 0; kc < nkc; kc++) {
                const int st = kc % kNS;
                if (kc >= kNS) mbar_wait(&sm.empty[st], ((kc / kNS) - 1) & 1);
                mbar_expect_tx(&sm.full[st], kABytes + kBBytes);
                bulk_g2s(sm.a[st], ga + (size_t)kc * L.rp * 256, kABytes, &sm.full[st]);
                bulk_g2s(sm.b[st], gb + (size_t)kc * L.rp * 128, kBBytes, &sm.full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = idesc_i8(kTM, kTN);
            for (int kc = 0; kc < nkc; kc++) {
                const int st = kc % kNS;
                mbar_wait(&sm.full[st], (kc / kNS) & 1);
                tc_fence_after();
                const uint32_t sa = smem_u32(sm.a[st]), sb = smem_u32(sm.b[st]);
#pragma unroll
                for (int p = 0; p < 2; p++)
#pragma unroll
                    for (int s = 0; s < kSl; s++)
#pragma unroll
                        for (int t = 0; t + s < kSl; t++) {
                            const uint64_t ad = smem_desc(sa + (p * kSl + s) * 256, 128, 2048);
                            const uint64_t bd = smem_desc(sb + t * 256, 128, 1024);
                            mma_i8(tmem + (uint32_t)((p * kSl + s + t) * kTN), ad, bd, idesc,
                                   (kc > 0 || s > 0) ? 1u : 0u);
                        }
                mma_commit(&sm.empty[st]);  // frees the ring slot when these MMAs complete
            }
            mma_commit(&sm.tmem_full);
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (= tile rows); its 32 rows are one
        // row block of A~ (sp is a multiple of 32), the tile's 32 columns one column block
        const int q = warp & 3;
        const int il = q * 32 + lane;
        const int i = tl.y * kTM + il;
        const int j0 = tl.z * kTN;
        const int T = L.sp >> 5;
        const bool blk_ok = (tl.y * kTM + q * 32) < L.sp && j0 < L.sp;   // warp-uniform
        const double inv_m2 = 1.0 / ((double)M * (double)M);
        const double inv_dr = 1.0 / ((double)M * (double)M - (double)M);
        float *Ab = Aout + L.a_off;
        const int et = threadIdx.x - 64;   // 0..127
        if (et < kTN) sm.rcol[et] = rsc[L.r_off + min(j0 + et, L.rp - 1)];
        mbar_wait(&sm.tmem_full, 0);
        tc_fence_after();
        // diagonal removal (R20): Q_ij = sum_m |e_mi|^2 |e_mj|^2 in fp64 (row i per lane, the
        // 8 columns of a chunk are warp-uniform loads)
        const double *wb = kDR ? wt + (size_t)L.r_off * M : nullptr;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (blk_ok) {
            const double ri = rsc[L.r_off + i];
            // stored tiles of block (i/32, j0/32) and of its mirror: resolved once per warp
            int td[3], tm[3];
            const int nd = sym_targets(T, L.g, i >> 5, j0 >> 5, td);
            const int nm = sym_targets(T, L.g, j0 >> 5, i >> 5, tm);
#pragma unroll 1
            for (int jc = 0; jc < kTN; jc += 8) {
                int32_t acc[2 * kSl][8];
#pragma unroll
                for (int a = 0; a < 2 * kSl; a++)
                    tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * kTN + jc), acc[a]);
                tmem_ld_wait();
                float v[8];
                double q4[8];
#pragma unroll
                for (int c = 0; c < 8; c++) q4[c] = 0.0;
                if (kDR) {
                    for (int m = 0; m < M; m++) {
                        const double wi = wb[(size_t)m * L.rp + i];
                        const double2 *wc = reinterpret_cast<const double2 *>(wb + (size_t)m * L.rp + j0 + jc);
#pragma unroll
                        for (int c = 0; c < 4; c++) {
                            const double2 w2 = __ldg(wc + c);
                            q4[2 * c] = fma(wi, w2.x, q4[2 * c]);
                            q4[2 * c + 1] = fma(wi, w2.y, q4[2 * c + 1]);
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const long long gre = ((long long)acc[0][c] << 21) + ((long long)acc[1][c] << 14) +
                                          ((long long)acc[2][c] << 7) + (long long)acc[3][c];
                    const long long gim = ((long long)acc[4][c] << 21) + ((long long)acc[5][c] << 14) +
                                          ((long long)acc[6][c] << 7) + (long long)acc[7][c];
                    const double dre = (double)gre, dim = (double)gim;
                    const double sq = dre * dre + dim * dim;
                    if (kDR) {
                        const double a = (sq * ri * sm.rcol[jc + c] - q4[c]) * inv_dr;
                        v[c] = (float)(a > 0.0 ? a : 0.0);
                    } else {
                        v[c] = (float)(sq * ri * sm.rcol[jc + c] * inv_m2);
                    }
                }
                // direct (i, j0+jc..+7): coalesced over lanes; mirror (j0+jc..+7, i): two float4 per lane
#pragma unroll
                for (int u = 0; u < 3; u++) {
                    if (u >= nd) break;
                    float *dst = Ab + (size_t)td[u] * 1024 + (i & 31) + jc * 32;
#pragma unroll
                    for (int c = 0; c < 8; c++) dst[c * 32] = v[c];
                }
#pragma unroll
                for (int u = 0; u < 3; u++) {
                    if (u >= nm) break;
                    float4 *mir = reinterpret_cast<float4 *>(Ab + (size_t)tm[u] * 1024 + (i & 31) * 32 + jc);
                    mir[0] = make_float4(v[0], v[1], v[2], v[3]);
                    mir[1] = make_float4(v[4], v[5], v[6], v[7]);
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, kTmemCols);
}

int psf_kp(int m) { return ((2 * m + 31) / 32) * 32; }
size_t psf_opa_bytes(int m, int64_t rows) { return (size_t)rows * psf_kp(m) * kAMat; }
size_t psf_opb_bytes(int m, int64_t rows) { return (size_t)rows * psf_kp(m) * kBMat; }
int psf_tile_rows() { return kTM; }
int psf_tile_cols() { return kTN; }

int launch_psf(const Geo &g, const double *dist, const double *amp, int n_bins, const double *freq,
               const BinLayout *lay, const int32_t *keep_idx, const double *b, int max_rp, int n_tiles,
               const int4 *tiles, int8_t *opA, int8_t *opB, double *rsc, double *bt, double *wt, float *A,
               cudaStream_t st) {
    const int kp = psf_kp(g.m);
    dim3 grid((max_rp + 7) / 8, n_bins);
    psf_slice_kernel<<<grid, 256, 0, st>>>(g, dist, amp, freq, lay, keep_idx, b, kp, opA, opB, rsc, bt, wt);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    if (n_tiles <= 0) return 1;
    const size_t smem = sizeof(PsfSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(psf_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                cudaSuccess ||
            cudaFuncSetAttribute(psf_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                cudaSuccess)
            return -1;
        attr = true;
    }
    if (wt)
        psf_tc_kernel<true><<<n_tiles, kPsfThreads, smem, st>>>(g.m, kp, tiles, lay, opA, opB, rsc, wt, A);
    else
        psf_tc_kernel<false><<<n_tiles, kPsfThreads, smem, st>>>(g.m, kp, tiles, lay, opA, opB, rsc, nullptr, A);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace dwc
