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
//  psf_tc_kernel     persistent, one CTA per SM over the list of 128 x 32 output tiles (bin, I, J):
//                    warp 0 streams the K steps (32 bytes of K per step: 16 KB of A digits, 8 KB
//                    of B digits, two bulk copies) into an 8-deep ring, running ahead across
//                    tiles; one thread of warp 1 issues the 10 MMAs (128x64x32, int8 -> s32) per
//                    step into 4 TMEM level accumulators (Re | Im) of one of two buffers (2 x 256);
//                    8 epilogue warps drain the other buffer (TMEM reads, 64 B/cycle per SM, are
//                    the epilogue's bound) and write A~ in the GS tile layout (symmetric tile
//                    layout, dwc_internal.cuh) from (i, j) and the mirror (j, i); the target tiles
//                    of a warp's 32x32 block are resolved once per tile.
//
// Operand layout (per bin; rp = nk rounded up to 128 rows, kp = 2M rounded up to 32 bytes).
// Z sits on the B side (Im G_ij = -X_i . Z_j; only its square is used), and one MMA per digit
// pair (s, t) multiplies A = X_s (128 rows) with B = [X_t ; Z_t] (2 x 32 rows, N = 64), so its
// 64 accumulator columns hold Re (0..31) and Im (32..63) of digit level w = s + t:
//   A side (4 matrices s = X_0..X_3), byte of (s, row r, k):
//     (k/32)*(rp*128) + (r/8)*1024 + s*256 + ((k/16)%2)*128 + (r%8)*16 + k%16
//   B side (per 32-row block: digit t, part p = X / Z), byte of (t, p, row r, k):
//     (k/32)*(rp*256) + (r/32)*8192 + t*2048 + p*1024 + ((r/8)%4)*256 + ((k/16)%2)*128 + (r%8)*16 + k%16
// so a 128-row A tile (32-row B block) of one K step is a single contiguous 16 KB (8 KB) block,
// and in shared memory every operand is the canonical K-major no-swizzle UMMA layout with
// LBO = 128 B and SBO = 1024 B (A) / 256 B (B: the 64 rows of [X_t ; Z_t] are 8 groups of 8).
// Per K step 10 MMAs of 128x64x32 read 60 KB of shared memory (20 MMAs of 128x32x32 with Z on
// the A side read 100 KB: the tensor pipe was bound by the shared-memory operand reads).
#include <math.h>

#include "dwc_internal.cuh"
#include "sm100.cuh"

namespace dwc {

using namespace sm100;

constexpr int kSl = 4;                     // int8 digits per value
constexpr int kTM = 128;                   // output tile rows (MMA M)
constexpr int kTN = 32;                    // output tile cols (MMA N) = one 32-column block
constexpr int kAMat = kSl;                 // X_s
constexpr int kBMat = 2 * kSl;             // X_t, Z_t
constexpr int kABytes = kTM * 32 * kAMat;  // 16 KB per K step
constexpr int kBBytes = kTN * 32 * kBMat;  //  8 KB per K step
constexpr int kNS = 8;                     // ring depth (K steps in flight, across tiles)
constexpr int kTmemCols = kSl * 2 * kTN;   // 4 levels x (Re | Im) 64 columns = 256 (x 2 buffers)
constexpr int kPsfThreads = 320;   // producer, MMA, 8 epilogue warps
// TMEM column of accumulator a = p * kSl + w (p: Re / Im, w: digit level)
__device__ __forceinline__ constexpr int acc_col(int a) { return (a % kSl) * 2 * kTN + (a / kSl) * kTN; }

__host__ __device__ inline size_t opa_index(int rp, int s, int r, int k) {
    return (size_t)(k >> 5) * ((size_t)rp * 128) + (size_t)(r >> 3) * 1024 + s * 256 + ((k >> 4) & 1) * 128 +
           (r & 7) * 16 + (k & 15);
}
__host__ __device__ inline size_t opb_index(int rp, int t, int p, int r, int k) {
    return (size_t)(k >> 5) * ((size_t)rp * 256) + (size_t)(r >> 5) * 8192 + t * 2048 + p * 1024 +
           ((r >> 3) & 3) * 256 + ((k >> 4) & 1) * 128 + (r & 7) * 16 + (k & 15);
}

// int64 -> fp64 for |x| < 2^51 without the conversion unit (I2F.F64.S64 runs on the XU pipe,
// which ncu showed saturated in the epilogue): x + (2^52 + 2^51) as the bit pattern of a double
// in [2^52, 2^53) holds x exactly in its mantissa; subtracting 2^52 + 2^51 is exact.  The Gram
// accumulators combine to |G| < 2^46 (K <= 1024 products of |digit| <= 127, scaled by <= 2^21).
__device__ __forceinline__ double exact_i64_to_f64(long long x) {
    constexpr long long kMagic = 0x4338000000000000LL;   // bits of 2^52 + 2^51
    return __longlong_as_double(x + kMagic) - 6755399441055744.0;
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
                 double *__restrict__ bt, double *__restrict__ wt, const double *__restrict__ ampb,
                 double *__restrict__ rscb) {
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
        // power-of-two row scale from the amplitude bound |Re e|, |Im e| <= amp (per side: the
        // paper-literal PSF has v on the A side and g on the B side)
        auto scale_of = [&](const double *ap) {
            double amax = 0.0;
            for (int m = lane; m < M; m += 32) amax = fmax(amax, ap[(size_t)m * g.S + s]);
#pragma unroll
            for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            int e;
            const double f = frexp(amax, &e);         // amax = f 2^e, f in [0.5, 1)
            return (f > 127.0 / 128.0) ? -e - 1 : -e;  // |v| 2^q <= 127/128
        };
        const double *apb = ampb ? ampb : amp;
        const int q = scale_of(amp), qb = ampb ? scale_of(ampb) : q;
        const double kpi = 2.0 * freq[bin] / g.c0;   // k / pi: phase in half-turns
        for (int m = lane; m < M; m += 32) {
            const double d = dist[(size_t)m * g.S + s], a = amp[(size_t)m * g.S + s];
            double sn, cs;
            sincospi(kpi * d, &sn, &cs);
            int dr[kSl], di[kSl], gr[kSl], gi[kSl];
            const double er = a * cs, ei = -(a * sn);
            digits(ldexp(er, q), dr);
            digits(ldexp(ei, q), di);
            if (ampb) {
                const double ab = apb[(size_t)m * g.S + s];
                digits(ldexp(ab * cs, qb), gr);
                digits(ldexp(-(ab * sn), qb), gi);
            } else {
#pragma unroll
                for (int t = 0; t < kSl; t++) { gr[t] = dr[t]; gi[t] = di[t]; }
            }
            if (wt) wt[(size_t)L.r_off * M + (size_t)m * L.rp + r] = er * er + ei * ei;   // |e_mr|^2 (R20)
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, m)] = (int8_t)dr[t];            // X_t = [Re; Im]
                A[opa_index(L.rp, t, r, M + m)] = (int8_t)di[t];
                B[opb_index(L.rp, t, 0, r, m)] = (int8_t)gr[t];
                B[opb_index(L.rp, t, 0, r, M + m)] = (int8_t)gi[t];
                B[opb_index(L.rp, t, 1, r, m)] = (int8_t)(-gi[t]);      // Z_t = [-Im; Re]
                B[opb_index(L.rp, t, 1, r, M + m)] = (int8_t)gr[t];
            }
        }
        for (int kk = 2 * M + lane; kk < kp; kk += 32) {
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, kk)] = 0;
                B[opb_index(L.rp, t, 0, r, kk)] = 0;
                B[opb_index(L.rp, t, 1, r, kk)] = 0;
            }
        }
        if (lane == 0) {
            rsc[L.r_off + r] = ldexp(1.0, -2 * q - 35);
            if (rscb) rscb[L.r_off + r] = ldexp(1.0, -2 * qb - 35);
            if (b) bt[L.v_off + r] = b[(size_t)bin * g.S + s];
        }
    } else {
        if (wt)
            for (int m = lane; m < M; m += 32) wt[(size_t)L.r_off * M + (size_t)m * L.rp + r] = 0.0;
        for (int kk = lane; kk < kp; kk += 32) {
#pragma unroll
            for (int t = 0; t < kSl; t++) {
                A[opa_index(L.rp, t, r, kk)] = 0;
                B[opb_index(L.rp, t, 0, r, kk)] = 0;
                B[opb_index(L.rp, t, 1, r, kk)] = 0;
            }
        }
        if (lane == 0) {
            rsc[L.r_off + r] = 0.0;
            if (rscb) rscb[L.r_off + r] = 0.0;
            if (b && r < L.sp) bt[L.v_off + r] = 0.0;
        }
    }
}

struct __align__(1024) PsfSmem {
    int8_t a[kNS][kABytes];
    int8_t b[kNS][kBBytes];
    double rcol[2][kTN];                   // row scales of the tile's columns, per TMEM buffer
    unsigned long long full[kNS], empty[kNS], tmem_full[2], tmem_empty[2];
    uint32_t tmem_base;
};

// Persistent: CTA c takes tiles c, c + gridDim.x, ... (neighbouring CTAs work on neighbouring
// tiles at the same time, so a 128-row A block is read from HBM once and shared through L2).
// Two TMEM accumulator sets (2 x 256 columns): the MMAs of tile n+1 run while the epilogue
// warps drain tile n; the producer runs up to kNS K steps ahead across tile boundaries.
template <bool kDR>
__global__ void __launch_bounds__(kPsfThreads, 1)
psf_tc_kernel(int M, int kp, int n_tiles, const int4 *__restrict__ tiles, const BinLayout *__restrict__ lay,
              const int8_t *__restrict__ opA, const int8_t *__restrict__ opB, const double *__restrict__ rsc,
              const double *__restrict__ wt, float *__restrict__ Aout, float *__restrict__ Adense,
              const double *__restrict__ rscb) {
    const bool paper = rscb != nullptr;   // asymmetric paper-literal PSF: every tile, transposed out
    const double *rscc = paper ? rscb : rsc;   // column scales
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    PsfSmem &sm = *reinterpret_cast<PsfSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkc = kp >> 5;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kNS; i++) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&sm.tmem_full[b], 1);
            mbar_init(&sm.tmem_empty[b], 8);   // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 2 * kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        if (lane == 0) {  // producer: one K step = one 16 KB A block + one 8 KB B block
            int it = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int4 tl = tiles[tile];   // (bin, I: 128-row block, J: 32-column block)
                const BinLayout L = lay[tl.x];
                const int8_t *ga = opA + (size_t)L.r_off * kp * kAMat + (size_t)tl.y * kABytes;
                const int8_t *gb = opB + (size_t)L.r_off * kp * kBMat + (size_t)tl.z * kBBytes;
                for (int kc = 0; kc < nkc; kc++, it++) {
                    const int st = it % kNS;
                    if (it >= kNS) mbar_wait(&sm.empty[st], ((it / kNS) - 1) & 1);
                    mbar_expect_tx(&sm.full[st], kABytes + kBBytes);
                    bulk_g2s(sm.a[st], ga + (size_t)kc * L.rp * 32 * kAMat, kABytes, &sm.full[st]);
                    bulk_g2s(sm.b[st], gb + (size_t)kc * L.rp * 32 * kBMat, kBBytes, &sm.full[st]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = idesc_i8(kTM, 2 * kTN);
            int it = 0, n = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, n++) {
                const int bf = n & 1;
                if (n >= 2) mbar_wait(&sm.tmem_empty[bf], ((n >> 1) - 1) & 1);   // tile n-2 drained
                tc_fence_after();
                const uint32_t td = tmem + (uint32_t)(bf * kTmemCols);
                for (int kc = 0; kc < nkc; kc++, it++) {
                    const int st = it % kNS;
                    mbar_wait(&sm.full[st], (it / kNS) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(sm.a[st]), sb = smem_u32(sm.b[st]);
#pragma unroll
                    for (int s = 0; s < kSl; s++)
#pragma unroll
                        for (int t = 0; t + s < kSl; t++) {   // level s + t; (0, w) first initialises it
                            const uint64_t ad = smem_desc(sa + s * 256, 128, 1024);
                            const uint64_t bd = smem_desc(sb + t * 2048, 128, 256);
                            mma_i8(td + (uint32_t)((s + t) * 2 * kTN), ad, bd, idesc, (kc > 0 || s > 0) ? 1u : 0u);
                        }
                    mma_commit(&sm.empty[st]);  // frees the ring slot when these MMAs complete
                }
                mma_commit(&sm.tmem_full[bf]);
            }
        }
    } else {
        // epilogue, 8 warps: warp w reads TMEM lanes 32*(w%4) .. +31 (= tile rows; one row block of
        // A~, sp is a multiple of 32) and columns 16h .. 16h+15 of the tile's 32-column block,
        // h = (w-2)/4, as two 8-column chunks; the second chunk's TMEM loads are in flight while
        // the first is converted and stored (TMEM reads are the epilogue's bound)
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int et = threadIdx.x - 64;   // 0..255
        const double inv_m2 = 1.0 / ((double)M * (double)M);
        const double inv_dr = 1.0 / ((double)M * (double)M - (double)M);
        int n = 0;
        // tile metadata one tile ahead (two dependent global loads per tile, off the critical path)
        int4 tl_nx = make_int4(0, 0, 0, 0);
        BinLayout L_nx = {0, 0, 0, 0, 0, 0, 0, 0};
        if (blockIdx.x < n_tiles) {
            tl_nx = tiles[blockIdx.x];
            L_nx = lay[tl_nx.x];
        }
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, n++) {
            const int bf = n & 1;
            const int4 tl = tl_nx;
            const BinLayout L = L_nx;
            if (tile + (int)gridDim.x < n_tiles) {
                tl_nx = tiles[tile + gridDim.x];
                L_nx = lay[tl_nx.x];
            }
            const int i = tl.y * kTM + q * 32 + lane;
            const int j0 = tl.z * kTN;
            const int T = L.sp >> 5;
            const bool blk_ok = (tl.y * kTM + q * 32) < L.sp && j0 < L.sp;   // warp-uniform
            float *Ab = Aout + L.a_off;
            // rcol[bf] was last read for tile n-2, before every epilogue warp passed tile n-1's barrier
            if (et < kTN) sm.rcol[bf][et] = rscc[L.r_off + min(j0 + et, L.rp - 1)];
            asm volatile("bar.sync 1, 256;" ::: "memory");
            // diagonal removal (R20): Q_ij = sum_m |e_mi|^2 |e_mj|^2 in fp64 (row i per lane, the
            // 8 columns of a chunk are warp-uniform loads)
            const double *wb = kDR ? wt + (size_t)L.r_off * M : nullptr;
            mbar_wait(&sm.tmem_full[bf], (n >> 1) & 1);
            tc_fence_after();
            if (blk_ok) {
                const double ri = rsc[L.r_off + i];
                // stored tiles of block (i/32, j0/32) and of its mirror: resolved once per tile
                int td[3], tm[3], nd, nm;
                float *Dn = Adense ? Adense + L.d_off : nullptr;
                if (Adense) {
                    nd = nm = 0;   // residual-GS layout: the dense matrix holds everything
                } else {
                    nd = sym_targets_g(T, L.g, i >> 5, j0 >> 5, td);
                    nm = sym_targets_g(T, L.g, j0 >> 5, i >> 5, tm);
                }
                const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(bf * kTmemCols);
                auto emit = [&](int32_t (&acc)[2 * kSl][8], int jc) {
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
                        const double dre = exact_i64_to_f64(gre), dim = exact_i64_to_f64(gim);
                        const double sq = dre * dre + dim * dim;
                        if (kDR) {
                            const double a = (sq * ri * sm.rcol[bf][jc + c] - q4[c]) * inv_dr;
                            v[c] = (float)(a > 0.0 ? a : 0.0);
                        } else {
                            v[c] = (float)(sq * ri * sm.rcol[bf][jc + c] * inv_m2);
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
                    if (Dn) {
                        // dense row-major: row i (two float4 per lane; not for the asymmetric
                        // paper-literal PSF, which is stored transposed), and column i (rows
                        // j0+jc..+7, coalesced over the lanes: the mirror, or the transpose)
                        if (!paper) {
                            float4 *drow = reinterpret_cast<float4 *>(Dn + (size_t)i * L.sp + j0 + jc);
                            drow[0] = make_float4(v[0], v[1], v[2], v[3]);
                            drow[1] = make_float4(v[4], v[5], v[6], v[7]);
                        }
#pragma unroll
                        for (int c = 0; c < 8; c++) Dn[(size_t)(j0 + jc + c) * L.sp + i] = v[c];
                    }
                };
                // the registers of a tcgen05.ld are valid only after tcgen05.wait::ld: tie them to it
                auto settle = [](int32_t (&acc)[2 * kSl][8]) {
#pragma unroll
                    for (int a = 0; a < 2 * kSl; a++)
#pragma unroll
                        for (int c = 0; c < 8; c++) asm volatile("" : "+r"(acc[a][c]));
                };
                const int jA = 16 * h, jB = 16 * h + 8;
                int32_t acc0[2 * kSl][8], acc1[2 * kSl][8];
#pragma unroll
                for (int a = 0; a < 2 * kSl; a++) tmem_ld8(tb + (uint32_t)(acc_col(a) + jA), acc0[a]);
                tmem_ld_wait();
                settle(acc0);
#pragma unroll
                for (int a = 0; a < 2 * kSl; a++) tmem_ld8(tb + (uint32_t)(acc_col(a) + jB), acc1[a]);
                emit(acc0, jA);
                tmem_ld_wait();
                settle(acc1);
                emit(acc1, jB);
            }
            // TMEM buffer bf is free for tile n+2
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&sm.tmem_empty[bf]);
        }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * kTmemCols);
}

int psf_kp(int m) { return ((2 * m + 31) / 32) * 32; }
size_t psf_opa_bytes(int m, int64_t rows) { return (size_t)rows * psf_kp(m) * kAMat; }
size_t psf_opb_bytes(int m, int64_t rows) { return (size_t)rows * psf_kp(m) * kBMat; }
int psf_tile_rows() { return kTM; }
int psf_tile_cols() { return kTN; }

int launch_psf(const Geo &g, const double *dist, const double *amp, int n_bins, const double *freq,
               const BinLayout *lay, const int32_t *keep_idx, const double *b, int max_rp, int n_tiles,
               const int4 *tiles, int8_t *opA, int8_t *opB, double *rsc, double *bt, double *wt, float *A,
               float *Adense, cudaStream_t st, const double *ampb, double *rscb) {
    const int kp = psf_kp(g.m);
    dim3 grid((max_rp + 7) / 8, n_bins);
    psf_slice_kernel<<<grid, 256, 0, st>>>(g, dist, amp, freq, lay, keep_idx, b, kp, opA, opB, rsc, bt, wt, ampb,
                                           rscb);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    if (n_tiles <= 0) return 1;
    const size_t smem = sizeof(PsfSmem) + 1024;
    // queried and set on every call: both are per device, and a process may drive several
    int dev = 0, num_sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || num_sms < 1)
        return -1;
    const int n_cta = n_tiles < num_sms ? n_tiles : num_sms;
    if (raise_smem_limit(wt ? psf_tc_kernel<true> : psf_tc_kernel<false>, smem) != cudaSuccess)
        return -1;
    if (wt)
        psf_tc_kernel<true><<<n_cta, kPsfThreads, smem, st>>>(g.m, kp, n_tiles, tiles, lay, opA, opB, rsc, wt, A, Adense,
                                                              nullptr);
    else
        psf_tc_kernel<false><<<n_cta, kPsfThreads, smem, st>>>(g.m, kp, n_tiles, tiles, lay, opA, opB, rsc, nullptr, A,
                                                               Adense, rscb);
    return cudaPeekAtLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace dwc
