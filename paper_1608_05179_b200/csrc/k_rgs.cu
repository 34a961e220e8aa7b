// k_rgs.cu -- S7 DAMAS Gauss-Seidel sweeps (+ S8 embed) in residual-update form.
//
// Eq. 13-14, readings R4, R11, R12, R18: for n = 1..sweeps, i ascending,
//   r_i = sum_j A_ij x_j - b_i   (x_j of this sweep for j < i, of the previous one for j > i)
//   x_i <- max(x_i - r_i / A_ii, 0),   x^0 = 0.
// The row order and the sweep order are kept exactly.  Instead of recomputing every row dot
// from A (S~^2 multiply-adds per sweep), the kernel keeps the residual vector r = A x - b of
// the current iterate on chip, in fp64, and whenever x_c changes by dx_c adds dx_c * A[c, :]
// (row c = column c, A is symmetric, reading R1) to it.  In exact arithmetic this is the same
// sequence of iterates; r only receives products of A (fp32) with exact x differences (fp64), so
// it equals A x - b of the fp32 iterate to fp64 rounding -- more accurate than an fp32 row dot.
// The memory traffic per sweep is (rows whose x changes) x S~ instead of S~^2: DAMAS solutions
// are sparse (cfg2-cfg5: 5-25 % of the kept nodes change per sweep, fewer as the sweeps
// converge), and a row whose x does not change is not read at all.
//
// Block formulation (B = 32 rows, T = sp/32 blocks, global step s solves block k = s mod T; for
// alternating sweeps (reading R21) the visit sequence k = pos or T-1-pos):
//  * solver (warp 4; forward sweeps: lane l = row 32k + 31 - l, so the next row in order is the
//    highest ballot bit): the block's residuals are the stored r plus the carried contributions
//    of the changes of the last W = min(kRgsWin, T-1) steps, which the solver accumulates itself
//    (fp32, for its own residuals only).  In row order, the next row whose x changes is found
//    with one ballot over the block (the rows in between keep x exactly); its change is broadcast
//    and applied to every row's fp32 update w = -r/A_ii (from the block's diagonal tile, the only
//    load on the row-to-row chain) and to the carries of the blocks of the next W steps (from
//    row t's "panel": row t of A~ = column t, symmetric, over the columns of those blocks;
//    consumed one change later, off the chain).  A block with q changing rows takes q + 1
//    ballot rounds instead of a 32-row chain.  The changes (row, x before / after) are
//    published as the step's change list.
//  * panel producer (warp 0 beside the solver on its SM sub-partition; cluster mode warp 5): per step, cp.async copies of the block's 32x32 diagonal tile and of
//    the panels of the rows PREDICTED to change: those that changed at the block's previous visit
//    (before the first visit: the rows with b > 0, exactly the rows sweep 1 changes).  The carries
//    of a change outside the prediction are added after the block from global memory.
//  * row producer (warp 6): the exact fp64 dx of every listed change; bulk copies of the rows of
//    A~ (dense row-major) of every change into a 3-slot shared-memory ring, as batches.
//  * stream (warps 1..3, 5, 7; cluster mode 0..3, 7; 128-column chunks owned by warps, so every element of r has one
//    writer and a fixed update order): apply dx_c * A[c, :] (fp64) to r.  REGR (systems up to
//    kRegMaxSp points): r in the stream warps' registers; after its step j the owner of a block
//    publishes that block's r (fp32) for the solver step that reads "r after stream step j".
//    Otherwise r in shared memory, and the W blocks the solver carries accumulate into a pending
//    buffer added to r when the solver has read the block.  The solver of step s needs stream
//    step s - W - 1 complete: W steps of slack for the row fetch.
//  * cluster mode (CLU, systems above kRegMaxSp up to 8 x kRegMaxSp): the G CTAs of a cluster
//    share a bin, CTA c holding r of a contiguous range of chunks (REGR); only the leader runs
//    the solver and the panel producer; change lists go to the other CTAs, published r back to
//    the leader, by st.async completing on mbarriers (relaxed cross-CTA arrivals).
// One CTA (cluster) per bin; bins are taken in descending S~ order from a global counter.
// Numerics: the stream accumulates A~ (fp32, widened exactly) x dx (fp64) into r in fp64; the
// solver's carries and its row recurrence are fp32.
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dwc_internal.cuh"

namespace dwc {

namespace {

#ifndef RGS_NSTREAM
#define RGS_NSTREAM 5
#endif
constexpr int kNStream = RGS_NSTREAM;          // stream warps 1..3, 5, 7.. or 0..3, 7.. (see panel_warp)
constexpr int kRThreads = 32 * (kNStream + 3);
constexpr int kRMinBlocks = kNStream > 5 ? 1 : 2;
// warp roles: the latency-critical warps take the higher warp of each SMSP pair (w, w+4): the
// issue arbiter prefers the higher warp id
#ifndef RGS_PANEL_WARP
#define RGS_PANEL_WARP 0
#endif
constexpr int kWSolver = 4, kWRows = 6;
// the panel producer's warp: warps w and w + 4 share an SM sub-partition.  One CTA per bin: warp 0,
// beside the solver instead of a stream warp (a few copies per step; cut the solver's chain by
// 2 %: cfg3 bin 249 alone 20.85 -> 20.48 ms, band GS 20.98 -> 20.59 ms), warp 5 then streams.
// Cluster mode: warp 5 (warp 0 measured 5 % slower on cfg4's full grid, whose non-leader CTAs
// have no solver).  RGS_PANEL_WARP=5 keeps warp 5 everywhere (experiment).
template <bool CLU>
__device__ __forceinline__ constexpr int panel_warp() { return (CLU || RGS_PANEL_WARP == 5) ? 5 : 0; }
static_assert(RGS_PANEL_WARP == 5 || RGS_PANEL_WARP == 0, "panel producer: warp 0 or warp 5");
// stream warp index: warps 0..3, 7, 8, ... -> 0..3, 4, 5, ...; warp 5 takes index 0 when the panel
// producer is on warp 0
template <bool CLU>
__device__ __forceinline__ int stream_index(int wid) { return (panel_warp<CLU>() == 0 && wid == 5) ? 0 : (wid < 4 ? wid : wid - 3); }
#ifndef RGS_STG
#define RGS_STG 4
#endif
#ifndef RGS_NP
#define RGS_NP 8
#endif
#ifndef RGS_NLIST
#define RGS_NLIST 16
#endif
#ifndef RGS_NSLOT
#define RGS_NSLOT 3
#endif
constexpr int kRStg = RGS_STG;       // panel staging depth (steps)
constexpr int kNP = RGS_NP;          // panels staged per step (predicted rows beyond: loaded on demand)
constexpr int kPW = kRgsWin * 32;   // panel floats: blocks of steps s+1..s+W of one row
constexpr int kPPL = (kRgsWin * 8 + 31) / 32;   // 16-byte panel pieces per producer lane
// pending-buffer slots: the contributions to a block wait in the slot of the step that will read
// it, (step mod 16).  At stream step s the pending visits are those of steps s .. s + nsub; a slot is
// written for the visit at step S + 16 from stream step S + 16 - nsub >= S + 9 on, and the stream
// warps are at most nsub steps apart (the solver of step s waited for all of them to finish step
// s - nsub - 1), so a slot is never written for its next visit before the owner warp of the
// previous visit's block has committed it.
constexpr int kPendBlk = 16;
constexpr int kPendF = kPendBlk * 32;
static_assert(kRgsWin + 2 <= kPendBlk, "pending / published slots are reused after kPendBlk steps");
constexpr int kNList = RGS_NLIST;    // change-list ring (steps; > kRgsWin + 2)
static_assert(kNList > kRgsWin + 2, "the row producer must stay within the change-list ring");
constexpr int kCP = 2;               // stream: chunks held in registers per pass
constexpr int kNSlot = RGS_NSLOT;    // row ring: batches in flight
// register-resident r: 128-column chunks per stream warp -- kRegCh for systems up to kRegMaxSp
// points (and per CTA in cluster mode), kRegChWide for a single CTA up to kRegMaxSpWide (twice
// the registers: measured 3 % slower on cfg3's small systems, so only where it saves a cluster)
constexpr int kRegCh = 4, kRegChWide = 8, kRegChPair = 2;
constexpr int kRegMaxSpPair = 128 * kRegChPair * kNStream;    // 1280: two CTAs per SM (128 registers)
constexpr int kRegMaxSp = 128 * kRegCh * kNStream;            // 2560
constexpr int kRegMaxSpWide = 128 * kRegChWide * kNStream;    // 5120

struct __align__(16) RgsEntry {
    float xn, xo;   // x of the row after / before the change (dx = xn - xo, exact in fp64)
    int c;          // row (bin-relative)
    int pad;
};
__device__ __forceinline__ double entry_dx(const RgsEntry &e) { return (double)e.xn - (double)e.xo; }

struct __align__(128) RgsSmem {
    float diag[kRStg][32 * 32];       // the block's diagonal tile, row t: A[32k+t][32k .. 32k+31]
    float panel[kRStg][kNP][kPW];     // staged panels (ascending row), segment d-1: the block of step s+d
    unsigned smask[kRStg];            // rows (bits) whose panels a stage holds
    float sinv[kRStg][32];            // 1/A_ii of the stage's block (0 for padding rows)
    RgsEntry list[kNList][32];
    double dxs[kNList][32];           // dx of each listed change (written by the row producer)
    int cnt[kNList];
    unsigned long long stg_full[kRStg], stg_empty[kRStg];
    unsigned long long dready[kNList], sdone[kNList], dxready[kNList];
    unsigned long long rfull[kNSlot], rempty[kNSlot];   // row ring slots
    int item;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
#if defined(RGS_WATCHDOG) || defined(DWC_CHECKED)
// debug / checked build: a wait that has not completed after ~2^24 polls reports itself and traps
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    for (unsigned it = 0;; it++) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        if (it == (1u << 24)) {
            printf("[rgs watchdog] block %d warp %d lane %d stuck on barrier smem+%u parity %u\n", blockIdx.x,
                   threadIdx.x / 32, threadIdx.x % 32, smem_u32(b), parity);
            __trap();
        }
    }
}
#else
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "R_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra R_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
// ---- cluster mode (systems above kRegMaxSp: the residual's columns split over the CTAs of a cluster)
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_map(const void *p, uint32_t rank) {   // this smem address in CTA `rank`
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cl_s32(uint32_t raddr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}
// st.async: registers -> another CTA's shared memory, the bytes completing on its mbarrier
__device__ __forceinline__ void st_async_v4b32(uint32_t raddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                               uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t a, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(a), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t rbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx_cl(uint32_t rbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
                 : "memory");
}
// relaxed: the data the waiter reads travels by st.async on the same barrier, so the arrival needs
// no release (a release at cluster scope waits for the thread's outstanding stores)
__device__ __forceinline__ void mbar_arrive_tx_cl_relaxed(uint32_t rbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// fp32 -> fp64 for a non-negative float (every PSF: |.|^2 times positive scales) without the F2F
// unit (~15 lanes/clk/SM, the stream's bottleneck): the float's bits placed in a double with the
// exponent left at its fp32 bias, i.e. the value f * 2^-896 exactly -- zero and fp32 subnormals
// (as fp64 subnormals) included.  One ALU shift and one FMA-pipe shift.  The stream's dx carries
// the 2^896 (kDxScale): the DFMA forms the product D * dx * 2^896 = f * dx exactly, as before.
constexpr double kDxScale = 0x1p896;
__device__ __forceinline__ double nn_scaled(float f) {
    const unsigned u = __float_as_uint(f);
    return __hiloint2double((int)(u >> 3), (int)(u << 29));   // (IMAD.WIDE.U32 u * 2^29 measured slower)
}
__device__ __forceinline__ unsigned long long clk() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}

// The visit sequence (reading R21 for alternating sweeps): global step s visits block
// blk(s) = pos or T-1-pos (pos = s mod T; descending on odd sweeps when alt).  win_blk gives the
// block of step s+d (0 <= d < T) from s's (sweep p, position pos) without a division.
__device__ __forceinline__ bool sweep_fwd(int p, int alt) { return !(alt && (p & 1)); }
__device__ __forceinline__ int win_blk(int p, int pos, int d, int T, int alt) {
    int q = pos + d, pp = p;
    if (q >= T) { q -= T; pp++; }
    return sweep_fwd(pp, alt) ? q : T - 1 - q;
}

// Row-ring batching, identical in the row producer and the stream warps: the changes of a step
// are cut into units (row e, segment g) of seg floats (the last segment of a row shorter); one
// batch = up to upb units = one ring slot.
struct RingGeom {
    int seg;    // floats per unit slot (sp, or a multiple of 128 when rows are cut)
    int nseg;   // segments per row
    int upb;    // units per batch
};
__device__ __forceinline__ RingGeom ring_geom(int sp, int slot_floats) {
    RingGeom g;
    // whole rows when a row fits a slot (units of sp floats, 128-byte aligned), else segments
    // that start on 128-column chunk boundaries
    g.seg = (sp <= slot_floats) ? sp : (slot_floats / 128) * 128;
    g.nseg = (sp + g.seg - 1) / g.seg;
    g.upb = slot_floats / g.seg;
    return g;
}

}  // namespace

// Profile slots (DWC_RGS_PROF=1), item 0 = the largest bin: solver [0] tile wait, [1] stream
// wait, [2] ballot loop, [3] rest, [4] steps, [5] changes; stream warp 0 [8] list wait, [9]
// batch wait, [10] apply, [11] batches; row producer [12] ring wait, [13] issue; [14] total.
constexpr int kProfSlots = 24;
constexpr int kProfItems = 1024;   // then per item: start, end (globaltimer ns), bin, changes

// r (fp64, sp), the pending carried contributions (fp64, 16 blocks), x (fp32, sp), the prediction
// masks (T words) and the row ring (kNSlot slots of slot_floats) follow RgsSmem.
// Register-resident stream: the rows of one ring batch applied to the NC chunks a warp owns (all
// loads of a row issued together, independent fp64 chains per chunk element).
template <int NC, bool NN, int RC>
__device__ __forceinline__ void apply_rows(double (&r)[RC][4], const float *src, int sp, int nb, const double *dxs,
                                           int w) {
#pragma unroll 4
    for (int j = 0; j < nb; j++) {
        const double dx = dxs[j];
        const float *rowp = src + (size_t)j * sp;
        float4 v[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) v[c] = *reinterpret_cast<const float4 *>(rowp + 128 * (w + kNStream * c));
#pragma unroll
        for (int c = 0; c < NC; c++) {
            r[c][0] = fma(NN ? nn_scaled(v[c].x) : (double)v[c].x, dx, r[c][0]);
            r[c][1] = fma(NN ? nn_scaled(v[c].y) : (double)v[c].y, dx, r[c][1]);
            r[c][2] = fma(NN ? nn_scaled(v[c].z) : (double)v[c].z, dx, r[c][2]);
            r[c][3] = fma(NN ? nn_scaled(v[c].w) : (double)v[c].w, dx, r[c][3]);
        }
    }
}

// nch = the chunks a warp owns (0: a small system leaves this warp none)
template <bool NN, int RC>
__device__ __forceinline__ void apply_dispatch(int nch, double (&r)[RC][4], const float *src, int stride, int nb,
                                               const double *dxb, int w) {
    switch (nch) {
        case 1: apply_rows<1, NN, RC>(r, src, stride, nb, dxb, w); break;
        case 2: apply_rows<2, NN, RC>(r, src, stride, nb, dxb, w); break;
        case 3: apply_rows<3, NN, RC>(r, src, stride, nb, dxb, w); break;
        case 4: apply_rows<4, NN, RC>(r, src, stride, nb, dxb, w); break;
        default:
            if constexpr (RC > 4) {
                switch (nch) {
                    case 5: apply_rows<5, NN, RC>(r, src, stride, nb, dxb, w); break;
                    case 6: apply_rows<6, NN, RC>(r, src, stride, nb, dxb, w); break;
                    case 7: apply_rows<7, NN, RC>(r, src, stride, nb, dxb, w); break;
                    case 8: apply_rows<8, NN, RC>(r, src, stride, nb, dxb, w); break;
                    default: break;
                }
            }
            break;
    }
}

template <bool ALT, bool REGR, bool CLU, int RC = kRegCh>
#ifndef RGS_PAIR_MINB
#define RGS_PAIR_MINB kRMinBlocks
#endif
__global__ void __launch_bounds__(kRThreads, (REGR && RC > kRegChPair) ? 1 : (REGR ? RGS_PAIR_MINB : kRMinBlocks))
rgs_kernel(int n_items, const int *__restrict__ order, const BinLayout *__restrict__ lay, int *__restrict__ counter,
           const float *__restrict__ Adense, const double *__restrict__ bt, int sweeps, float *__restrict__ x_out,
           float *__restrict__ x_map, const int32_t *__restrict__ keep_idx, int S, int max_sp, int slot_floats,
           int use_ivs, int nonneg,
           unsigned long long *__restrict__ n_updates, unsigned long long *__restrict__ prof) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    RgsSmem &sh = *reinterpret_cast<RgsSmem *>(smem_raw);
    // r (shared-memory residual path only: registers when REGR)
    double *rs = reinterpret_cast<double *>(smem_raw + sizeof(RgsSmem));
    // carried contributions not yet in r (the visit at step S in slot S mod kPendBlk); with r in
    // registers: the published fp32 r of the block each solver step reads
    double *pend = rs + (REGR ? 0 : max_sp);
    float *xs = reinterpret_cast<float *>(pend + kPendF);
    // 1/A_ii of every row when shared memory allows (use_ivs), else per stage from the panel producer
    float *ivs = xs + max_sp;
    unsigned *pmask = reinterpret_cast<unsigned *>(ivs + (use_ivs ? max_sp : 0));   // per block: rows predicted to change
    float *ring = reinterpret_cast<float *>(pmask + ((max_sp / 32 + 31) & ~31));   // 128-byte aligned
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long my_updates = 0, my_bytes = 0;
    constexpr int alt = ALT ? 1 : 0;   // forward sweeps: the visit sequence folds to pos, pos+1, ...
    // cluster mode: the G CTAs of a cluster solve one bin; CTA c holds r of a contiguous range of
    // 128-column chunks (registers), fetches that slice of every changed row and applies it; the
    // leader (rank 0) also runs the solver and the panel producer.  The change lists reach the
    // other CTAs by st.async (completing on their dready barriers), the published r of each
    // block reaches the leader by st.async (completing on its sdone barriers).
    const uint32_t crank = CLU ? cl_rank() : 0u;
    const int G = CLU ? (int)cl_size() : 1;
    const bool leader = crank == 0;

    for (;;) {
        if (CLU) {
            if (leader && tid == 0) {
                const int it = atomicAdd(counter, 1);
                for (int c = 0; c < G; c++) st_cl_s32(cl_map(&sh.item, c), it);
            }
            cl_sync();
        } else {
            if (tid == 0) sh.item = atomicAdd(counter, 1);
            __syncthreads();
        }
        const int item = sh.item;
        if (item >= n_items) break;
        const int bin = order[item];
        const BinLayout L = lay[bin];
        const int sp = L.sp, nk = L.nk, T = sp >> 5;
        const int nsub = min(kRgsWin, T - 1);      // blocks the solver carries
        const int pw = nsub * 32;                  // panel floats
        const int total = sweeps * T;
        // this CTA's columns: chunks [q_lo, q_hi) of the nq 128-column chunks (all of them unless CLU)
        const int nq = (sp + 127) >> 7;
        const int nqc = CLU ? (nq + G - 1) / G : nq;
        const int q_lo = min(nq, (int)crank * nqc), q_hi = min(nq, q_lo + nqc);
        const int col0 = 128 * q_lo;
        const int swid = max(0, min(sp, 128 * q_hi) - col0);   // floats of a row this CTA applies
        const int rstride = CLU ? 128 * nqc : sp;               // floats per row in the ring
        const bool pf = prof != nullptr && item == 0 && leader;
        const unsigned long long t_item = pf ? clk() : 0ull;
        if (prof && leader && tid == 0 && item < kProfItems) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[kProfSlots + 4 * item] = t;
        }
        const float *Ad = Adense + L.d_off;    // dense row-major sp x sp
        for (int i = tid; i < sp; i += kRThreads) {
            const double b = bt[L.v_off + i];
            if (!REGR) rs[i] = -b;   // r = A x0 - b with x0 = 0 (b~ zero padded)
            xs[i] = 0.f;
            if (use_ivs) ivs[i] = (i < nk) ? __frcp_rn(Ad[(size_t)i * sp + i]) : 0.f;
            // sweep 1 from x0 = 0 changes exactly the rows with b~ > 0
            const unsigned m = __ballot_sync(0xffffffffu, i < nk && b > 0.0);
            if ((i & 31) == 0) pmask[i >> 5] = m;
        }
        for (int i = tid; i < kPendF; i += kRThreads) pend[i] = 0.0;
        if (nsub < kRgsWin) {   // the panel columns beyond the window stay 0 (the solver reads all segments)
            float *pz = &sh.panel[0][0][0];
            for (int i = tid; i < kRStg * kNP * kPW; i += kRThreads) pz[i] = 0.f;
        }
        if (tid == 0) {
            for (int i = 0; i < kRStg; i++) {
                mbar_init(&sh.stg_full[i], 33);   // 32 cp.async arrivals + the mask publisher
                mbar_init(&sh.stg_empty[i], 1);
            }
            for (int i = 0; i < kNList; i++) {
                mbar_init(&sh.dready[i], 1);
                mbar_init(&sh.sdone[i], kNStream * G);   // (CLU: every CTA's stream warps, at the leader)
                mbar_init(&sh.dxready[i], 1);
            }
            for (int h = 0; h < kNSlot; h++) {
                mbar_init(&sh.rfull[h], 1);
                mbar_init(&sh.rempty[h], kNStream);
            }
            fence_mbar_init();
        }
        if (CLU)
            cl_sync();   // every CTA's barriers initialised before any remote arrival
        else
            __syncthreads();
        const RingGeom rg = ring_geom(rstride, slot_floats);

        if (wid == panel_warp<CLU>()) {
            if (!CLU || leader) {   // (cluster: the leader's)
            // ================= panel producer: the panels of the rows predicted to change, as
            // 16-byte cp.async copies spread over the warp's lanes (a 1 KB panel is 2 instructions;
            // one bulk copy per panel cost ~80 cycles of issue on a single lane)
            unsigned long long pw_wait = 0, pw_issue = 0;
            float dnext = (!use_ivs && lane < nk) ? __ldg(Ad + (size_t)lane * sp + lane) : 1.f;
            for (int s = 0, p = 0, pos = 0; s < total; s++, pos = (pos + 1 == T) ? 0 : pos + 1, p += (pos == 0)) {
                const int k = sweep_fwd(p, alt) ? pos : T - 1 - pos;
                const int sl = s % kRStg;
                const unsigned long long t0 = pf ? clk() : 0ull;
                mbar_wait(&sh.stg_empty[sl], ((s / kRStg) & 1) ^ 1);
                const unsigned long long t1 = pf ? clk() : 0ull;
                // the mask of block k as the solver left it at its previous visit, when that visit
                // is certainly complete (>= kRStg steps ago: this stage slot was released by the
                // solver's step s - kRStg); a visit closer than that (systems of T < kRStg blocks,
                // the turn of alternating sweeps) may still be running, and which value a racing read
                // saw would decide which carries take the panel path and which the miss path -- a
                // different fp32 summation order, so results would depend on timing.  Those steps
                // stage the block's first kNP rows instead (deterministic).
                const int dprev = ALT ? 2 * pos + 1 : T;   // steps since block k's previous visit
                unsigned m = (p == 0 || dprev >= kRStg) ? *(volatile unsigned *)&pmask[k] : ~0u;
                DWC_DCHECK(k >= 0 && k < T, "panel producer: block");
                unsigned st = 0;
                for (int n = 0; m && n < kNP; n++) {
                    st |= m & (0u - m);   // lowest set bit
                    m &= m - 1;
                }
                // the diagonal tile: 32 rows x 128 B, 8 pieces of 16 B per lane (row offsets in 32
                // bits from the block's row base: t * sp < 2^31)
                const float *blk = Ad + (size_t)(32 * k) * sp;
                {
                    const float *dg = blk + 32 * k + 4 * (lane & 7);
                    const uint32_t sd = smem_u32(&sh.diag[sl][32 * (lane >> 3) + 4 * (lane & 7)]);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int r = 4 * i + (lane >> 3);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sd + 4 * 128 * i), "l"(dg + r * sp)
                                     : "memory");
                    }
                }
                // panel segment d-1 (pieces 8(d-1) .. 8(d-1)+7) holds the columns of the block of step s+d
                const int q4 = pw >> 2;   // 16-byte pieces per panel
                // lane piece 32i + lane (i < kPPL) is segment 4i + (lane >> 3)
                const float *pc[kPPL];
                bool on[kPPL];
#pragma unroll
                for (int i = 0; i < kPPL; i++) {
                    const int d = 1 + 4 * i + (lane >> 3);
                    pc[i] = blk + 32 * win_blk(p, pos, d < T ? d : 0, T, alt) + 4 * (lane & 7);
                    on[i] = 32 * i + lane < q4;
                }
                const uint32_t sp0 = smem_u32(&sh.panel[sl][0][4 * lane]);
                unsigned mm = st;
                for (int j = 0; mm; j++) {
                    const int t = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const int ro = t * sp;
#pragma unroll
                    for (int i = 0; i < kPPL; i++)
                        if (on[i])
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sp0 + 4 * kPW * j + 512 * i),
                                         "l"(pc[i] + ro)
                                         : "memory");
                }
                // 1/A_ii of the block's rows, as the dense-stream kernel forms it (padding rows: 0);
                // the diagonal of the next step's block is loaded one step ahead
                if (!use_ivs) {
                    const int rw = 32 * k + lane;
                    sh.sinv[sl][lane] = (rw < nk) ? __frcp_rn(dnext) : 0.f;
                    const int rn = 32 * win_blk(p, pos, 1 < T ? 1 : 0, T, alt) + lane;
                    dnext = (rn < nk) ? __ldg(Ad + (size_t)rn * sp + rn) : 1.f;
                }
                // each lane's copies complete on stg_full (32 async arrivals + lane 0's below)
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sh.stg_full[sl]))
                             : "memory");
                __syncwarp();
                if (lane == 0) {
                    sh.smask[sl] = st;
                    mbar_arrive(&sh.stg_full[sl]);
                }
                if (pf) { pw_wait += t1 - t0; pw_issue += clk() - t1; }
            }
            if (pf && lane == 0) { prof[7] = pw_wait; prof[15] = pw_issue; }
            }
        } else if (wid == kWRows) {
            // ================= row producer: the exact dx of every change (all lanes), then the rows
            // of every step's changes into the ring (one bulk copy per lane: issued from one lane
            // they took ~170 cycles each)
            unsigned long long tw = 0, ti = 0;
            int b = 0;   // global batch counter (ring slot = b % kNSlot)
            for (int s = 0; s < total; s++) {
                const int li = s % kNList;
                mbar_wait(&sh.dready[li], (s / kNList) & 1);
                const int n = sh.cnt[li];
                DWC_DCHECK(n >= 0 && n <= 32, "row producer: change-list length");
                if (lane < n) sh.dxs[li][lane] = entry_dx(sh.list[li][lane]) * ((REGR && nonneg) ? kDxScale : 1.0);   // exact
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.dxready[li]);
                const int nu = swid > 0 ? n * rg.nseg : 0;   // (a CTA without columns fetches nothing)
                for (int u0 = 0; u0 < nu; u0 += rg.upb, b++) {
                    const int h = b % kNSlot;
                    const unsigned long long t0 = pf ? clk() : 0ull;
                    const int nb = min(rg.upb, nu - u0);
                    float *dst = ring + (size_t)h * slot_floats;
                    if (lane == 0) {
                        mbar_wait(&sh.rempty[h], ((b / kNSlot) & 1) ^ 1);
                        DWC_DCHECK(h < kNSlot && nb >= 1 && (rg.nseg > 1 || nb * rstride <= slot_floats) &&
                                       (rg.nseg == 1 || nb * rg.seg <= slot_floats),
                                   "row producer: ring slot overflow");
                    }
                    const unsigned long long t1 = pf ? clk() : 0ull;
                    if (rg.nseg == 1) {   // whole rows (CLU: this CTA's slice of them), one copy per lane
                        if (lane == 0) mbar_expect_tx(&sh.rfull[h], (uint32_t)nb * swid * 4);
                        __syncwarp();   // (the slot is free: every lane's copy may start)
                        if (lane < nb)
                            bulk_g2s(dst + (size_t)lane * rstride, Ad + (size_t)sh.list[li][u0 + lane].c * sp + col0,
                                     (uint32_t)swid * 4, &sh.rfull[h]);
                    } else if (lane == 0) {
                        uint32_t bytes = 0;
                        for (int j = 0; j < nb; j++) {
                            const int u = u0 + j, e = u / rg.nseg, g = u - e * rg.nseg;
                            bytes += (uint32_t)min(rg.seg, sp - g * rg.seg) * 4;
                        }
                        mbar_expect_tx(&sh.rfull[h], bytes);
                        for (int j = 0; j < nb; j++) {
                            const int u = u0 + j, e = u / rg.nseg, g = u - e * rg.nseg;
                            const int c = sh.list[li][e].c;
                            bulk_g2s(dst + (size_t)j * rg.seg, Ad + (size_t)c * sp + (size_t)g * rg.seg,
                                     (uint32_t)min(rg.seg, sp - g * rg.seg) * 4, &sh.rfull[h]);
                        }
                    }
                    if (pf) { tw += t1 - t0; ti += clk() - t1; }
                }
                __syncwarp();
            }
            if (pf && lane == 0) { prof[12] = tw; prof[13] = ti; }
        } else if (wid == kWSolver) {
          if (!CLU || leader) {   // (cluster: the leader's)
            // ================= solver: lane = row 32k + rl of the current block, rl = 31 - lane for
            // forward sweeps (the next changing row in order is then the HIGHEST set ballot bit: one
            // FLO instead of BREV + FLO on the row-to-row chain), rl = lane in the alternating
            // kernel.  Its carries are
            // fp32 (the residual only needs fp32 for the chain); the exact fp64 contributions are
            // committed to r by the stream warps (pending buffer, see below).
            const int rl = ALT ? lane : (lane ^ 31);   // this lane's row in the block
            float carry[kRgsWin];
#pragma unroll
            for (int d = 0; d < kRgsWin; d++) carry[d] = 0.f;
            unsigned long long tt = 0, tsd = 0, tl = 0, tr = 0, nch = 0, nmiss = 0, e_sd = 0, e_l = 0, e_ch = 0, nzero = 0, nwait = 0;
            for (int s = 0, p = 0, pos = 0; s < total; s++, pos = (pos + 1 == T) ? 0 : pos + 1, p += (pos == 0)) {
                const unsigned long long t0 = pf ? clk() : 0ull;
                const bool fwd = sweep_fwd(p, alt);
                const int k = fwd ? pos : T - 1 - pos;
                const int sl = s % kRStg, li = s % kNList;
                const int row = 32 * k + rl;
                const float x0 = xs[row];   // this row's x before the step (its list entry's xo)
                float xo = x0;
                // the carry of step s + d goes to the block of step s + d only at its first occurrence
                // in the window (a block visited twice in the window -- the turn of alternating
                // sweeps -- gets the contribution committed at its first visit)
                unsigned vmask = (1u << nsub) - 1u;   // bit d-1: step s+d is the first visit of its block in the window
                // alternating sweeps (the window holds at most one turn, nsub < T): step s+dt is the
                // first of the next sweep, which walks the blocks back, so step s+d (d >= dt) revisits
                // the block of step s+2dt-1-d: not a first occurrence for dt <= d <= 2dt-2.  Block k
                // itself was last visited at step s-2pos-1 (the previous sweep's mirror position).
                int vprev = -1;   // the last visit of block k within the window behind, else -1
                if (ALT) {
                    const int dt = T - pos;
                    if (dt <= nsub && dt >= 2) vmask &= ~(((1u << (dt - 1)) - 1u) << (dt - 1));
                    if (p >= 1 && 2 * pos + 1 <= nsub) vprev = s - 2 * pos - 1;
                }
                mbar_wait(&sh.stg_full[sl], (s / kRStg) & 1);
                const unsigned smk = sh.smask[sl];
                const float invd = use_ivs ? ivs[row] : sh.sinv[sl][rl];
                const unsigned long long t1 = pf ? clk() : 0ull;
                const int sw = max(s - nsub - 1, vprev);   // the stream step the stored r of this block needs
                if (sw >= 0) mbar_wait(&sh.sdone[sw % kNList], (sw / kNList) & 1);
                const unsigned long long t2 = pf ? clk() : 0ull;
                // r of the block as of stream step sw (before any stream step: r = -b~)
                const float ac = (REGR ? (sw >= 0 ? reinterpret_cast<const float *>(pend)[32 * (s & (kPendBlk - 1)) + rl]
                                                  : (float)-bt[L.v_off + row])
                                       : (float)rs[row]) + carry[0];
                float acc[kRgsWin];
#pragma unroll
                for (int d = 0; d < kRgsWin; d++) acc[d] = 0.f;
                RgsEntry *lst = sh.list[li];
                int pos_r = fwd ? 0 : 31, q = 0;   // next row of the block in sweep order
                unsigned chg = 0;
                // the projected update is carried as w = -ac/A_ii: a change dv of row t moves it by
                // -(dv/A_ii) A[row][32k+t], read from the staged diagonal tile (row t, by symmetry /
                // the transposed store) -- the only shared-memory load on the row-to-row chain
                float w = -ac * invd;
                const float *dgt = sh.diag[sl] + rl;
                const float *dgt_last = dgt + 32 * 31;
                // the previous change's panel values and dv: consumed one iteration later, after the
                // next ballot, so that the chain never waits for the panel loads
                float pvp[kRgsWin], dvp = 0.f;
#pragma unroll
                for (int d = 0; d < kRgsWin; d++) pvp[d] = 0.f;
                for (;;) {
                    const float xn = xo + fmaxf(w, -xo);   // = max(xo - ac/A_ii, 0)
                    const float dl = xn - xo;              // this row's change if it is the next one
                    const unsigned m = __ballot_sync(0xffffffffu, (fwd ? rl >= pos_r : rl <= pos_r) && xn != xo);
                    // the row (in the block) of the next change: forward sweeps take the lowest row,
                    // i.e. (ALT = false, rl = 31 - lane) the highest ballot bit
                    int tl;   // the highest ballot bit (bfind = FLO; -1 when m == 0): the lane of the next
                    // change for forward sweeps, used as is on the chain (shuffle source, own-lane test)
                    asm("bfind.u32 %0, %1;" : "=r"(tl) : "r"(m));
                    const int t = !ALT ? 31 - tl : fwd ? __ffs(m) - 1 : tl;
                    DWC_DCHECK(m == 0u || (t >= 0 && t < 32 && !((chg >> t) & 1u)), "solver: a row changes twice in one visit");
#pragma unroll
                    for (int d = 0; d < kRgsWin; d++)   // (forward: pv = 0 beyond nsub)
                        if (!ALT || ((vmask >> d) & 1u)) acc[d] = fmaf(pvp[d], dvp, acc[d]);
                    if (m == 0u) break;
                    const float dv = __shfl_sync(0xffffffffu, dl, ALT ? t : tl);
                    const float a0 = ALT ? dgt[32 * t] : dgt_last[-32 * tl];   // (row t = 31 - tl: one IMAD)
                    if (ALT ? rl == t : lane == tl) xo = xn;   // (the list entry is written after the block, below)
#ifdef RGS_SCALE_A0
                    w = fmaf(dv, a0 * -invd, w);   // (the scale of the tile entry off the shuffle's path)
#else
                    w = fmaf(-invd * dv, a0, w);
#endif
                    // off the chain: the carries, from row t's staged panel (element 32(d-1) + lane =
                    // A[32k+t][32 blk(s+d) + lane] = A[32 blk(s+d) + lane][32k+t]; segments beyond nsub
                    // are zero); a row not staged is added after the block from global memory
                    const bool stg = (smk >> t) & 1u;
                    const float *pr = sh.panel[sl][stg ? __popc(smk & ((1u << t) - 1u)) : 0] + rl;
                    dvp = stg ? dv : 0.f;
#pragma unroll
                    for (int d = 0; d < kRgsWin; d++) pvp[d] = pr[32 * d];
                    chg |= 1u << t;
                    pos_r = fwd ? t + 1 : t - 1;
                    q++;
                }
                // the carries of the changed rows that were not staged (the prediction missed: 1 % of
                // the changes on cfg3, 30 % on the noisy cfg5), from global memory, four rows' loads
                // in flight at a time
                for (unsigned mm = chg & ~smk; mm; mm &= mm - 1) {
                    const int t = __ffs(mm) - 1;
                    const float dv = __shfl_sync(0xffffffffu, xo - x0, ALT ? t : t ^ 31);
                    const float *rw = Ad + (size_t)(32 * k + t) * sp + rl;
#pragma unroll
                    for (int d = 0; d < kRgsWin; d++)
                        if (d < nsub && (!ALT || ((vmask >> d) & 1u)))
                            acc[d] = fmaf(__ldg(rw + 32 * win_blk(p, pos, d + 1, T, alt)), dv, acc[d]);
                    nmiss++;
                }
                const unsigned long long t3 = pf ? clk() : 0ull;
                xs[row] = xo;
                DWC_DCHECK(q == __popc(chg) && q <= 32, "solver: change count");
                DWC_DCHECK(sw < s && (sw < 0 || sw >= s - nsub - 1), "solver: stored-residual step");
                // the block's changes in sweep order (each row changes at most once per visit)
                if ((chg >> rl) & 1u) {
                    const int e = fwd ? __popc(chg & ((1u << rl) - 1u)) : __popc(chg >> rl) - 1;
                    lst[e].xn = xo;
                    lst[e].xo = x0;
                    lst[e].c = row;
                    if (CLU)   // the other CTAs' copies, completing on their dready[li]
                        for (int c = 1; c < G; c++)
                            st_async_v4b32(cl_map(&lst[e], c), __float_as_uint(xo), __float_as_uint(x0), (uint32_t)row, 0u,
                                           cl_map(&sh.dready[li], c));
                }
                if (lane == 0) {
                    sh.cnt[li] = q;
                    pmask[k] = chg;   // the prediction for the next visit
                }
                if (CLU && lane >= 1 && lane < G) {   // lane c: CTA c's count and dready arrival (the list
                    // bytes complete on it too; the arrival needs no release: everything CTA c reads
                    // arrives by st.async)
                    st_async_b32(cl_map(&sh.cnt[li], lane), (uint32_t)q, cl_map(&sh.dready[li], lane));
                    mbar_arrive_tx_cl_relaxed(cl_map(&sh.dready[li], lane), 16u * (uint32_t)q + 4u);
                }
                my_updates += (unsigned long long)q;
                my_bytes += (unsigned long long)q * sp * 4;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sh.dready[li]);
                    mbar_arrive(&sh.stg_empty[sl]);
                }
#pragma unroll
                for (int d = 0; d + 1 < kRgsWin; d++) carry[d] = carry[d + 1] + acc[d];
                carry[kRgsWin - 1] = acc[kRgsWin - 1];
                if (pf) {
                    tt += t1 - t0; tsd += t2 - t1; tl += t3 - t2; tr += clk() - t3;
                    if (10 * s < total) { e_sd += t2 - t1; e_l += t3 - t2; e_ch += q; }   // the first 10 % of the steps
                    nzero += (q == 0);
                    nwait += (t2 - t1 > 100);
                }
                nch += q;
            }
            if (CLU)   // the last steps' published-r bytes (st.async) have landed before the barriers are re-initialised
                for (int s = max(0, total - kNList); s < total; s++) mbar_wait(&sh.sdone[s % kNList], (s / kNList) & 1);
            if (prof && lane == 0 && item < kProfItems) prof[kProfSlots + 4 * item + 3] = nch;
            if (pf && lane == 0) { prof[0] = tt; prof[1] = tsd; prof[2] = tl; prof[3] = tr; prof[4] = total; prof[5] = nch; prof[6] = nmiss;
                                    prof[16] = e_sd; prof[17] = e_l; prof[18] = e_ch; prof[19] = nzero; prof[20] = nwait; }
          }
        } else if (REGR) {
            // ================= stream warps, r in registers (sp <= kRegMaxSp, whole rows in the
            // ring): r += dx_c A[c, :] for every change of every step.  Warp w owns the 128-column
            // chunks q = w, w + 5, ... (at most kRegCh); lane l columns 128q + 4l .. +3.  After its
            // step j the owner of each block publishes that block's r (8 lanes x 4 fp64) for the
            // solver step s' whose stored residual is "r after stream step j" (s' = j + nsub + 1,
            // or for alternating sweeps the revisit s' whose last visit was step j), in the
            // step-indexed slot s' mod 16 (the pend buffer)
            // (CLU: the chunks of this CTA's slice, local index ql = q - q_lo)
            const int w = stream_index<CLU>(wid);
            const int nch = max(0, (q_hi - q_lo - w + kNStream - 1) / kNStream);   // chunks this warp owns
            DWC_DCHECK(nch <= RC && rg.nseg == 1, "stream: register chunks");
            unsigned long long tlw = 0, tbw = 0, tap = 0, nb_all = 0;
            uint32_t pub_bytes = 0;   // (CLU) bytes this warp published during the current step
            double r[RC][4];
#pragma unroll
            for (int c = 0; c < RC; c++) {
                const int col = col0 + 128 * (w + kNStream * c) + 4 * lane;
#pragma unroll
                for (int e = 0; e < 4; e++) r[c][e] = (col + e < sp) ? -bt[L.v_off + col + e] : 0.0;
            }
            // the stored r of solver step s' = s + d: r after stream step s'-nsub-1, or for a revisit
            // whose last visit v > s'-nsub-1 (alternating sweeps; the solver carries step v's
            // changes) r before stream step v.  `before`: called before step s's changes (d <= nsub)
            // for the revisits with v = s, else after them for s' = s + nsub + 1
            auto publish = [&](int s0, int p0, int pos0, int d, bool before) {
                int q2 = pos0 + d, p2 = p0;   // step s0 + d without a division (d <= T)
                if (q2 >= T) { q2 -= T; p2++; }
                const int vp = (ALT && p2 >= 1 && 2 * q2 + 1 <= nsub) ? s0 + d - 2 * q2 - 1 : -1;
                const bool rev = vp > s0 + d - nsub - 1;
                if (before ? !(rev && vp == s0) : rev) return;
                const int bb = sweep_fwd(p2, alt) ? q2 : T - 1 - q2;   // its block
                const int qb = bb >> 2, oc = CLU ? qb / nqc : 0, ql = qb - oc * nqc;   // owner CTA, local chunk
                DWC_DCHECK(bb >= 0 && bb < T && ql / kNStream < RC && oc < G, "stream: published block");
                if (oc == (int)crank && (ql % kNStream) == w) {
                    if ((lane >> 3) == (bb & 3)) {
                        const int cb = ql / kNStream;
                        // rounded to fp32 here (the solver's recurrence is fp32), off the solver's path
                        float *dst = reinterpret_cast<float *>(pend) + 32 * ((s0 + d) & (kPendBlk - 1)) + 4 * (lane & 7);
#pragma unroll
                        for (int c = 0; c < RC; c++)
                            if (c == cb) {
                                const float4 v = make_float4((float)r[c][0], (float)r[c][1], (float)r[c][2], (float)r[c][3]);
                                if (CLU)   // into the leader's slot, completing on its sdone of this stream step
                                    st_async_v4b32(cl_map(dst, 0), __float_as_uint(v.x), __float_as_uint(v.y),
                                                   __float_as_uint(v.z), __float_as_uint(v.w),
                                                   cl_map(&sh.sdone[s0 % kNList], 0));
                                else
                                    *reinterpret_cast<float4 *>(dst) = v;
                            }
                    }
                    pub_bytes += 128;   // (8 lanes x 16 B)
                }
            };
            int b = 0;
            for (int s = 0, p = 0, pos = 0; s < total; s++, pos = (pos + 1 == T) ? 0 : pos + 1, p += (pos == 0)) {
                const int li = s % kNList;
                const unsigned long long t0 = pf ? clk() : 0ull;
                mbar_wait(&sh.dxready[li], (s / kNList) & 1);
                if (pf) tlw += clk() - t0;
                const int n = sh.cnt[li];
                // alternating sweeps: a revisit s' = s + d of block k whose last visit is this step
                // carries this step's changes itself, so its stored r is the one before them
                if (ALT)
                    for (int d = 1; d <= nsub; d++) publish(s, p, pos, d, true);
                for (int u0 = 0; u0 < (swid > 0 ? n : 0); u0 += rg.upb, b++) {
                    const int h = b % kNSlot;
                    const unsigned long long t1 = pf ? clk() : 0ull;
                    mbar_wait(&sh.rfull[h], (b / kNSlot) & 1);
                    const unsigned long long t2 = pf ? clk() : 0ull;
                    const int nb = min(rg.upb, n - u0);
                    const float *src = ring + (size_t)h * slot_floats + 4 * lane;
                    const double *dxb = &sh.dxs[li][u0];
                    if (nonneg)
                        apply_dispatch<true, RC>(nch, r, src, rstride, nb, dxb, w);
                    else
                        apply_dispatch<false, RC>(nch, r, src, rstride, nb, dxb, w);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sh.rempty[h]);
                    if (pf) { tbw += t2 - t1; tap += clk() - t2; nb_all++; }
                }
                // publish the r of block blk(s + nsub + 1) after this step -- unless that visit is an
                // alternating-sweep revisit whose last visit is inside its window (published then)
                publish(s, p, pos, nsub + 1, false);
                __syncwarp();
                if (lane == 0) {
                    if (CLU)   // the leader's sdone: one arrival plus the bytes this warp published (by
                        // st.async: no release needed; the slots it reuses were consumed steps ago)
                        mbar_arrive_tx_cl_relaxed(cl_map(&sh.sdone[li], 0), pub_bytes);
                    else
                        mbar_arrive(&sh.sdone[li]);
                }
                pub_bytes = 0;
            }
            if (pf && w == 0 && lane == 0) { prof[8] = tlw; prof[9] = tbw; prof[10] = tap; prof[11] = nb_all; }
        } else {
            // ================= stream warps: r += dx_c A[c, :] for every change of every step;
            // warp w owns the 128-column chunks q = w, w + 5, ...; lane l columns 128q + 4l..+3
            const int w = stream_index<CLU>(wid);
            unsigned long long tlw = 0, tbw = 0, tap = 0, nb_all = 0;
            int b = 0;
            for (int s = 0, p = 0, pos = 0; s < total; s++, pos = (pos + 1 == T) ? 0 : pos + 1, p += (pos == 0)) {
                const int k = sweep_fwd(p, alt) ? pos : T - 1 - pos;
                // the blocks of the next nsub steps (their contributions wait in pend for that
                // step's visit; first occurrence only, see the solver)
                int wb[kRgsWin + 1];
                if (ALT) {
#pragma unroll
                    for (int d = 1; d <= kRgsWin; d++) wb[d] = (d <= nsub) ? win_blk(p, pos, d, T, alt) : -1;
                }
                const int li = s % kNList;
                const unsigned long long t0 = pf ? clk() : 0ull;
                // the row producer arrives dxready after it observed the solver's dready (the list
                // and its dx are then visible); waiting on it every step, also without changes, keeps
                // the row producer within kNList steps of the solver (which runs at most nsub + 1
                // steps ahead of the stream)
                mbar_wait(&sh.dxready[li], (s / kNList) & 1);
                if (pf) tlw += clk() - t0;
                const int n = sh.cnt[li];
                const int nu = n * rg.nseg;
                // the solver has read block k: commit the contributions the solver carried for it
                // (steps s-nsub .. s-1, held in pend) -- by the owner warp of block k's chunk
                if ((((k >> 2) % kNStream) == w) && (lane >> 3) == (k & 3)) {
                    const int col = 32 * k + 4 * (lane & 7);
                    double2 *rp = reinterpret_cast<double2 *>(rs + col);
                    double2 *pp = reinterpret_cast<double2 *>(pend + 32 * (s & (kPendBlk - 1)) + 4 * (lane & 7));
                    double2 r0 = rp[0], r1 = rp[1];
                    const double2 p0 = pp[0], p1 = pp[1];
                    r0.x += p0.x; r0.y += p0.y; r1.x += p1.x; r1.y += p1.y;
                    rp[0] = r0; rp[1] = r1;
                    pp[0] = make_double2(0.0, 0.0);
                    pp[1] = make_double2(0.0, 0.0);
                }
                for (int u0 = 0; u0 < nu; u0 += rg.upb, b++) {
                    const int h = b % kNSlot;
                    const unsigned long long t1 = pf ? clk() : 0ull;
                    mbar_wait(&sh.rfull[h], (b / kNSlot) & 1);
                    const unsigned long long t2 = pf ? clk() : 0ull;
                    const int nb = min(rg.upb, nu - u0);
                    const float *src = ring + (size_t)h * slot_floats;
                    // the warp's chunks of each segment, kCP at a time: their r in registers while
                    // every unit of that segment is applied (independent DFMA chains per chunk)
                    for (int g = 0; g < rg.nseg; g++) {
                        const int q0 = (g * rg.seg) >> 7, q1 = (min(sp, (g + 1) * rg.seg) + 127) >> 7;
                        const int qs = q0 + ((w - q0) % kNStream + kNStream) % kNStream;
                        for (int qp = qs; qp < q1; qp += kCP * kNStream) {
                            // loads and fp64 updates run unconditionally on clamped addresses
                            // (no divergence, all kCP chunks in flight); only the stores are masked
                            // blocks k+1..k+nsub (carried by the solver) accumulate into pend until
                            // the solver has read them; the others into r
                            double2 ra[kCP], rb[kCP];
                            bool on[kCP];
                            int cc[kCP];
                            double *tg[kCP];
#pragma unroll
                            for (int i = 0; i < kCP; i++) {
                                const int qq = qp + i * kNStream, col = 128 * qq + 4 * lane;
                                on[i] = qq < q1 && col < sp;
                                cc[i] = (qq < q1) ? 128 * qq : 128 * qp;   // a chunk of this segment
                                const int ce = cc[i] + 4 * lane, blk = ce >> 5;
                                int o = 0;   // the first step s+o (1 <= o <= nsub) that visits blk, else 0
                                if (ALT) {
#pragma unroll
                                    for (int d = kRgsWin; d >= 1; d--)
                                        if (wb[d] == blk) o = d;
                                } else {   // forward: step s+o visits block k+o (mod T)
                                    o = blk - k;
                                    if (o < 0) o += T;
                                    if (o > nsub) o = 0;
                                }
                                tg[i] = (o >= 1) ? pend + 32 * ((s + o) & (kPendBlk - 1)) + (ce & 31) : rs + ce;
                                const double2 *rp = reinterpret_cast<const double2 *>(tg[i]);
                                ra[i] = rp[0];
                                rb[i] = rp[1];
                            }
                            for (int j = 0; j < nb; j++) {
                                int e = u0 + j;
                                if (rg.nseg > 1) {
                                    const int u = e;
                                    e = u / rg.nseg;
                                    if (u - e * rg.nseg != g) continue;
                                }
                                const double dx = sh.dxs[li][e];
                                const float *rowp = src + ((long)j - g) * rg.seg + 4 * lane;   // + chunk column
                                float4 v[kCP];
#pragma unroll
                                for (int i = 0; i < kCP; i++) v[i] = *reinterpret_cast<const float4 *>(rowp + cc[i]);
#pragma unroll
                                for (int i = 0; i < kCP; i++) {
                                    ra[i].x = fma((double)v[i].x, dx, ra[i].x);
                                    ra[i].y = fma((double)v[i].y, dx, ra[i].y);
                                    rb[i].x = fma((double)v[i].z, dx, rb[i].x);
                                    rb[i].y = fma((double)v[i].w, dx, rb[i].y);
                                }
                            }
#pragma unroll
                            for (int i = 0; i < kCP; i++) {
                                if (!on[i]) continue;
                                double2 *rp = reinterpret_cast<double2 *>(tg[i]);
                                rp[0] = ra[i];
                                rp[1] = rb[i];
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sh.rempty[h]);
                    if (pf) { tbw += t2 - t1; tap += clk() - t2; nb_all++; }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.sdone[li]);
            }
            if (pf && w == 0 && lane == 0) { prof[8] = tlw; prof[9] = tbw; prof[10] = tap; prof[11] = nb_all; }
        }
        __syncthreads();
        if (pf && tid == 0) prof[14] = clk() - t_item;
        if (prof && leader && tid == 0 && item < kProfItems) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[kProfSlots + 4 * item + 1] = t;
            prof[kProfSlots + 4 * item + 2] = (unsigned long long)bin;
        }
        // ---- output: x~ and the embedded full-grid map (S8)
        if (leader)
            for (int i = tid; i < nk; i += kRThreads) {
                const float v = xs[i];
                if (x_out) x_out[L.v_off + i] = v;
                if (x_map) x_map[(size_t)bin * S + keep_idx[(size_t)bin * S + i]] = v;
            }
        if (CLU)
            cl_sync();   // no CTA re-initialises its barriers while another still signals them
        else
            __syncthreads();
    }
    if (n_updates && wid == kWSolver && lane == 0 && my_updates) {
        atomicAdd(n_updates, my_updates);        // row updates
        atomicAdd(n_updates + 1, my_bytes);      // bytes of the rows they streamed
    }
}

namespace {
// RgsSmem, r (fp64; none when r lives in registers), the pending / published slots, x, the masks
size_t rgs_base_bytes(int max_sp, bool regr = false) {
    return sizeof(RgsSmem) + kPendF * 8 + (size_t)max_sp * ((regr ? 0 : 8) + 4) + (((size_t)max_sp / 32 + 31) & ~(size_t)31) * 4;
}
}  // namespace

// The automatic kernel choice: the residual kernel up to 8 x kRegMaxSp points (r in registers, one
// CTA -- or a cluster of up to 8 -- per bin), else the dense-stream kernel.  Measured (one B200):
// cfg3 GS 24.5 ms vs 45.2 dense-stream; cfg4 full grid (S = 10201, clusters of 4) 496 vs 2107 ms;
// cfg5 (S~ up to 9k, per-size-class launches) 1156 vs 1697 ms.
int rgs_auto_max_sp() {
    static const int v = getenv("DWC_RGS_AUTO_MAX_SP") ? atoi(getenv("DWC_RGS_AUTO_MAX_SP")) : 8 * kRegMaxSp;
    return v;
}

size_t rgs_smem_bytes(int max_sp) { return rgs_base_bytes(max_sp, max_sp <= 8 * kRegMaxSp) + kNSlot * 128 * 4 + 512; }


// wide: clusters of CTAs with 8 chunks per stream warp (5120 columns each) rather than 4 (2560):
// fewer SMs per bin, more stream work per CTA -- better when many rows change per sweep (the
// compressed grid: cfg5 GS 801 -> 665 ms), worse when few do (cfg4's full grid: 183 -> 200 ms)
int rgs_cluster_size(int sp, bool wide) {
    static const bool no_regr = getenv("DWC_RGS_NO_REGR") != nullptr;       // experiment: r in shared memory
    static const bool no_cluster = getenv("DWC_RGS_NO_CLUSTER") != nullptr; // experiment
    static const int force_g = getenv("DWC_RGS_CLUSTER_G") ? atoi(getenv("DWC_RGS_CLUSTER_G")) : 0;   // experiment
    if (force_g > 1 && force_g <= 8 && !no_regr) return force_g;
    if (no_regr || no_cluster || sp <= kRegMaxSpWide) return 1;   // (one CTA: r in registers, wide above kRegMaxSp)
    const int per = wide ? kRegMaxSpWide : kRegMaxSp;
    const int g = (sp + per - 1) / per;
    return g <= 8 ? g : 1;   // (portable cluster sizes; beyond: one CTA with r in shared memory)
}

// Small systems of a band with more bins than SMs run two CTAs per SM, so that every bin starts
// at once instead of the late-started ones forming the band's tail: the bins whose padded size
// is at most 2/3 of the band's largest (a bin's time grows about linearly with S~, and sharing an
// SM at most doubles it).  cfg3 (largest 1344): one band alone 24.0 ms at 2/3 (896) as at 1/2
// (672), bands in flight 14.2 -> 15.6 k bins/s; 1024 and 1280 gain more in flight (16.0 k) but
// lose alone (25.9, 28.6 ms).  throughput (DWC_THROUGHPUT: bands in flight): every system up to
// kRegMaxSpPair, whatever the band's size.
int rgs_pair_max_sp(int band_max_sp, int n_bins, int num_sms, bool throughput) {
    static const int env = getenv("DWC_RGS_PAIR_MAX_SP") ? atoi(getenv("DWC_RGS_PAIR_MAX_SP")) : -1;   // experiment
    if (env >= 0) return std::min(env, kRegMaxSpPair);
    if (throughput) return kRegMaxSpPair;
    if (n_bins <= num_sms) return 0;
    return std::min((2 * band_max_sp / 3) & ~31, kRegMaxSpPair);
}

int rgs_size_class(int sp, bool wide, int pair_max_sp) {
    const int g = rgs_cluster_size(sp, wide);
    // 0: two CTAs per SM, 1: one CTA, 2: one CTA with wide registers, 2+G: clusters
    return g > 1 ? 2 + g : (sp > kRegMaxSp ? 2 : (sp > pair_max_sp ? 1 : 0));
}

int launch_rgs(int n_bins, const int *order_dev, const BinLayout *lay_dev, int max_sp, int *counter,
               const float *Adense, const double *bt, int sweeps, float *x_out, float *x_map,
               const int32_t *keep_idx, int S, int num_sms, unsigned long long *n_updates, cudaStream_t st,
               GsLaunchInfo *info, int alt, int nonneg, int wide_clusters, int pair_max_sp) {
    static const int ring_env = getenv("DWC_RGS_RING_KB") ? atoi(getenv("DWC_RGS_RING_KB")) : 0;   // experiment
    static const int per_sm_env = getenv("DWC_RGS_PER_SM") ? atoi(getenv("DWC_RGS_PER_SM")) : 0;   // experiment
    static const bool no_regr = getenv("DWC_RGS_NO_REGR") != nullptr;   // experiment: r in shared memory
    // r in registers (one CTA per SM: up to 255 registers) when the system fits the stream warps'
    // chunks; above that, split over a cluster of G CTAs (<= 8, portable) -- both need a ring slot
    // that holds a whole row (slice); else r in shared memory
    const int nq_max = (max_sp + 127) / 128;
    int G = rgs_cluster_size(max_sp, wide_clusters);
    const bool regr_try = !no_regr && (max_sp <= kRegMaxSpWide || G > 1);
    // 8 chunks per stream warp: one CTA above kRegMaxSp, or the wide clusters
    const bool wide = regr_try && (G == 1 ? max_sp > kRegMaxSp : (bool)wide_clusters);
    const bool pair = regr_try && G == 1 && max_sp <= pair_max_sp && n_bins > 1;   // two CTAs per SM
    const int rstride_max = G > 1 ? 128 * ((nq_max + G - 1) / G) : max_sp;   // floats of a ring row
    // the configuration: base shared memory, 1/A_ii copy (when a ring of >= 24 KB still fits), ring
    auto layout = [&](bool regr, int &use_ivs, size_t &base, bool allow_ivs) {
        use_ivs = (allow_ivs && rgs_base_bytes(max_sp, regr) + (size_t)max_sp * 4 + 24 * 1024 + 1536 <= 227 * 1024) ? 1 : 0;
        base = (rgs_base_bytes(max_sp, regr) + (use_ivs ? (size_t)max_sp * 4 : 0) + 127) / 128 * 128;
    };
    auto slot_of = [&](size_t ring) { return (int)(ring / (4 * kNSlot)) / 128 * 128; };
    auto ring_of = [&](size_t base) {
        size_t ring = base + 1536 <= 227 * 1024 ? (227 * 1024 - base - 512) / 1024 * 1024 : 0;
        if (ring_env > 0 && (size_t)ring_env * 1024 < ring) ring = (size_t)ring_env * 1024;
        return ring;
    };
    int use_ivs;
    size_t base;
    bool regr = regr_try;
    layout(regr, use_ivs, base, true);
    if (regr && slot_of(ring_of(base)) < rstride_max)   // a slot must hold a whole row (slice): drop the 1/A_ii copy
        layout(regr, use_ivs, base, false);
    if (regr && slot_of(ring_of(base)) < rstride_max) {   // still not: r in shared memory
        regr = false;
        G = 1;
        layout(regr, use_ivs, base, true);
    }
    if (base + 1536 > 227 * 1024) return -1;
    // shared-memory r: two CTAs per SM (2 x (smem + 1 KB reserved) <= 228 KB) when the band has
    // more bins than SMs and every ring slot still holds 2 rows
#ifndef RGS_PAIR_PER_SM
#define RGS_PAIR_PER_SM 2
#endif
    const size_t per2 = 114 * 1024 - 1024;
    // the small register class: RGS_PAIR_PER_SM CTAs per SM (shared memory split that many ways;
    // 3, with RGS_PAIR_MINB=3 for 80 registers, measured 31 % slower for bands in flight)
    const size_t perp = 228 * 1024 / RGS_PAIR_PER_SM - 1024;
    const bool two = regr ? (pair && perp > base + 3 * 4 * (size_t)max_sp + 1024)   // (r in registers: the small class)
                     : kRMinBlocks < 2 ? false
                     : per_sm_env ? per_sm_env == 2 && per2 > base + 2048
                                : n_bins > num_sms && per2 > base && (per2 - base) / (4 * kNSlot) >= 2 * (size_t)max_sp;
    size_t ring = two ? ((regr ? perp : per2) - base - 512) / 1024 * 1024 : (227 * 1024 - base - 512) / 1024 * 1024;
    if (ring_env > 0 && (size_t)ring_env * 1024 < ring) ring = (size_t)ring_env * 1024;
    const int slot_floats = slot_of(ring);   // floats per ring slot
    if (slot_floats < 128) return -1;
    const size_t smem = base + (size_t)slot_floats * 4 * kNSlot + 512;   // + slack: a row's last chunk reads past it
    const bool clu = G > 1;
    const auto kern =
        alt ? (clu ? (wide ? rgs_kernel<true, true, true, kRegChWide> : rgs_kernel<true, true, true>)
                   : regr ? (wide ? rgs_kernel<true, true, false, kRegChWide>
                                  : two ? rgs_kernel<true, true, false, kRegChPair> : rgs_kernel<true, true, false>)
                          : rgs_kernel<true, false, false>)
            : (clu ? (wide ? rgs_kernel<false, true, true, kRegChWide> : rgs_kernel<false, true, true>)
                   : regr ? (wide ? rgs_kernel<false, true, false, kRegChWide>
                                  : two ? rgs_kernel<false, true, false, kRegChPair> : rgs_kernel<false, true, false>)
                          : rgs_kernel<false, false, false>);
    if (raise_smem_limit(kern, smem) != cudaSuccess)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(kRThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    int grid;
    if (clu) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(G * std::min(n_bins, std::max(1, num_sms / G)));
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            ncl = std::max(1, num_sms / G);
        }
        grid = G * std::min(n_bins, ncl);
    } else {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRThreads, smem) != cudaSuccess || per_sm < 1) {
            cudaGetLastError();
            per_sm = 1;
        }
        grid = std::min(n_bins, num_sms * per_sm);
        static const int cta_env = getenv("DWC_RGS_CTAS") ? atoi(getenv("DWC_RGS_CTAS")) : 0;   // experiment
        if (cta_env > 0 && cta_env < grid) grid = cta_env;
        if (grid < 1) grid = 1;
    }
    cfg.gridDim = dim3(grid);
    if (info) {
        info->kernel = DWC_GS_KERNEL_RESIDUAL;
        info->xtra_tiles = 0;
        info->ctas = grid;
        info->max_group = G;
    }
    // DWC_RGS_PROF=1: clock64 breakdown of the largest bin (stderr)
    static const bool profile = getenv("DWC_RGS_PROF") != nullptr;
    unsigned long long *prof = nullptr;
    if (profile) {
        const size_t pb = (kProfSlots + 4 * kProfItems + 2) * sizeof(unsigned long long);
        if (cudaMalloc(&prof, pb) != cudaSuccess) return -1;
        cudaMemsetAsync(prof, 0, pb, st);
    }
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, n_bins, order_dev, lay_dev, counter, Adense, bt, sweeps, x_out,
                                             x_map, keep_idx, S, max_sp, slot_floats, use_ivs, nonneg, n_updates, prof);
    if (profile) {
        static unsigned long long h[kProfSlots + 4 * kProfItems + 2];
        cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        {   // the items that ended last (the band's tail) and when
            const int ni = std::min(n_bins, kProfItems);
            unsigned long long t0 = ~0ull;
            for (int i = 0; i < ni; i++) t0 = std::min(t0, h[kProfSlots + 4 * i]);
            std::vector<int> idx(ni);
            for (int i = 0; i < ni; i++) idx[i] = i;
            std::sort(idx.begin(), idx.end(), [&](int a, int b) { return h[kProfSlots + 4 * a + 1] > h[kProfSlots + 4 * b + 1]; });
            fprintf(stderr, "[rgs-prof] last items to end (item bin: start..end ms, changes):");
            for (int j = 0; j < std::min(ni, 8); j++) {
                const unsigned long long *r = h + kProfSlots + 4 * idx[j];
                fprintf(stderr, " %d b%llu: %.2f..%.2f (%llu)", idx[j], r[2], (r[0] - t0) * 1e-6, (r[1] - t0) * 1e-6, r[3]);
            }
            fprintf(stderr, "\n");
        }
        const double n = h[4] ? (double)h[4] : 1.0;
        fprintf(stderr,
                "[rgs-prof] grid %d x %zu B smem (ring %d x %d floats), steps %llu, changes %llu (%.2f/step), item %.0f cyc"
                " | solver cyc/step: tiles %.0f stream %.0f loop %.0f rest %.0f | stream0: list %.0f batch %.0f apply %.0f"
                " (%llu batches) | rowprod: ring wait %.0f issue %.0f | panel misses %llu | panelprod wait %.0f issue %.0f\n",
                grid, smem, kNSlot, slot_floats, h[4], h[5], h[5] / n, (double)h[14], h[0] / n, h[1] / n, h[2] / n, h[3] / n,
                h[8] / n, h[9] / n, h[10] / n, h[11], h[12] / n, h[13] / n, h[6], h[7] / n, h[15] / n);
        fprintf(stderr, "[rgs-prof] first 10%% of the steps: stream wait %.0f, loop %.0f cyc/step, %.2f changes/step; "
                        "steps without a change: %.1f %%; stream waits over 100 cycles: %.1f %% of the steps\n",
                h[16] / (0.1 * n), h[17] / (0.1 * n), h[18] / (0.1 * n), 100.0 * h[19] / n, 100.0 * h[20] / n);
        cudaFree(prof);
    }
    return e == cudaSuccess ? 1 : -1;
}

// dwc_gs input conversion: dense row-major n x n -> the padded dense sp x sp matrix of the
// residual kernel: symmetric (reading R1): the upper triangle is read; general (the paper-literal
// PSF): the transpose (the kernel reads column c of A as row c).
__global__ void rgs_convert_kernel(int n, int sp, const float *__restrict__ src, float *__restrict__ dense, int general) {
    const long total = (long)sp * sp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / sp), j = (int)(e - (long)(e / sp) * sp);
        if (general) {
            dense[e] = (i < n && j < n) ? src[(size_t)j * n + i] : 0.f;
        } else {
            const int lo = min(i, j), hi = max(i, j);
            dense[e] = (hi < n) ? src[(size_t)lo * n + hi] : 0.f;
        }
    }
}

int launch_rgs_convert(int n, int sp, const float *src, float *dense, cudaStream_t st, int general) {
    const long total = (long)sp * sp;
    const int blocks = (int)std::min<long>((total + 255) / 256, 148L * 32);
    rgs_convert_kernel<<<blocks, 256, 0, st>>>(n, sp, src, dense, general);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// dwc_psf (paper-literal): out[i][j] = src[j][i] (transpose = 1) or src[i][j], n x n out of the
// padded sp x sp dense layout.
__global__ void dense_extract_kernel(int n, int sp, const float *__restrict__ src, float *__restrict__ out, int transpose) {
    const long total = (long)n * n;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e - (long)(e / n) * n);
        out[e] = transpose ? src[(size_t)j * sp + i] : src[(size_t)i * sp + j];
    }
}

int launch_dense_extract(int n, int sp, const float *src, float *out, int transpose, cudaStream_t st) {
    const long total = (long)n * n;
    const int blocks = (int)std::min<long>((total + 255) / 256, 148L * 32);
    dense_extract_kernel<<<blocks, 256, 0, st>>>(n, sp, src, out, transpose);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
