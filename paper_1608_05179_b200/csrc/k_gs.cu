// k_gs.cu -- S7 DAMAS non-negative Gauss-Seidel sweeps (+ S8 embed), the time sink.
//
// Eq. 13-14, readings R4, R11, R12, R18:
//   r_i = sum_{j<i} A_ij x_j^(n+1) + sum_{j>=i} A_ij x_j^(n) - b_i,
//   x_i^(n+1) = max(x_i^(n) - r_i / A_ii, 0),  i ascending, x^0 = 0, fixed sweep count.
// Row order and sweep order are kept exactly; only the summation order of each row dot
// differs from the oracle (fp32 A~ and fp32 partial dots; residual against fp64 b~).
//
// Block formulation (B = 32 rows, T = sp/32 blocks): solver step j solves block k = j mod T
// with the residual r_{I_k} = P_k + (increments of the blocks solved in the last two steps)
// - b_{I_k}.  P_k is produced by "stream" warps ahead of the solver.  A~ is symmetric and only
// its upper tiles are stored (dwc_internal.cuh layout), so the contributions to row block kn are
//   row use   U(kn, J) x_J^old, J > kn (minus the two blocks below)      stream, step kn
//   scatter   U(kn-3, J)^T x_{kn-3}^new, J >= kn  -> P_kn (J = kn) or y_J stream, step kn
//   L, LL     A[kn, kn-1], A[kn, kn-2]: old-x products by the leader's L warp, increments by
//             the solver's role-1 / role-2 lanes while it solves those blocks
//   D         old-x product by the leader's D warp; the in-block recurrence by the solver
// so the stream depends only on x of solver step s-3 and runs up to two steps ahead.
// In-block recurrence, one warp, "step form":
//   w_l = -r_l / A_ll;  delta_t = max(w_t, -x_t)  (x_t + delta_t = max(x_t + w_t, 0))
//   w_l -= (A_lt / A_ll) delta_t for all lanes;   x_t += delta_t.
//
// B200 mapping
//  * A CTA = warp 0 solver, warp 1 bulk-copy producer (in the leader also of the solver's staged
//    blocks), warp 4 helper (leader: sums the g*kCons partial vectors of each step so the
//    solver reads P as one float4 per lane, and forwards each new x block to the other CTAs
//    as soon as the solver publishes it), warps 2,3,5,6,7 consumers (in the leader 6 = D
//    product, 7 = L/LL products).  The producer streams this CTA's runs of each step with
//    cp.async.bulk (<= 6 tiles per copy, mbarrier complete_tx) into a shared-memory ring (2 slots
//    of 24 KB; non-leader CTAs also use the staging area: 3), running ahead across steps (tiles
//    do not depend on x); an L2 prefetch of the runs n steps ahead is available with -DGS_PF=n
//    (off by default: measured not to pay).
//  * Clusters of kCl = 4 CTAs.  A work item gives the cluster either one large bin (sub-group of
//    g = 4 CTAs), two medium bins (g = 2) or four small bins (g = 1).  Inside a sub-group every
//    CTA keeps a full copy of x in shared memory; column blocks are owned by CTAs in a periodic
//    pattern weighted by stream warps (dwc_internal.cuh own_of); every consumer warp sends its 32
//    partial row sums to the leader with st.async (DSMEM, complete_tx on the leader's
//    P-ready barrier); the leader's helper warp forwards each new x block the same way.  No grid or
//    cluster barrier inside the sweep loop; cluster barriers only between work items.
//  * g depends on S~ only (host), so a bin's result is bit-identical whatever else is in the
//    batch (and on however many GPUs the band is sharded); items run largest first (LPT).
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dwc_internal.cuh"

namespace dwc {

constexpr int kCl = 4;             // cluster size
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kCons = kWarps - 3;  // consumer warps (3..7)
#ifndef GS_CHUNK
#define GS_CHUNK 6
#endif
#ifndef GS_RING
#define GS_RING 2
#endif
constexpr int kChunk = GS_CHUNK;   // tiles per ring slot (one contiguous bulk copy)
constexpr int kRing = GS_RING;     // stream ring slots of the leader
#ifndef GS_PF
#define GS_PF 0
#endif
// L2 prefetch distance of the stream runs, in steps.  Off: with the current CTA-per-bin
// thresholds it no longer pays (cfg3 GS 48.3 ms without, 49.3 with 4 steps, 51.0 with 6; cfg2,
// cfg5 neutral; scripts/ab_multi.sh); -DGS_PF=n re-enables it.
constexpr int kPf = GS_PF;
constexpr double kL2WindowBytes = 48.0 * 1024 * 1024;   // L2 share the prefetch window may use
constexpr int kTile = 1024;        // floats per tile
#ifndef GS_KSTG
#define GS_KSTG 3
#endif
constexpr int kStg = GS_KSTG;            // solver tiles (L, D) prefetched this many steps ahead

// Per-block solver packet (precomputed once per bin by gs_prep_kernel, staged with L/D):
// invd[r] = 1/A_rr (0 for padding rows), wg[L][0..5] = within-group A[r][t]/A[r][r] for
// lane L's rows r = 4L+i' > t = 4L+i  (order: 10 20 30 21 31 32), and b~ of the block as an
// fp32 pair b = bhi + blo (the residual (acc - bhi) - blo keeps b~'s fp64 accuracy: an fp32
// b~ would shift the fixed point the sweeps converge to).
struct __align__(16) GsPacket {
    float invd[32];
    float wg[8][8];
    float bhi[32];
    float blo[32];
};
constexpr int kPacketBytes = (int)sizeof(GsPacket);

struct GsItem {
    int g;          // CTAs per bin: 1, 2 or 4
    int bin[kCl];   // bins of the sub-groups (-1 = idle)
};

constexpr int kRsTiles = kRing * kChunk + kStg * 3;   // stream ring + staging area (tiles)
// Non-leader CTAs have no staging slots and use the whole area as 3 slots of 7 tiles (6-tile
// slots left 3 tiles idle): cfg3 GS 45.9-46.0 -> 45.5-45.9 ms, cubic band 35.7 -> 34.5 ms
// (5 tiles: 45.5-45.9 / 35.9-36.5, 4: 46.0 / 36.4-37.2, 3: 47.0 / 39.1-39.5; scripts/ab_modes.sh).
#ifndef GS_NLCHUNK
#define GS_NLCHUNK 7
#endif
constexpr int kChunkNL = GS_NLCHUNK;                  // tiles per slot of a non-leader CTA
constexpr int kNringNL = kRsTiles / kChunkNL;         // stream slots of a non-leader CTA
// Systems whose x, y and tables already keep the kernel at one CTA per SM (cfg4, cfg5) get the
// shared memory left over as extra ring slots after the dynamic tables (launch_gs: xtra tiles).
constexpr int kNringMax = 8;
static_assert(kNringNL <= kNringMax && kRing <= kNringMax, "ring barrier arrays");
struct __align__(128) GsSmem {
    // stream slot p = tiles [p*kChunk, (p+1)*kChunk); in the leader the tiles from kRing*kChunk on
    // are the staging slots (slot q = 3 tiles: L_j, D_j, LL_{j+2}), in the other CTAs more stream slots
    float rs[kRsTiles][kTile];
    GsPacket pk[kStg];                 // solver packet of the staged block
    float pr[2][kCl][kCons][32];       // leader: partial row sums of every consumer warp of the sub-group
    unsigned long long full[kNringMax], empty[kNringMax];
    unsigned long long stg_full[kStg], stg_empty[kStg];
    unsigned long long pready[2];      // leader: 1 arrival + g*kCons*128 tx bytes per step
    unsigned long long xr[2];          // leader: solver arrival; others: 1 arrival + 128 tx
    float psum[2][32];                 // leader: P of the step, summed by the helper warp
    unsigned long long psum_full[2];   // leader: helper arrival
    int item;
    unsigned long long issue_t[kNringMax];   // profiling: clock64 at which each slot's copy was issued
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
#ifdef DWC_CHECKED
// checked build: waits that have not completed after ~2^24 polls report and trap
template <bool kCluster>
__device__ __forceinline__ void mbar_wait_checked(unsigned long long *b, uint32_t parity) {
    for (unsigned it = 0;; it++) {
        uint32_t ok;
        if (kCluster)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
        else
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
        if (ok) return;
        DWC_DCHECK(it < (1u << 24), "gs: mbarrier wait never completes");
    }
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) { mbar_wait_checked<true>(b, parity); }
__device__ __forceinline__ void mbar_wait_cta(unsigned long long *b, uint32_t parity) { mbar_wait_checked<false>(b, parity); }
#else
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// CTA-scope acquire, for barriers completed only by this CTA's own threads or by its own bulk
// copies (ring, staging, the leader's x-ready): no L1 invalidation (ptxas emits CCTL.IVALL for
// the cluster-scope acquire above, which the barriers completed by other CTAs -- partial sums,
// the non-leaders' x-ready -- need).
__device__ __forceinline__ void mbar_wait_cta(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "C_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra C_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void mbar_arrive_local(unsigned long long *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
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
__device__ __forceinline__ void st_remote_f32(uint32_t raddr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(raddr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_remote_s32(uint32_t raddr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}
// shared::cta -> shared::cluster (another CTA) bulk copy, completing on the remote mbarrier
__device__ __forceinline__ void bulk_s2s(uint32_t dst_cluster, const void *src, uint32_t bytes, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
        "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
        : "memory");
}
// st.async: register -> another CTA's shared memory, completing tx bytes on its mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(raddr), "f"(v),
                 "r"(rbar)
                 : "memory");
}
// L2 prefetch of a global range (no shared-memory destination, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// The stream tiles of one step (row block kn) for CTA rg of a g-CTA sub-group, in ring order:
// two contiguous runs of the symmetric layout (dwc_internal.cuh), each cut into chunks of
// <= kChunk tiles:
//  seg 0  row use      U(kn, J), J > kn, J = rg mod g, x_J old -- minus J = (kn-1) mod T and
//                      (kn-2) mod T (kn <= 1), which are L_kn / LL_kn
//  seg 1  scatter      U(kn-3, J)^T x_{kn-3}^new for J >= kn (kn >= 3): J = kn into P_kn, J > kn
//                      into the warp's y_J (the lower part of row J, consumed at step J)
// The first and second sub-diagonal blocks A[kn, kn-1] = L_kn and A[kn, kn-2] = LL_kn are done
// by the leader: its L warp multiplies them with the old x (LL one step early) and the solver
// adds their increments while it solves blocks kn-1 / kn-2.  So the stream needs only x of solver
// step s-3 and older, and runs up to two steps ahead of the solver.
// The runs are computed once per work item into shared memory (seg_table) so the per-step cost
// is two LDS.128.
struct __align__(16) Seg {
    int t0, len, j0, ord0;   // first tile (bin-relative), tiles, J of the first tile, its ordinal
};                           // among the CTA's owned column blocks (own_nth)
__device__ Seg seg_run(int T, int g, int rg, int kn, int seg) {
    Seg r{0, 0, 0, 0};
    const int I = (seg == 0) ? kn : kn - 3;
    if (I < 0) return r;
    int len = sym_run_len(T, g, I, rg), st = sym_run_start(T, g, I, rg), ord = sym_cnt(I, rg, g);
    if (seg == 0) {
        const int kx = (kn + T - 1) % T, kl = (kn + T - 2) % T;
        while (len > 0) {
            const int jl = own_nth(g, rg, ord + len - 1);
            if (jl != kx && jl != kl) break;
            len--;
        }
    } else {
        while (len > 0 && own_nth(g, rg, ord) < kn) { ord++; st++; len--; }
    }
    r.t0 = st; r.len = len; r.j0 = len > 0 ? own_nth(g, rg, ord) : 0; r.ord0 = ord;
    return r;
}

// Consumer: acc[q] (rows 4*rq+q) += sum over columns c = cq + 4i of tile[c][4rq+q] * x[c].
__device__ __forceinline__ void tile_dot(const float *__restrict__ tile, const float *__restrict__ xcol, int rq,
                                         int cq, float acc[4]) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int c = cq + 4 * i;
        const float4 v = *reinterpret_cast<const float4 *>(tile + c * 32 + 4 * rq);
        const float xv = xcol[c];
        // packed fp32x2 FMA (FFMA2): the same two correctly rounded FMAs in one instruction
        const float2 xx = make_float2(xv, xv);
        const float2 a01 = __ffma2_rn(make_float2(v.x, v.y), xx, make_float2(acc[0], acc[1]));
        const float2 a23 = __ffma2_rn(make_float2(v.z, v.w), xx, make_float2(acc[2], acc[3]));
        acc[0] = a01.x; acc[1] = a01.y; acc[2] = a23.x; acc[3] = a23.y;
    }
}

// Consumer, transposed tile: returns, in lane o, (U^T x)[o] = sum_r tile[o][r] x[r] -- the whole
// column o of the column-major tile, read as 8 float4 in the lane-rotated order (k + o) mod 8 so
// every quarter-warp touches 8 distinct 16-byte bank groups (x likewise).  No cross-lane reduction.
__device__ __forceinline__ float tile_tdot(const float *__restrict__ tile, const float *__restrict__ x, int lane) {
    float2 t2 = make_float2(0.f, 0.f);   // two interleaved partial sums, packed FMAs
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int r0 = 4 * ((k + lane) & 7);
        const float4 v = *reinterpret_cast<const float4 *>(tile + lane * 32 + r0);
        const float4 xv = *reinterpret_cast<const float4 *>(x + r0);
        t2 = __ffma2_rn(make_float2(v.x, v.y), make_float2(xv.x, xv.y), t2);
        t2 = __ffma2_rn(make_float2(v.z, v.w), make_float2(xv.z, xv.w), t2);
    }
    return t2.x + t2.y;
}

// Stream step s computes P for block kn = s mod T excluding kx = (s-1) mod T.  Stream tiles
// of sub-group rank rg: J in [0,T), J mod g == rg, J != kx, J != kn.  The leader also stages
// tile (kn,kx) (L, for the solver) and (kn,kn) (D, solver + its old-x product).
#ifndef GS_MINB
#define GS_MINB 2
#endif
template <bool kXtra>   // extra ring slots in use (an instantiation of its own: no cost otherwise)
__global__ void __launch_bounds__(kThreads, GS_MINB)
gs_cluster_kernel(int n_items, const GsItem *__restrict__ items, const BinLayout *__restrict__ lay,
                  int *__restrict__ counter, const float *__restrict__ A, const GsPacket *__restrict__ packets,
                  int sweeps, float *__restrict__ x_out, float *__restrict__ x_map,
                  const int32_t *__restrict__ keep_idx, int S, int xcap, int ystride, int pf,
                  int xtra_off, int xtra_tiles, unsigned long long *__restrict__ prof) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *xtra = reinterpret_cast<float *>(smem_raw + xtra_off);   // extra ring tiles (may be none)
    GsSmem &sh = *reinterpret_cast<GsSmem *>(smem_raw);
    float *xs = reinterpret_cast<float *>(smem_raw + sizeof(GsSmem));
    float *ys = xs + xcap;   // per stream warp: y_J (lower part of row J) for the owned J, J/g-indexed
    Seg *segt = reinterpret_cast<Seg *>(ys + kCons * ystride);   // [kn][2] runs of this CTA
    int *ownJ = reinterpret_cast<int *>(segt + 2 * (xcap / 32));  // ordinal -> owned column block J
    int *ordOf = ownJ + (xcap / 32);                             // J -> ordinal (-1: not owned)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t crank = cluster_rank();
    auto gtime = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    if (prof && tid == 0 && blockIdx.x < 1024) prof[32 + 2 * blockIdx.x] = gtime();   // CTA start (ns)

    for (;;) {
        // ---- the cluster's next item: rank 0 pops and writes it into every CTA
        if (crank == 0 && tid == 0) {
            const int it = atomicAdd(counter, 1);
            for (uint32_t q = 0; q < kCl; q++) st_remote_s32(mapa(smem_u32(&sh.item), q), it);
        }
        cluster_sync();
        const int item = sh.item;
        if (item >= n_items) {
            if (prof && tid == 0 && blockIdx.x < 1024) prof[33 + 2 * blockIdx.x] = gtime();   // CTA idle from here
            break;
        }
        const GsItem IT = items[item];
        const int g = IT.g;   // 1, 2 or 4
        const int sg = (int)crank / g, rg = (int)crank % g;
        const uint32_t leader = (uint32_t)(sg * g);
        const bool is_leader = (rg == 0);
        const int chunk = is_leader ? kChunk : kChunkNL;
        const int nbase = is_leader ? kRing : kNringNL;    // non-leaders stream into the staging area too
        const int nring = kXtra ? min(kNringMax, nbase + xtra_tiles / chunk) : nbase;
        // first tile of ring slot sl: the fixed area, then the extra tiles
        auto slot_ptr = [&](uint32_t sl) -> float * {
            if constexpr (!kXtra) return &sh.rs[sl * chunk][0];
            return (int)sl < nbase ? &sh.rs[sl * chunk][0] : xtra + (size_t)((int)sl - nbase) * chunk * kTile;
        };
        const int bin = IT.bin[sg];
        BinLayout L = {0, 0, 0, 0, 0, 0, 0};
        if (bin >= 0) L = lay[bin];
        const int sp = L.sp, nk = L.nk, T = sp >> 5;
        const int total = (bin >= 0) ? sweeps * T : 0;
        const float *Ab = A + L.a_off;
        const GsPacket *pkb = packets + (L.v_off >> 5);

        for (int i = tid; i < sp; i += kThreads) xs[i] = 0.f;
        for (int i = tid; i < kCons * ystride; i += kThreads) ys[i] = 0.f;
        for (int i = tid; i < 2 * T; i += kThreads) segt[i] = seg_run(T, g, rg, i >> 1, i & 1);
        for (int J = tid; J < T; J += kThreads) {
            const bool mine = own_of(g, J) == rg;
            const int o = sym_cnt(J - 1, rg, g);
            ordOf[J] = mine ? o : -1;
            if (mine) ownJ[o] = J;
        }
        if (tid == 0) {
            const int n_sw = is_leader ? kCons - 2 : kCons;
            for (int i = 0; i < kNringMax; i++) {
                mbar_init(&sh.full[i], 1);
                mbar_init(&sh.empty[i], (uint32_t)n_sw);   // every stream warp releases every chunk
            }
            for (int b = 0; b < kStg; b++) {
                mbar_init(&sh.stg_full[b], 1);
                mbar_init(&sh.stg_empty[b], 3);   // solver, L-product warp, D-product warp
            }
            for (int b = 0; b < 2; b++) {
                mbar_init(&sh.pready[b], 1);
                mbar_init(&sh.xr[b], 1);
                mbar_init(&sh.psum_full[b], 1);
            }
            fence_mbar_init();
        }
        cluster_sync();

        if (wid == 1) {
            // ================= stream producer (one lane): this CTA's tiles of each row block
            if (lane == 0) {
                uint32_t seq = 0, slot = 0, ph = 0;
                const bool ppf = prof && item == 0 && crank == 0;   // item 0 = the largest bin (LPT)
                unsigned long long t0 = 0, p_wait = 0, p_issue = 0;
                // the row runs of step s + pf are prefetched into L2 while step s is copied into the
                // ring: the ring then only has to cover L2 latency, not HBM latency
                for (int s = 0, kn = 0, kp = (T > 0 ? pf % T : 0); s < total;
                     s++, kn = (kn + 1 == T) ? 0 : kn + 1, kp = (kp + 1 == T) ? 0 : kp + 1) {
                    if (pf > 0 && s + pf < total) {
                        const Seg *sp = segt + 2 * kp;
                        for (int sg = 0; sg < 2; sg++)
                            if (sp[sg].len > 0)
                                bulk_prefetch_l2(Ab + (size_t)sp[sg].t0 * kTile, (uint32_t)sp[sg].len * kTile * 4);
                    }
                    if (is_leader) {
                        // the solver's staged block of step s: L = (kn,kx), D = (kn,kn), LL_{kn+2}, packet
                        const int sl = s % kStg;
                        const int kn2 = (kn + 2 >= T) ? kn + 2 - T : kn + 2;   // (mod T again for T < 2)
                        mbar_wait_cta(&sh.stg_empty[sl], ((s / kStg) & 1) ^ 1);
                        mbar_expect_tx(&sh.stg_full[sl], 3 * kTile * 4 + kPacketBytes);
                        bulk_g2s(sh.rs[kRing * kChunk + 3 * (sl) + 0], Ab + (size_t)(T + kn) * kTile, kTile * 4, &sh.stg_full[sl]);   // L_kn
                        bulk_g2s(sh.rs[kRing * kChunk + 3 * (sl) + 1], Ab + (size_t)kn * kTile, kTile * 4, &sh.stg_full[sl]);         // D_kn
                        bulk_g2s(sh.rs[kRing * kChunk + 3 * (sl) + 2], Ab + (size_t)(2 * T + kn2 % T) * kTile, kTile * 4,
                                 &sh.stg_full[sl]);                                                      // LL_{kn+2}
                        bulk_g2s(&sh.pk[sl], pkb + kn, kPacketBytes, &sh.stg_full[sl]);
                    }
                    const Seg *sd = segt + 2 * kn;
                    for (int sg = 0; sg < 2; sg++)
                    for (int off = 0; off < sd[sg].len; off += chunk) {
                        const int tt = sd[sg].t0 + off, nt = min(chunk, sd[sg].len - off);
                        if (ppf) t0 = clock64();
                        mbar_wait_cta(&sh.empty[slot], ph ^ 1);
                        if (ppf) { const unsigned long long t = clock64(); p_wait += t - t0; t0 = t; }
                        DWC_DCHECK(slot < (uint32_t)nring && nt >= 1 && nt <= chunk, "gs producer: ring slot / chunk");
                        DWC_DCHECK(!kXtra || (int)slot < nbase || ((int)slot - nbase + 1) * chunk <= xtra_tiles,
                                   "gs producer: extra ring slot beyond its tiles");
                        mbar_expect_tx(&sh.full[slot], (uint32_t)nt * kTile * 4);
                        if (prof) sh.issue_t[slot] = clock64();
                        bulk_g2s(slot_ptr(slot), Ab + (size_t)tt * kTile, (uint32_t)nt * kTile * 4, &sh.full[slot]);
                        if (ppf) { const unsigned long long t = clock64(); p_issue += t - t0; }
                        seq++;
                        if (++slot == (uint32_t)nring) { slot = 0; ph ^= 1; }
                    }
                }
                if (ppf) { prof[12] = p_wait; prof[13] = p_issue; prof[14] = seq; }
            }
        } else if (wid == 4) {
            // ================= partial-sum helper (leader): P of step j = the g*kCons partial
            // vectors, lane r summing row r, so the solver finds it summed (one float4 per lane)
            // -- off the solver's path whenever the stream is ahead of it
            // It also forwards each new x block to the sub-group's other CTAs (st.async completes
            // 128 bytes on their x-ready barrier) as soon as the solver publishes it: the solver
            // publishes x of step j-1 once it has consumed P_j, so the others have finished step j
            // and observed x of step j-3, the previous phase of the slot this store completes.
            if (is_leader) {
                const int np = g * kCons;
                auto push_x = [&](int jj) {
                    mbar_wait_cta(&sh.xr[jj & 1], (jj >> 1) & 1);
                    if (lane < 8) {
                        const int r0 = 32 * (jj % T) + 4 * lane;
                        const float4 xv = *reinterpret_cast<const float4 *>(xs + r0);
                        const uint32_t xa = smem_u32(xs + r0), xra = smem_u32(&sh.xr[jj & 1]);
                        for (int q = 1; q < g; q++) st_async_v4(mapa(xa, leader + q), xv, mapa(xra, leader + q));
                    }
                };
                for (int j = 0; j < total; j++) {
                    const int b = j & 1;
                    mbar_wait(&sh.pready[b], (j >> 1) & 1);
                    const float *prb = &sh.pr[b][0][0][lane];
                    float v = 0.f;
                    for (int idx = 0; idx < np; idx++) v += prb[idx * 32];
                    sh.psum[b][lane] = v;
                    __syncwarp();
                    if (lane == 0) mbar_arrive_local(&sh.psum_full[b]);
                    if (g > 1 && j >= 1) push_x(j - 1);
                }
                if (g > 1 && total > 0) push_x(total - 1);
            }
        } else if (wid >= 2) {
            // ================= consumers: P_s = sum over J != kn of A[I_kn, I_J] x_J (old x for the
            // blocks being solved: the solver adds their increments)
            // warps 2,3,5,6,7 (none on the solver's sub-partition 0).  In the leader, consumer 4
            // computes L_kn x_kx^old (+ LL_kn x_{kn-2}^old, computed one step early as LL_{kn+1} x_kx^old)
            // and consumer 3 the in-block D product; the stream tiles (SegIter) go to the others.
            // Every warp sends its 32 partial row sums to the leader with st.async.
            const int c = (wid < 4) ? wid - 2 : wid - 3;
            const int rq = lane & 7, cq = lane >> 3;
            const int n_sw = is_leader ? kCons - 2 : kCons;   // warps taking stream tiles
            const bool do_L = is_leader && c == kCons - 1, do_D = is_leader && c == kCons - 2;
            uint32_t slot = 0, ph = 0;
            float lcarry[4] = {0.f, 0.f, 0.f, 0.f};   // L warp: LL_{kn+1} x_kx^old for the next step
            // profile item 0 (the largest bin): consumer 0 of the leader and of cluster rank 1
            const bool pf = prof && item == 0 && c == 0 && lane == 0 && crank <= 1;
            unsigned long long *pc = prof + (crank == 0 ? 5 : 16);
            unsigned long long tA = 0, cw_x = 0, cw_full = 0, c_comp = 0, c_red = 0, lat_sum = 0, lat_n = 0;
            for (int s = 0, kn = 0, kx = T - 1; s < total; s++, kx = kn, kn = (kn + 1 == T) ? 0 : kn + 1) {
                if (pf) tA = clock64();
                // x of solver step s-3 (the newest any stream tile needs).  The solver publishes it
                // only after it consumed P_{s-2}, so this step's partials cannot land in the
                // previous phase of P-ready[s&1].  At s = 2 that guarantee needs x of step 0.
                // Non-leader: arm x-ready for solver step s-2 first (its previous phase, step s-4,
                // was observed by this warp at step s-1), since the waits below may target it.
                if (!is_leader && c == 0 && lane == 0 && s >= 2) mbar_expect_tx(&sh.xr[s & 1], 128);
                if (s >= 3) {
                    if (is_leader) mbar_wait_cta(&sh.xr[(s - 3) & 1], ((s - 3) >> 1) & 1);
                    else mbar_wait(&sh.xr[(s - 3) & 1], ((s - 3) >> 1) & 1);
                } else if (s == 2) {
                    if (is_leader) mbar_wait_cta(&sh.xr[0], 0);
                    else mbar_wait(&sh.xr[0], 0);
                }
                // leader: arm this step's P-ready (its previous phase, step s-2, is complete)
                if (is_leader && c == 0 && lane == 0) mbar_expect_tx(&sh.pready[s & 1], (uint32_t)(g * kCons * 128));
                if (pf) { const unsigned long long t = clock64(); cw_x += t - tA; tA = t; }
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                float acc_t = 0.f;   // row `lane` of P_kn from transposed tiles and y
                if (do_L || do_D) {
                    const int b = s % kStg;
                    mbar_wait_cta(&sh.stg_full[b], (s / kStg) & 1);
                    // L: x_kx^old (last updated at step s-1-T); D: x_kn^old (step s-T).  With T <= 2
                    // those may be step s-2.
                    if (T <= 2 && s >= 2) mbar_wait_cta(&sh.xr[s & 1], ((s - 2) >> 1) & 1);
                    if (do_L) {
                        // L_kn x_kx^old + the carried LL_kn x_{kn-2}^old; then LL_{kn+1} x_kx^old
                        // (tile staged at step s-1) for the next step, while x_kx is still old
#pragma unroll
                        for (int q = 0; q < 4; q++) { acc[q] = lcarry[q]; lcarry[q] = 0.f; }
                        tile_dot(sh.rs[kRing * kChunk + 3 * (b) + 0], xs + 32 * kx, rq, cq, acc);
                        if (T >= 3 && s >= 1) tile_dot(sh.rs[kRing * kChunk + 3 * ((s - 1) % kStg) + 2], xs + 32 * kx, rq, cq, lcarry);
                        __syncwarp();
                        if (lane == 0 && s >= 1) mbar_arrive_local(&sh.stg_empty[(s - 1) % kStg]);
                    } else {
                        if (T >= 2) tile_dot(sh.rs[kRing * kChunk + 3 * (b) + 1], xs + 32 * kn, rq, cq, acc);
                        __syncwarp();
                        if (lane == 0) mbar_arrive_local(&sh.stg_empty[b]);
                    }
                } else {
                    // chunks of this step (seg_table): the step's i-th tile goes to stream warp i mod n_sw
                    float *yw = ys + c * ystride;
                    const Seg *sd = segt + 2 * kn;
                    // the lower part of row kn this warp accumulated from earlier steps' scatters
                    if (ordOf[kn] >= 0) {
                        float *yp = yw + ordOf[kn] * 32 + lane;
                        acc_t += *yp;
                        *yp = 0.f;
                    }
                    const float *x3 = xs + 32 * (kn - 3);   // scatter: x_{kn-3}^new
                    int first = c;   // index (within the next chunk) of this warp's first tile
                    for (int sg = 0; sg < 2; sg++) {
                        const Seg sr = sd[sg];
                        for (int off = 0; off < sr.len; off += chunk) {
                            const int nt = min(chunk, sr.len - off);
                            // every warp observes and releases every chunk (parity-tracked barriers: no
                            // warp may fall a ring lap behind or run one ahead)
                            const unsigned long long tw0 = pf ? clock64() : 0ull;
                            mbar_wait_cta(&sh.full[slot], ph);
                            if (pf) {
                                const unsigned long long t = clock64();
                                cw_full += t - tA; tA = t;
                                if (t - tw0 > 40) { lat_sum += t - sh.issue_t[slot]; lat_n++; }   // waited: ~ latency
                            }
                            int t = first;
                            for (; t < nt; t += n_sw) {
                                const int ord = sr.ord0 + off + t, J = ownJ[ord];
                                DWC_DCHECK(slot < (uint32_t)nring && J >= 0 && J < T, "gs consumer: slot / owned block");
                                const float *tile = slot_ptr(slot) + t * kTile;
                                if (sg == 0) {
                                    tile_dot(tile, xs + 32 * J, rq, cq, acc);
                                } else {
                                    const float v = tile_tdot(tile, x3, lane);
                                    if (J == kn) {
                                        acc_t += v;
                                    } else {
                                        yw[ord * 32 + lane] += v;
                                    }
                                }
                            }
                            first = t - nt;
                            if (pf) { const unsigned long long t = clock64(); c_comp += t - tA; tA = t; }
                            __syncwarp();
                            if (lane == 0) mbar_arrive_local(&sh.empty[slot]);
                            if (++slot == (uint32_t)nring) { slot = 0; ph ^= 1; }
                        }
                    }
                }
                // reduce over the 4 column groups: lanes (rq, cq) then hold rows 4rq..4rq+3; add the
                // per-lane (row = lane) transposed / y contributions
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 8);
                    acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 16);
                    acc[q] += __shfl_sync(0xffffffffu, acc_t, 4 * rq + q);
                }
                if (cq == 0)
                    st_async_v4(mapa(smem_u32(&sh.pr[s & 1][rg][c][4 * rq]), leader),
                                make_float4(acc[0], acc[1], acc[2], acc[3]), mapa(smem_u32(&sh.pready[s & 1]), leader));
                if (pf) { const unsigned long long t = clock64(); c_red += t - tA; tA = t; }
            }
            if (!is_leader && c == 0 && total > 0) {
                // observe every remaining x-ready phase (steps total-3 .. total-1; the last two are
                // armed here) so no async store lands after this item: barriers are re-initialised
                for (int j = total - 3; j < total; j++) {
                    if (j < 0) continue;
                    if (j >= total - 2 && lane == 0) mbar_expect_tx(&sh.xr[j & 1], 128);
                    mbar_wait(&sh.xr[j & 1], (j >> 1) & 1);
                }
            }
            if (pf) {
                pc[0] = cw_x; pc[1] = cw_full; pc[2] = c_comp; pc[3] = c_red;
                prof[crank == 0 ? 24 : 20] = lat_sum;
                prof[crank == 0 ? 25 : 21] = lat_n;
                if (crank == 0) prof[9] = total;
            }
        } else if (is_leader && total > 0) {
            // ================= solver (warp 0 of the leader) =================
            // Lane l: group L = l & 7 (rows 4L..4L+3), role = l >> 3.  Role 0 (lanes 0-7) solves
            // the current block; role 1 (lanes 8-15) executes the same instruction stream on the
            // next block's sub-diagonal tile, accumulating A[I_{k+1}, I_k] delta_k (lres, used at
            // the next step); role 2 (lanes 16-23) on LL_{k+2} = A[I_{k+2}, I_k], accumulating
            // A[I_{k+2}, I_k] delta_k (used two steps later); role 3 mirrors role 0.  x_k^new is
            // published (xs + x-ready) only once P_{k+1} has arrived, so the L warp reads x_k^old.
            const int L4 = 4 * (lane & 7);
            const bool role1 = (lane >> 3) == 1, role2 = (lane >> 3) == 2;
            float xprev[4] = {0.f, 0.f, 0.f, 0.f};
            float lres[4] = {0.f, 0.f, 0.f, 0.f};
            float ll0[4] = {0.f, 0.f, 0.f, 0.f}, ll1[4] = {0.f, 0.f, 0.f, 0.f};   // LL increments by step parity
            const bool use_ll = T >= 3;
            float invd[4], xo[4], wg10, wg20, wg30, wg21, wg31, wg32;
            float bhi[4], blo[4];
            int prev_row0 = -1;
            const bool pf = prof && item == 0 && lane == 0;
            unsigned long long tA = 0, w_p = 0, w_s = 0, c_set = 0, c_rec = 0, c_bc = 0, c_pub = 0, c_post = 0;
            auto publish = [&](int jj, int r0) {
                // x of solver step jj (block at r0) -> own xs + x-ready; bulk copies to the others
                // local only: the leader's D-product warp pushes the block to the other CTAs
                if (lane < 8) *reinterpret_cast<float4 *>(xs + r0 + L4) = make_float4(xprev[0], xprev[1], xprev[2], xprev[3]);
                __syncwarp();
                if (lane == 0) mbar_arrive_local(&sh.xr[jj & 1]);
            };
            // per-block operands of the own rows from the staged packet (+ x^old)
            auto prepare = [&](int jj) {
                const GsPacket &P = sh.pk[jj % kStg];
                const float4 iv = *reinterpret_cast<const float4 *>(&P.invd[L4]);
                invd[0] = iv.x; invd[1] = iv.y; invd[2] = iv.z; invd[3] = iv.w;
                const float4 w0 = *reinterpret_cast<const float4 *>(&P.wg[L4 >> 2][0]);
                const float4 w1 = *reinterpret_cast<const float4 *>(&P.wg[L4 >> 2][4]);
                wg10 = w0.x; wg20 = w0.y; wg30 = w0.z; wg21 = w0.w; wg31 = w1.x; wg32 = w1.y;
                const float4 bh = *reinterpret_cast<const float4 *>(&P.bhi[L4]);
                const float4 bl = *reinterpret_cast<const float4 *>(&P.blo[L4]);
                bhi[0] = bh.x; bhi[1] = bh.y; bhi[2] = bh.z; bhi[3] = bh.w;
                blo[0] = bl.x; blo[1] = bl.y; blo[2] = bl.z; blo[3] = bl.w;
                if (T == 1) {
#pragma unroll
                    for (int i = 0; i < 4; i++) xo[i] = xprev[i];
                } else {
                    const float4 v = *reinterpret_cast<const float4 *>(xs + 32 * (jj % T) + L4);
                    xo[0] = v.x; xo[1] = v.y; xo[2] = v.z; xo[3] = v.w;
                }
            };
            mbar_wait_cta(&sh.stg_full[0], 0);
            prepare(0);
            for (int j = 0, k = 0, sl = 0; j < total;
                 j++, k = (k + 1 == T) ? 0 : k + 1, sl = (sl + 1 == kStg) ? 0 : sl + 1) {
                const int b = j & 1, row0 = 32 * k, sl1 = (sl + 1 == kStg) ? 0 : sl + 1;

                const bool has_next = (j + 1 < total);
                if (pf) tA = clock64();
                const float *Dt = sh.rs[kRing * kChunk + 3 * (sl) + 1];
                // role 1 streams the next block's L tile (with no next step it re-reads Dt, unused),
                // role 2 the LL tile staged with this step
                const float *tp = (role1 && has_next) ? sh.rs[kRing * kChunk + 3 * (sl1) + 0] : (role2 ? sh.rs[kRing * kChunk + 3 * (sl) + 2] : Dt);
                // ---- critical path: P_k -> residual -> publish x_{k-1} -> recurrence
                mbar_wait_cta(&sh.psum_full[b], (j >> 1) & 1);
                if (pf) { const unsigned long long t = clock64(); w_p += t - tA; tA = t; }
                float ac[4];
                {
                    // P_j, summed by the helper warp
                    const float4 pv = *reinterpret_cast<const float4 *>(&sh.psum[b][L4]);
                    float a[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        a[i] += lres[i];
                        if (use_ll) a[i] += (j & 1) ? ll1[i] : ll0[i];
                        const float r = (a[i] - bhi[i]) - blo[i];   // residual against b~ = bhi + blo
                        ac[i] = (role1 || role2) ? 0.f : r;
                    }
                }
                // partials of P_j are consumed: x of step j-1 may now release the stream warps
                if (prev_row0 >= 0) publish(j - 1, prev_row0);
                if (pf) { const unsigned long long t = clock64(); c_pub += t - tA; tA = t; }
                // the next block's staged slot must have landed before the recurrence: role-1 lanes
                // read its L tile during it (its operands are loaded after the recurrence)
                if (has_next) mbar_wait_cta(&sh.stg_full[sl1], ((j + 1) / kStg) & 1);
                if (pf) { const unsigned long long t = clock64(); c_set += t - tA; tA = t; }
#pragma unroll
                for (int G = 0; G < 8; G++) {
                    const float m = (lane == G) ? 1.f : 0.f;
                    // this group's 4 tile columns (role 0/3: D, role 1: L_{k+1}, role 2: LL_{k+2})
                    float4 v[4];
#pragma unroll
                    for (int i = 0; i < 4; i++) v[i] = *reinterpret_cast<const float4 *>(tp + (4 * G + i) * 32 + L4);
                    // rows 4G..4G+3, sequential inside lane G, on temporaries taken before this
                    // group's updates; every delta is broadcast and applied to all lanes' residuals
                    // as soon as it is known (only the last one is on the path to the next group)
                    const float w0 = -ac[0] * invd[0], w1 = -ac[1] * invd[1], w2 = -ac[2] * invd[2],
                                w3 = -ac[3] * invd[3];
                    auto apply = [&](const float4 &t, float d) {
                        ac[0] = fmaf(t.x, d, ac[0]);
                        ac[1] = fmaf(t.y, d, ac[1]);
                        ac[2] = fmaf(t.z, d, ac[2]);
                        ac[3] = fmaf(t.w, d, ac[3]);
                    };
                    const float c0 = fmaxf(w0, -xo[0]);
                    apply(v[0], __shfl_sync(0xffffffffu, c0, G));
                    float u1 = fmaf(-wg10, c0, w1);
                    float u2 = fmaf(-wg20, c0, w2);
                    float u3 = fmaf(-wg30, c0, w3);
                    const float c1 = fmaxf(u1, -xo[1]);
                    apply(v[1], __shfl_sync(0xffffffffu, c1, G));
                    u2 = fmaf(-wg21, c1, u2);
                    u3 = fmaf(-wg31, c1, u3);
                    const float c2 = fmaxf(u2, -xo[2]);
                    apply(v[2], __shfl_sync(0xffffffffu, c2, G));
                    u3 = fmaf(-wg32, c2, u3);
                    const float c3 = fmaxf(u3, -xo[3]);
                    apply(v[3], __shfl_sync(0xffffffffu, c3, G));
                    xo[0] = fmaf(m, c0, xo[0]);
                    xo[1] = fmaf(m, c1, xo[1]);
                    xo[2] = fmaf(m, c2, xo[2]);
                    xo[3] = fmaf(m, c3, xo[3]);
                }
                if (pf) { asm volatile("" ::"f"(xo[3])); const unsigned long long t = clock64(); c_rec += t - tA; tA = t; }
                // role-1 accumulators (lanes 8-15) -> lres; role-2 (lanes 16-23) -> LL increment of
                // step j+2 (same parity slot as this step's, already consumed)
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    lres[i] = __shfl_sync(0xffffffffu, ac[i], (lane & 7) + 8);
                    const float v = __shfl_sync(0xffffffffu, ac[i], (lane & 7) + 16);
                    if (j & 1) ll1[i] = v;
                    else ll0[i] = v;
                    xprev[i] = xo[i];
                }
                prev_row0 = row0;
                __syncwarp();
                if (lane == 0) mbar_arrive_local(&sh.stg_empty[sl]);
                if (pf) { const unsigned long long t = clock64(); c_post += t - tA; tA = t; }
                // the next block's operands, after the recurrence: their load latency overlaps the
                // wait for the next P (the solver's registers stay free during the recurrence)
                if (has_next) prepare(j + 1);
                if (pf) { const unsigned long long t = clock64(); c_bc += t - tA; tA = t; }
            }
            publish(total - 1, prev_row0);
            if (pf) { prof[0] = w_p; prof[1] = w_s; prof[2] = c_set; prof[3] = c_rec; prof[4] = c_bc; prof[10] = c_pub; prof[11] = c_post; }
        }
        __syncthreads();
        // ---- output (leader): x~ and the embedded full-grid map (S8)
        if (is_leader && bin >= 0) {
            for (int i = tid; i < nk; i += kThreads) {
                const float v = xs[i];
                if (x_out) x_out[L.v_off + i] = v;
                if (x_map) x_map[(size_t)bin * S + keep_idx[(size_t)bin * S + i]] = v;
            }
        }
        cluster_sync();
    }
}

// Solver packets: one per (bin, block); reads the diagonal tile of A~ and b~.
__global__ void gs_prep_kernel(const BinLayout *__restrict__ lay, const float *__restrict__ A,
                               const double *__restrict__ bt, GsPacket *__restrict__ packets) {
    const int bin = blockIdx.y;
    const BinLayout L = lay[bin];
    const int T = L.sp >> 5, k = blockIdx.x, r = threadIdx.x;
    if (k >= T) return;
    const float *D = A + L.a_off + (size_t)k * kTile;   // D_k = tile (k,k), [c][r]
    GsPacket &P = packets[(L.v_off >> 5) + k];
    const int row = 32 * k + r;
    const float inv = (row < L.nk) ? __frcp_rn(D[r * 32 + r]) : 0.f;
    P.invd[r] = inv;
    const double bv = bt[L.v_off + row];
    const float bh = (float)bv;
    P.bhi[r] = bh;
    P.blo[r] = (float)(bv - (double)bh);
    __shared__ float sinv[32];
    sinv[r] = inv;
    __syncwarp();
    if (r < 8) {
        const int q = 4 * r;   // rows q+i', columns q+i, i < i'
        const float *c0 = D + (q + 0) * 32, *c1 = D + (q + 1) * 32, *c2 = D + (q + 2) * 32;
        P.wg[r][0] = c0[q + 1] * sinv[q + 1];
        P.wg[r][1] = c0[q + 2] * sinv[q + 2];
        P.wg[r][2] = c0[q + 3] * sinv[q + 3];
        P.wg[r][3] = c1[q + 2] * sinv[q + 2];
        P.wg[r][4] = c1[q + 3] * sinv[q + 3];
        P.wg[r][5] = c2[q + 3] * sinv[q + 3];
        P.wg[r][6] = 0.f;
        P.wg[r][7] = 0.f;
    }
}

int gs_packet_bytes() { return kPacketBytes; }

int launch_gs_prep(int n_bins, int max_sp, const BinLayout *lay_dev, const float *A, const double *bt,
                   void *packets, cudaStream_t st) {
    dim3 grid(max_sp >> 5, n_bins);
    gs_prep_kernel<<<grid, 32, 0, st>>>(lay_dev, A, bt, (GsPacket *)packets);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Layout conversions for the stage entry points: dense row-major n x n <-> symmetric tiles.
// to_sym: every (i, j) of the padded sp x sp matrix writes the stored tiles of its block with
// the upper-triangle value src[min(i,j)][max(i,j)] (0 outside n).
__global__ void tile_convert_kernel(int to_sym, int n, int sp, int g, const float *__restrict__ src,
                                    float *__restrict__ dst) {
    const int T = sp >> 5;
    const long total = (long)sp * sp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int i = (int)(e / sp), j = (int)(e - (long)(e / sp) * sp);
        const int lo = min(i, j), hi = max(i, j);
        if (to_sym) {
            const float v = (hi < n) ? src[(size_t)lo * n + hi] : 0.f;
            int t[2];
            const int nt = sym_targets(T, g, i >> 5, j >> 5, t);
            for (int u = 0; u < nt; u++) dst[(size_t)t[u] * kTile + (j & 31) * 32 + (i & 31)] = v;
        } else if (i < n && j < n) {
            const int tl = (lo >> 5) == (hi >> 5) ? (lo >> 5) : sym_u_tile(T, g, lo >> 5, hi >> 5);
            dst[(size_t)i * n + j] = src[(size_t)tl * kTile + (hi & 31) * 32 + (lo & 31)];
        }
    }
}

int launch_tile_convert(int to_sym, int n, int sp, int g, const float *src, float *dst, cudaStream_t st) {
    long total = (long)sp * sp;
    int blocks = (int)std::min<long>((total + 255) / 256, 148L * 32);
    tile_convert_kernel<<<blocks, 256, 0, st>>>(to_sym, n, sp, g, src, dst);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

size_t gs_smem_bytes(int max_sp, int ystride) {
    return sizeof(GsSmem) + (size_t)max_sp * 4 + (size_t)kCons * ystride * 4 + sizeof(Seg) * 2 * (size_t)(max_sp / 32) +
           2 * sizeof(int) * (size_t)(max_sp / 32);
}

// floats of y per stream warp: 32 per owned column block
int gs_ystride(int nk) {
    const int T = (nk + 31) / 32, g = gs_group_size(nk);
    int mx = 0;
    for (int o = 0; o < g; o++) mx = std::max(mx, sym_cnt(T - 1, o, g));
    return mx * 32;
}

int gs_cluster_size() { return kCl; }

int gs_item_ints() { return (int)(sizeof(GsItem) / sizeof(int)); }

// CTAs per bin from S~ alone (batch-independent => bit-identical per-bin results).
// Thresholds 832 / 448 (26 / 14 row blocks), measured on two bands with different S~ spreads
// (scripts/gs_group_variants.sh, GS ms): cfg3 linear predictor 768/384 47.2, 800/416 45.6-46.3,
// 832/448 45.5, 864/448 44.9-45.1, 896/448 45.2-45.8; cfg3 cubic predictor (3.5 % kept) 33.8-34.4,
// 34.6, 36.1-36.5, 40.6-41.7, 42.2-42.9.  The band is bound both by the largest bin's chain and
// by the CTA-steps all bins occupy: more CTAs per medium bin shorten chains that are not the
// longest but cost slots, so the best split depends on the S~ distribution; 832 / 448 is within
// 1 % of the best on the linear band and 6 % on the cubic one.  DWC_GS_G4 / DWC_GS_G2 override.
int gs_group_size(int nk) {
    static const int t4 = getenv("DWC_GS_G4") ? atoi(getenv("DWC_GS_G4")) : 832;
    static const int t2 = getenv("DWC_GS_G2") ? atoi(getenv("DWC_GS_G2")) : 448;
    return nk >= t4 ? 4 : (nk >= t2 ? 2 : 1);
}

int launch_gs(int n_items, const int *items, const BinLayout *lay_dev, int max_sp, int ystride, int *counter,
              const float *A,
              const void *packets, int sweeps, float *x_out, float *x_map, const int32_t *keep_idx, int S,
              int num_sms, const int *items_host, const BinLayout *lay_host, cudaStream_t st,
              GsLaunchInfo *info) {
    // DWC_GS_PROFILE=1: clock64 breakdown of the first CTA's solver / consumer warp (stderr).
    static const bool profile = getenv("DWC_GS_PROFILE") != nullptr;
    unsigned long long *prof = nullptr;
    if (profile) {
        if (cudaMalloc(&prof, (32 + 2048) * sizeof(unsigned long long)) != cudaSuccess) return -1;
        cudaMemsetAsync(prof, 0, (32 + 2048) * sizeof(unsigned long long), st);
    }
    // one CTA per SM anyway (two would need 2 x (smem + 1 KB) <= 228 KB): the rest of the 227 KB
    // becomes extra ring tiles
    const size_t base = (gs_smem_bytes(max_sp, ystride) + 127) / 128 * 128;
    int xtra_tiles = 0;
    if (2 * (base + 1024) > 228 * 1024) xtra_tiles = (int)std::min<size_t>((227 * 1024 - base) / (kTile * 4), 4 * kChunkNL);
    static const int xt_env = getenv("DWC_GS_XTRA") ? atoi(getenv("DWC_GS_XTRA")) : -1;   // experiment
    if (xt_env >= 0 && xt_env < xtra_tiles) xtra_tiles = xt_env;
    const size_t smem = base + (size_t)xtra_tiles * kTile * 4;
    auto kern = xtra_tiles > 0 ? gs_cluster_kernel<true> : gs_cluster_kernel<false>;
    if (raise_smem_limit(kern, smem) != cudaSuccess) {
        if (prof) cudaFree(prof);
        return -1;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n_clusters = 0;
    cfg.gridDim = dim3(num_sms * 2);
    if (cudaOccupancyMaxActiveClusters(&n_clusters, kern, &cfg) != cudaSuccess || n_clusters < 1) {
        cudaGetLastError();
        n_clusters = num_sms / kCl;
    }
    static const int cl_env = getenv("DWC_GS_CLUSTERS") ? atoi(getenv("DWC_GS_CLUSTERS")) : 0;   // experiment
    if (cl_env > 0 && cl_env < n_clusters) n_clusters = cl_env;
    if (n_clusters > n_items) n_clusters = n_items;
    if (n_clusters < 1) n_clusters = 1;
    cfg.gridDim = dim3(n_clusters * kCl);
    // L2 prefetch distance: the runs are prefetched kPf steps ahead only while the prefetch and
    // scatter windows ((kPf + 3) steps of row runs) of the bins running at once fit in a share of
    // L2.  Full-grid systems (cfg4: 64 bins of T = 319) do not fit: the prefetched tiles were
    // evicted before use and DRAM read 3.3x the algorithmic bytes (profiles/r01/next).
    int pf = kPf;
    if (kPf > 0 && items_host && lay_host) {
        const int ni = gs_item_ints();
        double win = 0.0;
        for (int it = 0; it < std::min(n_items, n_clusters); it++)
            for (int q = 0; q < kCl; q++) {
                const int b = items_host[it * ni + 1 + q];
                if (b < 0) continue;
                const int T = lay_host[b].sp >> 5;
                win += (kPf + 3) * (double)kTile * 4.0 * 0.5 * (T - 1);
            }
        if (win > kL2WindowBytes) pf = 0;
    }
    if (info) {
        info->kernel = xtra_tiles > 0 ? DWC_GS_KERNEL_CLUSTER_XTRA : DWC_GS_KERNEL_CLUSTER;
        info->xtra_tiles = xtra_tiles;
        info->ctas = n_clusters * kCl;
        info->max_group = 0;
        if (items_host)
            for (int it = 0; it < n_items; it++) info->max_group = std::max(info->max_group, items_host[it * gs_item_ints()]);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, n_items, (const GsItem *)items, lay_dev, counter, A,
                                       (const GsPacket *)packets, sweeps, x_out, x_map, keep_idx, S, max_sp, ystride,
                                       pf, (int)base, xtra_tiles, prof);
    if (profile) {
        static unsigned long long h[32 + 2048];
        cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        {   // when each CTA ran out of items, relative to the first CTA start: the band's tail
            const int nc = std::min(n_clusters * kCl, 1024);
            unsigned long long t0 = ~0ull;
            std::vector<double> idle;
            for (int c = 0; c < nc; c++) t0 = std::min(t0, h[32 + 2 * c]);
            for (int c = 0; c < nc; c++) idle.push_back((h[33 + 2 * c] - t0) * 1e-6);
            std::sort(idle.begin(), idle.end());
            if (!idle.empty())
                fprintf(stderr, "[gs-prof] CTAs out of items at (ms): min %.2f p10 %.2f median %.2f p90 %.2f max %.2f\n",
                        idle.front(), idle[idle.size() / 10], idle[idle.size() / 2], idle[idle.size() * 9 / 10], idle.back());
        }
        const double n = h[9] ? (double)h[9] : 1.0;
        fprintf(stderr,
                "[gs-prof] steps=%llu grid=%d | solver cyc/step: wait_P %.0f wait_stg %.0f sum+publish %.0f fetch %.0f recur %.0f post %.0f prep %.0f"
                " | consumer0: wait_x %.0f wait_tile %.0f compute %.0f reduce+send %.0f\n",
                h[9], n_clusters * kCl, h[0] / n, h[1] / n, h[10] / n, h[2] / n, h[3] / n, h[11] / n,
                (h[4] - h[11]) / n, h[5] / n, h[6] / n, h[7] / n, h[8] / n);
        fprintf(stderr, "[gs-prof] dynamic smem %zu B per CTA (GsSmem %zu, %d extra ring tiles), %d clusters of %d\n", smem, sizeof(GsSmem), xtra_tiles,
                n_clusters, kCl);
        fprintf(stderr, "[gs-prof] producer: chunks=%llu (%.1f/step) wait_empty %.0f issue %.0f cyc/chunk\n", h[14],
                h[14] / n, h[14] ? (double)h[12] / h[14] : 0.0, h[14] ? (double)h[13] / h[14] : 0.0);
        fprintf(stderr, "[gs-prof] rank-1 consumer0: wait_x %.0f wait_tile %.0f compute %.0f reduce+send %.0f\n",
                h[16] / n, h[17] / n, h[18] / n, h[19] / n);
        fprintf(stderr, "[gs-prof] copy issue->arrival when a consumer had to wait: leader %.0f cyc (%llu waits), rank-1 %.0f cyc (%llu waits)\n",
                h[25] ? (double)h[24] / h[25] : 0.0, h[25], h[21] ? (double)h[20] / h[21] : 0.0, h[21]);
        cudaFree(prof);
    }
    return e == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
