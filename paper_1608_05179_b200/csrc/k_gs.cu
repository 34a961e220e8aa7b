// k_gs.cu -- S7 DAMAS non-negative Gauss-Seidel sweeps (+ S8 embed), the time sink.
//
// Eq. 13-14, readings R4, R11, R12, R18:
//   r_i = sum_{j<i} A_ij x_j^(n+1) + sum_{j>=i} A_ij x_j^(n) - b_i,
//   x_i^(n+1) = max(x_i^(n) - r_i / A_ii, 0),  i ascending, x^0 = 0, fixed sweep count.
// Row order and sweep order are kept exactly; only the summation order of each row dot
// differs from the oracle (fp32 A~ and fp32 partial dots; residual against fp64 b~).
//
// Block formulation (B = 32 rows, T = sp/32 blocks): solver step j solves block k = j mod T.
//   r_{I_k} = P_k + A[I_k, I_{k-1}] x_{k-1}^new - b_{I_k},
//   P_k    = sum over column blocks J != k-1 of A[I_k, I_J] x_J   (in-block: old values)
// P_k is produced by "stream" warps WHILE block k-1 is being solved (stream step s = k runs
// concurrently with solver step s-1); only the 32x32 sub-diagonal product and the in-block
// recurrence are on the critical path.  In-block recurrence, one warp, "step form":
//   w_l = -r_l / A_ll;  delta_t = max(w_t, -x_t)  (x_t + delta_t = max(x_t + w_t, 0))
//   w_l -= (A_lt / A_ll) delta_t for all lanes;   x_t += delta_t.
//
// B200 mapping
//  * A~_k stored as 32x32 fp32 tiles, column-major inside a tile, row-block-major:
//    tile (I,J) at ((I*T + J) * 1024) floats, element (32I+r, 32J+c) at [c*32 + r].
//  * A CTA = warp 0 solver, warp 1 TMA producer, warps 2..7 consumers.  The producer
//    streams this CTA's tiles of each row block with cp.async.bulk (4 KB, mbarrier
//    complete_tx) into a kStages-deep shared-memory ring, running ahead of the consumers
//    across steps (tiles do not depend on x); consumers compute 32-row partial dots with
//    LDS.128 (conflict-free on the column-major tile) and release the slots.
//  * Clusters of kCl = 4 CTAs.  A work item gives the cluster either one large bin
//    (sub-group of g = 4 CTAs), two medium bins (g = 2) or four small bins (g = 1).
//    Inside a sub-group every CTA keeps a full copy of x in shared memory; stream tiles of
//    a row block are dealt round-robin over the g CTAs; each CTA reduces its consumer
//    warps' partials and pushes 32 floats into the leader CTA's shared memory over DSMEM
//    (st.shared::cluster + remote mbarrier arrive, release.cluster); the leader's solver
//    broadcasts each new x block the same way.  No grid-wide or cluster barrier inside the
//    sweep loop; cluster barriers only between work items.
//  * g depends on S~ only (host), so a bin's result is bit-identical whatever else is in
//    the batch (and on however many GPUs the band is sharded); items run largest first.
#include <stdint.h>

#include <algorithm>

#include "dwc_internal.cuh"

namespace dwc {

constexpr int kCl = 4;             // cluster size
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kCons = kWarps - 2;  // consumer warps (2..7)
constexpr int kStages = 16;        // ring depth (4 KB tiles)
constexpr int kTile = 1024;        // floats per tile

struct GsItem {
    int g;          // CTAs per bin: 1, 2 or 4
    int bin[kCl];   // bins of the sub-groups (-1 = idle)
};

struct __align__(128) GsSmem {
    float ring[kStages][kTile];
    float stg[2][2][kTile];            // [buf][0 = L tile, 1 = D tile]
    float pw[2][kCons][32];            // consumer partials (double-buffered by step)
    float pr[2][kCl][32];              // sub-group partials (leader)
    unsigned long long full[kStages], empty[kStages];
    unsigned long long stg_full[2], stg_empty[2];
    unsigned long long pready[2];      // leader: g*32 arrivals per step
    unsigned long long xr[2];          // every CTA: 32 arrivals per solver step
    int item;
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
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
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
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Consumer: acc[q] (rows 4*rq+q) += sum over columns c = cq + 4i of tile[c][4rq+q] * x[c].
__device__ __forceinline__ void tile_dot(const float *__restrict__ tile, const float *__restrict__ xcol, int rq,
                                         int cq, float acc[4]) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int c = cq + 4 * i;
        const float4 v = *reinterpret_cast<const float4 *>(tile + c * 32 + 4 * rq);
        const float xv = xcol[c];
        acc[0] = fmaf(v.x, xv, acc[0]);
        acc[1] = fmaf(v.y, xv, acc[1]);
        acc[2] = fmaf(v.z, xv, acc[2]);
        acc[3] = fmaf(v.w, xv, acc[3]);
    }
}

// Stream step s computes P for block kn = s mod T excluding kx = (s-1) mod T.  Stream tiles
// of sub-group rank rg: J in [0,T), J mod g == rg, J != kx, J != kn.  The leader also stages
// tile (kn,kx) (L, for the solver) and (kn,kn) (D, solver + its old-x product).
__global__ void __launch_bounds__(kThreads, 2)
gs_cluster_kernel(int n_items, const GsItem *__restrict__ items, const BinLayout *__restrict__ lay,
                  int *__restrict__ counter, const float *__restrict__ A, const double *__restrict__ bt,
                  int sweeps, float *__restrict__ x_out, float *__restrict__ x_map,
                  const int32_t *__restrict__ keep_idx, int S) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    GsSmem &sh = *reinterpret_cast<GsSmem *>(smem_raw);
    float *xs = reinterpret_cast<float *>(smem_raw + sizeof(GsSmem));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t crank = cluster_rank();

    for (;;) {
        // ---- the cluster's next item: rank 0 pops and writes it into every CTA
        if (crank == 0 && tid == 0) {
            const int it = atomicAdd(counter, 1);
            for (uint32_t q = 0; q < kCl; q++) st_remote_s32(mapa(smem_u32(&sh.item), q), it);
        }
        cluster_sync();
        const int item = sh.item;
        if (item >= n_items) break;
        const GsItem IT = items[item];
        const int g = IT.g;
        const int sg = (int)crank / g, rg = (int)crank % g;
        const uint32_t leader = (uint32_t)(sg * g);
        const bool is_leader = (rg == 0);
        const int bin = IT.bin[sg];
        BinLayout L = {0, 0, 0, 0};
        if (bin >= 0) L = lay[bin];
        const int sp = L.sp, nk = L.nk, T = sp >> 5;
        const int total = (bin >= 0) ? sweeps * T : 0;
        const float *Ab = A + L.a_off;
        const double *btb = bt + L.v_off;

        for (int i = tid; i < sp; i += kThreads) xs[i] = 0.f;
        if (tid == 0) {
            for (int i = 0; i < kStages; i++) {
                mbar_init(&sh.full[i], 1);
                mbar_init(&sh.empty[i], 1);
            }
            for (int b = 0; b < 2; b++) {
                mbar_init(&sh.stg_full[b], 1);
                mbar_init(&sh.stg_empty[b], 2);
                mbar_init(&sh.pready[b], (uint32_t)g * 32);
                mbar_init(&sh.xr[b], 32);
            }
            fence_mbar_init();
        }
        cluster_sync();

        if (wid == 1) {
            // ================= TMA producer (one lane) =================
            if (lane == 0) {
                uint32_t seq = 0;
                for (int s = 0; s < total; s++) {
                    const int kn = s % T, kx = (s + T - 1) % T;
                    const float *rowb = Ab + (size_t)kn * T * kTile;
                    if (is_leader) {
                        const int b = s & 1;
                        mbar_wait(&sh.stg_empty[b], ((s >> 1) & 1) ^ 1);
                        mbar_expect_tx(&sh.stg_full[b], 2 * kTile * 4);
                        bulk_g2s(sh.stg[b][0], rowb + (size_t)kx * kTile, kTile * 4, &sh.stg_full[b]);
                        bulk_g2s(sh.stg[b][1], rowb + (size_t)kn * kTile, kTile * 4, &sh.stg_full[b]);
                    }
                    for (int J = rg; J < T; J += g) {
                        if (J == kx || J == kn) continue;
                        const uint32_t slot = seq % kStages;
                        mbar_wait(&sh.empty[slot], ((seq / kStages) & 1) ^ 1);
                        mbar_expect_tx(&sh.full[slot], kTile * 4);
                        bulk_g2s(sh.ring[slot], rowb + (size_t)J * kTile, kTile * 4, &sh.full[slot]);
                        seq++;
                    }
                }
            }
        } else if (wid >= 2) {
            // ================= consumers =================
            const int c = wid - 2;
            const int rq = lane & 7, cq = lane >> 3;
            uint32_t seq = 0;
            const uint32_t pr_base = smem_u32(&sh.pr[0][0][0]);
            for (int s = 0; s < total; s++) {
                const int kn = s % T, kx = (s + T - 1) % T;
                if (s >= 2) mbar_wait(&sh.xr[s & 1], ((s - 2) >> 1) & 1);
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                int i = 0;
                for (int J = rg; J < T; J += g) {
                    if (J == kx || J == kn) continue;
                    if (i == c) {
                        const uint32_t slot = seq % kStages;
                        mbar_wait(&sh.full[slot], (seq / kStages) & 1);
                        tile_dot(sh.ring[slot], xs + 32 * J, rq, cq, acc);
                        __syncwarp();
                        if (lane == 0) mbar_arrive_local(&sh.empty[slot]);
                    }
                    i = (i + 1 == kCons) ? 0 : i + 1;
                    seq++;
                }
                if (is_leader && c == kCons - 1) {
                    const int b = s & 1;
                    mbar_wait(&sh.stg_full[b], (s >> 1) & 1);
                    if (T >= 2) tile_dot(sh.stg[b][1], xs + 32 * kn, rq, cq, acc);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_local(&sh.stg_empty[b]);
                }
                // reduce over the 4 column groups: every lane then holds rows 4rq..4rq+3
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 8);
                    acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 16);
                }
                if (cq == 0)
                    *reinterpret_cast<float4 *>(&sh.pw[s & 1][c][4 * rq]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
                named_bar(1, kCons * 32);
                if (c == 0) {
                    float v = 0.f;
#pragma unroll
                    for (int w = 0; w < kCons; w++) v += sh.pw[s & 1][w][lane];
                    const uint32_t off = (uint32_t)((((s & 1) * kCl + rg) * 32 + lane) * 4);
                    st_remote_f32(mapa(pr_base + off, leader), v);
                    mbar_arrive_remote(mapa(smem_u32(&sh.pready[s & 1]), leader));
                }
            }
        } else if (is_leader && total > 0) {
            // ================= solver (warp 0 of the leader) =================
            float xprev = 0.f;
            double bnext = btb[lane];
            const uint32_t xs_base = smem_u32(xs);
            for (int j = 0; j < total; j++) {
                const int k = j % T, b = j & 1, row0 = 32 * k;
                const double bk = bnext;
                bnext = btb[32 * ((j + 1) % T) + lane];
                mbar_wait(&sh.pready[b], (j >> 1) & 1);
                mbar_wait(&sh.stg_full[b], (j >> 1) & 1);
                float acc = 0.f;
                for (int q = 0; q < g; q++) acc += sh.pr[b][q][lane];
                const float *Lt = sh.stg[b][0];
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
                    a0 = fmaf(Lt[(t + 0) * 32 + lane], __shfl_sync(0xffffffffu, xprev, t + 0), a0);
                    a1 = fmaf(Lt[(t + 1) * 32 + lane], __shfl_sync(0xffffffffu, xprev, t + 1), a1);
                    a2 = fmaf(Lt[(t + 2) * 32 + lane], __shfl_sync(0xffffffffu, xprev, t + 2), a2);
                    a3 = fmaf(Lt[(t + 3) * 32 + lane], __shfl_sync(0xffffffffu, xprev, t + 3), a3);
                }
                acc += (a0 + a1) + (a2 + a3);
                // residual in fp64 against the fp64 b~ (an fp32 b~ would shift the fixed point)
                const double r = (double)acc - bk;
                const float *Dt = sh.stg[b][1];
                const float dii = Dt[lane * 32 + lane];
                const float invd = (row0 + lane < nk) ? 1.0f / dii : 0.f;
                float w = (float)(-r * (double)invd);
                float xo = xs[row0 + lane];
                float dp[32];
#pragma unroll
                for (int t = 0; t < 32; t++) dp[t] = Dt[t * 32 + lane] * invd;
#pragma unroll
                for (int t = 0; t < 32; t++) {
                    const float cand = fmaxf(w, -xo);
                    const float d = __shfl_sync(0xffffffffu, cand, t);
                    w = fmaf(-dp[t], d, w);
                    xo = (lane == t) ? xo + d : xo;
                }
                xprev = xo;
                __syncwarp();
                if (lane == 0) mbar_arrive_local(&sh.stg_empty[b]);
                // broadcast the new block to every CTA of the sub-group (self included)
                const uint32_t xa = xs_base + (uint32_t)(row0 + lane) * 4;
                const uint32_t xra = smem_u32(&sh.xr[b]);
                for (int q = 0; q < g; q++) {
                    st_remote_f32(mapa(xa, leader + q), xo);
                    mbar_arrive_remote(mapa(xra, leader + q));
                }
            }
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

// Layout conversions for the stage entry points: dense row-major n x n <-> tiled.
__global__ void tile_convert_kernel(int to_tiled, int n, int sp, const float *__restrict__ src,
                                    float *__restrict__ dst) {
    const int T = sp >> 5;
    const long total = (long)sp * sp;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
        const int tile = (int)(e >> 10), w = (int)(e & 1023);
        const int I = tile / T, J = tile - (tile / T) * T, c = w >> 5, r = w & 31;
        const int i = 32 * I + r, j = 32 * J + c;
        if (to_tiled)
            dst[e] = (i < n && j < n) ? src[(size_t)i * n + j] : 0.f;
        else if (i < n && j < n)
            dst[(size_t)i * n + j] = src[e];
    }
}

int launch_tile_convert(int to_tiled, int n, int sp, const float *src, float *dst, cudaStream_t st) {
    long total = (long)sp * sp;
    int blocks = (int)std::min<long>((total + 255) / 256, 148L * 32);
    tile_convert_kernel<<<blocks, 256, 0, st>>>(to_tiled, n, sp, src, dst);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

size_t gs_smem_bytes(int max_sp) { return sizeof(GsSmem) + (size_t)max_sp * 4; }

int gs_cluster_size() { return kCl; }

int gs_item_ints() { return (int)(sizeof(GsItem) / sizeof(int)); }

// CTAs per bin from S~ alone (batch-independent => bit-identical per-bin results).
int gs_group_size(int nk) { return nk >= 768 ? 4 : (nk >= 384 ? 2 : 1); }

int launch_gs(int n_items, const int *items, const BinLayout *lay_dev, int max_sp, int *counter, const float *A,
              const double *bt, int sweeps, float *x_out, float *x_map, const int32_t *keep_idx, int S,
              int num_sms, cudaStream_t st) {
    const size_t smem = gs_smem_bytes(max_sp);
    cudaFuncSetAttribute(gs_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    if (cudaOccupancyMaxActiveClusters(&n_clusters, gs_cluster_kernel, &cfg) != cudaSuccess || n_clusters < 1) {
        cudaGetLastError();
        n_clusters = num_sms / kCl;
    }
    if (n_clusters > n_items) n_clusters = n_items;
    if (n_clusters < 1) n_clusters = 1;
    cfg.gridDim = dim3(n_clusters * kCl);
    cudaError_t e = cudaLaunchKernelEx(&cfg, gs_cluster_kernel, n_items, (const GsItem *)items, lay_dev, counter, A,
                                       bt, sweeps, x_out, x_map, keep_idx, S);
    return e == cudaSuccess ? 1 : -1;
}

}  // namespace dwc
