// dwc_api.cu -- host side of the C ABI (include/dwc.h): validation, workspace pool,
// per-call layout of the compressed systems, LPT schedule, stage orchestration, stats.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "dwc_internal.cuh"

using namespace dwc;

cudaError_t dwc::raise_smem_limit(const void *fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> set;   // (device, kernel) -> limit set
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t &cur = set[{dev, fn}];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

namespace {

thread_local std::string g_err;

dwc_status fail(dwc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

struct PinBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// PSF output tiles (bin, I, J) of 128 rows x 32 columns (psf_tile_rows x psf_tile_cols) that touch
// the upper triangle of the sp x sp system (the kernel writes each computed entry and its mirror).
void append_psf_tiles(std::vector<int4> &tiles, int bin, int sp, bool all = false) {
    const int TR = dwc::psf_tile_rows(), TC = dwc::psf_tile_cols();
    for (int I = 0; I * TR < sp; I++)
        for (int J = 0; J * TC < sp; J++)
            if (all || J * TC + TC - 1 >= I * TR) tiles.push_back(make_int4(bin, I, J, 0));
}

enum FlagBits { kFlagNonFinite = 1, kFlagSingular = 4 };

}  // namespace

struct dwc_ctx {
    int device = 0;
    int num_sms = 148;
    size_t total_bytes = 0;
    DevBuf mic, freq, dist, amp, herm, bint, opa, opb, rsc, wt, bt, A, lay, order, counter, tiles, flag, items, packets,
        csm_h, nk_h, keep_h, xmap_h, bmap_h, gs_x, gs_b, Ad, upd, ampv, ampg, rscb;
    PinBuf stage, readback;
    size_t stage_off = 0;
    cudaEvent_t stage_done = nullptr;
    cudaStream_t copy_st = nullptr;         // host API: early keep-set readback (overlaps S5-S7)
    cudaEvent_t keep_ready = nullptr, copy_done = nullptr;
    // residual GS on a band whose systems need different cluster sizes: one launch per size class,
    // the classes on their own streams (forked from and joined back into the call's stream)
    static constexpr int kMaxClasses = 8;
    cudaStream_t class_st[kMaxClasses] = {};
    cudaEvent_t class_fork = nullptr, class_join[kMaxClasses] = {};
    int geo_m = -1, geo_n = -1;
    bool timing = false;
    cudaEvent_t ev[8] = {};
    // the end of the last call's work on this context: every call's stream waits for it first,
    // so calls on different streams never overlap on the shared workspace
    cudaEvent_t last_done = nullptr;
    bool last_valid = false;
    dwc_stats stats{};
    bool stats_events_valid = false;
    bool stats_upd_valid = false;   // the residual kernel's update counter belongs to the last call
};

namespace {

#define CU(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(e_ == cudaErrorMemoryAllocation ? DWC_ENOMEM : DWC_ECUDA,      \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define LAUNCH(expr)                                                                   \
    do {                                                                               \
        int n_ = (expr);                                                               \
        if (n_ < 0) {                                                                  \
            cudaError_t e_ = cudaGetLastError();                                       \
            return fail(DWC_ECUDA, "launch %s: %s", #expr, cudaGetErrorString(e_));   \
        }                                                                              \
        launches += n_;                                                                \
    } while (0)

dwc_status ensure(dwc_ctx *ctx, DevBuf &b, size_t bytes) {
    if (bytes <= b.bytes) return DWC_OK;
    // 25 % headroom, also on the first allocation: consecutive bands' sizes differ by a few per
    // cent (the kept counts), and a regrowth costs a device-wide synchronisation (cudaFree), which
    // stalls every other context's work on the device too
    bytes = std::max(bytes + bytes / 4, b.bytes + b.bytes / 4);
    if (b.p) {
        CU(cudaDeviceSynchronize());
        CU(cudaFree(b.p));
        ctx->total_bytes -= b.bytes;
        b.p = nullptr;
        b.bytes = 0;
    }
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWC_ENOMEM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    }
    b.bytes = bytes;
    ctx->total_bytes += bytes;
    return DWC_OK;
}

dwc_status ensure_pin(PinBuf &b, size_t bytes) {
    if (bytes <= b.bytes) return DWC_OK;
    bytes = std::max(bytes + bytes / 4, (size_t)64 << 10);   // (headroom: see ensure)
    if (b.p) CU(cudaFreeHost(b.p));
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMallocHost(&b.p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWC_ENOMEM, "pinned allocation of %zu bytes failed", bytes);
    }
    b.bytes = bytes;
    return DWC_OK;
}

// Staging of small host arrays into device buffers through a pinned bump buffer.  The
// buffer is reused only after the previous call's copies completed (event).
dwc_status stage_begin(dwc_ctx *ctx, size_t need) {
    CU(cudaEventSynchronize(ctx->stage_done));
    dwc_status s = ensure_pin(ctx->stage, need + 4096);
    if (s) return s;
    ctx->stage_off = 0;
    return DWC_OK;
}

dwc_status stage_upload(dwc_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return DWC_OK;
    size_t off = (ctx->stage_off + 255) & ~(size_t)255;
    if (off + bytes > ctx->stage.bytes) return fail(DWC_ECUDA, "internal: staging overflow");
    char *p = (char *)ctx->stage.p + off;
    memcpy(p, src, bytes);
    CU(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, st));
    ctx->stage_off = off + bytes;
    return DWC_OK;
}

dwc_status stage_end(dwc_ctx *ctx, cudaStream_t st) {
    CU(cudaEventRecord(ctx->stage_done, st));
    return DWC_OK;
}

bool finite(double v) { return std::isfinite(v); }

dwc_status check_ctx(dwc_ctx *ctx) {
    if (!ctx) return fail(DWC_EINVAL, "ctx is NULL");
    int cur = -1;
    CU(cudaGetDevice(&cur));
    if (cur != ctx->device) CU(cudaSetDevice(ctx->device));
    return DWC_OK;
}

// Order a call after the previous call on this context (whatever stream that used) and mark its
// end; the workspace is shared by every call.
dwc_status enter_stream(dwc_ctx *ctx, cudaStream_t st) {
    if (ctx->last_valid) CU(cudaStreamWaitEvent(st, ctx->last_done, 0));
    return DWC_OK;
}
struct StreamScope {   // marks the end of the call's work (also on an error return)
    dwc_ctx *ctx;
    cudaStream_t st;
    ~StreamScope() {
        if (cudaEventRecord(ctx->last_done, st) == cudaSuccess) ctx->last_valid = true;
        else cudaGetLastError();
    }
};
#define STREAM_SCOPE(ctx_, st_)                              \
    if ((s = enter_stream((ctx_), (st_)))) return s;         \
    StreamScope scope_{(ctx_), (st_)}

dwc_status check_array(const dwc_array *a) {
    if (!a) return fail(DWC_EINVAL, "array is NULL");
    if (a->m < 2 || a->m > DWC_MAX_MICS) return fail(DWC_EINVAL, "m = %d outside [2, %d]", a->m, DWC_MAX_MICS);
    if (!a->mic_xyz) return fail(DWC_EINVAL, "mic_xyz is NULL");
    if (!(a->c0 > 0.0) || !finite(a->c0)) return fail(DWC_EINVAL, "c0 must be > 0 and finite");
    for (int i = 0; i < 3 * a->m; i++)
        if (!finite(a->mic_xyz[i])) return fail(DWC_EINVAL, "mic_xyz[%d] is not finite", i);
    return DWC_OK;
}

dwc_status check_grid(const dwc_grid *g) {
    if (!g) return fail(DWC_EINVAL, "grid is NULL");
    if (g->n < 2 || g->n > 46340) return fail(DWC_EINVAL, "n = %d outside [2, 46340]", g->n);
    if (!(g->side_len > 0.0) || !finite(g->side_len)) return fail(DWC_EINVAL, "side_len must be > 0");
    if (!(g->z0 > 0.0) || !finite(g->z0)) return fail(DWC_EINVAL, "z0 must be > 0");
    if (!finite(g->cx) || !finite(g->cy)) return fail(DWC_EINVAL, "plane centre not finite");
    return DWC_OK;
}

dwc_status check_params(const dwc_params *p) {
    if (!p) return fail(DWC_EINVAL, "params is NULL");
    if (!(p->epsilon > 0.0) || !finite(p->epsilon)) return fail(DWC_EINVAL, "epsilon must be > 0");
    if (p->eps_mode != 0 && p->eps_mode != 1) return fail(DWC_EINVAL, "eps_mode must be 0 or 1");
    if (p->sweeps < 1) return fail(DWC_EINVAL, "sweeps must be >= 1");
    if (p->flags & ~(DWC_FULL_GRID | DWC_CUBIC | DWC_DIAG_REMOVAL | DWC_ALT_SWEEPS | DWC_GS_DENSE_STREAM | DWC_GS_RESIDUAL |
                     DWC_PAPER_PSF | DWC_THROUGHPUT))
        return fail(DWC_EINVAL, "unknown flags 0x%x", p->flags);
    if ((p->flags & DWC_GS_DENSE_STREAM) && (p->flags & DWC_GS_RESIDUAL))
        return fail(DWC_EINVAL, "DWC_GS_DENSE_STREAM and DWC_GS_RESIDUAL exclude each other");
    if ((p->flags & DWC_PAPER_PSF) && (p->flags & (DWC_DIAG_REMOVAL | DWC_GS_DENSE_STREAM)))
        return fail(DWC_EINVAL, "DWC_PAPER_PSF runs on the residual kernel, without diagonal removal");
    return DWC_OK;
}

dwc_status check_freqs(int n_bins, const double *f) {
    if (n_bins < 1) return fail(DWC_EINVAL, "n_bins must be >= 1");
    if (!f) return fail(DWC_EINVAL, "freq_hz is NULL");
    for (int k = 0; k < n_bins; k++)
        if (!(f[k] > 0.0) || !finite(f[k])) return fail(DWC_EINVAL, "freq_hz[%d] must be > 0", k);
    return DWC_OK;
}

// Full-grid mode knows S~ = S before any launch: reject a grid beyond the Gauss-Seidel kernels'
// on-chip capacity up front (compressed bands can only be checked once S~ is known).
dwc_status check_capacity_upfront(const dwc_grid *g, const dwc_params *p) {
    if (!(p->flags & DWC_FULL_GRID)) return DWC_OK;
    const int sp = (g->n * g->n + 31) & ~31;
    const bool fits = (p->flags & DWC_ALT_SWEEPS) ? true
                      : (rgs_smem_bytes(sp) <= 227 * 1024 || gs_smem_bytes(sp, gs_ystride(sp)) <= 227 * 1024);
    if (!fits) return fail(DWC_EINVAL, "full grid of %d points exceeds the on-chip capacity of the Gauss-Seidel kernels", sp);
    return DWC_OK;
}

Geo make_geo(dwc_ctx *ctx, const dwc_array *a, const dwc_grid *g) {
    Geo G;
    G.m = a->m;
    G.n = g->n;
    G.S = g->n * g->n;
    G.L = g->side_len;
    G.z0 = g->z0;
    G.cx = g->cx;
    G.cy = g->cy;
    G.dx = g->side_len / (double)(g->n - 1);
    G.c0 = a->c0;
    G.mic = (const double *)ctx->mic.p;
    return G;
}

// Upload mic + frequencies, build the steering tables.  Returns the launch count via *launches.
dwc_status prepare_geometry(dwc_ctx *ctx, const dwc_array *a, const dwc_grid *g, int n_freq,
                            const double *freq, Geo &G, int &launches, cudaStream_t st, bool paper = false) {
    dwc_status s;
    const size_t S = (size_t)g->n * g->n;
    if (paper && ((s = ensure(ctx, ctx->ampv, sizeof(double) * a->m * S)) || (s = ensure(ctx, ctx->ampg, sizeof(double) * a->m * S))))
        return s;
    if ((s = ensure(ctx, ctx->mic, sizeof(double) * 3 * a->m))) return s;
    if ((s = ensure(ctx, ctx->freq, sizeof(double) * std::max(n_freq, 1)))) return s;
    if ((s = ensure(ctx, ctx->dist, sizeof(double) * a->m * S))) return s;
    if ((s = ensure(ctx, ctx->amp, sizeof(double) * a->m * S))) return s;
    if ((s = ensure(ctx, ctx->flag, 64))) return s;
    if ((s = stage_begin(ctx, sizeof(double) * (3 * a->m + n_freq) + 1024))) return s;
    if ((s = stage_upload(ctx, ctx->mic.p, a->mic_xyz, sizeof(double) * 3 * a->m, st))) return s;
    if (n_freq > 0 && (s = stage_upload(ctx, ctx->freq.p, freq, sizeof(double) * n_freq, st))) return s;
    if ((s = stage_end(ctx, st))) return s;
    CU(cudaMemsetAsync(ctx->flag.p, 0, 64, st));
    G = make_geo(ctx, a, g);
    LAUNCH(launch_geom_tables(G, (double *)ctx->dist.p, (double *)ctx->amp.p, (int *)ctx->flag.p, st,
                              paper ? (double *)ctx->ampv.p : nullptr, paper ? (double *)ctx->ampg.p : nullptr));
    return DWC_OK;
}

// Work items of the GS cluster kernel: bins in descending S~ order, grouped by their
// per-bin CTA count g (batch independent): one g=4 bin, two g=2 bins or four g=1 bins per
// item; items stay in descending-work order (LPT).
std::vector<int> build_gs_items(const std::vector<int32_t> &order, const int32_t *nk) {
    const int cl = gs_cluster_size(), w = gs_item_ints();
    std::vector<int> items;
    std::vector<int> cur;
    int cur_g = 0;
    auto flush = [&]() {
        if (cur.empty()) return;
        items.push_back(cur_g);
        for (int q = 0; q < cl; q++) items.push_back(q < (int)cur.size() ? cur[q] : -1);
        for (int q = cl + 1; q < w; q++) items.push_back(-1);
        cur.clear();
    };
    for (int b : order) {
        const int g = gs_group_size(nk[b]);
        if (g != cur_g) {
            flush();
            cur_g = g;
        }
        cur.push_back(b);
        if ((int)cur.size() == cl / g) flush();
    }
    flush();
    return items;
}

void ev(dwc_ctx *ctx, int i, cudaStream_t st) {
    if (ctx->timing) cudaEventRecord(ctx->ev[i], st);
}

// The batched path on device buffers.  Input: the CSMs (csm) or, when snap != NULL, the
// snapshot spectra [n_bins][M][n_snap] from which Eq. 1 forms them on the device.
dwc_status solve_band_dev(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, const dwc_params *p,
                          int n_bins, const double *freq, const double *csm, int32_t *n_keep,
                          int32_t *keep_idx, float *x_map, double *b_map, uint32_t *warn,
                          cudaStream_t st, const double *snap = nullptr, int n_snap = 0,
                          int32_t *early_nk_host = nullptr, int32_t *early_keep_host = nullptr) {
    dwc_status s;
    int launches = 0;
    const int M = arr->m, n = grid->n;
    const int S = n * n;
    const bool paper = (p->flags & DWC_PAPER_PSF) != 0;   // NEXT-4: Eq. 4 / Eq. 7 as printed
    ev(ctx, 0, st);
    Geo G;
    if ((s = prepare_geometry(ctx, arr, grid, n_bins, freq, G, launches, st, paper))) return s;
    // S2 DAS on the Hermitian part of each CSM
    if ((s = ensure(ctx, ctx->herm, sizeof(double) * 2 * (size_t)n_bins * das_mpad(M) * das_mpad(M)))) return s;
    double *b = b_map;
    if (!b) {
        if ((s = ensure(ctx, ctx->bint, sizeof(double) * (size_t)n_bins * S))) return s;
        b = (double *)ctx->bint.p;
    }
    const int dr = (p->flags & DWC_DIAG_REMOVAL) ? 1 : 0;
    if (snap)
        LAUNCH(launch_csm(M, n_bins, n_snap, snap, (double *)ctx->herm.p, 1, dr, st));   // Eq. 1 -> Ch
    else
        LAUNCH(launch_hermitize(M, n_bins, csm, (double *)ctx->herm.p, dr, st));
    LAUNCH(launch_das(G, (double *)ctx->dist.p, (double *)(paper ? ctx->ampv.p : ctx->amp.p), n_bins,
                      (double *)ctx->freq.p, (double *)ctx->herm.p, b, dr, st));
    ev(ctx, 1, st);
    // S3+S4
    LAUNCH(launch_compress(n, n_bins, b, p->epsilon, p->eps_mode, (p->flags & DWC_FULL_GRID) ? 1 : 0, (p->flags & DWC_CUBIC) ? 3 : 1,
                           n_keep, keep_idx, nullptr, (int *)ctx->flag.p, st));
    ev(ctx, 2, st);
    // the single device->host read: kept counts (+ error flags)
    if ((s = ensure_pin(ctx->readback, sizeof(int32_t) * (n_bins + 16)))) return s;
    int32_t *hk = (int32_t *)ctx->readback.p;
    CU(cudaMemcpyAsync(hk, n_keep, sizeof(int32_t) * n_bins, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(hk + n_bins, ctx->flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const int flags = hk[n_bins];
    if (flags & kFlagSingular) return fail(DWC_ESINGULAR, "a scan-grid node coincides with a microphone");
    if (flags & kFlagNonFinite) return fail(DWC_ENUMERIC, "non-finite value in the CSM / DAS map");
    // host layout of the compressed systems
    std::vector<BinLayout> lay(n_bins);
    // GS kernel of the band (forward sweeps): DWC_GS_RESIDUAL / DWC_GS_DENSE_STREAM force one, else
    // the residual kernel when the band's largest system is at most rgs_auto_max_sp() points (one
    // SM streams a residual bin's changed rows; the dense-stream kernel spreads a large bin's
    // stream over 4 SMs)
    int band_sp = 0;
    for (int k = 0; k < n_bins; k++) band_sp = std::max(band_sp, (hk[k] + 31) & ~31);
    // (alternating sweeps: the residual kernel's visit sequence; the one-CTA-per-bin alternating
    // kernel only when the dense-stream kernel is asked for or the systems are too large)
    const bool resid = paper ||
                       ((p->flags & DWC_GS_RESIDUAL) || (!(p->flags & DWC_GS_DENSE_STREAM) && band_sp <= rgs_auto_max_sp()));
    const int alt = (p->flags & DWC_ALT_SWEEPS) ? 1 : 0;
    int64_t a_off = 0, v_off = 0, r_off = 0, d_off = 0;
    int max_sp = 0, max_rp = 0, ystride = 0;
    double sum_sq = 0.0, sum_sym = 0.0;
    int64_t sum_k = 0;
    const int TR = psf_tile_rows();
    for (int k = 0; k < n_bins; k++) {
        const int nk = hk[k];
        const int sp = (nk + 31) & ~31;
        const int rp = (nk + TR - 1) / TR * TR;
        lay[k] = {nk, sp, a_off, v_off, rp, gs_group_size(nk), r_off, d_off};
        if (!resid) a_off += sym_tiles(sp / 32) * 1024;
        if (resid) d_off += (int64_t)sp * sp;
        ystride = std::max(ystride, gs_ystride(nk));
        sum_sym += (double)nk * (nk + 1) / 2.0;
        v_off += sp;
        r_off += rp;
        max_sp = std::max(max_sp, sp);
        max_rp = std::max(max_rp, rp);
        sum_sq += (double)nk * nk;
        sum_k += nk;
    }
    if (resid ? rgs_smem_bytes(max_sp) > 227 * 1024 : gs_smem_bytes(max_sp, ystride) > 227 * 1024)
        return fail(DWC_EINVAL,
                    "compressed grid of %d points exceeds the on-chip capacity of the Gauss-Seidel kernels "
                    "(b_map, n_keep and keep_idx hold the S2-S4 results; x_map is not written)", max_sp);
    std::vector<int32_t> order(n_bins);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b2) { return hk[a] > hk[b2]; });
    std::vector<int> items = build_gs_items(order, hk);
    const int n_items = (int)items.size() / gs_item_ints();
    std::vector<int4> tiles;
    for (int k = 0; k < n_bins; k++) append_psf_tiles(tiles, k, lay[k].sp, paper);
    if ((s = ensure(ctx, ctx->lay, sizeof(BinLayout) * n_bins))) return s;
    if ((s = ensure(ctx, ctx->items, sizeof(int) * items.size()))) return s;
    if ((s = ensure(ctx, ctx->tiles, sizeof(int4) * std::max<size_t>(tiles.size(), 1)))) return s;
    if ((s = ensure(ctx, ctx->counter, 64))) return s;
    if ((s = ensure(ctx, ctx->opa, psf_opa_bytes(M, r_off))) || (s = ensure(ctx, ctx->opb, psf_opb_bytes(M, r_off))) ||
        (s = ensure(ctx, ctx->rsc, sizeof(double) * (size_t)r_off)))
        return s;
    if (dr && (s = ensure(ctx, ctx->wt, sizeof(double) * (size_t)r_off * M))) return s;
    if (paper && (s = ensure(ctx, ctx->rscb, sizeof(double) * (size_t)r_off))) return s;
    if ((s = ensure(ctx, ctx->bt, sizeof(double) * (size_t)v_off))) return s;
    if ((s = ensure(ctx, ctx->A, sizeof(float) * (size_t)std::max<int64_t>(a_off, 1024)))) return s;
    if (resid && ((s = ensure(ctx, ctx->Ad, sizeof(float) * (size_t)d_off)) || (s = ensure(ctx, ctx->upd, 64)) ||
                  (s = ensure(ctx, ctx->order, sizeof(int32_t) * n_bins))))
        return s;
    if ((s = ensure(ctx, ctx->packets, (size_t)gs_packet_bytes() * (size_t)(v_off / 32)))) return s;
    if ((s = stage_begin(ctx, sizeof(BinLayout) * n_bins + sizeof(int) * items.size() +
                                  sizeof(int4) * tiles.size() + 4096))) return s;
    if ((s = stage_upload(ctx, ctx->lay.p, lay.data(), sizeof(BinLayout) * n_bins, st))) return s;
    if ((s = stage_upload(ctx, ctx->items.p, items.data(), sizeof(int) * items.size(), st))) return s;
    if ((s = stage_upload(ctx, ctx->tiles.p, tiles.data(), sizeof(int4) * tiles.size(), st))) return s;
    if (resid && (s = stage_upload(ctx, ctx->order.p, order.data(), sizeof(int32_t) * n_bins, st))) return s;
    if ((s = stage_end(ctx, st))) return s;
    if (early_keep_host) {
        // the keep set is final: read it back on the copy stream while S5-S7 run (queued only now
        // that every check and allocation of the call has passed: no copy into the caller's
        // buffer outlives a failed call)
        if (!ctx->copy_st) {
            CU(cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&ctx->keep_ready, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
        }
        CU(cudaEventRecord(ctx->keep_ready, st));
        CU(cudaStreamWaitEvent(ctx->copy_st, ctx->keep_ready, 0));
        memcpy(early_nk_host, hk, sizeof(int32_t) * n_bins);
        CU(cudaMemcpyAsync(early_keep_host, keep_idx, sizeof(int32_t) * (size_t)n_bins * S, cudaMemcpyDeviceToHost,
                           ctx->copy_st));
        CU(cudaEventRecord(ctx->copy_done, ctx->copy_st));
        CU(cudaStreamWaitEvent(st, ctx->copy_done, 0));   // the call's stream covers the copy too
    }
    ev(ctx, 3, st);
    // S5 (+S6)
    LAUNCH(launch_psf(G, (double *)ctx->dist.p, (double *)(paper ? ctx->ampv.p : ctx->amp.p), n_bins,
                      (double *)ctx->freq.p, (BinLayout *)ctx->lay.p, keep_idx, b, max_rp, (int)tiles.size(),
                      (int4 *)ctx->tiles.p, (int8_t *)ctx->opa.p, (int8_t *)ctx->opb.p, (double *)ctx->rsc.p,
                      (double *)ctx->bt.p, dr ? (double *)ctx->wt.p : nullptr, (float *)ctx->A.p,
                      resid ? (float *)ctx->Ad.p : nullptr, st, paper ? (double *)ctx->ampg.p : nullptr,
                      paper ? (double *)ctx->rscb.p : nullptr));
    ev(ctx, 4, st);
    // S7 + S8
    CU(cudaMemsetAsync(x_map, 0, sizeof(float) * (size_t)n_bins * S, st));
    CU(cudaMemsetAsync(ctx->counter.p, 0, 64, st));
    ev(ctx, 5, st);
    GsLaunchInfo gsi;
    if (resid) {
        CU(cudaMemsetAsync(ctx->upd.p, 0, 64, st));
        // size classes of the bins (order = descending S~): the CTAs and registers each system
        // needs (rgs_size_class); one launch per class, the classes concurrently on their own streams
        // (wide clusters -- 5120 columns per CTA -- on the compressed grid, where many rows change
        // per sweep; narrow ones on the full grid, where few do)
        const bool wide_cl = !(p->flags & DWC_FULL_GRID);
        const int pair_sp = rgs_pair_max_sp(max_sp, n_bins, ctx->num_sms, (p->flags & DWC_THROUGHPUT) != 0);
        std::vector<std::pair<int, int>> cls;   // [begin, end) in `order`
        for (int i = 0; i < n_bins; i++) {
            const int g = rgs_size_class((hk[order[i]] + 31) & ~31, wide_cl, pair_sp);
            if (cls.empty() || rgs_size_class((hk[order[cls.back().first]] + 31) & ~31, wide_cl, pair_sp) != g)
                cls.push_back({i, i + 1});
            else
                cls.back().second = i + 1;
        }
        if ((int)cls.size() > dwc_ctx::kMaxClasses) {   // merge the smallest classes into the last one kept
            cls[dwc_ctx::kMaxClasses - 1].second = n_bins;
            cls.resize(dwc_ctx::kMaxClasses);
        }
        const int ncls = (int)cls.size();
        if (ncls > 1) {
            if (!ctx->class_fork) CU(cudaEventCreateWithFlags(&ctx->class_fork, cudaEventDisableTiming));
            for (int c = 1; c < ncls; c++) {
                if (!ctx->class_st[c]) CU(cudaStreamCreateWithFlags(&ctx->class_st[c], cudaStreamNonBlocking));
                if (!ctx->class_join[c]) CU(cudaEventCreateWithFlags(&ctx->class_join[c], cudaEventDisableTiming));
            }
            CU(cudaEventRecord(ctx->class_fork, st));
        }
        gsi = GsLaunchInfo{DWC_GS_KERNEL_RESIDUAL, 0, 0, 1};
        // every forked stream joins back into the call's stream, also when a launch fails midway
        // (no work of this call may outlive it on a stream the caller does not see)
        struct Join {
            dwc_ctx *ctx;
            cudaStream_t st;
            int forked = 0;
            ~Join() {
                for (int c = 1; c <= forked; c++) {
                    cudaEventRecord(ctx->class_join[c], ctx->class_st[c]);
                    cudaStreamWaitEvent(st, ctx->class_join[c], 0);
                }
            }
        } join{ctx, st};
        for (int c = 0; c < ncls; c++) {
            cudaStream_t cs = c == 0 ? st : ctx->class_st[c];
            if (c > 0) {
                CU(cudaStreamWaitEvent(cs, ctx->class_fork, 0));
                join.forked = c;
            }
            const int b0 = cls[c].first, nb = cls[c].second - cls[c].first;
            const int csp = (hk[order[b0]] + 31) & ~31;   // the class's largest system
            GsLaunchInfo ci;
            LAUNCH(launch_rgs(nb, (int *)ctx->order.p + b0, (BinLayout *)ctx->lay.p, csp, (int *)ctx->counter.p + c,
                              (float *)ctx->Ad.p, (double *)ctx->bt.p, p->sweeps, nullptr, x_map, keep_idx,
                              S, ctx->num_sms, (unsigned long long *)ctx->upd.p, cs, &ci, alt,
                              /*nonneg: every PSF is |.|^2 times positive scales*/ 1, wide_cl ? 1 : 0, pair_sp));
            gsi.ctas += ci.ctas;
            gsi.max_group = std::max(gsi.max_group, ci.max_group);
        }
    } else if (p->flags & DWC_ALT_SWEEPS) {
        gsi.kernel = DWC_GS_KERNEL_ALT;
        gsi.ctas = n_bins;
        gsi.max_group = 1;
        LAUNCH(launch_gs_alt(n_bins, (BinLayout *)ctx->lay.p, max_sp, (float *)ctx->A.p, (double *)ctx->bt.p,
                             p->sweeps, nullptr, x_map, keep_idx, S, st));
    } else {
    LAUNCH(launch_gs_prep(n_bins, max_sp, (BinLayout *)ctx->lay.p, (float *)ctx->A.p, (double *)ctx->bt.p,
                          ctx->packets.p, st));
    LAUNCH(launch_gs(n_items, (int *)ctx->items.p, (BinLayout *)ctx->lay.p, max_sp, ystride, (int *)ctx->counter.p,
                     (float *)ctx->A.p, ctx->packets.p, p->sweeps, nullptr, x_map, keep_idx, S,
                     ctx->num_sms, items.data(), lay.data(), st, &gsi));
    }
    ev(ctx, 6, st);
    // warnings (host, Eq. 24)
    if (warn) {
        double rmax = 0.0;
        for (int i = 0; i < M; i++)
            rmax = std::max(rmax, sqrt(arr->mic_xyz[3 * i] * arr->mic_xyz[3 * i] +
                                       arr->mic_xyz[3 * i + 1] * arr->mic_xyz[3 * i + 1]));
        const double phi = atan(grid->side_len / (2.0 * grid->z0));
        const double dx = grid->side_len / (double)(n - 1);
        for (int k = 0; k < n_bins; k++) {
            const double cp = cos(phi);
            const double B = 1.22 * grid->z0 * arr->c0 / (cp * cp * cp * 2.0 * rmax * freq[k]);
            warn[k] = (dx / B > 0.2) ? 1u : 0u;
        }
    }
    dwc_stats &stt = ctx->stats;
    stt = dwc_stats{};
    stt.n_bins = n_bins;
    stt.sum_keep = sum_k;
    stt.sum_keep_sq = sum_sq;
    stt.gs_bytes = 4.0 * sum_sym * p->sweeps;   // the symmetric-packed A~ (fp32) once per sweep
    stt.psf_flops = 8.0 * M * sum_sq;
    stt.das_flops = 8.0 * (double)M * M * S * n_bins;
    stt.launches = launches;
    stt.gs_kernel = gsi.kernel;
    stt.gs_xtra_tiles = gsi.xtra_tiles;
    stt.gs_ctas = gsi.ctas;
    stt.gs_max_group = gsi.max_group;
    ctx->stats_upd_valid = resid;
    ctx->stats_events_valid = ctx->timing;
    return DWC_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

const char *dwc_version(void) { return "dwc 0.1 (sm_100a)"; }

const char *dwc_last_error(void) { return g_err.c_str(); }

size_t dwc_workspace_bytes(const dwc_ctx *ctx) { return ctx ? ctx->total_bytes : 0; }

dwc_status dwc_create(int device, dwc_ctx **out) {
    if (!out) return fail(DWC_EINVAL, "out is NULL");
    *out = nullptr;
    int count = 0;
    CU(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(DWC_EINVAL, "device %d not present (%d devices)", device, count);
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(DWC_ESTATE, "device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
                    prop.major, prop.minor);
    CU(cudaSetDevice(device));
    dwc_ctx *c = new dwc_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    if (cudaEventCreateWithFlags(&c->stage_done, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return fail(DWC_ECUDA, "event creation failed");
    }
    for (auto &e : c->ev) cudaEventCreate(&e);
    if (cudaEventCreateWithFlags(&c->last_done, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return fail(DWC_ECUDA, "event creation failed");
    }
    *out = c;
    return DWC_OK;
}

dwc_status dwc_destroy(dwc_ctx *ctx) {
    if (!ctx) return DWC_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    DevBuf *bufs[] = {&ctx->mic, &ctx->freq, &ctx->dist, &ctx->amp, &ctx->herm, &ctx->bint, &ctx->opa, &ctx->opb, &ctx->rsc, &ctx->wt,
                      &ctx->bt, &ctx->A, &ctx->lay, &ctx->order, &ctx->counter, &ctx->tiles, &ctx->flag,
                      &ctx->items, &ctx->packets, &ctx->csm_h, &ctx->nk_h, &ctx->keep_h, &ctx->xmap_h, &ctx->bmap_h, &ctx->gs_x, &ctx->gs_b,
                      &ctx->Ad, &ctx->upd, &ctx->ampv, &ctx->ampg, &ctx->rscb};
    for (DevBuf *b : bufs)
        if (b->p) cudaFree(b->p);
    if (ctx->stage.p) cudaFreeHost(ctx->stage.p);
    if (ctx->readback.p) cudaFreeHost(ctx->readback.p);
    if (ctx->stage_done) cudaEventDestroy(ctx->stage_done);
    if (ctx->copy_st) cudaStreamDestroy(ctx->copy_st);
    if (ctx->keep_ready) cudaEventDestroy(ctx->keep_ready);
    if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
    for (int c = 0; c < dwc_ctx::kMaxClasses; c++) {
        if (ctx->class_st[c]) cudaStreamDestroy(ctx->class_st[c]);
        if (ctx->class_join[c]) cudaEventDestroy(ctx->class_join[c]);
    }
    if (ctx->class_fork) cudaEventDestroy(ctx->class_fork);
    if (ctx->last_done) cudaEventDestroy(ctx->last_done);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
    return DWC_OK;
}

dwc_status dwc_set_timing(dwc_ctx *ctx, int enable) {
    if (!ctx) return fail(DWC_EINVAL, "ctx is NULL");
    ctx->timing = enable != 0;
    return DWC_OK;
}

dwc_status dwc_get_stats(dwc_ctx *ctx, dwc_stats *out) {
    if (!ctx || !out) return fail(DWC_EINVAL, "NULL argument");
    dwc_stats s = ctx->stats;
    if (ctx->stats_upd_valid) {
        // residual kernel: rows of A~ the sweeps had to read (x changes), read back once
        unsigned long long u[2] = {0, 0};
        CU(cudaMemcpy(u, ctx->upd.p, sizeof u, cudaMemcpyDeviceToHost));
        s.gs_updates = (int64_t)u[0];
        s.gs_row_bytes = (double)u[1];
        ctx->stats.gs_updates = s.gs_updates;
        ctx->stats.gs_row_bytes = s.gs_row_bytes;
        ctx->stats_upd_valid = false;
    }
    if (ctx->stats_events_valid) {
        CU(cudaEventSynchronize(ctx->ev[6]));
        cudaEventElapsedTime(&s.ms_total, ctx->ev[0], ctx->ev[6]);
        cudaEventElapsedTime(&s.ms_das, ctx->ev[0], ctx->ev[1]);
        cudaEventElapsedTime(&s.ms_compress, ctx->ev[1], ctx->ev[2]);
        cudaEventElapsedTime(&s.ms_psf, ctx->ev[3], ctx->ev[4]);
        cudaEventElapsedTime(&s.ms_gs, ctx->ev[5], ctx->ev[6]);
    }
    *out = s;
    return DWC_OK;
}

dwc_status dwc_solve_band(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, const dwc_params *p,
                          int32_t n_bins, const double *freq_hz, const double *csm, int32_t *n_keep,
                          int32_t *keep_idx, float *x_map, double *b_map, uint32_t *warn,
                          void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_params(p)) ||
        (s = check_freqs(n_bins, freq_hz)))
        return s;
    if (!csm || !n_keep || !keep_idx || !x_map) return fail(DWC_EINVAL, "NULL device buffer");
    if ((s = check_capacity_upfront(grid, p))) return s;
    STREAM_SCOPE(ctx, (cudaStream_t)cuda_stream);
    return solve_band_dev(ctx, arr, grid, p, n_bins, freq_hz, csm, n_keep, keep_idx, x_map, b_map, warn,
                          (cudaStream_t)cuda_stream);
}

dwc_status dwc_solve_band_snapshots(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid,
                                    const dwc_params *p, int32_t n_bins, const double *freq_hz, int32_t n_snap,
                                    const double *snap, int32_t *n_keep, int32_t *keep_idx, float *x_map,
                                    double *b_map, uint32_t *warn, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_params(p)) ||
        (s = check_freqs(n_bins, freq_hz)))
        return s;
    if (n_snap < 1) return fail(DWC_EINVAL, "n_snap must be >= 1");
    if (!snap || !n_keep || !keep_idx || !x_map) return fail(DWC_EINVAL, "NULL device buffer");
    if ((s = check_capacity_upfront(grid, p))) return s;
    STREAM_SCOPE(ctx, (cudaStream_t)cuda_stream);
    return solve_band_dev(ctx, arr, grid, p, n_bins, freq_hz, nullptr, n_keep, keep_idx, x_map, b_map, warn,
                          (cudaStream_t)cuda_stream, snap, n_snap);
}

dwc_status dwc_csm(dwc_ctx *ctx, int32_t m, int32_t n_bins, int32_t n_snap, const double *snap, double *csm,
                   void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx))) return s;
    if (m < 1 || m > DWC_MAX_MICS || n_bins < 1 || n_snap < 1)
        return fail(DWC_EINVAL, "m = %d, n_bins = %d, n_snap = %d", m, n_bins, n_snap);
    if (!snap || !csm) return fail(DWC_EINVAL, "NULL device buffer");
    STREAM_SCOPE(ctx, (cudaStream_t)cuda_stream);
    int launches = 0;
    LAUNCH(launch_csm(m, n_bins, n_snap, snap, csm, 0, 0, (cudaStream_t)cuda_stream));
    return DWC_OK;
}

dwc_status dwc_solve_band_host(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid,
                               const dwc_params *p, int32_t n_bins, const double *freq_hz,
                               const double *csm, int32_t *n_keep, int32_t *keep_idx, float *x_map,
                               double *b_map, uint32_t *warn, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_params(p)) ||
        (s = check_freqs(n_bins, freq_hz)))
        return s;
    if (!csm || !n_keep || !keep_idx || !x_map) return fail(DWC_EINVAL, "NULL host buffer");
    if ((s = check_capacity_upfront(grid, p))) return s;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    const size_t S = (size_t)grid->n * grid->n, M = arr->m;
    const size_t csm_b = sizeof(double) * 2 * M * M * n_bins;
    if ((s = ensure(ctx, ctx->csm_h, csm_b)) || (s = ensure(ctx, ctx->nk_h, sizeof(int32_t) * n_bins)) ||
        (s = ensure(ctx, ctx->keep_h, sizeof(int32_t) * S * n_bins)) ||
        (s = ensure(ctx, ctx->xmap_h, sizeof(float) * S * n_bins)))
        return s;
    if (b_map && (s = ensure(ctx, ctx->bmap_h, sizeof(double) * S * n_bins))) return s;
    CU(cudaMemcpyAsync(ctx->csm_h.p, csm, csm_b, cudaMemcpyHostToDevice, st));
    // a pinned keep_idx buffer is filled while the PSF and Gauss-Seidel run (the keep set is final
    // after S4); pageable buffers are copied at the end (an early async copy would block the host)
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, keep_idx) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    s = solve_band_dev(ctx, arr, grid, p, n_bins, freq_hz, (double *)ctx->csm_h.p, (int32_t *)ctx->nk_h.p,
                       (int32_t *)ctx->keep_h.p, (float *)ctx->xmap_h.p,
                       b_map ? (double *)ctx->bmap_h.p : nullptr, warn, st, nullptr, 0,
                       pinned ? n_keep : nullptr, pinned ? keep_idx : nullptr);
    if (s) return s;
    if (!pinned) {
        CU(cudaMemcpyAsync(n_keep, ctx->nk_h.p, sizeof(int32_t) * n_bins, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(keep_idx, ctx->keep_h.p, sizeof(int32_t) * S * n_bins, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaMemcpyAsync(x_map, ctx->xmap_h.p, sizeof(float) * S * n_bins, cudaMemcpyDeviceToHost, st));
    if (b_map) CU(cudaMemcpyAsync(b_map, ctx->bmap_h.p, sizeof(double) * S * n_bins, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return DWC_OK;
}

dwc_status dwc_steer(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, double freq_hz,
                     int32_t n_pts, const int32_t *idx, double *E, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_freqs(1, &freq_hz)))
        return s;
    if (n_pts < 0 || (n_pts > 0 && (!idx || !E))) return fail(DWC_EINVAL, "bad n_pts / NULL buffer");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    int launches = 0;
    Geo G;
    if ((s = prepare_geometry(ctx, arr, grid, 1, &freq_hz, G, launches, st))) return s;
    LAUNCH(launch_steer(G, (double *)ctx->dist.p, (double *)ctx->amp.p, (double *)ctx->freq.p, n_pts, idx, E, st));
    return DWC_OK;
}

dwc_status dwc_das(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, int32_t n_bins,
                   const double *freq_hz, const double *csm, int32_t flags, double *b_map, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_freqs(n_bins, freq_hz)))
        return s;
    if (!csm || !b_map) return fail(DWC_EINVAL, "NULL device buffer");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    int launches = 0;
    if (flags & ~(DWC_DIAG_REMOVAL | DWC_PAPER_PSF)) return fail(DWC_EINVAL, "unknown flags 0x%x", flags);
    if ((flags & DWC_DIAG_REMOVAL) && (flags & DWC_PAPER_PSF))
        return fail(DWC_EINVAL, "DWC_PAPER_PSF excludes DWC_DIAG_REMOVAL");
    const bool paper = (flags & DWC_PAPER_PSF) != 0;
    Geo G;
    if ((s = prepare_geometry(ctx, arr, grid, n_bins, freq_hz, G, launches, st, paper))) return s;
    if ((s = ensure(ctx, ctx->herm, sizeof(double) * 2 * (size_t)n_bins * das_mpad(arr->m) * das_mpad(arr->m))))
        return s;
    const int dr = (flags & DWC_DIAG_REMOVAL) ? 1 : 0;
    LAUNCH(launch_hermitize(arr->m, n_bins, csm, (double *)ctx->herm.p, dr, st));
    LAUNCH(launch_das(G, (double *)ctx->dist.p, (double *)(paper ? ctx->ampv.p : ctx->amp.p), n_bins,
                      (double *)ctx->freq.p, (double *)ctx->herm.p, b_map, dr, st));
    return DWC_OK;
}

dwc_status dwc_compress(dwc_ctx *ctx, const dwc_grid *grid, const dwc_params *p, int32_t n_bins,
                        const double *b_map, int32_t *n_keep, int32_t *keep_idx, uint8_t *level,
                        void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_grid(grid)) || (s = check_params(p))) return s;
    if (n_bins < 1) return fail(DWC_EINVAL, "n_bins must be >= 1");
    if (!b_map || !n_keep || !keep_idx) return fail(DWC_EINVAL, "NULL device buffer");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    int launches = 0;
    if ((s = ensure(ctx, ctx->flag, 64))) return s;
    LAUNCH(launch_compress(grid->n, n_bins, b_map, p->epsilon, p->eps_mode, (p->flags & DWC_FULL_GRID) ? 1 : 0, (p->flags & DWC_CUBIC) ? 3 : 1,
                           n_keep, keep_idx, level, (int *)ctx->flag.p, st));
    return DWC_OK;
}

dwc_status dwc_psf(dwc_ctx *ctx, const dwc_array *arr, const dwc_grid *grid, double freq_hz,
                   int32_t n_keep, const int32_t *keep_idx, int32_t flags, float *A, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx)) || (s = check_array(arr)) || (s = check_grid(grid)) || (s = check_freqs(1, &freq_hz)))
        return s;
    const int S = grid->n * grid->n;
    if (n_keep < 1 || n_keep > S) return fail(DWC_EINVAL, "n_keep = %d outside [1, S]", n_keep);
    if (!keep_idx || !A) return fail(DWC_EINVAL, "NULL device buffer");
    if (flags & ~(DWC_DIAG_REMOVAL | DWC_PAPER_PSF)) return fail(DWC_EINVAL, "unknown flags 0x%x", flags);
    if ((flags & DWC_DIAG_REMOVAL) && (flags & DWC_PAPER_PSF))
        return fail(DWC_EINVAL, "DWC_PAPER_PSF excludes DWC_DIAG_REMOVAL");
    const int dr = (flags & DWC_DIAG_REMOVAL) ? 1 : 0;
    const bool paper = (flags & DWC_PAPER_PSF) != 0;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    int launches = 0;
    Geo G;
    if ((s = prepare_geometry(ctx, arr, grid, 1, &freq_hz, G, launches, st, paper))) return s;
    const int sp = (n_keep + 31) & ~31;
    const int rp = (n_keep + psf_tile_rows() - 1) / psf_tile_rows() * psf_tile_rows();
    BinLayout lay{n_keep, sp, 0, 0, rp, gs_group_size(n_keep), 0, 0};
    std::vector<int4> tiles;
    append_psf_tiles(tiles, 0, sp, paper);
    if (paper && ((s = ensure(ctx, ctx->rscb, sizeof(double) * rp)) || (s = ensure(ctx, ctx->Ad, sizeof(float) * (size_t)sp * sp))))
        return s;
    if ((s = ensure(ctx, ctx->lay, sizeof(BinLayout))) || (s = ensure(ctx, ctx->tiles, sizeof(int4) * tiles.size())) ||
        (s = ensure(ctx, ctx->opa, psf_opa_bytes(arr->m, rp))) || (s = ensure(ctx, ctx->opb, psf_opb_bytes(arr->m, rp))) ||
        (s = ensure(ctx, ctx->rsc, sizeof(double) * rp)) || (s = ensure(ctx, ctx->bt, sizeof(double) * sp)) ||
        (s = ensure(ctx, ctx->A, sizeof(float) * 1024 * (size_t)sym_tiles(sp / 32))))
        return s;
    if (dr && (s = ensure(ctx, ctx->wt, sizeof(double) * (size_t)rp * arr->m))) return s;
    if ((s = stage_begin(ctx, sizeof(BinLayout) + sizeof(int4) * tiles.size() + 1024))) return s;
    if ((s = stage_upload(ctx, ctx->lay.p, &lay, sizeof(BinLayout), st))) return s;
    if ((s = stage_upload(ctx, ctx->tiles.p, tiles.data(), sizeof(int4) * tiles.size(), st))) return s;
    if ((s = stage_end(ctx, st))) return s;
    if (paper) {
        // asymmetric: every tile, written transposed into the dense scratch, then A = its transpose
        LAUNCH(launch_psf(G, (double *)ctx->dist.p, (double *)ctx->ampv.p, 1, (double *)ctx->freq.p,
                          (BinLayout *)ctx->lay.p, keep_idx, nullptr, rp, (int)tiles.size(), (int4 *)ctx->tiles.p,
                          (int8_t *)ctx->opa.p, (int8_t *)ctx->opb.p, (double *)ctx->rsc.p, (double *)ctx->bt.p,
                          nullptr, (float *)ctx->A.p, (float *)ctx->Ad.p, st, (double *)ctx->ampg.p,
                          (double *)ctx->rscb.p));
        LAUNCH(launch_dense_extract(n_keep, sp, (float *)ctx->Ad.p, A, 1, st));
        return DWC_OK;
    }
    LAUNCH(launch_psf(G, (double *)ctx->dist.p, (double *)ctx->amp.p, 1, (double *)ctx->freq.p,
                      (BinLayout *)ctx->lay.p, keep_idx, nullptr, rp, (int)tiles.size(), (int4 *)ctx->tiles.p,
                      (int8_t *)ctx->opa.p, (int8_t *)ctx->opb.p, (double *)ctx->rsc.p, (double *)ctx->bt.p,
                      dr ? (double *)ctx->wt.p : nullptr, (float *)ctx->A.p, nullptr, st));
    LAUNCH(launch_tile_convert(0, n_keep, sp, lay.g, (float *)ctx->A.p, A, st));
    return DWC_OK;
}

dwc_status dwc_gs(dwc_ctx *ctx, int32_t n, const float *A, const double *b, int32_t sweeps, int32_t flags,
                  float *x, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx))) return s;
    if (n < 1) return fail(DWC_EINVAL, "n must be >= 1");
    if (sweeps < 1) return fail(DWC_EINVAL, "sweeps must be >= 1");
    if (!A || !b || !x) return fail(DWC_EINVAL, "NULL device buffer");
    if (flags & ~(DWC_ALT_SWEEPS | DWC_GS_DENSE_STREAM | DWC_GS_RESIDUAL | DWC_PAPER_PSF))
        return fail(DWC_EINVAL, "unknown flags 0x%x", flags);
    if ((flags & DWC_GS_DENSE_STREAM) && (flags & DWC_GS_RESIDUAL))
        return fail(DWC_EINVAL, "DWC_GS_DENSE_STREAM and DWC_GS_RESIDUAL exclude each other");
    // DWC_PAPER_PSF: A is a general (asymmetric) matrix, read in full; residual kernel
    const bool general = (flags & DWC_PAPER_PSF) != 0;
    if (general && (flags & DWC_GS_DENSE_STREAM))
        return fail(DWC_EINVAL, "a general (DWC_PAPER_PSF) matrix runs on the residual kernel");
    const int sp = (n + 31) & ~31;
    const bool resid = general || (flags & DWC_GS_RESIDUAL) || (!(flags & DWC_GS_DENSE_STREAM) && sp <= rgs_auto_max_sp());
    if (resid ? rgs_smem_bytes(sp) > 227 * 1024 : gs_smem_bytes(sp, gs_ystride(n)) > 227 * 1024)
        return fail(DWC_EINVAL, "n = %d exceeds the on-chip x capacity", n);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    STREAM_SCOPE(ctx, st);
    int launches = 0;
    // precondition A_ii > 0: checked on the device, read back before the sweeps
    if ((s = ensure(ctx, ctx->flag, 64)) || (s = ensure_pin(ctx->readback, 64))) return s;
    CU(cudaMemsetAsync(ctx->flag.p, 0, sizeof(int), st));
    LAUNCH(launch_diag_check(n, A, (int *)ctx->flag.p, st));
    CU(cudaMemcpyAsync(ctx->readback.p, ctx->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (*(int *)ctx->readback.p & 2) return fail(DWC_ENUMERIC, "A has a diagonal entry <= 0 or non-finite");
    const int nonneg = (*(int *)ctx->readback.p & 4) ? 0 : 1;   // no entry with its sign bit set, all finite
    BinLayout lay{n, sp, 0, 0, 0, gs_group_size(n), 0, 0};
    std::vector<int32_t> order{0};
    int32_t nk0 = n;
    std::vector<int> items = build_gs_items(order, &nk0);
    const size_t a_floats = 1024 * (size_t)(resid ? 1 : sym_tiles(sp / 32));
    if ((s = ensure(ctx, ctx->lay, sizeof(BinLayout))) || (s = ensure(ctx, ctx->items, sizeof(int) * items.size())) ||
        (s = ensure(ctx, ctx->counter, 64)) || (s = ensure(ctx, ctx->gs_b, sizeof(double) * sp)) ||
        (s = ensure(ctx, ctx->gs_x, sizeof(float) * a_floats)) ||
        (s = ensure(ctx, ctx->packets, (size_t)gs_packet_bytes() * (size_t)(sp / 32))) ||
        (s = ensure(ctx, ctx->order, sizeof(int32_t))))
        return s;
    if (resid && ((s = ensure(ctx, ctx->Ad, sizeof(float) * (size_t)sp * sp)) || (s = ensure(ctx, ctx->upd, 64))))
        return s;
    if ((s = stage_begin(ctx, 1024 + sizeof(int) * items.size()))) return s;
    if ((s = stage_upload(ctx, ctx->lay.p, &lay, sizeof(BinLayout), st))) return s;
    if ((s = stage_upload(ctx, ctx->items.p, items.data(), sizeof(int) * items.size(), st))) return s;
    if ((s = stage_upload(ctx, ctx->order.p, order.data(), sizeof(int32_t), st))) return s;
    if ((s = stage_end(ctx, st))) return s;
    float *Ap = (float *)ctx->gs_x.p;
    if (resid)
        LAUNCH(launch_rgs_convert(n, sp, A, (float *)ctx->Ad.p, st, general));
    else
        LAUNCH(launch_tile_convert(1, n, sp, lay.g, A, Ap, st));
    CU(cudaMemsetAsync(ctx->gs_b.p, 0, sizeof(double) * sp, st));
    CU(cudaMemcpyAsync(ctx->gs_b.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemsetAsync(ctx->counter.p, 0, 64, st));
    dwc_stats &stt = ctx->stats;
    stt = dwc_stats{};
    ctx->stats_events_valid = false;
    ctx->stats_upd_valid = false;
    stt.n_bins = 1;
    stt.sum_keep = n;
    stt.sum_keep_sq = (double)n * n;
    stt.gs_bytes = 2.0 * (double)n * (n + 1) * sweeps;
    if ((flags & DWC_ALT_SWEEPS) && !resid) {
        LAUNCH(launch_gs_alt(1, (BinLayout *)ctx->lay.p, sp, Ap, (double *)ctx->gs_b.p, sweeps, x, nullptr, nullptr,
                             0, st));
        stt.gs_kernel = DWC_GS_KERNEL_ALT;
        stt.gs_ctas = stt.gs_max_group = 1;
        stt.launches = launches;
        return DWC_OK;
    }
    GsLaunchInfo gsi;
    if (resid) {
        CU(cudaMemsetAsync(ctx->upd.p, 0, 64, st));
        LAUNCH(launch_rgs(1, (int *)ctx->order.p, (BinLayout *)ctx->lay.p, sp, (int *)ctx->counter.p,
                          (float *)ctx->Ad.p, (double *)ctx->gs_b.p, sweeps, x, nullptr, nullptr, 0, ctx->num_sms,
                          (unsigned long long *)ctx->upd.p, st, &gsi, (flags & DWC_ALT_SWEEPS) ? 1 : 0, nonneg));
        ctx->stats_upd_valid = true;
    } else {
        LAUNCH(launch_gs_prep(1, sp, (BinLayout *)ctx->lay.p, Ap, (double *)ctx->gs_b.p, ctx->packets.p, st));
        LAUNCH(launch_gs((int)items.size() / gs_item_ints(), (int *)ctx->items.p, (BinLayout *)ctx->lay.p, sp,
                         gs_ystride(n), (int *)ctx->counter.p, Ap, ctx->packets.p, sweeps, x, nullptr, nullptr, 0,
                         ctx->num_sms, items.data(), &lay, st, &gsi));
    }
    stt.launches = launches;
    stt.gs_kernel = gsi.kernel;
    stt.gs_xtra_tiles = gsi.xtra_tiles;
    stt.gs_ctas = gsi.ctas;
    stt.gs_max_group = gsi.max_group;
    return DWC_OK;
}

dwc_status dwc_keep_mask(dwc_ctx *ctx, int32_t n_bins, int32_t S, const int32_t *n_keep, const int32_t *keep_idx,
                         uint32_t *mask, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx))) return s;
    if (S < 1 || n_bins < 0) return fail(DWC_EINVAL, "S = %d, n_bins = %d", S, n_bins);
    if (n_bins == 0) return DWC_OK;
    if (!n_keep || !keep_idx || !mask) return fail(DWC_EINVAL, "NULL device buffer");
    STREAM_SCOPE(ctx, (cudaStream_t)cuda_stream);
    int launches = 0;
    LAUNCH(launch_keep_mask(n_bins, S, n_keep, keep_idx, mask, (cudaStream_t)cuda_stream));
    return DWC_OK;
}

dwc_status dwc_keep_unmask(dwc_ctx *ctx, int32_t n_bins, int32_t S, const uint32_t *mask, int32_t *n_keep,
                           int32_t *keep_idx, void *cuda_stream) {
    dwc_status s;
    if ((s = check_ctx(ctx))) return s;
    if (S < 1 || n_bins < 0) return fail(DWC_EINVAL, "S = %d, n_bins = %d", S, n_bins);
    if (n_bins == 0) return DWC_OK;
    if (!n_keep || !keep_idx || !mask) return fail(DWC_EINVAL, "NULL device buffer");
    STREAM_SCOPE(ctx, (cudaStream_t)cuda_stream);
    int launches = 0;
    LAUNCH(launch_keep_unmask(n_bins, S, mask, n_keep, keep_idx, (cudaStream_t)cuda_stream));
    return DWC_OK;
}

}  // extern "C"
