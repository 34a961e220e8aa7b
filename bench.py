#!/usr/bin/env python
"""bench.py -- DAMAS on the wavelet-compressed grid, batched over frequency bins, on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]
                  [--scaling weak|strong]

One *step* = one pass of the whole hot path (S1..S8 of SURVEY §8(a): steering, fp64 DAS,
fp64 wavelet threshold + compaction, PSF on the kept points, Gauss-Seidel sweeps, embed)
over one band of synthetic input (BASELINE.json configs[2] = cfg3: 64 mics, 101x101 grid,
256 bins 0.5-10 kHz, ~5% kept, 1000 sweeps) already resident in HBM.

Two measurements, both bracketed by barrier + cuda.synchronize and timed with CUDA events:
  * sequential (`sequential` in the line): the same band K times, one at a time on one stream,
    each step timed alone with the L2 flushed (256 MiB write) between steps;
  * pipelined (the line's `value`, default; --no-pipeline keeps the sequential one): K
    consecutive bands -- new measurement blocks of the same scene, as a stream of acoustic
    data delivers them -- on several contexts and streams (3 on one GPU, 8 for a rank's shard of
    a sharded band; --contexts), each call with the DWC_THROUGHPUT hint, so that a band's DAS /
    compress / PSF and sweeps run beside the previous bands' sweeps; one event pair around the K
    steps, every step reading a band no earlier step read (no L2 reuse; the L2 is flushed
    once before).  e2e likewise, one host thread per context (the host call returns with
    its outputs in host memory).

Multi-GPU (torchrun, one rank per GPU, NCCL): bins are independent.  --scaling strong
(default for N > 1, the north_star's "256-bin workload ... bins sharded over 1/2/4/8 GPUs"):
the band's bins are strided over ranks (bin k -> rank k mod N) and the maps are gathered once
with a single all_gather_into_tensor at the end, inside the timed region; value = the band's
bins / max-over-ranks step time.  --scaling weak (explicit option): every rank solves its own
full band (per-rank seed), no data-path collective; value = N * bins / max-rank time.
`chain_floor_ms`: the slowest of the band's 16 largest bins solved alone in the same run -- the
sequential Gauss-Seidel chain that bounds any sharding of the band.

--impl reference: the fp64 CPU oracle (oracle/) as it stands, on this host's cores, timed
on a bounded strided sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "DAMAS freq-bins/s and PSF-stream HBM GB/s (compressed grid) at 1/2/4/8 B200"
UNIT = "freq-bins/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_desc(cfg):
    kept = {"cfg2": "~10%", "cfg3": "~5%", "cfg5": "~8%"}.get(cfg.name, "full grid" if cfg.full_grid else "")
    return (f"{cfg.name}: {cfg.m} mics ({cfg.aperture} m spiral), {cfg.n}x{cfg.n} grid (S={cfg.S}), "
            f"{cfg.n_bins} bins {cfg.f_lo:g}-{cfg.f_hi:g} Hz, "
            f"{'exact' if cfg.csm == 'exact' else f'{cfg.snapshots}-snapshot {cfg.snr_db:g} dB'} CSM, "
            f"eps={cfg.epsilon} ({kept} kept), {cfg.sweeps} sweeps")


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    # each step: a bounded strided sample (~4 bins per core, a few seconds on the box)
    nb = args.ref_bins or min(cfg.n_bins, 4 * cores)
    bins = synth.strided_bins(cfg.n_bins, nb)
    band = synth.make_band(cfg, bins=bins)
    oracle.build()
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.solve_band_cfg(band, n_threads=cores)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    ms = 1000.0 * float(np.mean(times))
    value = len(bins) / (ms / 1000.0)
    sample = f"{len(bins)} strided bins of {cfg.n_bins} (full {cfg.sweeps} sweeps each), fp64 oracle, pthread pool"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "bins_per_step": len(bins)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, budget_bins=None):
    """The oracle as it stands on the host cores, on a bounded strided sample."""
    import oracle
    cores = os.cpu_count() or 1
    # bounded sample sized for ~10-30 s of CPU work on the box (cfg3: 256 bins ~ 13 s on 16 cores)
    nb = budget_bins or min(cfg.n_bins, 16 * cores)
    bins = synth.strided_bins(cfg.n_bins, nb)
    band = synth.make_band(cfg, bins=bins)
    oracle.build()
    t0 = time.perf_counter()
    oracle.solve_band_cfg(band, n_threads=cores)
    dt = time.perf_counter() - t0
    return {"value": len(bins) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{len(bins)} strided bins of {cfg.n_bins}, full {cfg.sweeps} sweeps, {dt:.1f} s wall"}


# ------------------------------------------------------------------------------ our arm
FP64_PEAK_TFLOPS = 36.0   # DFMA and DMMA, measured on B200 by scripts/ubench/fp64.cu
KERNEL_FLAG = {"auto": None, "residual": False, "dense": True}   # dwc.py dense_stream argument


def step_roofline(st, sweeps, hbm_gbs, ms_step):
    """Lower bound of one step from the method's algorithmic work (per step, whole band)."""
    stream_ms = st["gs_bytes"] / (hbm_gbs * 1e9) * 1e3
    write_ms = st["gs_bytes"] / sweeps / (hbm_gbs * 1e9) * 1e3
    das_ms = 0.5 * st["das_flops"] / (FP64_PEAK_TFLOPS * 1e12) * 1e3
    total = stream_ms + write_ms + das_ms
    return {"gs_stream_ms": stream_ms, "psf_write_ms": write_ms, "das_fp64_ms": das_ms, "roofline_ms": total,
            "measured_ms": ms_step, "frac": total / ms_step}


def bench_value(n_bins_band: int, k_local: int, world: int, scaling: str, ms_max: float) -> float:
    """freq-bins/s of the whole job: strong = the band's bins / the max-over-ranks step time;
    weak = every rank's own band (world * k_local bins) / the same time."""
    total = n_bins_band if (scaling == "strong" and world > 1) else k_local * world
    return total / (ms_max / 1000.0)


def variant_key(cfg, args) -> str:
    """Key of profiles/gs_traffic.json: the ncu DRAM bytes of a GS launch are only reported for
    the exact config and variant they were captured on."""
    return (f"{cfg.name}|order{args.order}|dr{int(bool(args.dr))}|alt{int(bool(args.alt))}|{args.input}"
            f"{'|paper' if getattr(args, 'paper', False) else ''}"
            f"{'' if getattr(args, 'kernel', 'auto') == 'auto' else '|' + args.kernel}"
            f"|{args.scaling if int(os.environ.get('WORLD_SIZE', '1')) > 1 else 'n1'}"
            f"|g{int(os.environ.get('WORLD_SIZE', '1'))}")


def run_pipelined(args, cfg, band, geom, ctx, dev, world, rank, strong, flush, gather_band):
    """Consecutive bands on several contexts / streams (see run_ours).  Returns the per-step times of
    the device path and of the host path (CSMs from pinned host memory, outputs to pinned host
    memory, one host thread per context)."""
    import threading as th
    from concurrent.futures import ThreadPoolExecutor

    import torch
    import torch.distributed as dist

    from paper_1608_05179_b200 import Context
    K = args.steps
    # bands in flight: 3 for the whole band on one GPU (with the DWC_THROUGHPUT hint: 16.9 k
    # bins/s against 16.0 k with 2 and 16.6 k with 4); a rank's shard of a sharded band is smaller,
    # so more shards in flight fill its SMs (profiles/r02/shard_pipeline_projection.json: 8 best
    # for 128-, 64- and 32-bin shards)
    nc = args.contexts or (3 if not strong else 8)
    # warm-up: W steps, and at least one band per context (its workspace and first launches are
    # set up untimed)
    W = max(args.warmup, nc)
    n = W + K
    # exact-CSM configs have no measurement noise: their consecutive "blocks" are new scenes
    exact = cfg.csm == "exact"
    seed0 = rank if (args.scaling == "weak" or world == 1) else 0

    def mk(j):
        return synth.make_band(cfg, seed=seed0 + 1000 * (j + 1) if exact else seed0, bins=band.bins, block=0 if exact else j + 1)
    with ThreadPoolExecutor(8) as ex:
        pool = list(ex.map(mk, range(2 * n)))   # device path: bands 0..n-1; host path: n..2n-1
    ctxs = [ctx] + [Context(dev.index) for _ in range(nc - 1)]
    sts = [torch.cuda.Stream(dev) for _ in range(nc)]
    nb, S = len(band.freqs), cfg.S
    kw = dict(full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt, paper=args.paper,
              dense_stream=KERNEL_FLAG[args.kernel], throughput=args.throughput)

    def outs(device):
        mk_ = (lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)) if device else \
              (lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory())
        return {"n_keep": mk_(nb, torch.int32), "keep_idx": mk_((nb, S), torch.int32),
                "x_map": mk_((nb, S), torch.float32), "b_map": None}

    cur = torch.cuda.current_stream(dev)

    def timed(run_steps):
        if world > 1:
            dist.barrier()
        flush.zero_()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for s_ in sts:
            s_.wait_stream(cur)
        run_steps()
        for s_ in sts:
            cur.wait_stream(s_)
        e1.record(cur)
        torch.cuda.synchronize(dev)
        t = e0.elapsed_time(e1) / K
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    # device path: inputs resident in HBM
    csm_dev = [torch.from_numpy(pool[i].csm).to(dev) for i in range(n)]
    dout = [outs(True) for _ in range(nc)]

    def dstep(i, j):   # band i on context / stream j
        o = ctxs[j].solve_band(geom, pool[i].freqs, csm_dev[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                               out=dout[j], stream=sts[j], **kw)
        if strong:
            with torch.cuda.stream(sts[j]):
                mask = ctxs[j].keep_mask(o["n_keep"], o["keep_idx"], stream=sts[j])
                gather_band(o["x_map"], o["n_keep"], mask, cfg.n_bins)
    def drun(first, last):
        # one host thread per context, each waiting for its band before it starts its next one:
        # at most two bands in flight, the next band's DAS / compress / PSF taking the SMs the
        # previous band's sweeps free.  (Bands queued without that wait -- one host thread, the
        # calls return once the sweeps are launched -- overlapped unevenly: 9.6-11.9 k bins/s
        # from run to run against 11.9 k steady here.)
        def worker(j):
            for i in range(first + j, last, nc):
                t0 = time.perf_counter()
                if trace is not None:
                    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ea.record(sts[j])
                    wb = ctxs[j].workspace_bytes()
                dstep(i, j)
                t1 = time.perf_counter()
                if trace is not None:
                    eb.record(sts[j])
                sts[j].synchronize()
                if trace is not None:
                    trace.append((j, i, t0, t1, time.perf_counter(), ea.elapsed_time(eb),
                                  ctxs[j].workspace_bytes() - wb, float(dout[j]["x_map"].double().sum())))
        if strong:   # (the collectives must be issued in the same order on every rank: one thread)
            for i in range(first, last):
                dstep(i, (i - first) % nc)
            return
        ths = [th.Thread(target=worker, args=(j,)) for j in range(nc)]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
    trace = [] if os.environ.get("DWC_BENCH_TRACE") else None
    drun(0, W)
    torch.cuda.synchronize(dev)
    if trace is not None:
        trace.clear()
    ms_dev = timed(lambda: drun(W, n))
    if trace:   # (diagnostic: host-side band start / call return / band done, ms from the first)
        for i in range(W, n):
            o = ctxs[0].solve_band(geom, pool[i].freqs, csm_dev[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode, **kw)
            torch.cuda.synchronize(dev)
            print(f"alone band {i}: sum x {float(o['x_map'].double().sum())!r}", file=sys.stderr)
        t00 = min(x[2] for x in trace)
        for j, i, t0, t1, t2, dev_ms, grow, xs in sorted(trace, key=lambda x: x[2]):
            print(f"trace ctx {j} band {i}: start {1e3 * (t0 - t00):8.2f} ret {1e3 * (t1 - t00):8.2f} "
                  f"done {1e3 * (t2 - t00):8.2f} device {dev_ms:7.2f} ms, workspace +{grow} B, sum x {xs!r}",
                  file=sys.stderr)

    # host path: one host thread per context (the host call returns with the outputs in host
    # memory), CSMs from pinned host memory
    csm_host = [torch.from_numpy(pool[n + i].csm).pin_memory() for i in range(n)]
    hout = [outs(False) for _ in range(nc)]

    def hstep(i, j):
        ctxs[j].solve_band_host(geom, pool[n + i].freqs, csm_host[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                                cfg.full_grid, out=hout[j], stream=sts[j], order=args.order, dr=args.dr,
                                alt=args.alt, paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel],
                                throughput=args.throughput)

    def hrun(first, last):
        ths = [th.Thread(target=lambda j=j: [hstep(i, j) for i in range(first + j, last, nc)]) for j in range(nc)]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
    hrun(0, W)
    torch.cuda.synchronize(dev)
    ms_host = timed(lambda: hrun(W, n)) if not strong else None
    for c_ in ctxs[1:]:
        c_.close()
    mb = sum(p_.csm.nbytes for p_ in pool[W:n]) / 1e6
    return {"ms_per_step": ms_dev, "e2e_ms_per_step": ms_host if ms_host is not None else float("nan"),
            "desc": (f"consecutive bands (new measurement blocks of the same scene) on {nc} contexts and {nc} streams, "
                     + ("one host thread per context waiting for its band before the next" if not strong else
                        "this rank's shard of each band, issued in band order from one host thread (the gathers in "
                        "the same order on every rank), each call waiting for its context's previous band")
                     + f": at most {nc} bands in flight, a band's DAS/compress/PSF overlapping the previous band's "
                       "Gauss-Seidel tail"),
            "l2": (f"none between steps: each of the {K} timed steps reads its own band ({mb:.0f} MB of CSMs in "
                   f"all, never re-read); 256 MiB write before the timed region")}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1608_05179_b200 import Context, Geometry
    from paper_1608_05179_b200.band_parallel import gather_band, shard_bins

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    # inputs: weak = own full band per rank (seed = rank); strong = strided shard of one band
    if args.scaling is None:
        args.scaling = "strong" if world > 1 else "weak"
    if args.scaling == "weak" or world == 1:
        band = synth.make_band(cfg, seed=rank)
    else:
        band = synth.make_band(cfg, bins=shard_bins(cfg.n_bins, rank, world))
    K = len(band.freqs)
    geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    snapshots = args.input == "snapshots"
    if snapshots:   # NEXT-3: the CSMs are formed on the device from the snapshot spectra (Eq. 1)
        snap_np = synth.make_snapshots(cfg, seed=rank if (args.scaling == "weak" or world == 1) else 0,
                                       bins=band.bins)
        snap_dev = torch.from_numpy(snap_np).to(dev)
    else:
        csm_dev = torch.from_numpy(band.csm).to(dev)
    ctx = Context(dev.index)
    ctx.set_timing(True)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    S = cfg.S
    strong = args.scaling == "strong" and world > 1

    def step():
        if snapshots:
            out = ctx.solve_band_snapshots(geom, band.freqs, snap_dev, cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                                           full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt, stream=stream,
                                           paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel])
        else:
            out = ctx.solve_band(geom, band.freqs, csm_dev, cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                                 full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt, stream=stream,
                                           paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel])
        if strong:
            # the one collective: maps + keep bitmasks + counts, all ranks
            mask = ctx.keep_mask(out["n_keep"], out["keep_idx"], stream=stream)
            out["gathered"] = gather_band(out["x_map"], out["n_keep"], mask, cfg.n_bins)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(dev.index)
    clocks.start()
    ms_steps, st_list = [], []
    for it in range(args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_steps.append(e0.elapsed_time(e1))
        st_list.append(ctx.stats())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = clocks.stop()

    ms = float(np.mean(ms_steps))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = bench_value(cfg.n_bins, K, world, args.scaling, ms)

    # roofline of the dominant kernel (GS sweep stream), per launch, CUDA-event timed
    st = st_list[-1]
    gs_ms = float(np.mean([s["ms_gs"] for s in st_list]))
    algo_bytes = st["gs_bytes"]
    achieved = algo_bytes / (gs_ms / 1000.0) / 1e9
    peak, peak_src = load_peaks()
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "gs_traffic.json")
    if os.path.exists(tp):
        try:
            rec = json.load(open(tp)).get(variant_key(cfg, args))
            if rec is not None and rec.get("gs_kernel") == st.get("gs_kernel"):
                traffic, traffic_src = rec["dram_bytes"], rec["source"]
        except Exception:
            traffic = None
    launches = int(sum(s["launches"] for s in st_list))

    # e2e through the C ABI with host buffers (pinned), copies inside the timed region
    h_out = {"n_keep": torch.empty(K, dtype=torch.int32).pin_memory(),
             "keep_idx": torch.empty((K, S), dtype=torch.int32).pin_memory(),
             "x_map": torch.empty((K, S), dtype=torch.float32).pin_memory(), "b_map": None}
    if snapshots:
        snap_host = torch.from_numpy(snap_np).pin_memory()

        def e2e_call():
            snap_dev.copy_(snap_host, non_blocking=True)
            out = ctx.solve_band_snapshots(geom, band.freqs, snap_dev, cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                                           full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt, stream=stream,
                                           paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel])
            for key in ("n_keep", "keep_idx", "x_map"):
                h_out[key].copy_(out[key], non_blocking=True)
    else:
        csm_host = torch.from_numpy(band.csm).pin_memory()

        def e2e_call():
            ctx.solve_band_host(geom, band.freqs, csm_host, cfg.epsilon, cfg.sweeps, cfg.eps_mode, cfg.full_grid,
                                out=h_out, stream=stream, order=args.order, dr=args.dr, alt=args.alt,
                                paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel])
    e2e_call()
    e2e_ms = []
    for it in range(args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_call()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms.append(e0.elapsed_time(e1))
    ems = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([ems], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e_value = bench_value(cfg.n_bins, K, world, args.scaling, ems)

    # chain floor: the slowest of this rank's bins solved alone (same kernels, same stream, timing
    # on).  The chain length is the bin's number of changes, not its size, so the 16 largest bins
    # are each solved once alone and the slowest of them is re-timed.
    last = step()
    nk_last = last["n_keep"].cpu().numpy()

    def alone(kb):
        torch.cuda.synchronize(dev)
        if snapshots:
            ctx.solve_band_snapshots(geom, band.freqs[kb:kb + 1], snap_dev[kb:kb + 1], cfg.epsilon, cfg.sweeps,
                                     cfg.eps_mode, full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt,
                                     stream=stream)
        else:
            ctx.solve_band(geom, band.freqs[kb:kb + 1], csm_dev[kb:kb + 1], cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                           full_grid=cfg.full_grid, order=args.order, dr=args.dr, alt=args.alt, stream=stream,
                           paper=args.paper, dense_stream=KERNEL_FLAG[args.kernel])
        torch.cuda.synchronize(dev)
        return ctx.stats()

    cand = [int(k) for k in np.argsort(-nk_last, kind="stable")[:16]]
    first = {kb: alone(kb) for kb in cand}
    kbig = max(cand, key=lambda kb: first[kb]["ms_total"])
    chain = [first[kbig]] + [alone(kbig) for _ in range(2)]
    chain_floor = {"bin": int(band.bins[kbig]), "n_keep": int(nk_last[kbig]),
                   "gs_updates": int(chain[0]["gs_updates"]), "candidates": "the 16 largest bins, each alone",
                   "gs_ms": float(np.min([c["ms_gs"] for c in chain])),
                   "total_ms": float(np.min([c["ms_total"] for c in chain]))}
    if world > 1:
        t = torch.tensor([chain_floor["gs_ms"], chain_floor["total_ms"]], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        chain_floor["gs_ms"], chain_floor["total_ms"] = float(t[0]), float(t[1])
    h2d = snap_np.nbytes if snapshots else band.csm.nbytes
    d2h = K * 4 + K * S * 4 + K * S * 4
    seq = {"value": value, "ms_per_step": ms, "e2e_value": e2e_value, "e2e_ms_per_step": ems}

    # pipelined: consecutive bands (new measurement blocks of the same scene) on several contexts
    # and streams, so that a band's DAS / compress / PSF and sweeps run beside the previous bands'
    # sweeps.  Every timed step reads a band no earlier step read (no L2 reuse).
    pipe = None
    if args.pipeline and not snapshots:
        pipe = run_pipelined(args, cfg, band, geom, ctx, dev, world, rank, strong, flush, gather_band)
        value = bench_value(cfg.n_bins, K, world, args.scaling, pipe["ms_per_step"])
        ms = pipe["ms_per_step"]
        if math.isfinite(pipe["e2e_ms_per_step"]):   # (sharded runs keep the one-band-at-a-time e2e)
            e2e_value = bench_value(cfg.n_bins, K, world, args.scaling, pipe["e2e_ms_per_step"])
            ems = pipe["e2e_ms_per_step"]

    cvf = None
    if world == 1 and not args.no_cvf:
        # compressed-grid vs full-grid DAMAS on the same bins (north_star), scripts/compressed_vs_full.py
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import compressed_vs_full
        cvf = compressed_vs_full.measure(ctx)
        ctx.set_timing(True)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, args.ref_bins)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
            "dtype": "f32 (PSF + Gauss-Seidel); f64 (DAS map + wavelet threshold)", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "bins_per_gpu": K,
                       "predictor": "cubic (R19)" if args.order == 3 else "linear (R7)",
                       "diagonal_removal": bool(args.dr), "alternating_sweeps": bool(args.alt),
                       "paper_literal_psf": bool(args.paper), "gs_kernel_choice": args.kernel,
                       "parallelism": f"bins-dp{world}",
                       "l2_flush": (pipe["l2"] if pipe else "256 MiB write between timed steps"),
                       "pipeline": (pipe["desc"] if pipe else "none: one band at a time"),
                       "throughput_hint": bool(pipe) and args.throughput,
                       "inputs": ("snapshot spectra resident in HBM, CSM formed on device (Eq. 1)" if snapshots
                                  else "CSMs resident in HBM")},
            "psf_stream_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": {1: "gs_cluster_kernel<false>", 2: "gs_cluster_kernel<true>",
                                    3: "gs_alt_kernel", 4: "rgs_kernel"}.get(int(st["gs_kernel"]), str(st["gs_kernel"])),
                         "algorithmic_bytes_per_launch": algo_bytes, "kernel_ms": gs_ms, "peak_source": peak_src,
                         **({"streamed_bytes_per_launch": st["gs_row_bytes"], "row_updates": int(st["gs_updates"]),
                             "streamed_gbs": st["gs_row_bytes"] / (gs_ms / 1000.0) / 1e9,
                             "streamed_frac": st["gs_row_bytes"] / (gs_ms / 1000.0) / 1e9 / peak,
                             "chain_bound_frac": chain_floor["gs_ms"] / gs_ms,
                             "note": ("residual-update Gauss-Seidel: reads only the rows of A~ whose x changes "
                                      "(streamed_bytes, streamed_frac of the HBM peak); achieved = the SURVEY 8(d) "
                                      "algorithmic stream (packed A~ once per sweep) / kernel time, i.e. the "
                                      "dense-equivalent rate, > peak because the skipped rows are never read.  The "
                                      "kernel is bound by its longest bin's sequential chain of changes: "
                                      "chain_bound_frac = that bin's GS time alone / the band's GS time")}
                            if int(st["gs_kernel"]) == 4 else {})},
            "chain_floor_ms": chain_floor["total_ms"], "chain_floor": chain_floor,
            "stage_ms": {"das": float(np.mean([s["ms_das"] for s in st_list])),
                         "compress": float(np.mean([s["ms_compress"] for s in st_list])),
                         "psf": float(np.mean([s["ms_psf"] for s in st_list])), "gs": gs_ms,
                         "total_events": float(np.mean([s["ms_total"] for s in st_list]))},
            # whole-step roofline: the method's own minimal work at the measured
            # peaks -- the packed A~ stream and the A~ write over HBM, the Hermitian-half DAS on the
            # fp64 pipes (36 TF/s, scripts/ubench/fp64.cu) -- against the measured step time
            "step_roofline": step_roofline(st, cfg.sweeps, peak, ms),
            "sum_keep": int(st["sum_keep"]), "mean_keep_frac": st["sum_keep"] / (K * S),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": ems},
            # one band at a time on one stream (L2 flushed between steps): the value the
            # pipelined line's ratio to the sequential work is judged against
            "sequential": seq,
            "gpu_launches": launches,
            "compressed_vs_full": cvf,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)   # (the pipelined value amortises its fill and drain over the steps)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: strong (default) shards one band over the ranks; weak gives every rank its own band")
    ap.add_argument("--ref-bins", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cvf", action="store_true", help="skip the compressed-vs-full-grid measurement")
    ap.add_argument("--input", default="csm", choices=["csm", "snapshots"],
                    help="csm: CSMs resident in HBM (default); snapshots: snapshot spectra, Eq. 1 on device")
    ap.add_argument("--dr", action="store_true", help="CSM diagonal removal (reading R20)")
    ap.add_argument("--alt", action="store_true", help="alternating sweep directions (reading R21, variant kernel)")
    ap.add_argument("--paper", action="store_true",
                    help="paper-literal beamformer and PSF (Eq. 4 v, Eq. 7 g; asymmetric, NEXT-4)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "residual", "dense"],
                    help="Gauss-Seidel kernel: automatic by system size (default), residual, dense-stream")
    ap.add_argument("--order", type=int, default=1, choices=[1, 3],
                    help="S3 predictor: 1 linear (reading R7, default), 3 cubic (R19)")
    ap.add_argument("--contexts", type=int, default=None,
                    help="pipelined: bands in flight (contexts / streams / host threads); default 3 on one GPU, "
                         "8 for a sharded band")
    ap.add_argument("--no-throughput-hint", dest="throughput", action="store_false",
                    help="pipelined: do not pass DWC_THROUGHPUT (bands in flight) to the library")
    ap.add_argument("--no-pipeline", dest="pipeline", action="store_false",
                    help="time one band at a time only (default: consecutive bands on several contexts and streams)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
