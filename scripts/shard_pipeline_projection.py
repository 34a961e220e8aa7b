"""Strong-scaling projection with streamed bands, on one B200: a G-GPU run gives rank r the
strided shard k = r, r + G, ... of every band (band_parallel.shard_bins); with bands streaming in
(new measurement blocks of the same scene, as bench.py's pipelined measurement) each rank solves
its shard of consecutive bands on C contexts / streams, one host thread per context waiting for
its band before its next one.  For each G this times, on this one GPU, the shard holding the
band's slowest chain (bin 249 of cfg3, in shard 1 for every G > 1), K consecutive bands after W
warm-up ones, for several C; the projected whole-job rate is 256 bins / the per-band interval
(what a G-GPU strong-scaling run would report, the final gather of ~1.3 MB per band aside).
No rank's kernels wait on another's: every rank's work is independent.
Usage: python scripts/shard_pipeline_projection.py [out.json]"""
import json
import os
import sys
import threading
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402
from paper_1608_05179_b200.band_parallel import shard_bins  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
W0, K = 3, int(os.environ.get("PROJ_STEPS", "16"))
GS = [int(x) for x in os.environ.get("PROJ_G", "1,2,4,8").split(",")]
CS = [int(x) for x in os.environ.get("PROJ_C", "2,3,4,6,8").split(",")]
TP = os.environ.get("PROJ_THROUGHPUT", "1") == "1"   # the DWC_THROUGHPUT hint (bench.py's pipelined default)
band0 = synth.make_band(cfg, bins=[0])
g = Geometry(band0.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ctxs = [Context(0) for _ in range(max(CS))]
sts = [torch.cuda.Stream(dev) for _ in range(max(CS))]
cur = torch.cuda.current_stream(dev)
res = {"workload": "cfg3 (256 bins, 1000 sweeps), consecutive bands (blocks 1..W+K)", "warmup": "max(3, bands in flight)", "steps": K,
       "throughput_hint": TP,
       "shards": {}}


def run(bins, nc):
    W = max(W0, nc)
    with ThreadPoolExecutor(8) as ex:
        pool = list(ex.map(lambda j: synth.make_band(cfg, bins=bins, block=j + 1), range(W + K)))
    csm = [torch.from_numpy(b.csm).to(dev) for b in pool]
    freqs = pool[0].freqs

    def drun(first, last):
        def worker(j):
            for i in range(first + j, last, nc):
                ctxs[j].solve_band(g, freqs, csm[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode, stream=sts[j],
                                   throughput=TP)
                sts[j].synchronize()
        ths = [threading.Thread(target=worker, args=(j,)) for j in range(nc)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    drun(0, W)   # (W >= nc: every context warmed)
    torch.cuda.synchronize()
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in sts[:nc]:
        s.wait_stream(cur)
    drun(W, W + K)
    for s in sts[:nc]:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for G in GS:
    bins = shard_bins(cfg.n_bins, 1 if G > 1 else 0, G)
    rows = {}
    for nc in CS:
        ms = run(bins, nc)
        rows[nc] = {"ms_per_band": ms, "projected_bins_per_s": cfg.n_bins / ms * 1e3}
        print(f"G={G} ({len(bins)} bins per rank) C={nc}: {ms:.2f} ms per band -> {cfg.n_bins / ms * 1e3:.0f} bins/s",
              file=sys.stderr, flush=True)
    best = min(rows, key=lambda c: rows[c]["ms_per_band"])
    res["shards"][G] = {"bins_per_rank": len(bins), "by_contexts": rows, "best_contexts": best,
                        "projected_bins_per_s": rows[best]["projected_bins_per_s"]}
txt = json.dumps(res, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(txt)
print(txt)
