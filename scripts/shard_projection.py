"""Strong-scaling projection on one B200: every rank's strided shard of the cfg3 band
(bins k = r, r + G, ...; band_parallel.shard_bins) solved on its own, G = 2, 4, 8, CUDA-event
timed with an L2 flush before each run.  For each G: the slowest shard's time (what a G-GPU run
waits for, without the final gather), the projected whole-band rate 256 / that time, and the
shard's chain floor (its slowest bin solved alone).  Writes the JSON to argv[1] (default stdout)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402
from paper_1608_05179_b200.band_parallel import shard_bins  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
band = synth.make_band(cfg)
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
csm = torch.from_numpy(band.csm).cuda()
ctx = Context(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cur = torch.cuda.current_stream()


def timed(idx, reps=3):
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        ctx.solve_band(g, band.freqs[idx], csm[idx], cfg.epsilon, cfg.sweeps, cfg.eps_mode, stream=cur)
        e1.record(cur)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.min(ts))


full = timed(list(range(cfg.n_bins)))   # (also sizes the context's workspace before the timings)
for k in range(cfg.n_bins):   # every single-bin workspace shape once, untimed
    ctx.solve_band(g, band.freqs[[k]], csm[[k]], cfg.epsilon, 1, cfg.eps_mode, stream=cur)
alone = {k: timed([k], reps=2) for k in range(cfg.n_bins)}   # every bin by itself (chain floors)
res = {"workload": "cfg3 (256 bins, 1000 sweeps)", "full_band_ms": full,
       "slowest_bin_alone_ms": max(alone.values()), "slowest_bin": int(max(alone, key=alone.get)), "shards": {}}
for G in (2, 4, 8):
    rows = []
    for r in range(G):
        idx = shard_bins(cfg.n_bins, r, G)
        ms = timed(idx)
        floor = max(alone[k] for k in idx)
        rows.append({"rank": r, "bins": len(idx), "ms": ms, "chain_floor_ms": floor, "ratio": ms / floor})
    worst = max(rows, key=lambda x: x["ms"])
    res["shards"][G] = {"max_rank_ms": worst["ms"], "projected_bins_per_s": cfg.n_bins / worst["ms"] * 1e3,
                        "speedup_vs_1": res["full_band_ms"] / worst["ms"], "ranks": rows}
    print(f"G={G}: max rank {worst['ms']:.2f} ms (chain floor {worst['chain_floor_ms']:.2f}, x{worst['ratio']:.2f}),"
          f" projected {cfg.n_bins / worst['ms'] * 1e3:.0f} bins/s, speedup {res['full_band_ms'] / worst['ms']:.2f}",
          file=sys.stderr, flush=True)
txt = json.dumps(res, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(txt)
else:
    print(txt)
