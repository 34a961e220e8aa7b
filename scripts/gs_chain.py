"""GS latency-chain study on cfg3: the S~ distribution of the band, the band's GS time, and the
GS time of the largest bin's system solved alone (same size, random SPD), i.e. whether the band
is bound by the largest bin's per-block chain.  Usage: python scripts/gs_chain.py [config]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
band = synth.make_band(cfg, seed=0)
geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
ctx.set_timing(True)
csm = torch.from_numpy(band.csm).cuda()
for _ in range(2):
    out = ctx.solve_band(geom, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid)
torch.cuda.synchronize()
st = ctx.stats()
nk = out["n_keep"].cpu().numpy()
srt = np.sort(nk)[::-1]
print("band: bins", len(nk), "sum", nk.sum(), "max", srt[:8], "median", int(np.median(nk)))
print("band GS ms %.2f" % st["ms_gs"], "total ms %.2f" % st["ms_total"])
rng = np.random.default_rng(0)
for n in sorted(set([int(srt[0]), int(srt[len(srt) // 8]), 768, 512])):
    Mx = rng.standard_normal((n, 48)).astype(np.float32)
    A = torch.from_numpy((Mx @ Mx.T) / 48 + np.eye(n, dtype=np.float32)).cuda()
    b = torch.from_numpy(rng.random(n)).cuda()
    ctx.gs(A, b, cfg.sweeps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.gs(A, b, cfg.sweeps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    T = (n + 31) // 32
    print("alone n=%d T=%d: %.2f ms = %.3f us/step" % (n, T, ms, ms * 1e3 / (T * cfg.sweeps)))

# the band restricted to its largest bins: how the chain of the largest bin stretches with the
# number of large bins running beside it
order = np.argsort(-nk, kind="stable")
for top in (1, 8, 16, 37, 74, 128):
    sel = np.sort(order[:top])
    sub = torch.from_numpy(band.csm[sel]).cuda()
    for _ in range(2):
        ctx.solve_band(geom, band.freqs[sel], sub, cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid)
    torch.cuda.synchronize()
    print("top %3d bins (S~ %d..%d): GS %.2f ms" % (top, nk[order[0]], nk[order[top - 1]], ctx.stats()["ms_gs"]))
