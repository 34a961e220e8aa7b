"""GS profiler (DWC_GS_PROFILE=1) on cfg3 sub-bands of the 16 / 74 / 256 largest bins: which per-step
bucket of the largest bin stretches when its SMs are shared."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_1608_05179_b200 import Context, Geometry
cfg = synth.CONFIGS["cfg3"]
band = synth.make_band(cfg, seed=0)
geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
csm = torch.from_numpy(band.csm).cuda()
out = ctx.solve_band(geom, band.freqs, csm, cfg.epsilon, 10, cfg.eps_mode)
nk = out["n_keep"].cpu().numpy()
order = np.argsort(-nk, kind="stable")
for top in (16, 74, 256):
    sel = np.sort(order[:top])
    print("=== top", top, flush=True)
    sys.stderr.flush()
    ctx.solve_band(geom, band.freqs[sel], torch.from_numpy(band.csm[sel]).cuda(), cfg.epsilon, cfg.sweeps, cfg.eps_mode)
    torch.cuda.synchronize()
    sys.stderr.flush()
