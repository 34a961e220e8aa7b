"""A/B helper (library chosen by DWC_LIB): the cfg3 band's GS time (median of 5 calls) and the
chain-floor bin alone (ALONE_BIN, default 249; median of 3), one line per library."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = synth.CONFIGS[cfgname]
band = synth.make_band(cfg)
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
ctx.set_timing(True)
csm = torch.from_numpy(band.csm).cuda()
kw = dict(full_grid=cfg.full_grid)
gs, xs = [], None
for rep in range(6):
    out = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, **kw)
    if rep:
        gs.append(ctx.stats()["ms_gs"])
    xs = out["x_map"].float().cpu().numpy()
kb = int(os.environ.get("ALONE_BIN", 249 if cfgname == "cfg3" else int(np.argmax(out["n_keep"].cpu().numpy()))))
al = []
for rep in range(3):
    ctx.solve_band(g, band.freqs[kb:kb + 1], csm[kb:kb + 1], cfg.epsilon, cfg.sweeps, cfg.eps_mode, **kw)
    al.append(ctx.stats()["ms_gs"])
print(f"{os.path.basename(os.environ.get('DWC_LIB', 'libdwc.so'))} {cfgname}: band gs median {np.median(gs):.2f} "
      f"(min {min(gs):.2f} max {max(gs):.2f}) | bin {kb} alone {np.median(al):.2f} ms | sum x {xs.sum():.6e} md5 {hashlib.md5(xs.tobytes()).hexdigest()[:12]}", flush=True)
