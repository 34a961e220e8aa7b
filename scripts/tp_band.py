"""One cfg3 band solved with the DWC_THROUGHPUT hint, twice (ncu target: the second call's
residual-GS launches -- the two-CTAs-per-SM class holds every system up to 1280 points)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
band = synth.make_band(cfg)
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
ctx.set_timing(True)
csm = torch.from_numpy(band.csm).cuda()
for rep in range(2):
    ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, throughput=True)
    torch.cuda.synchronize()
    st = ctx.stats()
    print(f"throughput hint: gs {st['ms_gs']:.2f} ms, ctas {st['gs_ctas']}", flush=True)
