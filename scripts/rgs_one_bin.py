"""cfg3's largest bin alone through dwc_solve_band (one rgs_kernel launch per call; for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 254
band = synth.make_band(cfg, bins=[kb])
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
csm = torch.from_numpy(band.csm).cuda()
for _ in range(2):
    out = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode)
torch.cuda.synchronize()
print("ok", int(out["n_keep"][0]))
