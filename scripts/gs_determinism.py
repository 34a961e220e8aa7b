"""Run-to-run determinism of the batched path on cfg3 (all 256 bins, full sweeps): x_map must be
bitwise identical across calls (fixed summation orders everywhere); prints the bins that differ."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
band = synth.make_band(cfg)
geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
csm = torch.from_numpy(band.csm).cuda()
ref = None
for r in range(reps):
    x = ctx.solve_band(geom, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode)["x_map"].cpu().numpy()
    if ref is None:
        ref = x
        continue
    bad = [k for k in range(x.shape[0]) if not np.array_equal(x[k], ref[k])]
    diff = max((float(np.abs(x[k] - ref[k]).max() / max(np.abs(ref[k]).max(), 1e-30)) for k in bad), default=0.0)
    print(f"rep {r}: {len(bad)} bins differ from rep 0 (max rel {diff:.2e}) {bad[:10]}", flush=True)
