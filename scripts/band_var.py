"""Per-band stage times of the bench's pool of consecutive cfg3 bands (bench.py run_pipelined:
new measurement blocks of one scene), each band alone on one context."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
band0 = synth.make_band(cfg)
g = Geometry(band0.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
ctx.set_timing(True)
for j in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    exact = cfg.csm == "exact"
    b = synth.make_band(cfg, seed=1000 * (j + 1) if exact else 0, bins=band0.bins, block=0 if exact else j + 1)
    csm = torch.from_numpy(b.csm).cuda()
    for rep in range(2):
        out = ctx.solve_band(g, b.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid)
        st = ctx.stats()
    nk = out["n_keep"].cpu()
    print(f"band {j}: total {st['ms_total']:.2f} das {st['ms_das']:.2f} psf {st['ms_psf']:.2f} gs {st['ms_gs']:.2f} ms, "
          f"sum S~ {int(nk.sum())} max {int(nk.max())} updates {st['gs_updates']} sum x {float(out['x_map'].double().sum())!r}",
          flush=True)
