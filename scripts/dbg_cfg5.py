"""Single bins through dwc_solve_band on the residual kernel, GS time of each (argv: cfg:bin ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

ctx = Context(0)
ctx.set_timing(True)
for spec in (sys.argv[1:] or ["cfg5:600"]):
    name, kb = spec.split(":")
    cfg = synth.CONFIGS[name]
    band = synth.make_band(cfg, bins=[int(kb)])
    g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    csm = torch.from_numpy(band.csm).cuda()
    for rep in range(2):
        out = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, dense_stream=False)
        torch.cuda.synchronize()
    st = ctx.stats()
    print(f"{spec}: S~={int(out['n_keep'][0])} gs {st['ms_gs']:.2f} ms, {st['gs_updates']} updates, "
          f"{st['gs_ctas']} CTAs", flush=True)
