"""Residual GS kernel profile (DWC_RGS_PROF=1 prints the clock64 breakdown of the largest bin):
cfg3's largest bin alone, then the whole cfg3 band, with the GS event times."""
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
dense = os.environ.get("DENSE", "0") == "1"
out = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid, dense_stream=dense)
st = ctx.stats()
nk = out["n_keep"].cpu().numpy()
kb = int(os.environ.get("ALONE_BIN", np.argmax(nk)))   # default: the largest bin
print(f"{cfgname} band: gs {st['ms_gs']:.2f} ms total {st['ms_total']:.2f} ms kernel {st['gs_kernel']} ctas {st['gs_ctas']} "
      f"updates {st['gs_updates']} ({st['gs_updates'] / max(1, st['sum_keep'] * cfg.sweeps):.3f} of rows x sweeps)", flush=True)
for rep in range(2):
    ctx.solve_band(g, band.freqs[kb:kb + 1], csm[kb:kb + 1], cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid,
                   dense_stream=dense)
    s1 = ctx.stats()
    print(f"{cfgname} bin {kb} (S~={nk[kb]}) alone: gs {s1['ms_gs']:.2f} ms updates {s1['gs_updates']}", flush=True)
if os.environ.get("ALL_BINS", "0") == "1":
    # every bin alone: the chain that bounds the band is the bin with the most changes, not the largest
    rows = []
    for kb in range(len(band.freqs)):
        ctx.solve_band(g, band.freqs[kb:kb + 1], csm[kb:kb + 1], cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                       full_grid=cfg.full_grid, dense_stream=dense)
        s1 = ctx.stats()
        rows.append((s1["ms_gs"], kb, int(nk[kb]), s1["gs_updates"]))
    if os.environ.get("ALL_BINS_JSON"):
        import json
        json.dump([{"ms": r[0], "bin": r[1], "nk": r[2], "updates": r[3], "freq": float(band.freqs[r[1]])} for r in rows],
                  open(os.environ["ALL_BINS_JSON"], "w"))
    rows.sort(reverse=True)
    print("slowest bins alone (gs ms, bin, S~, updates):", " ".join(f"{r[0]:.2f}/{r[1]}/{r[2]}/{r[3]}" for r in rows[:8]))
    print(f"sum of bins alone {sum(r[0] for r in rows):.1f} ms -> /148 SMs {sum(r[0] for r in rows) / 148:.2f} ms")
