"""Compressed-grid vs full-grid DAMAS on the same bins (north_star: "the compressed-grid
speedup over full-grid DAMAS is reported as well").  cfg2: all 8 bins; cfg3: a
strided 32-bin subset (the full-grid A~ of all 256 bins would be 54 GB).  CUDA-event time of
one dwc_solve_band call each (inputs resident, one warm-up).  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402


def timed(ctx, geom, band, full):
    cfg = band.cfg
    csm = torch.from_numpy(band.csm).cuda()
    run = lambda: ctx.solve_band(geom, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=full)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = run()
    e1.record()
    torch.cuda.synchronize()
    st = ctx.stats()
    return e0.elapsed_time(e1), st, out


def measure(ctx):
    ctx.set_timing(True)
    res = {}
    for name, bins in (("cfg2", list(range(8))), ("cfg3", synth.strided_bins(256, 32))):
        band = synth.make_band(name, bins=bins)
        cfg = band.cfg
        geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
        tc, sc, _ = timed(ctx, geom, band, False)
        tf, sf, _ = timed(ctx, geom, band, True)
        res[name] = {"bins": len(bins), "sweeps": cfg.sweeps, "S": cfg.S,
                     "mean_keep": sc["sum_keep"] / len(bins),
                     "ms_compressed": tc, "ms_full": tf, "speedup": tf / tc,
                     "gs_ms_compressed": sc["ms_gs"], "gs_ms_full": sf["ms_gs"],
                     "gs_gbs_full": sf["gs_bytes"] / (sf["ms_gs"] / 1e3) / 1e9}
        print(name, res[name], file=sys.stderr, flush=True)
    return res


def main():
    print(json.dumps({"compressed_vs_full": measure(Context(0))}))


if __name__ == "__main__":
    main()
