"""Prototype: a cfg3 band split into its NA highest-frequency bins (the longest Gauss-Seidel
chains) and the rest, solved concurrently by two contexts on two streams (the A half's GS runs on
NA SMs while the B half's DAS/compress/PSF use the others)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
band = synth.make_band(cfg)
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
csm = torch.from_numpy(band.csm).cuda()
K, S = len(band.freqs), g.S
ca, cb = Context(0), Context(0)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
out = {"n_keep": torch.empty(K, dtype=torch.int32, device="cuda"),
       "keep_idx": torch.empty((K, S), dtype=torch.int32, device="cuda"),
       "x_map": torch.empty((K, S), dtype=torch.float32, device="cuda"), "b_map": None}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(na):
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    if na == 0:
        ca.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, out=out, stream=cur)
    else:
        sa.wait_stream(cur)
        sb.wait_stream(cur)
        oa = {k: (v[K - na:] if v is not None else None) for k, v in out.items()}
        ob = {k: (v[:K - na] if v is not None else None) for k, v in out.items()}
        ca.solve_band(g, band.freqs[K - na:], csm[K - na:], cfg.epsilon, cfg.sweeps, cfg.eps_mode, out=oa, stream=sa)
        cb.solve_band(g, band.freqs[:K - na], csm[:K - na], cfg.epsilon, cfg.sweeps, cfg.eps_mode, out=ob, stream=sb)
        cur.wait_stream(sa)
        cur.wait_stream(sb)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


ref = None
for na in [0, 16, 24, 32, 48, 64]:
    ts = []
    for it in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        ts.append(run(na))
    x = out["x_map"].clone()
    if ref is None:
        ref = x
    print(f"NA={na}: {np.median(ts[1:]):.2f} ms/band  ({K / np.median(ts[1:]) * 1e3:.0f} bins/s)  "
          f"identical={bool(torch.equal(x, ref))}", flush=True)
