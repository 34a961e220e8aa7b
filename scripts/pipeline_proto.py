"""Prototype: consecutive cfg3 bands (distinct seeds) solved by two contexts on two streams,
alternating, so that one band's DAS/compress/PSF run in the tail of the previous band's GS.
Times K bands back to back (one event pair around all of them) against the same K bands
solved one after another on one stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
bands = [synth.make_band(cfg, seed=i) for i in range(K)]
g = Geometry(bands[0].mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
csms = [torch.from_numpy(b.csm).cuda() for b in bands]
ctxs = [Context(0), Context(0)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
S = g.S
outs = [{"n_keep": torch.empty(256, dtype=torch.int32, device="cuda"),
         "keep_idx": torch.empty((256, S), dtype=torch.int32, device="cuda"),
         "x_map": torch.empty((256, S), dtype=torch.float32, device="cuda"), "b_map": None} for _ in range(K)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(pipelined):
    cur = torch.cuda.current_stream()
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for st in sts:
        st.wait_stream(cur)
    for i in range(K):
        j = i % 2 if pipelined else 0
        ctxs[j].solve_band(g, bands[i].freqs, csms[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode, out=outs[i], stream=sts[j])
    for st in sts:
        cur.wait_stream(st)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(2):
    for pl in (False, True):
        ms = run(pl)
        print(f"{'pipelined' if pl else 'sequential'}: {ms / K:.2f} ms/band, {256 * K / ms * 1e3:.0f} bins/s", flush=True)
