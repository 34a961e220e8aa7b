"""Two contexts on two streams: are the outputs of each band those of the band solved alone?
(diagnostic for bench.py's pipelined measurement)"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1608_05179_b200 import Context, Geometry  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
band0 = synth.make_band(cfg)
g = Geometry(band0.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
NB = 8
bands = [synth.make_band(cfg, seed=0, bins=band0.bins, block=j + 1) for j in range(NB)]
csm = [torch.from_numpy(b.csm).cuda() for b in bands]
ctxs = [Context(0), Context(0)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
ref = []
for j in range(NB):
    o = ctxs[0].solve_band(g, bands[j].freqs, csm[j], cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid)
    torch.cuda.synchronize()
    ref.append(float(o["x_map"].double().sum()))
print("alone:", ref, flush=True)
mode = sys.argv[1] if len(sys.argv) > 1 else "threads"
res = {}
outs = [None, None]


def run(j, i):
    o = ctxs[j].solve_band(g, bands[i].freqs, csm[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode, full_grid=cfg.full_grid,
                           stream=sts[j])
    sts[j].synchronize()
    res[i] = float(o["x_map"].double().sum())


for rep in range(3):
    res.clear()
    if mode == "threads":
        ths = [threading.Thread(target=lambda j=j: [run(j, i) for i in range(j, NB, 2)]) for j in range(2)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    else:   # one thread, contexts alternating
        for i in range(NB):
            run(i % 2, i)
    bad = [i for i in range(NB) if res.get(i) != ref[i]]
    print(f"{mode} rep {rep}: mismatching bands {bad}", [(i, res.get(i)) for i in bad], flush=True)
