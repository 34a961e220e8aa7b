"""Band tail: with DWC_GS_PROFILE=1 the library prints when each GS CTA ran out of items."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_1608_05179_b200 import Context, Geometry
cfg = synth.CONFIGS["cfg3"]
band = synth.make_band(cfg, seed=0)
geom = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
ctx.set_timing(True)
csm = torch.from_numpy(band.csm).cuda()
ctx.solve_band(geom, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode)
torch.cuda.synchronize()
print("GS ms", ctx.stats()["ms_gs"])
