cd $GRAFT_REPO_ROOT
python - <<'PY' > gpurun_out/wd.log 2>&1
import sys, torch, numpy as np
sys.path.insert(0,'.')
import synth
from paper_1608_05179_b200 import Context, Geometry
from paper_1608_05179_b200 import dwc
band = synth.make_band("cfg2")
cfg = band.cfg
g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
ctx = Context(0)
# print the smem offsets of the barriers for decoding
out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, cfg.sweeps)
torch.cuda.synchronize()
print("done", ctx.stats())
PY
