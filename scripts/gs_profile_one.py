"""One synthetic system through dwc_gs with DWC_GS_PROFILE=1 (clock64 breakdown of the first
CTA's solver / consumer / producer warps, printed by the library to stderr).  N env = size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_05179_b200 import Context  # noqa: E402

n = int(os.environ.get("N", "1024"))
rng = np.random.default_rng(0)
M = rng.standard_normal((n, 48)).astype(np.float32)
A = torch.from_numpy((M @ M.T) / 48 + np.eye(n, dtype=np.float32)).cuda()
b = torch.from_numpy(rng.random(n)).cuda()
ctx = Context(0)
ctx.gs(A, b, int(os.environ.get("SWEEPS", "200")))
torch.cuda.synchronize()
