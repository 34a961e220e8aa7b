"""Per-step cost of the GS kernel on single synthetic systems (dwc_gs), to separate the
critical-path chain from streaming.  Prints n, T, g, ms, ns/step, GB/s."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_05179_b200 import Context  # noqa: E402


def main():
    ctx = Context(0)
    sweeps = int(os.environ.get("SWEEPS", "200"))
    rng = np.random.default_rng(0)
    for n in [32, 64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 4096]:
        M = rng.standard_normal((n, 48)).astype(np.float32)
        A = (M @ M.T) / 48 + np.eye(n, dtype=np.float32)
        A = torch.from_numpy(A).cuda()
        b = torch.from_numpy(rng.random(n)).cuda()
        ctx.gs(A, b, 5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.gs(A, b, sweeps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        T = (n + 31) // 32
        steps = sweeps * T
        g = 4 if n >= 896 else (2 if n >= 448 else 1)
        gbs = 4.0 * (32 * T) ** 2 * sweeps / (ms / 1e3) / 1e9
        print(f"n={n:5d} T={T:4d} g={g} ms={ms:9.3f} ns/step={1e6 * ms / steps:8.1f} GB/s={gbs:8.1f}", flush=True)


if __name__ == "__main__":
    main()
