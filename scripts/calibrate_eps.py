"""Calibrate each config's relative threshold eps with the ORACLE on seed 0 so the mean
kept fraction hits the target BASELINE.json names (cfg2 ~10%, cfg3 ~5%, cfg5 ~8%).
Calls only oracle/ and synth/ (the value is an oracle output, never a CUDA one).
Writes tests/golden/eps_calibration.txt.  Usage: python scripts/calibrate_eps.py"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

TARGETS = {"cfg2": 0.10, "cfg3": 0.05, "cfg5": 0.08}
SUBSET = {"cfg2": None, "cfg3": 64, "cfg5": 24}


def maps(cfg, bins):
    band = synth.make_band(cfg, bins=bins)
    def one(j):
        return oracle.das(band.mic_xyz, cfg.c0, cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy,
                          band.freqs[j], band.csm[j])
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        return list(ex.map(one, range(len(bins))))


def frac(cfg, bs, eps):
    return float(np.mean([len(oracle.compress(cfg.n, b, eps)[0]) for b in bs])) / cfg.S


def main():
    lines = ["# Relative thresholds calibrated with the oracle (scripts/calibrate_eps.py, seed 0).",
             "# cfg : eps : mean kept fraction : bins used"]
    for name, target in TARGETS.items():
        cfg = synth.CONFIGS[name]
        bins = synth.strided_bins(cfg.n_bins, SUBSET[name] or cfg.n_bins)
        bs = maps(cfg, bins)
        lo, hi = 1e-5, 0.5          # frac decreasing in eps
        for _ in range(40):
            mid = (lo * hi) ** 0.5
            if frac(cfg, bs, mid) > target:
                lo = mid
            else:
                hi = mid
        eps = float("%.3g" % hi)
        fr = frac(cfg, bs, eps)
        print(name, eps, fr, flush=True)
        lines.append(f"{name} : {eps} : {fr:.4f} : {len(bins)}")
    with open(os.path.join(ROOT, "tests", "golden", "eps_calibration.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
