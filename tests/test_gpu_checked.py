"""The device-checked library (libdwc_checked.so: -DDWC_CHECKED, device-side invariant checks on
the Gauss-Seidel kernels' ring slots, parities, change lists and indices, plus mbarrier
watchdogs that trap) runs the cfg3 band's longest-chain bins, its smallest systems with
alternating sweeps, and cfg5-shaped large systems on both GS kernels in a separate process.  It must finish without a trap and give results
bitwise identical to the production library's (the checks only observe)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1608_05179_b200", "libdwc_checked.so")

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth
from paper_1608_05179_b200 import Context, Geometry
import paper_1608_05179_b200.dwc as D
assert D.LIB_PATH.endswith({libname!r}), D.LIB_PATH
c = Context(0)
res = {{}}
for name, bins, sweeps, full, dense, alt in {cases!r}:
    band = synth.make_band(name, bins=bins)
    cfg = band.cfg
    g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    out = c.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, sweeps, cfg.eps_mode,
                       full_grid=full, dense_stream=dense, alt=alt)
    res[f"{{name}}_{{dense}}_{{alt}}"] = out["x_map"].cpu().numpy()
    res[f"{{name}}_{{dense}}_{{alt}}_k"] = np.array([c.stats()["gs_kernel"]])
np.savez({out!r}, **res)
"""

CASES = [("cfg3", [249, 255, 224, 10, 11, 12], 1000, False, False, False),
         ("cfg3", [249, 100], 300, False, True, False),
         ("cfg3", [0, 1, 2, 249], 300, False, False, True),   # systems of < 4 blocks, alternating sweeps
         ("cfg5", [1023], 20, False, False, False),
         ("cfg5", [1023], 20, False, True, False)]


def _run(lib, out, tmp_path):
    script = _SCRIPT.format(root=ROOT, libname=os.path.basename(lib), cases=CASES, out=str(out))
    # (two CTAs per SM for the systems of at most 640 points, as in a band with more bins than SMs)
    env = dict(os.environ, DWC_LIB=lib, DWC_RGS_PAIR_MAX_SP="640")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "[dwc checked]" not in r.stdout
    return np.load(out)


def test_checked_build_runs_clean_and_bitwise_equal(tmp_path):
    if not os.path.exists(CHECKED):
        pytest.fail("libdwc_checked.so is missing: run __graft_entry__.build() (builds both libraries)")
    a = _run(CHECKED, tmp_path / "checked.npz", tmp_path)
    b = _run(os.path.join(ROOT, "paper_1608_05179_b200", "libdwc.so"), tmp_path / "prod.npz", tmp_path)
    assert sorted(a.files) == sorted(b.files)
    for key in a.files:
        assert np.array_equal(a[key], b[key]), key
    # both GS kernels ran
    kinds = {int(a[k][0]) for k in a.files if k.endswith("_k")}
    assert 4 in kinds and (kinds & {1, 2})
