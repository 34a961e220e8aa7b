"""The PSF epilogue resolves the stored tiles of each 32x32 block with sym_targets_g (sub-group
size as a compile-time constant); it must equal the generic sym_targets of the symmetric tile
layout (dwc_internal.cuh) for every block, g in {1, 2, 4}, T <= 120.  Host-only program built
with nvcc (no GPU needed)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="nvcc not available")
def test_sym_targets_fast_equals_generic(tmp_path):
    exe = tmp_path / "sym_targets_check"
    src = os.path.join(ROOT, "tests", "native", "sym_targets_check.cu")
    inc = os.path.join(ROOT, "paper_1608_05179_b200", "csrc")
    nvcc = NVCC if os.path.exists(NVCC) else shutil.which("nvcc")
    subprocess.run([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-I", inc, "-o", str(exe), src], check=True,
                   capture_output=True, timeout=300)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
