"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads without a
GPU and exports every symbol include/dwc.h declares; the product never touches oracle/."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1608_05179_b200 import build
    return build.build()


def test_library_exports_header_symbols(libpath):
    from paper_1608_05179_b200 import dwc
    declared = dwc.exported_symbols_from_header()
    assert len(declared) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(dwc_\w+)", out))
    assert set(declared) == exported, (set(declared) ^ exported)
    L = dwc.lib()
    for name in declared:
        assert hasattr(L, name)
    assert L.dwc_version().startswith(b"dwc")


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_create_without_gpu_fails_cleanly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1608_05179_b200 import Context, DwcError
    with pytest.raises(DwcError):
        Context(0)


def test_product_does_not_reference_oracle():
    pkg = os.path.join(ROOT, "paper_1608_05179_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "dwc_oracle" not in src and "liboracle" not in src, f


def test_header_documents_every_entry_point():
    hdr = open(os.path.join(ROOT, "include", "dwc.h")).read()
    assert "PAPER.md" in hdr
    for name in ["dwc_solve_band", "dwc_das", "dwc_compress", "dwc_psf", "dwc_gs", "dwc_steer"]:
        i = hdr.index("DWC_API dwc_status " + name + "(")
        assert hdr[:i].rstrip().endswith("*/"), name      # a doc comment right above
