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
    """Every computing entry point has its own doc comment right above it, and that comment cites
    the PAPER.md passage (line numbers) it implements."""
    hdr = open(os.path.join(ROOT, "include", "dwc.h")).read()
    assert "PAPER.md" in hdr
    for name in ["dwc_solve_band", "dwc_solve_band_host", "dwc_solve_band_snapshots", "dwc_csm", "dwc_steer",
                 "dwc_das", "dwc_compress", "dwc_psf", "dwc_gs", "dwc_keep_mask", "dwc_keep_unmask"]:
        i = hdr.index("DWC_API dwc_status " + name + "(")
        before = hdr[:i].rstrip()
        assert before.endswith("*/"), name      # a doc comment right above
        comment = before[before.rindex("/*"):]
        if name in ("dwc_solve_band_host",):
            comment = hdr[hdr.rindex("/* ---- the batched hot path", 0, i):i]   # documented with the band call
        assert re.search(r"PAPER\.md:\d+", comment), name


def test_output_buffer_checks():
    """Caller-supplied output buffers are checked (shape, dtype, contiguity, residency) before
    their raw pointers reach the C call."""
    import torch

    from paper_1608_05179_b200.dwc import _check_out
    K, S = 3, 10
    ok = {"n_keep": torch.empty(K, dtype=torch.int32), "keep_idx": torch.empty((K, S), dtype=torch.int32),
          "x_map": torch.empty((K, S), dtype=torch.float32), "b_map": None}
    _check_out(ok, K, S, want_b=False, host=True)
    for key, bad in [("x_map", torch.empty((K, S + 1), dtype=torch.float32)),
                     ("x_map", torch.empty((K, S), dtype=torch.float64)),
                     ("keep_idx", torch.empty((S, K), dtype=torch.int32).t()),
                     ("n_keep", torch.empty(K + 1, dtype=torch.int32))]:
        with pytest.raises(ValueError):
            _check_out(dict(ok, **{key: bad}), K, S, want_b=False, host=True)
    with pytest.raises(ValueError):
        _check_out(ok, K, S, want_b=True, host=True)        # b_map wanted but missing
    with pytest.raises(ValueError):
        _check_out(ok, K, S, want_b=False, host=False)      # host tensors for the device path


def test_binding_flag_constants_match_header():
    """Every DWC_* flag / kernel id the binding names has the header's value (the binding passes
    them as raw bits through dwc_params.flags), and _flags composes them."""
    import re

    from paper_1608_05179_b200 import dwc
    hdr = open(os.path.join(ROOT, "include", "dwc.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(DWC_[A-Z0-9_]+)\s+(\d+)\b", hdr)}
    names = [n for n in dir(dwc) if n.startswith("DWC_") and isinstance(getattr(dwc, n), int)]
    assert "DWC_THROUGHPUT" in names and len(names) >= 8
    for n in names:
        assert n in defs and defs[n] == getattr(dwc, n), n
    f = dwc._flags(True, 3, dr=True, alt=True, dense_stream=False, throughput=True)
    assert f == (defs["DWC_FULL_GRID"] | defs["DWC_CUBIC"] | defs["DWC_DIAG_REMOVAL"] | defs["DWC_ALT_SWEEPS"] |
                 defs["DWC_GS_RESIDUAL"] | defs["DWC_THROUGHPUT"])
