"""B200-native DAMAS on the wavelet-compressed computational grid (arXiv 1608.05179).

The product is the C-ABI library libdwc.so (include/dwc.h) built in-tree for sm_100a by
`python -m paper_1608_05179_b200.build`; `dwc` is the thin ctypes binding over it.
"""
from .dwc import Context, DwcError, Geometry, lib  # noqa: F401

__all__ = ["Context", "DwcError", "Geometry", "lib"]
