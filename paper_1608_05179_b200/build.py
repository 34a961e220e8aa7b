"""Build the in-tree C-ABI library libdwc.so for sm_100a with nvcc (no JIT, no torch
extension machinery): `python -m paper_1608_05179_b200.build`.  `--checked` (or build(checked=True))
builds libdwc_checked.so with -DDWC_CHECKED: device-side invariant checks in the Gauss-Seidel
kernels and mbarrier watchdogs (tests/test_gpu_checked.py runs it)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libdwc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                 "-I", os.path.join(HERE, "..", "include"), "-Xptxas", "-v"]
# DWC_NVCC_EXTRA: extra nvcc flags for experiments (e.g. -DGS_KSTG=4); DWC_LIB: output path
COMMON += os.environ.get("DWC_NVCC_EXTRA", "").split()
LIB = os.environ.get("DWC_LIB", LIB)
BUILD = os.environ.get("DWC_BUILD_DIR", BUILD)
LIB_CHECKED = os.path.join(HERE, "libdwc_checked.so")
SOURCES = {
    "dwc_api.cu": [],
    "k_das.cu": [],
    "k_compress.cu": ["--fmad=false"],   # the fp64 threshold arithmetic must not contract
    "k_psf.cu": [],
    "k_gs.cu": [],
    "k_keep.cu": [],
    "k_csm.cu": [],
    "k_gs_alt.cu": [],
    "k_rgs.cu": [],
}


def _compile(name, extra, verbose, bdir=None, defs=()):
    bdir = bdir or BUILD
    src = os.path.join(CSRC, name)
    obj = os.path.join(bdir, name.replace(".cu", ".o"))
    cmd = [NVCC, *COMMON, *defs, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{r.stdout}\n{r.stderr}")
    with open(os.path.join(bdir, name + ".ptxas.txt"), "w") as f:
        f.write(r.stderr)
    if verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    bdir = BUILD + "_checked" if checked else BUILD
    defs = ("-DDWC_CHECKED",) if checked else ()
    os.makedirs(bdir, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "dwc.h")]
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps):
        return lib
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose, bdir, defs), SOURCES.items()))
    tmp = lib + ".tmp%d" % os.getpid()
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fvisibility=hidden"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, checked="--checked" in sys.argv))
