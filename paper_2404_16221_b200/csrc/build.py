"""Build the in-tree C-ABI library libvolray_b200.so for sm_100a with nvcc.

Every .cu under csrc/ is compiled separately (-lineinfo for ncu source pages) and
linked into one shared object next to the package; cudart is linked statically so
the library does not depend on which libcudart torch has loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
OUT = PKG / "libvolray_b200.so"
# checked build (device range checks, VR_CHECK in common.cuh): a separate library that
# _lib.load() picks when VR_CHECKED=1 is set in the environment
OUT_CHECKED = PKG / "libvolray_b200_checked.so"
BUILD = ROOT / "build" / "csrc"
SOURCES = ["capi.cu", "sampler.cu", "fields.cu", "composite.cu", "hashgrid.cu", "mlp.cu", "mlp_tc.cu",
           "interlevel.cu", "segapi.cu", "occupancy.cu", "rows.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _compile(src: str, verbose: bool, checked: bool = False) -> Path:
    obj = BUILD / (Path(src).stem + ("_checked.o" if checked else ".o"))
    cu = HERE / src
    deps = [cu, HERE / "common.cuh", ROOT / "include" / "vr_capi.h"]
    deps += list(HERE.glob("*.cuh"))
    if obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return obj
    cmd = [nvcc(), *ARCH, *FLAGS, *(["-DVR_CHECKED"] if checked else []), "-c", str(cu), "-o",
           str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, checked: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    out = OUT_CHECKED if checked else OUT
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, checked), SOURCES))
    if out.exists() and all(out.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return out
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, checked="--checked" in sys.argv))
