"""In-tree build of the sm_100a CUDA library (libcinr_b200.so).

Each .cu is compiled separately with nvcc for `-gencode arch=compute_100a,code=sm_100a`
and linked into one shared object next to this file, so the .so travels with
the repository snapshot to the GPU box.  march.cu (the parity-critical ray-march
arithmetic) is compiled with -fmad=false on top of its explicit _rn intrinsics.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
SO = OUT_DIR / ("libcinr_b200_stats.so" if os.environ.get("CINR_STATS") else "libcinr_b200.so")
INCLUDE = PKG.parent / "include"

SOURCES = {
    "capi.cu": [],
    "march.cu": ["-fmad=false"],
    "wave3.cu": ["-fmad=false"],
    "rays.cu": ["-fmad=false"],
    "pt.cu": ["-fmad=false"],
    "train.cu": [],
    "decode.cu": [],
    "cache.cu": [],
    "decode_tc.cu": [],
}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{INCLUDE}"]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build():
    if not SO.exists():
        return True
    mt = SO.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > mt for p in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return SO
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    logs = []
    for src, extra in SOURCES.items():
        obj = OUT_DIR / (Path(src).stem + (".stats.o" if os.environ.get("CINR_STATS") else ".o"))
        diag = ["-DCINR_STATS"] if os.environ.get("CINR_STATS") else []  # diagnostics build only
        cmd = [nvcc(), *ARCH, *COMMON, *diag, *extra, "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        objs.append(str(obj))
    tmp = SO.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, SO)
    (OUT_DIR / "ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return SO


if __name__ == "__main__":
    build(force=True, verbose=False)
    print(SO)
