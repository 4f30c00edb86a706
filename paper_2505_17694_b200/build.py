"""Build the in-tree shared library `_codec_b200.so` (C ABI, sm_100a).

    python -m paper_2505_17694_b200.build [-v] [--force]

nvcc compiles every csrc/*.cu for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (so ncu's source page maps to our code) and csrc/*.cpp as
host C++; host code is built with -ffp-contract=off because the planner
must reproduce the reference's float64 arithmetic bit for bit. The CUDA
runtime is linked statically so the library does not depend on which
libcudart torch loaded first. Objects go to build/ and are rebuilt only
when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
_TAG = os.environ.get("CODEC_BUILD_TAG", "")  # debug variants: build/obj_<tag>, _codec_b200_<tag>.so
OBJ = ROOT / "build" / ("obj_" + _TAG if _TAG else "obj")
OUT = PKG / ("_codec_b200_" + _TAG + ".so" if _TAG else "_codec_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden"]
DEV_FLAGS = ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"] + os.environ.get("CODEC_NVCC_EXTRA", "").split()


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers():
    return sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _compile(src: Path, force: bool, verbose: bool):
    obj = OBJ / (src.name + ".o")
    newest_dep = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if not force and obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj, ""
    cmd = [NVCC, *ARCH, *HOST_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd[1:1] = DEV_FLAGS
    else:
        cmd += ["-x", "c++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return obj, res.stderr if verbose else ""


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    # a failed compile must not leave the previous library in place (tests
    # and benches would silently run stale kernels)
    newest_dep = max([s.stat().st_mtime for s in srcs] + [h.stat().st_mtime for h in _headers()])
    if force or not OUT.exists() or OUT.stat().st_mtime < newest_dep:
        OUT.unlink(missing_ok=True)
    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, srcs):
            if log:
                print(f"== {s.name}\n{log}")
    newest = max(o.stat().st_mtime for o in objs)
    if force or not OUT.exists() or OUT.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(OUT), *map(str, objs),
               "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return OUT


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(out)
