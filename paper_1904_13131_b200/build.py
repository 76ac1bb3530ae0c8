"""Build libhf.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_1904_13131_b200.build [--force]

Each .cu translation unit is compiled in parallel, then linked into
``paper_1904_13131_b200/libhf.so`` which the ctypes loader (``_lib.py``) opens.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
DEBUG = os.environ.get("HF_DEBUG", "0") not in ("", "0")  # device bounds checks -> libhf_debug.so
TIMELINE = os.environ.get("HF_TIMELINE", "0") not in ("", "0")  # per-warp apply timeline -> libhf_tl.so
# A/B builds: HF_VARIANT_NAME=x HF_VARIANT_FLAGS="-DFOO=1" -> libhf_x.so
VARIANT = os.environ.get("HF_VARIANT_NAME", "")
_SUFFIX = "_debug" if DEBUG else ("_tl" if TIMELINE else (f"_{VARIANT}" if VARIANT else ""))
OBJ = os.path.join(PKG, "build_obj" + _SUFFIX)
LIB = os.path.join(PKG, f"libhf{_SUFFIX}.so")
SOURCES = ["hf_api.cu", "hf_cells2d.cu", "hf_cells3d.cu", "hf_assemble.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include")] + (["-DHF_DEBUG"] if DEBUG else []) + \
        (["-DHF_TIMELINE"] if TIMELINE else []) + os.environ.get("HF_VARIANT_FLAGS", "").split()


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps() -> list[str]:
    out = [os.path.join(ROOT, "include", "hf.h")]
    for f in os.listdir(CSRC):
        out.append(os.path.join(CSRC, f))
    return out


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: str) -> str:
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
