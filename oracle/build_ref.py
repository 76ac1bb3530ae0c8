"""Install the UNMODIFIED reference package into ``oracle/_ref`` (test infrastructure).

    python oracle/build_ref.py [--force]

The reference (``/root/reference/pkg``, package ``hyperfree`` 0.1.0) is pure
Python on numpy/scipy, so "building" it is a pip install of its own sources:
they are copied to a scratch directory (``/root/reference`` is read-only and
setuptools writes build metadata next to the sources), then installed with
``pip install --no-index --no-build-isolation --no-deps --target oracle/_ref``.
Nothing is edited.  ``oracle/_ref`` is git-ignored (no reference source enters
the history) but not gpurun-ignored, so the installed package travels with the
tree to the GPU box, where ``/root/reference`` does not exist.

Only ``tests/``, ``__graft_entry__`` and ``bench.py``'s reference / CPU-baseline
legs use it (``oracle/ref.py``), as the checker and the reference arm -- never
as the product path.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
TARGET = os.path.join(HERE, "_ref")
SOURCE = "/root/reference/pkg"
STAMP = os.path.join(TARGET, ".installed_from")


def _source_mtime() -> float:
    t = 0.0
    for d, _, files in os.walk(SOURCE):
        for f in files:
            t = max(t, os.path.getmtime(os.path.join(d, f)))
    return t


def build(force: bool = False) -> str | None:
    """Install the reference into oracle/_ref; returns the target, or None when
    the reference tree is absent (the GPU box uses the copy that travelled)."""
    if not os.path.isdir(SOURCE):
        return TARGET if os.path.isdir(os.path.join(TARGET, "hyperfree")) else None
    stamp = f"{SOURCE} {_source_mtime():.0f}"
    if not force and os.path.exists(STAMP) and open(STAMP).read().strip() == stamp:
        return TARGET
    with tempfile.TemporaryDirectory(prefix="hfref_") as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(SOURCE, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "*.egg-info", "build"))
        stage = os.path.join(tmp, "target")
        cmd = [sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation", "--no-deps",
               "--find-links", "/opt/wheelhouse", "--target", stage, src]
        r = subprocess.run(cmd, capture_output=True, text=True, env={**os.environ, "PYTHONDONTWRITEBYTECODE": "1"})
        if r.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{r.stdout}\n{r.stderr}")
        if os.path.isdir(TARGET):
            shutil.rmtree(TARGET)
        shutil.copytree(stage, TARGET)
    with open(STAMP, "w") as f:
        f.write(stamp + "\n")
    return TARGET


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
