"""In-tree build of the C-ABI shared library ``libdash_b200.so`` (sm_100a only).

    python -m paper_2602_02016_b200.build        # or __graft_entry__.build()

Every ``csrc/*.cu`` is compiled by nvcc with ``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and
linked into one shared library next to this file.  Objects are cached under ``build/`` and rebuilt
when a source or header is newer than its object.
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
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libdash_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted((ROOT / "include").glob("*.h"))


def _newest(paths) -> float:
    return max((p.stat().st_mtime for p in paths), default=0.0)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr_time = _newest(_headers())
    objs, cmds = [], []
    for src in sorted(CSRC.glob("*.cu")):
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_time):
            continue
        cmds.append([NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)])
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for proc in list(pool.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds)):
            sys.stderr.write(proc.stderr)
            if proc.returncode != 0:
                raise subprocess.CalledProcessError(proc.returncode, proc.args)
    if force or not LIB.exists() or LIB.stat().st_mtime < _newest(objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
