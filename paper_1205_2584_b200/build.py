"""In-tree build of the sm_100a engine (nvcc -> paper_1205_2584_b200/_lib/libcpfast_b200.so)."""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libcpfast_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "cpfast_b200.h"]


STAMP = OUT.with_suffix(".srchash")


def _extra_defs() -> list:
    """Diagnostic -D flags (CPF_NVCC_DEFS="-DCPF_PANEL_TIMING ..."); part of the build hash."""
    return os.environ.get("CPF_NVCC_DEFS", "").split()


def source_hash() -> str:
    """Content hash of every source the library is built from (mtimes do not survive snapshots)."""
    h = hashlib.sha256()
    h.update(" ".join(_extra_defs()).encode())
    for p in sources():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def up_to_date() -> bool:
    if not OUT.exists() or not STAMP.exists():
        return False
    return STAMP.read_text().strip() == source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    digest = source_hash()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-warn-spills" if not verbose else "-v",
           *_extra_defs(), "-o", str(tmp), str(CSRC / "engine.cu"), "-lnccl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building the B200 engine")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, OUT)
    STAMP.write_text(digest + "\n")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
