"""Build the sm_100a shared library ``lib/libw4a16moe.so`` in-tree with nvcc (no JIT cache).

``python -m paper_2504_16214_b200._build`` or ``__graft_entry__.build()``. Each ``csrc/*.cu`` is
compiled in parallel to an object, then linked with ``nvcc -shared``. Rebuilds only when a source
or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libw4a16moe.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", f"-I{INCLUDE}", f"-I{CSRC}"]
if os.environ.get("W4A16_TRACE"):  # debug build: per-stage clock64 timeline (w4a16_debug_trace)
    FLAGS.append("-DW4A16_TRACE")
for knob in ("W4A16_SPLITA", "W4A16_WAIT", "W4A16_DUAL", "W4A16_DECODE_NUMA", "W4A16_DECODE_MAXACC", "W4A16_EARLY_PDL", "W4A16_SMALL_TRIGGER", "W4A16_GEMM_TAIL_TRIGGER", "W4A16_SP_NUMA", "W4A16_SP_MAXACC", "W4A16_SP_MAXNTOK"):  # experiments (see w4a16_gemm.cu)
    if os.environ.get(knob):
        FLAGS.append(f"-D{knob}=" + os.environ[knob])
if os.environ.get("W4A16_KSPLIT"):  # experiment: k-split accumulators of the 16-token decode tile
    FLAGS.append("-DW4A16_KSPLIT=" + os.environ["W4A16_KSPLIT"])


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h")) + [Path(__file__)]


STAMP = LIBDIR / "build_flags.txt"


def up_to_date() -> bool:
    if not LIB.exists() or not STAMP.exists() or STAMP.read_text() != " ".join(ARCH + FLAGS):
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def _compile(src: Path, verbose: bool) -> Path:
    obj = LIBDIR / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    if verbose and r.stderr:
        (LIBDIR / (src.stem + ".ptxas.txt")).write_text(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(" ".join(ARCH + FLAGS))
    for o in objs:
        o.unlink(missing_ok=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
