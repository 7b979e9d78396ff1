"""Build the CUDA library in-tree: paper_2601_14980_b200/libpcb200.so (sm_100a only).

    python -m paper_2601_14980_b200.build [--force] [-j N]

Every translation unit is compiled by nvcc with `-gencode arch=compute_100a,code=sm_100a
-lineinfo`; the FP64 quantizers rely on `--fmad=false` (no contraction, quantize.cpp is built
without FMA on x86-64 — SURVEY.md §0 fact 6).  Objects are cached by content hash under
paper_2601_14980_b200/build/ so an unchanged tree relinks in a second.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "libpcb200.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXX = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
COMMON = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
          f"-I{CSRC}", f"-I{INCLUDE}", "-Xptxas", "-warn-spills"]

SOURCES = [
    "abi.cu",
    "paillier.cu",
    "side.cu",
    "side28.cu",
    "wide.cu",
    "rstream.cu",
    "imad_peak.cu",
    "rns.cu",
    "rnsx.cu",
    "wire.cu",
    "factor.cu",
    "prime.cu",
    "host/hbn.cpp",
]


def _deps() -> str:
    h = hashlib.sha256()
    for p in sorted(CSRC.rglob("*")):
        if p.suffix in (".cuh", ".h", ".hpp"):
            h.update(p.read_bytes())
    h.update((INCLUDE / "pcb200.h").read_bytes())
    return h.hexdigest()


def _obj(src: str, dep_hash: str, extra: list[str]) -> Path:
    s = CSRC / src
    key = hashlib.sha256(s.read_bytes() + dep_hash.encode() + " ".join(COMMON + ARCH + extra).encode())
    return BUILD / f"{src.replace('/', '_')}.{key.hexdigest()[:16]}.o"


def compile_one(src: str, dep_hash: str, extra: list[str], verbose: bool) -> Path:
    out = _obj(src, dep_hash, extra)
    if out.exists():
        return out
    cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", str(CSRC / src), "-o", str(out)]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-ccbin", CXX, *COMMON, *extra, "-x", "c++", "-c", str(CSRC / src), "-o", str(out)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    if "spill" in (r.stdout + r.stderr) and verbose:
        sys.stderr.write(r.stdout + r.stderr)
    return out


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, extra: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile (cached) and link the library.  `extra` adds nvcc flags (e.g. -DPCB_ROW_UNROLL=32)."""
    extra = list(extra or []) + os.environ.get("PCB_EXTRA_NVCC", "").split()
    lib_path = Path(out) if out else LIB
    BUILD.mkdir(exist_ok=True)
    if force:
        for p in BUILD.glob("*.o"):
            p.unlink()
    dep = _deps()
    jobs = jobs or min(len(SOURCES), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: compile_one(s, dep, extra, verbose), SOURCES))
    link_key = hashlib.sha256("".join(str(o) for o in objs).encode()).hexdigest()[:16]
    stamp = BUILD / f"link.{lib_path.name}.stamp"
    if lib_path.exists() and stamp.exists() and stamp.read_text() == link_key and not force:
        return lib_path
    tmp = lib_path.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-ccbin", CXX, "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib_path)
    stamp.write_text(link_key)
    return lib_path


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[], help="extra preprocessor define for nvcc")
    ap.add_argument("--out", default=None, help="alternative output .so (experiments)")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=a.v, extra=[f"-D{d}" for d in a.D], out=a.out))


if __name__ == "__main__":
    main()
