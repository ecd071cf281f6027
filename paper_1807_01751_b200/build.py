"""Build libbwm.so in-tree for sm_100a (B200).

Each ``csrc/*.cu`` translation unit is compiled with nvcc in parallel (one TU per
n_params family of kernel variants), then linked into ``paper_1807_01751_b200/libbwm.so``.
Rebuilds are incremental on source/header mtimes.  Used by ``__graft_entry__.build()``
and ``python -m paper_1807_01751_b200.build``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OBJ = PKG.parent / "build" / "obj"
LIB = PKG / "libbwm.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr", f"-I{INCLUDE}",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libbwm.so")
    return cand


def _deps_mtime() -> float:
    files = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    obj = OBJ / (src.stem + ".o")
    if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _deps_mtime()):
        return obj, ""
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj, res.stderr


def build(force: bool = False, verbose: bool = False, jobs: int | None = None, defines=(), out: Path | None = None,
          obj_dir: Path | None = None) -> Path:
    """Compile and link libbwm.so.  `defines` (e.g. ["BWM_STAGE_ROWS=16"]) and `out`/`obj_dir`
    build an experimental variant next to the default library (A/B runs via BWM_LIB)."""
    global OBJ, LIB
    if defines:
        NVCC_FLAGS.extend(f"-D{d}" for d in defines)
    if out is not None:
        LIB = Path(out)
    if obj_dir is not None:
        OBJ = Path(obj_dir)
    OBJ.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    jobs = jobs or min(len(sources), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=jobs) as pool:
        results = list(pool.map(lambda s: _compile(s, force), sources))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(tmp)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[], help="extra preprocessor define")
    ap.add_argument("--out", default=None, help="library path (default: in-tree libbwm.so)")
    args = ap.parse_args()
    obj = None
    if args.out:
        obj = Path(args.out).resolve().parent / ("obj_" + Path(args.out).stem)
    print(build(force=args.force, verbose=args.v, defines=args.D, out=args.out, obj_dir=obj))
