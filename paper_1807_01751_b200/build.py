"""Build libbwm.so in-tree for sm_100a (B200).

Each ``csrc/*.cu`` translation unit is compiled with nvcc in parallel (one TU per
n_params family of kernel variants), then linked into ``paper_1807_01751_b200/libbwm.so``.
Rebuilds are incremental on CONTENT: an object is recompiled when the SHA-256 of its
source, of every header it can include (``csrc/*.cuh``, ``csrc/*.h``, ``include/*.h``) or
of the nvcc command line changed; the library is relinked when its object set changed.
Used by ``__graft_entry__.build()`` and ``python -m paper_1807_01751_b200.build``.
"""

from __future__ import annotations

import hashlib
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

ARCH = ("-gencode", "arch=compute_100a,code=sm_100a")
NVCC_FLAGS = (
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr", f"-I{INCLUDE}",
)


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libbwm.so")
    return cand


def _headers_digest() -> str:
    h = hashlib.sha256()
    for f in sorted(list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()


def _compile(src: Path, obj_dir: Path, flags: tuple, headers: str, force: bool) -> tuple[Path, str, bool]:
    obj = obj_dir / (src.stem + ".o")
    stamp = obj.with_suffix(".sha256")
    cmd = [nvcc(), *ARCH, *flags, "-c", str(src), "-o", str(obj)]
    key = hashlib.sha256(src.read_bytes() + headers.encode() + "\0".join(cmd[1:]).encode()).hexdigest()
    if not force and obj.exists() and stamp.exists() and stamp.read_text() == key:
        return obj, "", False
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    stamp.write_text(key)
    return obj, res.stderr, True


def build(force: bool = False, verbose: bool = False, jobs: int | None = None, defines=(), out: Path | None = None,
          obj_dir: Path | None = None) -> Path:
    """Compile and link libbwm.so.  `defines` (e.g. ["BWM_STAGE_ROWS=16"]) and `out`/`obj_dir`
    build an experimental variant next to the default library (A/B runs via BWM_LIB); nothing
    module-global changes, so later default builds are unaffected."""
    lib = Path(out) if out is not None else LIB
    objs_dir = Path(obj_dir) if obj_dir is not None else OBJ
    flags = NVCC_FLAGS + tuple(f"-D{d}" for d in defines)
    objs_dir.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    headers = _headers_digest()
    jobs = jobs or min(len(sources), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=jobs) as pool:
        results = list(pool.map(lambda s: _compile(s, objs_dir, flags, headers, force), sources))
    objs = [o for o, _, _ in results]
    if verbose:
        for _, log, _ in results:
            if log:
                sys.stderr.write(log)
    link_key = hashlib.sha256(b"".join((o.with_suffix(".sha256")).read_bytes() for o in objs)).hexdigest()
    link_stamp = objs_dir / (lib.name + ".sha256")
    if force or not lib.exists() or not link_stamp.exists() or link_stamp.read_text() != link_key:
        tmp = lib.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(tmp)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        os.replace(tmp, lib)
        link_stamp.write_text(link_key)
    return lib


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
