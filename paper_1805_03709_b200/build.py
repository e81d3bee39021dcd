"""Build libvsb200.so (sm_100a) in-tree with nvcc.

Run as ``python -m paper_1805_03709_b200.build`` or through
``__graft_entry__.build()``.  Objects go to ``build/``; the shared library is
written next to this file so it travels with the repo snapshot to the GPU box.
No fast-math and no FTZ: the MC predicates must match IEEE compares on the
CPU.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "vsb200"
LIB = PKG / "libvsb200.so"
SOURCES = ["hash.cu", "mc.cu", "stream.cu", "fusion.cu", "shard.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "-Xptxas", "-v", f"-I{ROOT / 'include'}"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA extension cannot be built")
    return cand


def _deps() -> list[pathlib.Path]:
    return sorted(CSRC.glob("*.cu*")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "vsb200.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: pathlib.Path | None = None,
          defines: tuple = ()) -> pathlib.Path:
    """Compile to `out` (default: the in-tree libvsb200.so).  `defines` are
    extra -D flags for experiment variants (e.g. ("VSB_MC_STAGES=3",))."""
    lib = LIB if out is None else pathlib.Path(out)
    if out is None and not defines and not force and up_to_date():
        return LIB
    build_dir = BUILD if not defines else BUILD / ("v_" + "_".join(d.replace("=", "") for d in defines))
    build_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()

    def compile_one(src: str) -> tuple[str, str]:
        obj = build_dir / (src.rsplit(".", 1)[0] + ".o")
        cmd = [cc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        (build_dir / (src + ".ptxas.txt")).write_text(r.stderr)
        return str(obj), r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        for _, log in results:
            sys.stdout.write(log)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
