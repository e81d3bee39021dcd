"""Compile the C oracle (test infrastructure) with gcc into oracle/_build/.

IEEE-exact flags: no -ffast-math, -ffp-contract=off, so float compares and
the quantiser's float32 multiply match numpy / the reference bit for bit.
"""

from __future__ import annotations

import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
OUT = HERE / "_build"
LIB = OUT / "liboracle.so"
SOURCES = ["hash_oracle.c", "mc_oracle.c"]
FLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> pathlib.Path:
    srcs = [HERE / s for s in SOURCES]
    if not force and LIB.exists() and all(s.stat().st_mtime <= LIB.stat().st_mtime for s in srcs):
        return LIB
    OUT.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = ["gcc", *FLAGS, "-o", str(tmp), *map(str, srcs), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
