"""Build recipe for the oracle's C restatement (TEST INFRASTRUCTURE ONLY).

Compiles `oracle/ilu0.c` with gcc into `oracle/_build/liboracle_ilu0.so`.
`-ffp-contract=off` keeps products and differences separately rounded, which
matches the numba kernels of the reference (linalg.py:63-113).
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT_DIR = HERE / "_build"
LIB = OUT_DIR / "liboracle_ilu0.so"


def build(force: bool = False) -> Path:
    src = HERE / "ilu0.c"
    if LIB.exists() and not force and LIB.stat().st_mtime >= src.stat().st_mtime:
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
    subprocess.run(
        ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", str(tmp), str(src)],
        check=True,
    )
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
