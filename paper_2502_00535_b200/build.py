"""In-tree build of libparnms_b200.so (sm_100a) with nvcc.

The shared library is the C-ABI boundary declared in include/parnms_b200.h.  It is
built in place (next to this file) so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_NAME = "libparnms_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME
NOCDP_PATH = PKG_DIR / "build_tmp" / "libparnms_b200_nocdp.so"  # diagnostics only (see build())

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fopenmp",
    "-Xptxas", "-O3",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def sources() -> list[Path]:
    return (sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h"))
            + [REPO_DIR / "include" / "parnms_b200.h"])


def needs_build() -> bool:
    if not LIB_PATH.exists() or not NOCDP_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > built for p in sources())


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None) -> Path:
    """Compile csrc/*.cu into the in-tree shared library; returns its path."""
    if not force and not needs_build():
        return LIB_PATH
    # two units: pnms_devchain.cu with relocatable device code (device-side launches of the
    # binned path's fallback chain), pnms_capi.cu whole-program (its kernels keep their
    # register budgets); nvcc device-links the relocatable object into the shared library
    tmp = LIB_PATH.parent / "build_tmp"
    tmp.mkdir(exist_ok=True)
    # (+ a diagnostic variant without the relocatable unit, NOCDP_PATH: compute-sanitizer's
    # racecheck / synccheck / initcheck do not support dynamic parallelism)
    compiles = [
        [_nvcc(), *NVCC_FLAGS, *(extra or []), "-rdc=true", "-c", "-o", str(tmp / "devchain.o"),
         str(CSRC / "pnms_devchain.cu")],
        [_nvcc(), *NVCC_FLAGS, *(extra or []), "-c", "-o", str(tmp / "capi.o"), str(CSRC / "pnms_capi.cu")],
        [_nvcc(), *NVCC_FLAGS, *(extra or []), "-DPNMS_NO_DEVCHAIN", "-c", "-o", str(tmp / "capi_nocdp.o"),
         str(CSRC / "pnms_capi.cu")],
    ]
    links = [
        [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-shared",
         "-o", str(LIB_PATH) + ".tmp", str(tmp / "capi.o"), str(tmp / "devchain.o"), "-lcudadevrt", "-lgomp"],
        [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", "-shared",
         "-o", str(NOCDP_PATH), str(tmp / "capi_nocdp.o"), "-lgomp"],
    ]
    if verbose:
        for cmd in compiles + links:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
    procs = [subprocess.Popen(cmd) for cmd in compiles]  # the units compile in parallel
    for cmd, proc in zip(compiles, procs):
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, cmd)
    for cmd in links:
        subprocess.run(cmd, check=True)
    for obj in ("devchain.o", "capi.o", "capi_nocdp.o"):
        (tmp / obj).unlink(missing_ok=True)
    os.replace(str(LIB_PATH) + ".tmp", LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB_PATH)
