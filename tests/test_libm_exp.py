"""The device restatement of the host libm exp (csrc/pnms_libm.cuh), which makes gaussian
Soft-NMS bit-identical to the reference's math.exp (oracles.py:119): the same header built for
the host is compared with math.exp bit for bit here; the device build in the GPU tests."""

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def exp_ranges(n: int, seed: int = 7):
    """Arguments of every branch: the Soft-NMS domain -cov^2/sigma (cov in [0, 1], any sigma),
    tiny, large negative (subnormal results, the special case), positive, and random bits."""
    rng = np.random.default_rng(seed)
    cov = rng.random(n)
    sig = np.exp(rng.uniform(-8, 8, n))
    bits = rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64)
    return [-(cov * cov) / sig, -rng.random(n), -rng.random(n) * 2.0**-30, rng.uniform(-745.2, -700, n),
            rng.uniform(-710, 709.7, n), -np.abs(bits[np.isfinite(bits)]),
            np.array([0.0, -0.0, 2.0**-60, -2.0**-60, -745.13321910194122, -745.2, -708.4, 709.7, -np.inf,
                      -1e-300, -0.5, -1.0])]


def host_exp(x: np.ndarray) -> np.ndarray:
    return np.fromiter((math.exp(v) for v in x.tolist()), dtype=np.float64, count=x.size)


@pytest.fixture(scope="module")
def restated(tmp_path_factory):
    so = tmp_path_factory.mktemp("libm") / "libm_exp.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(so),
                    str(ROOT / "tests" / "libm_exp_host.cc")], check=True)
    lib = ctypes.CDLL(str(so))
    lib.libm_exp_restated.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]

    def run(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib.libm_exp_restated(x.ctypes.data, y.ctypes.data, x.size)
        return y
    return run


def test_restated_exp_is_bit_identical_to_host_libm(restated):
    for x in exp_ranges(1_000_000):
        got, want = restated(x), host_exp(x)
        bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
        assert bad.size == 0, [(float(x[i]).hex(), float(want[i]).hex(), float(got[i]).hex()) for i in bad[:5]]
