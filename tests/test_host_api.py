"""Host-side logic of the drop-in boundary (no GPU): config validation, data model,
C-ABI symbol table and argument checking that happens before any CUDA call."""

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2502_00535_b200 import (
    CapacityError, ConfigError, Detection, DetectionVector, NmsConfig, SuppressionMatrix, SurvivorMask,
    ValidationError, WorkCounters, _lib, mask_survivors,
)


def test_config_defaults_and_errors():
    c = NmsConfig()
    assert (c.theta, c.d_max, c.k, c.workers, c.tie_break) == (0.3, 4096, 32, 1, "paper_faithful")
    # messages of engine.py:57-71
    cases = [
        (dict(theta=1.5), "theta must be in [0, 1], got 1.5"),
        (dict(theta=-0.1), "theta must be in [0, 1], got -0.1"),
        (dict(d_max=0), "d_max must be positive, got 0"),
        (dict(k=0), "k must be positive, got 0"),
        (dict(d_max=100, k=32), "k=32 does not divide d_max=100"),
        (dict(workers=0), "workers must be positive, got 0"),
        (dict(tie_break="greedy"), "tie_break must be one of ('paper_faithful', 'by_index'), got 'greedy'"),
    ]
    for kw, msg in cases:
        with pytest.raises(ConfigError) as ei:
            NmsConfig(**kw)
        assert str(ei.value) == msg
    assert issubclass(ConfigError, ValueError)


def test_detection_validation():
    assert Detection(1, 2, 3, 0.5).validate() == Detection(1, 2, 3, 0.5)
    for d, frag in [(Detection(-1, 0, 3, 0.5), "x must be non-negative"), (Detection(0, 0, 0, 0.5), "side length"),
                    (Detection(0, 0, 2**24, 0.5), "exceeds the coordinate limit"),
                    (Detection(0, 0, 3, float("nan")), "finite"), (Detection(0, 0, 3, 0.0), "strictly positive"),
                    (Detection(0, 0, 3, True), "must be a number"), (Detection(1.5, 0, 3, 0.5), "integer")]:
        with pytest.raises(ValidationError, match=frag):
            d.validate()


def test_detection_vector_layout():
    v = DetectionVector([Detection(1, 2, 3, 0.5), Detection(4, 5, 6, 0.25)], 5)
    assert v.count == 2 and v.d_max == 5 and len(v) == 5
    assert v.xs.dtype == np.int64 and v.ss.dtype == np.float64
    assert v.xs.tolist() == [1, 4, 0, 0, 0] and v.ss.tolist() == [0.5, 0.25, 0, 0, 0]
    assert not v.xs.flags.writeable
    assert v.slot(3) == Detection(0, 0, 0, 0.0)
    assert v.repadded(8).d_max == 8 and v.repadded(8).valid() == v.valid()
    w = DetectionVector.from_arrays([1, 4], [2, 5], [3, 6], [0.5, 0.25], 5)
    assert w == v
    with pytest.raises(CapacityError):
        DetectionVector([Detection(1, 2, 3, 0.5)] * 3, 2)
    with pytest.raises(ValidationError):
        DetectionVector.from_arrays([1], [2], [0], [0.5])


def test_bit_containers_layout():
    m = SuppressionMatrix.all_ones(70)
    assert m.bits.shape == (70, 16)
    m.set(3, 65, False)
    assert not m.get(3, 65) and m.get(3, 64)
    assert m.bits[3, 8] == 0xFD
    v = SurvivorMask.from_bools(np.array([1, 0, 1, 1, 0, 0, 0, 0, 1], dtype=bool))
    assert v.bits.tolist() == [0b00001101, 1] and v.get(8) and not v.get(1)
    assert (WorkCounters(1, 2, 3) + WorkCounters(10, 20, 30)) == WorkCounters(11, 22, 33)


def test_mask_survivors_host():
    d = DetectionVector([Detection(10, 10, 20, 0.9), Detection(10, 10, 20, 0.8)], 4)
    r = mask_survivors(d, SurvivorMask.from_bools(np.array([1, 0, 1, 1], dtype=bool)))
    assert r.survivors == (Detection(10, 10, 20, 0.9),) and r.suppressed_count == 1
    with pytest.raises(ConfigError, match="mask dim 3 does not match vector capacity 4"):
        mask_survivors(d, SurvivorMask.from_bools(np.ones(3, dtype=bool)))


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    header = (ROOT / "include" / "parnms_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const char\*|int)\s+(pnms_\w+)\s*\(", header, flags=re.M))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    for sym in declared:
        assert getattr(lib, sym) is not None
    assert lib.pnms_version().decode().startswith("parnms_b200")


def test_c_abi_argument_errors_without_gpu():
    lib = _lib.load()
    assert _lib.strerror(_lib.PNMS_EINVAL_THETA) == "theta must be in [0, 1]"
    nb = _lib.workspace_bytes(256, 1024)
    assert nb >= 256 * 1024 * (32 + 4 + 4)
    # frames > 4096 slots add the chunked-sort scratch on top of the per-slot regions (the
    # fixed 64 KiB persistent head excluded)
    head = _lib.workspace_bytes(1, 1)
    assert _lib.workspace_bytes(1, 16384) - head > (_lib.workspace_bytes(1, 4096) - head) * 4
    out = ctypes.c_size_t()
    assert lib.pnms_workspace_bytes(1, _lib.MAX_SLOTS + 1, ctypes.byref(out)) == _lib.PNMS_ETOO_LARGE
    args = [None] * 5 + [1, 8, 8, 0.5, 0] + [None] * 5 + [0, None]
    a = list(args); a[8] = 1.5
    assert lib.pnms_run(*a) == _lib.PNMS_EINVAL_THETA
    a = list(args); a[8] = float("nan")
    assert lib.pnms_run(*a) == _lib.PNMS_EINVAL_THETA
    a = list(args); a[9] = 2
    assert lib.pnms_run(*a) == _lib.PNMS_EINVAL_TIE
    a = list(args); a[7] = 0
    assert lib.pnms_run(*a) == _lib.PNMS_EINVAL_DMAX
    assert lib.pnms_run(*args) == _lib.PNMS_EINVAL_ARG  # null planes
    assert lib.pnms_reduce_rows(None, 10, 3, None, None) == _lib.PNMS_EINVAL_K
    with pytest.raises(ConfigError):
        _lib.check(_lib.PNMS_EINVAL_THETA, "x")
    with pytest.raises(_lib.NativeLibraryError):
        _lib.check(_lib.PNMS_EWORKSPACE, "x")


def test_synth_distribution():
    from paper_2502_00535_b200.synth import random_frames

    x, y, z, s = random_frames(16, 2048, seed=1)
    assert x.dtype == np.int32 and s.dtype == np.float64 and x.shape == (16, 2048)
    assert z.min() >= 8 and z.max() <= 64
    assert (x + z <= 1920).all() and (y + z <= 1080).all() and x.min() >= 0
    assert s.min() >= 0.05 and s.max() < 1.0


def test_pack_box32_layout_and_domain():
    """pack_box32 word layout x | y<<12 | z<<24 and its domain checks (host side only)."""
    import numpy as np
    import pytest

    from paper_2502_00535_b200.tensor_api import pack_box32

    w = pack_box32(np.array([0, 4095, 7]), np.array([0, 4095, 9]), np.array([0, 255, 1])).view(np.uint32)
    assert list(w) == [0, 0xFFFFFFFF, 7 | (9 << 12) | (1 << 24)]
    for bad in ((4096, 0, 0), (0, -1, 0), (0, 0, 256)):
        with pytest.raises(ValueError):
            pack_box32(*(np.array([v]) for v in bad))


def test_pack_box32_host_matches_numpy_and_flags_the_domain():
    """pnms_pack_box32_host (the C ABI's multi-threaded host packer, no GPU needed): the same
    words as pack_box32 on the packable domain's edges and random planes, any thread count and
    ragged lengths; packable = 0 for any value outside it."""
    import ctypes

    import numpy as np

    from paper_2502_00535_b200 import _lib
    from paper_2502_00535_b200.tensor_api import pack_box32

    lib = _lib.load()
    rng = np.random.default_rng(3)
    ok = ctypes.c_int(-1)
    for n in (0, 1, 31, 1000, 100003):
        x = rng.integers(0, 4096, n).astype(np.int32)
        y = rng.integers(0, 4096, n).astype(np.int32)
        z = rng.integers(0, 256, n).astype(np.int32)
        if n >= 3:
            x[:3], y[:3], z[:3] = (0, 4095, 7), (0, 4095, 9), (0, 255, 1)
        for threads in (0, 1, 3, 16):
            out = np.full(n, -1, np.int32)
            assert lib.pnms_pack_box32_host(x.ctypes.data, y.ctypes.data, z.ctypes.data, n, out.ctypes.data,
                                            threads, ctypes.byref(ok)) == 0
            assert ok.value == 1 and np.array_equal(out, pack_box32(x, y, z)), (n, threads)
    x = np.zeros(64, np.int32); y = np.zeros(64, np.int32); z = np.ones(64, np.int32)
    out = np.zeros(64, np.int32)
    for arr, v in ((x, 4096), (y, -1), (z, 256), (x, -5), (z, -1)):
        arr[37] = v
        lib.pnms_pack_box32_host(x.ctypes.data, y.ctypes.data, z.ctypes.data, 64, out.ctypes.data, 4, ctypes.byref(ok))
        assert ok.value == 0, v
        arr[37] = 1 if arr is z else 0
    assert lib.pnms_pack_box32_host(None, None, None, 5, None, 0, ctypes.byref(ok)) != 0
