import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


class Case:
    __slots__ = ("x", "y", "z", "s", "count", "d_max", "keep", "writes", "mat", "by_index", "k", "theta", "note")

    @property
    def tie(self):
        return "by_index" if self.by_index else "paper_faithful"


def load_cases():
    g = np.load(GOLDEN / "cases.npz")
    out = []
    for i, (off, n, d_max, koff, klen, moff, mlen, by_index, k) in enumerate(g["meta"]):
        c = Case()
        c.x, c.y, c.z, c.s = (g[nm][off:off + n] for nm in ("x", "y", "z", "s"))
        c.count, c.d_max = int(n), int(d_max)
        c.keep = g["keep"][koff:koff + klen]
        c.writes = int(g["writes"][i])
        c.mat = g["mat"][moff:moff + mlen].reshape(d_max, -1) if mlen else None
        c.by_index, c.k = bool(by_index), int(k)
        c.theta = float(g["theta"][i])
        c.note = str(g["note"][i])
        out.append(c)
    return out


def load_configs():
    g = np.load(GOLDEN / "configs.npz")
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    return {nm: {f: g[f"{nm}_{f}"] for f in ("x", "y", "z", "s", "keep", "writes")} for nm in names}


@pytest.fixture(scope="session")
def golden_cases():
    return load_cases()


@pytest.fixture(scope="session")
def golden_configs():
    return load_configs()


def load_matrices():
    """Full-size reference SuppressionMatrix goldens (tests/golden/matrices.npz)."""
    g = np.load(GOLDEN / "matrices.npz")
    out = {}
    for nm in sorted({k.rsplit("_", 1)[0] for k in g.files}):
        d_max, by_index, writes = (int(v) for v in g[f"{nm}_meta"])
        out[nm] = dict(x=g[f"{nm}_x"], y=g[f"{nm}_y"], z=g[f"{nm}_z"], s=g[f"{nm}_s"], d_max=d_max,
                       tie="by_index" if by_index else "paper_faithful", writes=writes,
                       theta=float(g[f"{nm}_theta"][0]), bits=g[f"{nm}_bits"], mask=g[f"{nm}_mask"])
    return out


@pytest.fixture(scope="session")
def golden_matrices():
    return load_matrices()
