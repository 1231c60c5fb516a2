"""Build variants of the library with extra nvcc defines into build_tmp/var_<name>.so (A/B on
the GPU box through PNMS_LIB), then rebuild the default library.

    python tools/build_variants.py name=-DFOO=1,-DBAR=2 [name2=...]"""
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    build.build(force=True, extra=[f for f in flags.split(",") if f])
    shutil.copy(build.LIB_PATH, build.LIB_PATH.parent / "build_tmp" / f"var_{name}.so")
    print("built", name, flags)
build.build(force=True)
