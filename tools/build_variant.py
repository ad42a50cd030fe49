"""Build a tuning variant of the renderer library with extra -D flags into its
own directory, for A/B timing with NGPRT_LIB=<path> python bench.py.

  python tools/build_variant.py <name> [-DNGPRT_X=1 ...]
  -> paper_2407_10482_b200/_lib/var_<name>/libngprt_cuda.so
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_10482_b200 import _build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = _build.PKG / "_lib" / f"var_{name}"
_build.OBJ = out / "obj"
_build.LIB = out / "libngprt_cuda.so"
_build.COMMON = _build.COMMON + defines
print(_build.build())
