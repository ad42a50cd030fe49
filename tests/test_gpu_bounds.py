"""GPU: the renderer built with device-side bounds assertions on every gather and
per-ray store (NGPRT_DEBUG_BOUNDS=1, csrc/device_common.cuh NG_BOUNDS) runs the
golden parity cases, sharded renders, the f32 path and the skip-safety hook
without tripping one, and still matches the reference. This is the memory-safety
check of the render path: compute-sanitizer is closed on this GPU pool."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
VARIANT = ROOT / "paper_2407_10482_b200" / "_lib" / "var_bounds" / "libngprt_cuda.so"


def test_parity_suite_under_bounds_checks():
    if not VARIANT.exists():
        subprocess.run([sys.executable, str(ROOT / "tools" / "build_variant.py"), "bounds",
                        "-DNGPRT_DEBUG_BOUNDS=1"], check=True, capture_output=True)
    env = dict(os.environ, NGPRT_LIB=str(VARIANT))
    r = subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "-k",
                        "render_exact or render_tensor or c1_256 or axis_aligned or multi_camera",
                        "tests/test_gpu_shard.py", "tests/test_acceptance.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert "bounds check failed" not in r.stdout + r.stderr, tail
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
