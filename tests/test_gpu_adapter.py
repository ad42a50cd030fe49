"""GPU: the drop-in through the reference's own C++ types (include/ngprt_gpu.hpp).

tests/cpp/adapter_demo (built by `make -C oracle demo` where the reference
headers exist; the binary travels to the GPU box) builds a BakedScene with the
reference's functions, renders it with the reference's CPU path and through the
adapter on the B200, and reports the reference's own max_abs_diff / psnr."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

DEMO = Path(__file__).resolve().parent / "cpp" / "_build" / "adapter_demo"


def test_adapter_renders_reference_baked_scene():
    if not DEMO.exists():
        pytest.skip("adapter_demo not built (needs /root/reference at build time)")
    out = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["counter_mismatch"] == 0
    assert r["max_abs_exact"] == 0.0          # bit-exact in exact-MLP mode
    assert r["max_abs_tensor"] <= 1e-3        # north_star RGB tolerance
    assert r["psnr_tensor"] >= 60.0
    assert r["storage"] == 1                  # non-fp16-exact values -> f32 storage
    # ngprt::gpu::bake over a reference NgpRtModel == the reference's bake(), file for file
    assert r["bake_identical"] is True
    assert r["bake_corners"] > 0
    # ngprt::gpu::Scene::render_async + wait (ngprt_render_host_async) == render
    assert r["async_mismatch"] == 0
    # ngprt::gpu::MultiScene (ngprt_multi_*): NCCL on one device, peer copies for two
    # replicas on one device; tile and camera sharding == Scene::render
    assert r["multi_nccl"] is True
    assert r["multi_mismatch"] == 0
