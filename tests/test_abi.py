"""CPU: the C-ABI library loads, exports every function include/ngprt_cuda.h
declares, and the ctypes mirror has the C compiler's struct layouts. No GPU
compute is called here."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ngprt_cuda.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ngprt_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["ngprt_scene_create", "ngprt_scene_destroy", "ngprt_render", "ngprt_render_host",
                 "ngprt_build_pyramid", "ngprt_build_distance_grid", "ngprt_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(ng):
    L = C.CDLL(str(ng._abi.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert set(declared_functions()) <= set(ng._abi.SIGNATURES)
    assert L.ngprt_abi_version() == 2


def test_struct_layout_matches_c(tmp_path, ng):
    from paper_2407_10482_b200 import _abi
    src = tmp_path / "sz.c"
    structs = ["ngprt_scene_desc", "ngprt_camera", "ngprt_render_opts", "ngprt_ray_stats",
               "ngprt_scene_info", "ngprt_synth_params"]
    body = "\n".join(f'printf("%zu\\n", sizeof({s}));' for s in structs)
    src.write_text(f'#include <stdio.h>\n#include "ngprt_cuda.h"\nint main(){{{body}return 0;}}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    sizes = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                            check=True).stdout.split()]
    py = [_abi.SceneDesc, _abi.Camera, _abi.RenderOpts, _abi.RayStats, _abi.SceneInfo,
          _abi.SynthParams]
    assert [C.sizeof(t) for t in py] == sizes


def test_errors_without_device_are_loud(ng):
    """Scene creation with a bad descriptor fails with EINVAL and a message,
    before any device is touched."""
    d = ng._abi.SceneDesc()
    d.L = 7
    h = C.c_void_p()
    st = ng.lib().ngprt_scene_create(C.byref(d), 0, C.byref(h))
    assert st == ng._abi.EINVAL
    assert b"L out of range" in ng.lib().ngprt_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2407_10482_b200 import _abi
    monkeypatch.setattr(_abi, "LIB_PATH", tmp_path / "nope.so")
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _abi.lib()


def test_expf_port_table_matches_host_libm():
    """The device expf port's table (device_common.cuh) is glibc's __exp2f_data.tab."""
    import struct
    src = (ROOT / "paper_2407_10482_b200" / "csrc" / "device_common.cuh").read_text()
    tab = [int(v, 16) for v in re.findall(r"0x([0-9a-f]{16})ull", src)]
    assert len(tab) == 32
    libm = None
    for cand in ["/lib/x86_64-linux-gnu/libm.so.6", "/usr/lib/x86_64-linux-gnu/libm.so.6"]:
        if Path(cand).exists():
            libm = Path(cand).read_bytes()
            break
    if libm is None:
        pytest.skip("host libm not found")
    pat = b"".join(struct.pack("<Q", t) for t in tab)
    idx = libm.find(pat)
    assert idx >= 0, "table not found in host libm"
    after = struct.unpack("<9d", libm[idx + 256: idx + 256 + 72])
    # shift_scaled, poly[3], shift, invln2_scaled, poly_scaled[3] (e_exp2f_data.c)
    assert after[4] == float.fromhex("0x1.8p+52")
    assert after[5] == float.fromhex("0x1.71547652b82fep+5")
    assert after[6:9] == (float.fromhex("0x1.c6af84b912394p-20"),
                          float.fromhex("0x1.ebfce50fac4f3p-13"),
                          float.fromhex("0x1.62e42ff0c52d6p-6"))


def test_multi_and_shard_entry_points_validate_on_cpu(ng):
    """The multi-device and sharding entry points validate their arguments and fail
    loudly (no device here) instead of crashing; ngprt_shard_pixels is pure host
    arithmetic."""
    import ctypes as C
    L = ng.lib()
    h = C.c_void_p()
    assert L.ngprt_multi_create(None, None, 0, C.byref(h)) == ng._abi.EINVAL
    d = ng._abi.SceneDesc()
    d.L = 7
    devs = (C.c_int * 1)(0)
    assert L.ngprt_multi_create(C.byref(d), devs, 1, C.byref(h)) == ng._abi.EINVAL
    assert b"L out of range" in L.ngprt_last_error()
    assert L.ngprt_multi_uses_nccl(None) == 0
    assert L.ngprt_multi_scene(None, 0) is None
    # ceil(60 tiles / 7) = 9 tiles of 32 x 32 per rank for a 300 x 190 window
    assert L.ngprt_shard_pixels(300, 190, 7, 32) == 9 * 32 * 32
    assert L.ngprt_shard_pixels(300, 190, 0, 0) == 60 * 32 * 32  # world 0 => 1, tile 0 => 32
    assert L.ngprt_shard_assemble(None, 1, 1, 8, 8, 8, 3, None, None) == ng._abi.EINVAL
