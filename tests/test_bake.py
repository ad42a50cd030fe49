"""The bake (baking.hpp:107-202) on the GPU: ngprt_bake vs the reference's own bake.

Parity bar: the GPU-baked BakedScene, written with ngprt_baked_save, is the
reference's .ngrt file BYTE FOR BYTE (tests/golden/bake.json holds the SHA-256
of the file the reference's bake + save_baked wrote for each BAKE_CASE, made by
tests/golden/gen_bake_golden.py). That covers the density cull decisions,
dilation, the 512 render grid and its pyramid, the distance grid, the
retained corner keys and every bit of every evaluated corner row.

CPU: the synthetic-model generator is pinned, ngprt_baked_save reproduces the
reference's save_baked byte for byte, and invalid bakes fail with the
reference's messages (validation runs before any device work)."""
from __future__ import annotations

import ctypes as C
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from bake_util import baked_crcs, model_crc
from cases import BAKE_CASES, bake_opts
from checkers import CpuScene, ref

GOLDEN = json.loads((Path(__file__).parent / "golden" / "bake.json").read_text())
IDS = [c["name"] for c in BAKE_CASES]


@pytest.mark.parametrize("case", BAKE_CASES, ids=IDS)
def test_synth_model_pinned(ng, case):
    m = ng.SynthModel(**case["scene"])
    assert model_crc(m) == GOLDEN[case["name"]]["model_crc"]


def test_save_reproduces_reference_file(ng, tmp_path):
    """load_baked -> ngprt_baked_save of a reference-written file is the same file."""
    R = ref()
    if R is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    case = BAKE_CASES[3]
    m = ng.SynthModel(**case["scene"])
    src = tmp_path / "ref.ngrt"
    o = bake_opts(case["opts"])
    assert R.ref_bake(C.cast(m.desc_ptr, C.c_void_p), m.train_words().ctypes.data, m.train_res,
                      C.byref(o), str(src).encode()) == 0
    data = src.read_bytes()
    assert hashlib.sha256(data).hexdigest() == GOLDEN[case["name"]]["sha256"]
    dst = tmp_path / "resaved.ngrt"
    ng.BakedFile(src).save(dst)
    assert dst.read_bytes() == data


def _nan_model(ng):
    m = ng.SynthModel(occupancy="toy", occ_base_res=32, L=2, L_C=32, fine_table_len=1 << 10)
    fine = np.ctypeslib.as_array(C.cast(m.desc.fine_tables[1], C.POINTER(C.c_float)), shape=(8,))
    fine[5] = np.nan
    return m


ERRORS = [
    ("tres_not_dividing", dict(occupancy="toy", occ_base_res=48, L=2, L_C=48, fine_table_len=1 << 10),
     "bake: training grid must divide the 512 render grid"),
    ("lc_not_nesting", dict(occupancy="toy", occ_base_res=64, L=2, L_C=96, fine_table_len=1 << 10),
     "bake: L_C and the training grid must nest"),
    ("non_finite", None, "bake: non-finite parameter in group fine_l2"),
]


@pytest.mark.parametrize("name,scene,msg", ERRORS, ids=[e[0] for e in ERRORS])
def test_bake_errors_match_reference(ng, tmp_path, name, scene, msg):
    m = _nan_model(ng) if scene is None else ng.SynthModel(**scene)
    with pytest.raises(ng.NgprtError, match=msg):
        ng.bake(m)
    R = ref()
    if R is not None:  # the reference's bake raises the same text
        o = bake_opts({})
        assert R.ref_bake(C.cast(m.desc_ptr, C.c_void_p), m.train_words().ctypes.data,
                          m.train_res, C.byref(o), str(tmp_path / "x.ngrt").encode()) == 1
        assert R.ref_last_error().decode() == msg


@pytest.mark.gpu
@pytest.mark.parametrize("case", BAKE_CASES, ids=IDS)
def test_gpu_bake_is_the_reference_file(ng, tmp_path, case):
    m = ng.SynthModel(**case["scene"])
    b = ng.bake(m, **case["opts"])
    want = GOLDEN[case["name"]]
    got = baked_crcs(b)
    # per-array diagnostics first, then the whole file
    assert got["n_coarse"] == want["n_coarse"]
    assert got["occupied"] == want["occupied"]
    assert got["pyramid"] == want["pyramid"]
    assert got["dist"] == want["dist"]
    assert got["keys"] == want["keys"]
    assert got["rows"] == want["rows"]
    path = tmp_path / "gpu.ngrt"
    b.save(path)
    data = path.read_bytes()
    assert len(data) == want["size"]
    assert hashlib.sha256(data).hexdigest() == want["sha256"]


@pytest.mark.gpu
def test_gpu_baked_scene_renders_like_oracle(ng):
    """bake -> Scene -> render: the GPU-baked scene renders bit-exactly like the
    CPU oracle renders the same BakedScene."""
    import torch
    case = BAKE_CASES[1]
    m = ng.SynthModel(**case["scene"])
    b = ng.bake(m, **case["opts"])
    dev = ng.Scene(b)
    cam = ng.cameras(4, 48, 40)[2]
    opts = ng.Opts(mlp="exact")
    rgb, st = ng.render(dev, [cam], opts, stats=True)
    torch.cuda.synchronize()
    cs = CpuScene(b.desc_ptr, "oracle")
    want_rgb, want_st = cs.render(cam, opts.to_c(), nthreads=8)
    assert np.array_equal(st[0].cpu().numpy().view(np.uint32), want_st)
    assert np.array_equal(rgb[0].cpu().numpy().view(np.uint32), want_rgb.view(np.uint32))
    assert (want_st.reshape(-1, 4)[:, 1] > 0).any()  # some rays hit the baked scene
