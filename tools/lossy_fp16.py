"""Forced fp16 storage of an f32 scene (ngprt_storage F16 on values that are not
fp16-exact): speed and error against the exact f32 render (which is bit-exact vs
the reference). python tools/lossy_fp16.py [config] [cam]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_10482_b200 as ng  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_1080p_f32"
synth = ng.SynthScene(**ng.CONFIGS[cfg])
cams = ng.cameras(64, 1920, 1080)
res = {"config": cfg}
out = {}
for name, storage in [("f32", ng._abi.STORAGE_F32), ("fp16_lossy", ng._abi.STORAGE_F16)]:
    sc = ng.Scene(synth, storage=storage)
    rgbs, sts, ms = [], [], []
    for ci in range(5, 13):
        rgb, st = ng.render(sc, [cams[ci]], ng.Opts(mlp="exact"), stats=True)
        rgbs.append(rgb.cpu().numpy())
        sts.append(st.cpu().numpy())
    for rep in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ng.render(sc, [cams[5 + rep % 8]], ng.Opts())
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out[name] = (np.concatenate(rgbs), np.concatenate(sts))
    res[name + "_ms_per_frame"] = float(np.median(ms))
    del sc
a, b = out["f32"][0], out["fp16_lossy"][0]
d = np.abs(a - b)
mse = float(np.mean((a.astype(np.float64) - b) ** 2))
res.update(max_abs=float(d.max()), frac_pixels_over_1e3=float((d.max(-1) > 1e-3).mean()),
           psnr=99.0 if mse == 0 else float(10 * np.log10(1 / mse)),
           counter_rays_differing=float((out["f32"][1] != out["fp16_lossy"][1]).any(-1).mean()))
print(json.dumps(res))
