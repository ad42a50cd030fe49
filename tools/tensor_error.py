"""Max-abs RGB error of the tensor-MLP mode against the bit-exact mode (which
equals the reference bit for bit) on full frames of several configs:
  python tools/tensor_error.py  (NGPRT_LIB selects a build variant)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_10482_b200 as ng  # noqa: E402

out = {}
for cfg, w, h, cams in [("c3_1080p", 1920, 1080, [0, 13, 40]), ("c1_256", 256, 256, [0, 3]),
                        ("c2_blob800", 800, 800, [0, 7]), ("c3_mip360", 1920, 1080, [5])]:
    synth = ng.SynthScene(**dict(ng.CONFIGS[cfg]))
    dev = ng.Scene(synth)
    cs = ng.cameras(64, w, h)
    worst, se, npx = 0.0, 0.0, 0
    for i in cams:
        t, _ = ng.render(dev, [cs[i]], ng.Opts(mlp="tensor"), stats=True)
        e, _ = ng.render(dev, [cs[i]], ng.Opts(mlp="exact"), stats=True)
        torch.cuda.synchronize()
        d = (t[0] - e[0]).abs().double()
        worst = max(worst, float(d.max()))
        se += float((d * d).sum())
        npx += d.numel()
    mse = se / npx
    out[cfg] = {"max_abs": worst, "psnr_db": 99.0 if mse == 0 else min(99.0, -10 * np.log10(mse))}
print(json.dumps(out))
