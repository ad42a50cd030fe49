"""Time K3 (pyramid) and K4 (distance transform) on a config's occupancy
(CUDA events, best of N): python tools/bench_dt.py [config] [reps]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2407_10482_b200 as ng  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_1080p"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
synth = ng.SynthScene(**ng.CONFIGS[cfg])
r0 = int(synth.desc.occ_base_res)
words = torch.from_numpy(synth.base_words().view("int64").copy()).cuda()
out = {}
for name, fn in [("pyramid_K3", lambda: ng.build_pyramid(words, r0)),
                 ("distance_K4", None)]:
    if fn is None:
        lv = ng.build_pyramid(words, r0)
        fn = lambda: ng.build_distance_grid(lv[0], r0 // 2)  # noqa: E731
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[name + "_ms"] = best
out["config"] = cfg
out["grid"] = f"{r0}^3 base, distance grid {r0 // 2}^3"
out["occupancy"] = synth.occupancy_fraction()
print(json.dumps(out))
