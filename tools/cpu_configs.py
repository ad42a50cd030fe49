"""CPU reference throughput per BASELINE config (config 1 in
full, configs 2, 3 and 5 one full frame each): the compiled reference
(oracle/_ref, kind "reference") renders camera 0 of each config on all host
threads, and a 4-row band on one thread. Prints one JSON line per config.

  python tools/cpu_configs.py [--configs c1_256,c2_blob800,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2407_10482_b200 as ng  # noqa: E402
from checkers import REF_SO, CpuScene  # noqa: E402

DEFAULT = ["c1_256", "c2_blob800", "c3_1080p", "c5_2160p:n_boxes=10", "c5_2160p:n_boxes=140",
           "c5_2160p:n_boxes=2240"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(DEFAULT))
    a = ap.parse_args()
    kind = "reference" if REF_SO.exists() else "port"
    threads = os.cpu_count() or 1
    model = ""
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                     if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    for spec in a.configs.split(","):
        name, _, extra = spec.partition(":")
        cfg = dict(ng.CONFIGS[name])
        for kv in filter(None, extra.split(";")):
            k, v = kv.split("=")
            cfg[k] = int(v)
        W, H = cfg["width"], cfg["height"]
        synth = ng.SynthScene(**cfg)
        cam = ng.cameras(cfg.get("n_cams", 1), W, H)[0]
        cs = CpuScene(synth.desc_ptr, "ref" if kind == "reference" else "oracle")
        t = time.perf_counter()
        cs.render(cam, ng.Opts().to_c(), nthreads=threads)
        full = time.perf_counter() - t
        t = time.perf_counter()
        cs.render(cam, ng.Opts(window=(0, H // 2 - 2, W, 4)).to_c(), nthreads=1)
        one = time.perf_counter() - t
        cs.close()
        print(json.dumps({"config": spec, "kind": kind, "threads": threads, "cpu_model": model,
                          "frame_s": full, "fps": 1.0 / full, "mrays_per_s": W * H / full / 1e6,
                          "one_thread_mrays_per_s": W * 4 / one / 1e6}), flush=True)


if __name__ == "__main__":
    main()
