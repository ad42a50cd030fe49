"""BenchReport CSV (SPEC.md `bench` subcommand, "paired marcher comparison"):
the same rays marched with the occupancy pyramid only and with the distance
grid (Eq. 9), plus the max_step_rule variant, on the GPU renderer.

Columns (SPEC.md External Interfaces): scene, marcher, rays, mean_marching,
mean_occupied, mean_occ_accesses, mean_dist_accesses, ms_per_frame. The counter
columns are the bit-exact MarchCounters (identical to the reference's), so the
pairing is comparable by construction; ms_per_frame is the B200 device time of
a full render (CUDA events, best of 5).

  python tools/bench_report.py [--scenes slab,toy,bench,mip360] [--width 1920 --height 1080]
"""
from __future__ import annotations

import argparse
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2407_10482_b200 as ng  # noqa: E402

MARCHERS = [("occupancy", dict(use_dist_grid=False)),
            ("distance", dict(use_dist_grid=True)),
            ("distance_max_step_rule", dict(use_dist_grid=True, max_step_rule=True))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", default="slab,toy,bench,mip360")
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--out", default="-")
    a = ap.parse_args()
    f = sys.stdout if a.out == "-" else open(a.out, "w", newline="")
    w = csv.writer(f)
    w.writerow(["scene", "marcher", "rays", "mean_marching", "mean_occupied", "mean_occ_accesses",
                "mean_dist_accesses", "ms_per_frame"])
    for name in a.scenes.split(","):
        cfg = dict(ng.CONFIGS["c3_1080p"])
        cfg["occupancy"] = name
        if name != "mip360":
            cfg.update(sigma_lo=2.0, sigma_hi=6.0)
        scene = ng.Scene(ng.SynthScene(**cfg))
        cam = ng.cameras(64, a.width, a.height)[0]
        for marcher, kw in MARCHERS:
            opts = ng.Opts(mlp="tensor", **kw)
            _, st = ng.render(scene, [cam], opts, stats=True)
            m = st.reshape(-1, 4).double().mean(0).tolist()
            best = 1e30
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ng.render(scene, [cam], opts)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            w.writerow([name, marcher, a.width * a.height, f"{m[0]:.4f}", f"{m[1]:.4f}",
                        f"{m[2]:.4f}", f"{m[3]:.4f}", f"{best:.4f}"])
            f.flush()
        scene.close()


if __name__ == "__main__":
    main()
