"""BenchReport CSV (SPEC.md `bench`: paired marcher comparison, External
Interfaces columns) from tools/bench_report.py on the GPU renderer: both
marchers see the same rays, so the occupied-point column is identical, and on
the slab scene the distance grid removes >= 40 % of the marching points
(acceptance criterion 1)."""
from __future__ import annotations

import csv
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
COLUMNS = ["scene", "marcher", "rays", "mean_marching", "mean_occupied", "mean_occ_accesses",
           "mean_dist_accesses", "ms_per_frame"]


def test_bench_report_pairs(tmp_path):
    out = tmp_path / "report.csv"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "bench_report.py"), "--scenes",
                        "slab,toy", "--width", "256", "--height", "192", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(out.open()))
    assert list(rows[0].keys()) == COLUMNS
    by = {(x["scene"], x["marcher"]): x for x in rows}
    for scene in ("slab", "toy"):
        occ, dist = by[(scene, "occupancy")], by[(scene, "distance")]
        assert occ["rays"] == dist["rays"] == str(256 * 192)
        assert occ["mean_occupied"] == dist["mean_occupied"]          # same samples
        assert float(occ["mean_dist_accesses"]) == 0.0
        assert by[(scene, "distance_max_step_rule")]["mean_occupied"] == occ["mean_occupied"]
    slab_occ, slab_dist = by[("slab", "occupancy")], by[("slab", "distance")]
    assert float(slab_dist["mean_marching"]) <= 0.6 * float(slab_occ["mean_marching"])
