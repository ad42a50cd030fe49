"""Bake benchmark: ngprt_bake (GPU, csrc/bake.cu) against the reference's own
bake (baking.hpp:107-202, oracle/_ref's ref_bake, single-threaded as the
reference is) on the same synthetic model and training grid.

The GPU time is the whole C-ABI call: host model -> device, every kernel, the
BakedScene back in host memory (wall clock around a synchronous call, after
warm-up). Set NGPRT_BAKE_PROFILE=1 for the per-phase split.

  python tools/bench_bake.py --occupancy mip360 --tres 128 --lc 512 [--ref]
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2407_10482_b200 as ng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--occupancy", default="mip360")
    ap.add_argument("--tres", type=int, default=128)
    ap.add_argument("--lc", type=int, default=512)
    ap.add_argument("--L", type=int, default=2)
    ap.add_argument("--fine-log2", type=int, default=21)
    ap.add_argument("--sigma", type=float, default=-0.5)
    ap.add_argument("--fusion", default="separate_att_v")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--ref", action="store_true", help="also time the reference bake (CPU)")
    ap.add_argument("--check", action="store_true", help="compare the two .ngrt files")
    a = ap.parse_args()

    m = ng.SynthModel(occupancy=a.occupancy, occ_base_res=a.tres, L_C=a.lc, L=a.L,
                      fine_table_len=1 << a.fine_log2, sigma_lo=a.sigma, sigma_hi=a.sigma,
                      fusion_tag=a.fusion)
    for _ in range(a.warmup):
        ng.bake(m).close()
    times = []
    b = None
    for _ in range(a.steps):
        if b is not None:
            b.close()
        t0 = time.perf_counter()
        b = ng.bake(m)
        times.append((time.perf_counter() - t0) * 1e3)
    out = dict(metric="bake_ms", value=min(times), unit="ms", higher_is_better=False,
               steps=a.steps, warmup=a.warmup, all_ms=[round(t, 3) for t in times],
               config=dict(workload=f"bake {a.occupancy} train {a.tres}^3 L_C {a.lc}", L=a.L,
                           fine_table_len=1 << a.fine_log2, fusion=a.fusion),
               n_corners=int(b.desc.n_coarse))
    if a.ref:
        from cases import bake_opts
        from checkers import ref
        R = ref()
        with tempfile.TemporaryDirectory() as td:
            p = Path(td) / "ref.ngrt"
            o = bake_opts({})
            t0 = time.perf_counter()
            rc = R.ref_bake(C.cast(m.desc_ptr, C.c_void_p), m.train_words().ctypes.data,
                            m.train_res, C.byref(o), str(p).encode())
            out["cpu_ref_ms"] = (time.perf_counter() - t0) * 1e3
            assert rc == 0, R.ref_last_error()
            out["cpu_ref_cores"] = 1
            if a.check:
                g = Path(td) / "gpu.ngrt"
                b.save(g)
                out["identical"] = (hashlib.sha256(g.read_bytes()).hexdigest() ==
                                    hashlib.sha256(p.read_bytes()).hexdigest())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
