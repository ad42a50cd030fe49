"""Generate tests/golden/bake.json FROM THE REFERENCE ITSELF.

For every case of tests/cases.py:BAKE_CASES the reference's own bake()
(baking.hpp:107-202, via oracle/_ref's ref_bake) bakes the synthetic model and
writes it with save_baked (baking.hpp:266-349). The fixture records the SHA-256
of that .ngrt file plus per-array CRC-32s (corner keys and rows, pyramid
levels, distance grid) for diagnostics, and a CRC of the model's input arrays
to pin the synthetic-model generator. The GPU bake must reproduce the file byte
for byte (tests/test_bake.py). Runs only where /root/reference exists.
Usage: python tests/golden/gen_bake_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import paper_2407_10482_b200 as ng  # noqa: E402
from cases import BAKE_CASES, bake_opts  # noqa: E402
from checkers import ref  # noqa: E402
from bake_util import baked_crcs, model_crc  # noqa: E402


def main():
    R = ref()
    if R is None:
        raise SystemExit("reference not available")
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for case in BAKE_CASES:
            m = ng.SynthModel(**case["scene"])
            path = Path(td) / (case["name"] + ".ngrt")
            o = bake_opts(case["opts"])
            rc = R.ref_bake(C.cast(m.desc_ptr, C.c_void_p), m.train_words().ctypes.data,
                            m.train_res, C.byref(o), str(path).encode())
            if rc != 0:
                raise SystemExit(f"{case['name']}: {R.ref_last_error().decode()}")
            data = path.read_bytes()
            b = ng.BakedFile(path)
            out[case["name"]] = dict(sha256=hashlib.sha256(data).hexdigest(), size=len(data),
                                     model_crc=model_crc(m), **baked_crcs(b))
            print(case["name"], out[case["name"]]["n_coarse"], len(data))
    (HERE / "bake.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
