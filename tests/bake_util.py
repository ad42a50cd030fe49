"""CRC summaries of bake inputs (SynthModel) and outputs (BakedFile), shared by
tests/golden/gen_bake_golden.py and tests/test_bake.py."""
from __future__ import annotations

import ctypes as C

import numpy as np


def _crc(a) -> int:
    from paper_2407_10482_b200 import lib
    a = np.ascontiguousarray(a)
    return int(lib().ngprt_crc32(a.ctypes.data, a.nbytes, 0))


def _f32(ptr, n):
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(int(n),))


def model_crc(m) -> int:
    """CRC-32 over every input array of a SynthModel, in desc order."""
    d = m.desc
    L = int(d.L)
    crc = 0
    from paper_2407_10482_b200 import lib

    def add(a):
        nonlocal crc
        a = np.ascontiguousarray(a)
        crc = int(lib().ngprt_crc32(a.ctypes.data, a.nbytes, crc))

    for k in range(6):
        r = int(d.coarse_res[k])
        add(_f32(d.coarse_tables[k], min((r + 1) ** 3, int(d.coarse_table_len)) * 4))
    W = 8 + 2 * L
    add(_f32(d.aux_w[0], 64 * 24)); add(_f32(d.aux_b[0], 64))
    add(_f32(d.aux_w[1], W * 64)); add(_f32(d.aux_b[1], W))
    for l in range(L):
        add(_f32(d.fine_tables[l], int(d.fine_table_len[l]) * 8))
    add(m.train_words())
    return crc


def baked_crcs(b) -> dict:
    d = b.desc
    return dict(n_coarse=int(d.n_coarse), keys=_crc(b.coarse_keys()), rows=_crc(b.coarse_rows()),
                pyramid=[_crc(b.pyramid_words(k)) for k in range(5)], dist=_crc(b.dist_values()),
                occupied=[int(np.unpackbits(b.pyramid_words(k).view(np.uint8)).sum())
                          for k in range(5)])
