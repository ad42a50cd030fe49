"""CPU: the two column algorithms behind K4's u8 passes (occupancy.cu
dt_rmq_kernel / dt_deque_kernel), restated in numpy, reproduce the C oracle's
build_distance_grid (occupancy.hpp:136-194) on small grids. These check the
algorithms (u8 saturation with the all-empty flag, range-minimum bisection plus
1-Lipschitz steps along and across columns, monotone-deque sweeps), not the
kernels; the kernels are compared with the reference on the GPU
(test_gpu_parity.py::test_distance_grid_u8_passes_match_reference)."""
from __future__ import annotations

import numpy as np
import pytest

from cases import random_grid_words
from checkers import oracle


def _bits(words, r):
    return np.unpackbits(words.view(np.uint8), bitorder="little")[: r ** 3].reshape(r, r, r)  # z, y, x


def _x_pass(bits):
    """Saturated x-distance per voxel (255 for a row without occupied voxels)."""
    r = bits.shape[-1]
    x = np.arange(r)
    out = np.full(bits.shape, 255, np.int64)
    for z in range(r):
        for y in range(r):
            occ = np.nonzero(bits[z, y])[0]
            if occ.size:
                out[z, y] = np.minimum(np.abs(x[:, None] - occ[None, :]).min(1), 255)
    return out


def _rmq_pass(g, axis):
    """D(u) = min{d : min(g[u-d .. u+d]) <= d} along `axis`: bisection for the
    first column of each 4-column group (first element of each 8-element chunk),
    then 1-Lipschitz steps along the column and across x, as dt_rmq_kernel."""
    g = np.ascontiguousarray(np.moveaxis(g, axis, -1))  # (o, x, u): columns last
    r = g.shape[-1]
    out = np.empty_like(g)
    E = max(1, r // 32)

    def step(col, u, d):
        lo, hi = max(0, u - max(d - 1, 0)), min(r - 1, u + max(d - 1, 0))
        m1 = col[lo:hi + 1].min() if d >= 1 else 0xFFFF
        m2 = min(m1, col[max(u - d, 0)], col[min(u + d, r - 1)])
        return d - 1 if m1 <= d - 1 else (d if m2 <= d else d + 1)

    flat = g.reshape(-1, g.shape[-2], r)  # (o, x, u): x is the column index within a row
    res = out.reshape(-1, g.shape[-2], r)
    for o in range(flat.shape[0]):
        prev = None
        for x in range(flat.shape[1]):
            col = flat[o, x]
            if x % 4 == 0:
                cur = np.empty(r, np.int64)
                for u0 in range(0, r, E):
                    d = 0
                    for bit in (128, 64, 32, 16, 8, 4, 2, 1):
                        m = d + bit - 1
                        if col[max(0, u0 - m):min(r - 1, u0 + m) + 1].min() > m:
                            d += bit
                    cur[u0] = d
                    for u in range(u0 + 1, min(u0 + E, r)):
                        d = step(col, u, d)
                        cur[u] = d
            else:
                cur = np.array([step(col, u, int(prev[u])) for u in range(r)])
            res[o, x] = cur
            prev = cur
    return np.moveaxis(out, -1, axis)


def _deque_sweep(col):
    """min over i <= u of max(u - i, g_i) with the monotone deque (dt_sweep)."""
    dq, out = [], []
    for p, gp in enumerate(col):
        while dq and dq[-1][1] >= gp:
            dq.pop()
        dq.append((p, int(gp)))
        while len(dq) >= 2 and max(p - dq[0][0], dq[0][1]) >= max(p - dq[1][0], dq[1][1]):
            dq.pop(0)
        out.append(max(p - dq[0][0], dq[0][1]))
    return np.array(out)


def _deque_pass(g, axis):
    g = np.ascontiguousarray(np.moveaxis(g, axis, -1))
    out = np.empty_like(g)
    for idx in np.ndindex(g.shape[:-1]):
        col = g[idx]
        out[idx] = np.minimum(_deque_sweep(col), _deque_sweep(col[::-1])[::-1])
    return np.moveaxis(out, -1, axis)


def _final(d, bits):
    if not bits.any():
        return np.full(d.shape, 255, np.uint8)
    return np.maximum(d - 1, 0).astype(np.uint8)


GRIDS = [(32, 0.0, 31), (32, 0.002, 32), (32, 0.05, 33), (32, 0.5, 34), (64, 1e-4, 35)]


@pytest.mark.parametrize("res,dens,seed", GRIDS)
def test_rmq_and_deque_passes_match_oracle(ng, res, dens, seed):
    words = random_grid_words(ng, res, dens, seed)
    want = np.zeros(res ** 3, np.uint8)
    oracle().orc_build_distance_grid(words.ctypes.data, res, want.ctypes.data)
    bits = _bits(words, res)
    gx = _x_pass(bits)
    # axis order of the (z, y, x) array: y is axis 1, z is axis 0
    d_rmq = _rmq_pass(_rmq_pass(gx, 1), 0)
    d_deq = _deque_pass(_deque_pass(gx, 1), 0)
    assert np.array_equal(_final(d_rmq, bits).ravel(), want)
    assert np.array_equal(_final(d_deq, bits).ravel(), want)


def test_diagonal_plane_long_deques(ng):
    """A slope-2 plane: long monotone deques (the GPU ring overflows) and long
    Lipschitz runs; both restatements still equal the oracle."""
    r = 32
    bits = np.zeros((r, r, r), np.uint8)
    y = np.arange(r // 2)
    bits[: r // 2, y, 2 * y] = 1
    words = np.zeros(r ** 3 // 64, np.uint64)
    words.view(np.uint8)[:] = np.packbits(bits.ravel(), bitorder="little")
    want = np.zeros(r ** 3, np.uint8)
    oracle().orc_build_distance_grid(words.ctypes.data, r, want.ctypes.data)
    gx = _x_pass(bits)
    assert np.array_equal(_final(_rmq_pass(_rmq_pass(gx, 1), 0), bits).ravel(), want)
    assert np.array_equal(_final(_deque_pass(_deque_pass(gx, 1), 0), bits).ravel(), want)
