"""C3: shared-memory 2D Jacobi stencil (BASELINE.json configs[2]) — INPUT ONLY.

512x512 int grid, 1024 blocks x 256 threads (16x16 tiles).  Per block:
  load   the 18x18 halo tile: thread t loads cells t and t+256 (< 324):
         read in[gy*512+gx] (global, clamped at the border), write A[cell] (shared)
  __syncthreads
  K sweeps ping-ponging shared tiles A (words 0..323) and B (324..647):
         thread (ty, tx) reads src at its centre and 4 neighbours and writes dst
         at its centre, then __syncthreads (the barrier after sweep `removed`
         is dropped in the racy variant)
  final  read dst[centre] (shared), write out[gy*512+gx] (global, words 2^18..)
~256 checked accesses per thread, ~2^26 per launch.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from .format import (NOP, OP_READ, OP_WRITE, SPACE_GLOBAL, SPACE_SHARED, SYNCTHREADS, Trace,
                     kernel_from_rows, make_trace)

N = 512
T = 16
H = T + 2
TILE = H * H            # 324
A_BASE, B_BASE = 0, TILE
OUT_BASE = N * N
K_SWEEPS = 42


def _rec(op, space, word):
    return (np.uint64(op) << np.uint64(62)) | (np.uint64(space) << np.uint64(61)) | word.astype(np.uint64)


def stencil_trace(removed: Optional[int] = None, sweeps: int = K_SWEEPS, n: int = N) -> Trace:
    """The C3 trace; ``removed`` = index of the sweep whose trailing barrier is dropped."""
    tiles = n // T
    blocks = tiles * tiles
    ltid = np.arange(256)
    ty, tx = ltid // T, ltid % T
    centre = (ty + 1) * H + (tx + 1)
    bx = np.arange(blocks) % tiles
    by = np.arange(blocks) // tiles

    rows = []   # list of (blocks, 256) uint64 arrays, one per row step

    # load phase: two loads per thread (second only for cells < 324)
    for k in range(2):
        cell = ltid + 256 * k
        ok = cell < TILE
        hy, hx = np.minimum(cell, TILE - 1) // H, np.minimum(cell, TILE - 1) % H
        gy = np.clip(by[:, None] * T + hy[None, :] - 1, 0, n - 1)
        gx = np.clip(bx[:, None] * T + hx[None, :] - 1, 0, n - 1)
        rg = _rec(OP_READ, SPACE_GLOBAL, gy * n + gx)
        ws = np.broadcast_to(_rec(OP_WRITE, SPACE_SHARED, A_BASE + cell), (blocks, 256))
        rows.append(np.where(ok[None, :], rg, np.uint64(NOP)))
        rows.append(np.where(ok[None, :], ws, np.uint64(NOP)))
    rows.append(np.full((blocks, 256), SYNCTHREADS, dtype=np.uint64))

    src, dst = A_BASE, B_BASE
    for s in range(sweeps):
        for off in (0, -H, H, -1, 1):
            rows.append(np.broadcast_to(_rec(OP_READ, SPACE_SHARED, src + centre + off), (blocks, 256)))
        rows.append(np.broadcast_to(_rec(OP_WRITE, SPACE_SHARED, dst + centre), (blocks, 256)))
        if s != removed:
            rows.append(np.full((blocks, 256), SYNCTHREADS, dtype=np.uint64))
        src, dst = dst, src
    last = src                       # tile written by the final sweep
    gy = by[:, None] * T + ty[None, :]
    gx = bx[:, None] * T + tx[None, :]
    rows.append(np.broadcast_to(_rec(OP_READ, SPACE_SHARED, last + centre), (blocks, 256)))
    rows.append(_rec(OP_WRITE, SPACE_GLOBAL, OUT_BASE + gy * n + gx))

    r = np.stack([np.ascontiguousarray(x) for x in rows], axis=1)   # (blocks, nrows, 256)
    nr = r.shape[1]
    # (blocks, nrows, 8 warps, 32 lanes) -> (blocks*8 warps, nrows, 32)
    r = r.reshape(blocks, nr, 8, 32).transpose(0, 2, 1, 3).reshape(blocks * 8, nr, 32)
    return make_trace([kernel_from_rows(blocks, 8, 32, r, smem_words=2 * TILE)])


def expected_racy_shared_words(removed: Optional[int]) -> np.ndarray:
    """Closed form: with the barrier after sweep s removed, sweeps s and s+1
    share an epoch; every interior cell of both tiles is written by its own
    thread in one sweep and read by a neighbouring thread in the other."""
    if removed is None or removed >= K_SWEEPS - 1:
        return np.zeros(0, dtype=np.int64)
    ltid = np.arange(256)
    centre = (ltid // T + 1) * H + (ltid % T + 1)
    return np.sort(np.concatenate([A_BASE + centre, B_BASE + centre]))
