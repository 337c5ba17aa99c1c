"""Warp tiles (reading R8, exact part): a kernel that declares warp tiles of
2^tile_log2 lanes (kdesc[5]; cooperative-groups ``tiled_partition<T>().sync()``
= ``__syncwarp(tile mask)``) has each tile-aligned
``__syncwarp`` row replayed as one barrier per tile, exactly; the "Warp"
relation is "same tile".  GPU vs oracle through the C ABI on random tile
programs (both spaces, every encoding, the replay kernels a tile kernel may
take), the hand-pinned example of tests/test_oracle_pins.py, and the online
path (hr_set_warp_tile + hr_syncwarp_mask).
"""
import random

import numpy as np
import pytest

import oracle
from tests.test_gpu_parity import gpu_set, oracle_set
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu

# row 48/64 registers, forced pool (a tile kernel takes the row kernel), no
# coalescing, block-serial request (ignored for tiles), SMEM32, no fast exits
OPTIONS = [0, 16, 65536, 32, 256, 16384, 4096, 8192, 2048]


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def test_tile_example_exact():
    from tests.test_oracle_pins import _tile_example
    tr = _tile_example(True)
    want = oracle_set(tr)
    assert want[1] == 0 and len(want[0]) == 1          # word 1 only (pinned in test_oracle_pins)
    for o in OPTIONS:
        assert gpu_set(tr, options=o) == want, o
    und = _tile_example(False)
    assert gpu_set(und) == oracle_set(und)


@pytest.mark.parametrize("options", OPTIONS)
def test_random_tile_programs(options):
    rng = random.Random(7000 + options)
    for i in range(12):
        tl = rng.choice([1, 2, 3, 4])
        tr = tp.random_tile_program(rng, blocks=rng.randint(1, 3), warps=rng.randint(1, 3),
                                    lanes=rng.choice([32, 32, 24, 8]), tile_log2=tl, slots=rng.randint(4, 16),
                                    n_words=rng.choice([4, 24, 64]), spaces=(0, 1))
        want = oracle_set(tr)
        assert want[1] == 0
        assert gpu_set(tr, options=options) == want, (i, tl)


@pytest.mark.parametrize("fmt", ["c32", "packed"])
def test_random_tile_programs_encodings(fmt):
    rng = random.Random(71)
    for i in range(8):
        tr = tp.random_tile_program(rng, blocks=2, warps=2, lanes=32, tile_log2=rng.choice([1, 2, 3, 4]), slots=12,
                                    n_words=32, spaces=(0, 1))
        want = oracle_set(tr)
        assert gpu_set(tr, compact=fmt == "c32", packed=fmt == "packed") == want, i


def test_tile_kernel_rejected_by_pooled_format():
    rng = random.Random(3)
    tr = tp.random_tile_program(rng, blocks=1, warps=1, lanes=32, tile_log2=2, slots=4, n_words=4)
    with pytest.raises(hr().HiraceError):
        hr().check_trace(tr, pooled=True)


def test_tile_vs_whole_warp_differs():
    """The tile declaration matters: with tiles, a full __syncwarp row is one
    barrier per tile and does not order lanes of different tiles (same-block
    Block relation, same block epoch), so a cross-tile pair around it races;
    undeclared, the same row is a warp barrier and orders it."""
    rows = np.full((1, 3, 32), tf.NOP, dtype=np.uint64)
    rows[0, 0, 0] = tf.W(5)
    rows[0, 1, :] = tf.SYNCWARP
    rows[0, 2, 8] = tf.R(5)
    k = tf.kernel_from_rows(1, 1, 32, rows)
    k.tile_log2 = 2
    tiled = tf.make_trace([k])
    k2 = tf.kernel_from_rows(1, 1, 32, rows)
    plain = tf.make_trace([k2])
    assert len(oracle_set(tiled)[0]) == 1 and oracle_set(plain) == ([], 0)
    for o in (0, 16, 65536):
        assert gpu_set(tiled, options=o) == oracle_set(tiled)
        assert gpu_set(plain, options=o) == ([], 0)


def test_tile_syncwarp_online():
    """hr_syncwarp_mask over whole tiles in a real kernel (hr_set_warp_tile):
    the racy set equals the oracle's on the same access stream declared as a
    tile kernel, and carries no model-violation flag."""
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    rows = np.full((1, 3, 32), tf.NOP, dtype=np.uint64)
    for l in range(32):
        rows[0, 0, l] = tf.W(l)
        rows[0, 2, l] = tf.R((l & 16) | ((l + 1) & 15))
    rows[0, 1, :16] = tf.SYNCWARP
    k = tf.kernel_from_rows(1, 1, 32, rows)
    k.tile_log2 = 4
    tr = tf.make_trace([k])
    want = oracle_set(tr)
    assert want[1] == 0 and len(want[0]) == 16          # tile 0 ordered, tile 1 not
    data = torch.zeros(64, dtype=torch.int32, device="cuda")
    ck = h.Checker(32, 0)
    h.hr_set_warp_tile(ck.ctx, 4)
    online.masked_sync(ck.ctx, data)
    races, flags, _ = ck.report()
    ck.close()
    assert ([tuple(r) for r in races], flags) == want
