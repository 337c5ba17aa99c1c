"""Sticky device conditions (include/hr.h HR_F_*) and the control-record edge
cases, GPU vs oracle through the C ABI (VERDICT r1 "weak" 2):

* a control code the trace format does not define (word > 2) is no barrier:
  both sides set HR_F_MODEL_VIOLATION and advance no clock, so the racy set
  is the oracle's (which differs from the set with a __syncwarp there);
* a global access outside the registered region is not checked and sets
  HR_F_UNMONITORED: the set is the oracle's on the monitored words only;
* a barrier row on which the warp's lanes disagree sets
  HR_F_BARRIER_DIVERGENCE on both sides (its racy set is unspecified: CUDA
  leaves divergent barriers undefined).
Every replay kernel (row 64/32 registers, pooled, compacted, block-serial,
run-time options) and every record encoding (U64, C32, PACKED).
"""
import numpy as np
import pytest

import oracle
from tests.helpers import filter_trace_words
from tests.test_gpu_parity import gpu_set, oracle_set
from tracegen import format as tf

pytestmark = pytest.mark.gpu

KERNELS = [16, 65536, 32, 256, 32 | 16384, 4096]
UNDEFINED = tf.encode(tf.OP_CTRL, 0, 3)
UNDEFINED_BIG = tf.encode(tf.OP_CTRL, 0, 12345)


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def _undefined_code_trace(code):
    """2 blocks x 2 warps x 32 lanes.  Lane l of warp 0 writes word l (global)
    and shared word l; a uniform row of `code` in every warp; then lane l of
    warp 0 reads word (l+1) % 32 in both spaces.  Were `code` a __syncwarp,
    the same-warp pairs would be ordered; it is no barrier, so they race."""
    rows = np.full((4, 3, 32), tf.NOP, dtype=np.uint64)
    for b in range(2):
        w0 = b * 2
        for l in range(32):
            rows[w0, 0, l] = tf.W(l + 100 * b, 1 if l % 2 else 0)
            rows[w0, 2, l] = tf.R((l + 1) % 32 + 100 * b, 1 if (l + 1) % 2 else 0)
        rows[w0, 1, :] = code
        rows[w0 + 1, 1, :] = code
    return tf.make_trace([tf.kernel_from_rows(2, 2, 32, rows, smem_words=200)])


@pytest.mark.parametrize("code", [UNDEFINED, UNDEFINED_BIG])
@pytest.mark.parametrize("options", KERNELS)
def test_undefined_control_code(code, options):
    tr = _undefined_code_trace(code)
    want, wfl = oracle_set(tr)
    assert wfl == hr().HR_F_MODEL_VIOLATION and len(want) == 64
    # with a real __syncwarp the set is empty: the code must not act as one
    assert oracle_set(_undefined_code_trace(tf.SYNCWARP))[0] == []
    assert gpu_set(tr, options=options) == (want, wfl)


@pytest.mark.parametrize("fmt", ["c32", "packed"])
def test_undefined_control_code_encodings(fmt):
    tr = _undefined_code_trace(UNDEFINED)
    want = oracle_set(tr)
    assert gpu_set(tr, compact=fmt == "c32", packed=fmt == "packed") == want


@pytest.mark.parametrize("options", KERNELS)
def test_unmonitored_global_words(options):
    """Register words [0, 48) only.  Block 0 lane l writes words l and 63 - l,
    block 1 lane l reads word l: words 0..31 race (GRID), words 32..63 are
    written once; 48..63 are outside the region (flagged, not checked)."""
    h = hr()
    ev = {}
    for l in range(32):
        ev[(0, 0, l)] = [tf.W(l), tf.W(63 - l)]
        ev[(1, 0, l)] = [tf.R(l)]
    from tracegen import programs as tp
    tr = tp.from_thread_events(2, 1, 32, ev)
    ck = h.Checker(48, 0, options=options)
    ck.replay(h.DeviceTrace.from_trace(tr))
    races, fl, _ = ck.report()
    ck.close()
    assert fl == h.HR_F_UNMONITORED
    want = oracle.check(filter_trace_words(tr, set(range(48))))
    assert [tuple(r) for r in races] == [tuple(r) for r in want.races]
    assert len(want.races) == 32 and want.flags == 0


@pytest.mark.parametrize("options", KERNELS)
def test_barrier_divergence_flag_matches_oracle(options):
    # lane 0 meets a __syncthreads (resp. __syncwarp) that lanes 1 and 2 do not
    for bar in (tf.SYNCTHREADS, tf.SYNCWARP):
        rows = np.full((1, 2, 32), tf.NOP, dtype=np.uint64)
        rows[0, 0, 0] = bar
        rows[0, 1, 1] = tf.W(0)
        rows[0, 1, 2] = tf.W(0)
        tr = tf.make_trace([tf.kernel_from_rows(1, 1, 3, rows)])
        _, wfl = oracle_set(tr)
        # a __syncthreads on some lanes is divergence; a __syncwarp on some lanes is a
        # sub-warp mask (reading R8: model violation, no edge)
        assert wfl == (hr().HR_F_BARRIER_DIVERGENCE if bar == tf.SYNCTHREADS else hr().HR_F_MODEL_VIOLATION)
        _, fl = gpu_set(tr, options=options)
        assert fl == wfl


def test_mixed_barrier_and_undefined_row_flags():
    """Lanes split between __syncwarp and an undefined code: both flags."""
    rows = np.full((1, 1, 32), tf.SYNCWARP, dtype=np.uint64)
    rows[0, 0, 5] = UNDEFINED
    tr = tf.make_trace([tf.kernel_from_rows(1, 1, 32, rows)])
    _, wfl = oracle_set(tr)
    h = hr()
    assert wfl == h.HR_F_MODEL_VIOLATION | h.HR_F_BARRIER_DIVERGENCE
    for options in KERNELS:
        assert gpu_set(tr, options=options)[1] == wfl


# ---- sub-warp __syncwarp(mask) (reading R8: model violation, no happens-before edge) ----

def _masked_rows_trace(seed):
    """Random single-warp-row programs where some __syncwarp rows are held by
    a random subset of lanes (a sub-warp mask)."""
    import random
    rng = random.Random(seed)
    nw, nrows = 4, 10
    rows = np.full((2 * nw, nrows, 32), tf.NOP, dtype=np.uint64)
    for w in range(2 * nw):
        for r in range(nrows):
            if rng.random() < 0.3:
                lanes = [l for l in range(32) if rng.random() < 0.5] if rng.random() < 0.6 else list(range(32))
                for l in lanes:
                    rows[w, r, l] = tf.SYNCWARP
            else:
                for l in range(32):
                    if rng.random() < 0.6:
                        rows[w, r, l] = rng.choice([tf.R, tf.W, tf.A])(rng.randrange(40), rng.randrange(2))
    return tf.make_trace([tf.kernel_from_rows(2, nw, 32, rows, smem_words=40)])


@pytest.mark.parametrize("options", KERNELS)
def test_masked_syncwarp_replay_matches_oracle(options):
    from tests.test_oracle_pins import _masked_syncwarp_trace
    tr = _masked_syncwarp_trace()
    want = oracle_set(tr)
    assert want[1] == hr().HR_F_MODEL_VIOLATION and len(want[0]) == 2
    assert gpu_set(tr, options=options) == want
    for seed in range(3):
        tr = _masked_rows_trace(seed)
        want = oracle_set(tr)
        assert want[1] & hr().HR_F_MODEL_VIOLATION
        assert gpu_set(tr, options=options) == want, seed


def test_masked_syncwarp_online():
    """hr_syncwarp_mask in a real kernel: the racy set equals the oracle's on
    the same access stream (lanes 0..15 hold the masked __syncwarp row)."""
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    rows = np.full((1, 3, 32), tf.NOP, dtype=np.uint64)
    for l in range(32):
        rows[0, 0, l] = tf.W(l)
        rows[0, 2, l] = tf.R((l & 16) | ((l + 1) & 15))
    rows[0, 1, :16] = tf.SYNCWARP
    tr = tf.make_trace([tf.kernel_from_rows(1, 1, 32, rows)])
    want = oracle_set(tr)
    assert want[1] == h.HR_F_MODEL_VIOLATION and len(want[0]) == 32
    data = torch.zeros(64, dtype=torch.int32, device="cuda")
    ck = h.Checker(32, 0)
    online.masked_sync(ck.ctx, data)
    races, flags, _ = ck.report()
    ck.close()
    assert ([tuple(r) for r in races], flags) == want
