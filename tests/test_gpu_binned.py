"""Address-binned replay (csrc/hr_binned.cuh, DESIGN.md §5 "binned replay"):
every global access regrouped per (64 MB shadow bucket, simulated block) in
the block-serial happens-before order, checked bucket by bucket with per-entry
(tid, bc, wc) labels.  Opt-in (HR_OPT_BINNED); the racy set and flags must equal the
oracle's bit for bit: barriers of both kinds, sub-warp masks, clock overflow,
lazy reset, ring overflow, shards, representatives, hot words, and C5's
planted set at full generator settings."""
import random

import numpy as np
import pytest

from tests.test_gpu_parity import _concat, _only_representatives, _random_batch, gpu_set, oracle_set
from tracegen import c4, c5
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu
BINNED = 262144
LAZY = 8192


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("extra", [0, LAZY, 1 | 2])
def test_binned_random_programs(seed, extra):
    tr = _random_batch(700 + seed, 25, max_blocks=6, max_warps=8, max_lanes=32, max_slots=14, n_words=60,
                       spaces=(0,), p_barrier=0.25, p_skip=0.5)
    want = oracle_set(tr)
    assert gpu_set(tr, options=BINNED | extra) == want
    assert gpu_set(tr, options=BINNED | extra, compact=True) == want


def test_binned_hot_words_listings_and_ring_overflow():
    cases = [tp.listing1(3, 2, 32), tp.listing2(8, 4, 32), tp.listing4(2, 2, 32, 40)]
    rng = random.Random(4)
    hot = tp.random_program(rng, max_blocks=8, max_warps=8, max_lanes=32, max_slots=20, n_words=3,
                            spaces=(0,), p_barrier=0.2, n_kernels=3)
    cases.append(hot)
    for tr in cases:
        want = oracle_set(tr)
        assert gpu_set(tr, options=BINNED) == want
        got, fl = gpu_set(tr, options=BINNED, ring_capacity=3)
        assert got == want[0] and fl & ~hr().HR_F_RING_OVERFLOW == want[1]


def test_binned_clock_overflow_and_masks():
    ev = {(0, 0, 0): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)],
          (0, 0, 1): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)]}
    tr = tp.from_thread_events(1, 1, 2, ev)
    assert gpu_set(tr, options=BINNED, bc_bits=2, wc_bits=30) == oracle_set(tr, bc_bits=2, wc_bits=30)
    ev = {(0, 0, l): [tf.W(l)] + [tf.SYNCWARP] * 5 + [tf.R((l + 1) % 4)] for l in range(4)}
    tr = tp.from_thread_events(1, 1, 4, ev)
    assert gpu_set(tr, options=BINNED, bc_bits=29, wc_bits=3) == oracle_set(tr, bc_bits=29, wc_bits=3)
    from tests.test_oracle_pins import _masked_syncwarp_trace
    tr = _masked_syncwarp_trace()
    assert gpu_set(tr, options=BINNED) == oracle_set(tr)


def test_binned_shards_and_representatives():
    h = hr()
    tr = _random_batch(55, 10, max_blocks=4, max_warps=8, max_lanes=32, max_slots=10, n_words=3000, spaces=(0,))
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    for n in (2, 8):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), options=BINNED)
            ck.replay(h.DeviceTrace.from_trace(tr))
            union += [tuple(x) for x in ck.report()[0]]
            ck.close()
        assert sorted(union) == want
    for reps in ((2, 1), (1, 2)):
        assert gpu_set(tr, options=BINNED, representatives=reps) == oracle_set(_only_representatives(tr, *reps))


def test_binned_many_buckets_and_c4():
    """Words spread over several 2^23-word buckets (the bucket-major order and
    the bucket base of each entry), and C4 forced through the binned path."""
    rng = random.Random(8)
    span = 5 << 23
    def ev(b, w, l):
        out = []
        for s in range(6):
            out.append(rng.choice([tf.R, tf.W, tf.A])(rng.choice([rng.randrange(span), rng.randrange(64)])))
            if s == 2:
                out.append(tf.SYNCTHREADS)
        return out
    tr = tf.make_trace([tf.build_kernel(16, 4, 32, ev)])
    want = oracle_set(tr)
    assert len(want[0]) > 10
    assert gpu_set(tr, options=BINNED) == want
    g = c4.Graph(16)
    for racy in (True, False):
        t4 = g.trace(racy)
        assert gpu_set(t4, options=BINNED) == oracle_set(t4)


def test_binned_c5_planted():
    """C5 at 2^10 blocks with a 2^32-word region registered (a 32 GiB shadow,
    512 buckets) equals the planted closed form, over repeated steps with lazy
    reset."""
    h = hr()
    lb = 10
    r32, rop, woff, kd = c5.gpu_trace_c32(lb)
    dt = h.DeviceTrace(None, woff, kd, r32, rop)
    ck = h.Checker(1 << 32, 0, options=h.HR_OPT_LAZY_RESET | BINNED)
    for _ in range(3):
        ck.reset()
        ck.replay(dt)
        raw, fl = ck.report_raw()
        assert fl == 0
        assert [(int(x["word"]), int(x["scope"])) for x in raw] == c5.planted(lb)
    ck.close()
