"""Hybrid binned replay (csrc/hr_hybrid.cuh, HR_OPT_HYBRID): the row replay
appends the accesses of the binned shadow buckets to (bucket, block) runs in
happens-before order, and a bucket-major pass checks them.  The racy set and
the flags must equal the oracle's bit for bit: barriers of both kinds,
sub-warp masks, lazy reset, ring overflow, shards, representatives, hot
words, shared + global kernels, many buckets, and C5's planted set with the
buckets chosen by the scatter rule."""
import random

import pytest

from tests.test_gpu_parity import _only_representatives, _random_batch, gpu_set, oracle_set
from tracegen import c5
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu
HYB = 1048576
ALL = 2097152
LAZY = 8192
ROW_NARROW, ROW_WIDE = 65536, 512


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("extra", [0, LAZY, ROW_WIDE, ROW_NARROW | LAZY])
def test_hybrid_random_programs(seed, extra):
    tr = _random_batch(760 + seed, 25, max_blocks=6, max_warps=8, max_lanes=32, max_slots=14, n_words=60,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    want = oracle_set(tr)
    assert gpu_set(tr, options=HYB | ALL | extra) == want
    assert gpu_set(tr, options=HYB | ALL | extra, compact=True) == want


def test_hybrid_hot_words_listings_and_ring_overflow():
    cases = [tp.listing1(3, 2, 32), tp.listing2(8, 4, 32), tp.listing4(2, 2, 32, 40)]
    rng = random.Random(14)
    cases.append(tp.random_program(rng, max_blocks=8, max_warps=8, max_lanes=32, max_slots=20, n_words=3,
                                   spaces=(0,), p_barrier=0.2, n_kernels=3))
    for tr in cases:
        want = oracle_set(tr)
        assert gpu_set(tr, options=HYB | ALL) == want
        got, fl = gpu_set(tr, options=HYB | ALL, ring_capacity=3)
        assert got == want[0] and fl & ~hr().HR_F_RING_OVERFLOW == want[1]


def test_hybrid_masks_and_clock_fallback():
    from tests.test_oracle_pins import _masked_syncwarp_trace
    tr = _masked_syncwarp_trace()
    assert gpu_set(tr, options=HYB | ALL) == oracle_set(tr)
    # clocks that overflow: the kernel is replayed row by row (exact counts need no overflow)
    ev = {(0, 0, 0): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)],
          (0, 0, 1): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)]}
    tr = tp.from_thread_events(1, 1, 2, ev)
    assert gpu_set(tr, options=HYB | ALL, bc_bits=2, wc_bits=30) == oracle_set(tr, bc_bits=2, wc_bits=30)
    # more block barriers than an entry holds (bc > 127): row replay
    ev = {(b, 0, l): [tf.W(l)] + [tf.SYNCTHREADS] * 130 + [tf.R((l + 1) % 4)] for b in range(2) for l in range(4)}
    tr = tp.from_thread_events(2, 1, 4, ev)
    assert gpu_set(tr, options=HYB | ALL) == oracle_set(tr)


def test_hybrid_shards_and_representatives():
    h = hr()
    tr = _random_batch(65, 10, max_blocks=4, max_warps=8, max_lanes=32, max_slots=10, n_words=3000, spaces=(0,))
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    for n in (2, 8):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), options=HYB | ALL)
            ck.replay(h.DeviceTrace.from_trace(tr))
            union += [tuple(x) for x in ck.report()[0]]
            ck.close()
        assert sorted(union) == want
    for reps in ((2, 1), (1, 2)):
        assert gpu_set(tr, options=HYB | ALL, representatives=reps) == oracle_set(_only_representatives(tr, *reps))


def test_hybrid_many_buckets():
    """Words spread over several 2^22-word buckets and hot low words, both
    barrier kinds: bucket-major runs, bucket bases, runs spanning chunks."""
    rng = random.Random(18)
    span = 7 << 22
    def ev(b, w, l):
        out = []
        for s in range(8):
            out.append(rng.choice([tf.R, tf.W, tf.A])(rng.choice([rng.randrange(span), rng.randrange(64)])))
            if s == 2:
                out.append(tf.SYNCTHREADS)
            if s == 5:
                out.append(tf.SYNCWARP)
        return out
    tr = tf.make_trace([tf.build_kernel(64, 4, 32, ev), tf.build_kernel(8, 8, 32, ev)])
    want = oracle_set(tr)
    assert len(want[0]) > 10
    for extra in (0, LAZY):
        assert gpu_set(tr, options=HYB | ALL | extra) == want
        assert gpu_set(tr, options=HYB | ALL | extra, compact=True) == want


@pytest.mark.parametrize("lb", [8, 11])
def test_hybrid_c5_planted(lb):
    """C5 (device generator, C32): the scatter rule bins the random-read
    buckets; the set is the planted one (closed form), repeated replays on one
    ctx with lazy reset."""
    h = hr()
    r32, rop, woff, kd = c5.gpu_trace_c32(lb)
    dt = h.DeviceTrace(None, woff, kd, r32, rop)
    ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 16, options=HYB | LAZY)
    for _ in range(3):
        ck.reset(); ck.replay(dt)
        raw, fl = ck.report_raw()
        assert fl == 0
        assert [(int(r["word"]), int(r["scope"])) for r in raw] == c5.planted(lb)
    ck.close()
