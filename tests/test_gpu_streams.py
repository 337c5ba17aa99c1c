"""Stream-scheduled replay of barrier-free long-tailed kernels
(csrc/hr_streams.cuh, DESIGN.md §5 "hub fan-out"): the hub warps' accesses are
cut by word hash into helper streams that any CUDA warp replays, longest
first.  Parity with the oracle (bit-exact racy set + scope) on power-law
traces shaped like C4, on hub programs with hot words and every access kind,
under address shards and representative threads, and against the per-block
compacted replay (HR_OPT_NO_STREAMS)."""
import random

import numpy as np
import pytest

import oracle
from tests.test_gpu_parity import gpu_set, oracle_set
from tracegen import c4
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu
NO_STREAMS = 131072


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def hub_trace(seed, blocks=64, warps=8, hubs=3, hub_len=30000, n_words=5000, hot=16, n_kernels=2):
    """Thread-per-item kernels without barriers: every thread does a few
    accesses, `hubs` threads walk long lists (random words, a few hot ones),
    all kinds; several kernels (kernel boundaries order everything)."""
    rng = random.Random(seed)
    kernels = []
    for _ in range(n_kernels):
        hub_threads = {(rng.randrange(blocks), rng.randrange(warps), rng.randrange(32)) for _ in range(hubs)}

        def ev(b, w, l):
            n = hub_len if (b, w, l) in hub_threads else rng.randrange(0, 4)
            out = []
            for _ in range(n):
                word = rng.randrange(hot) if rng.random() < 0.05 else rng.randrange(n_words)
                kind = rng.choice("RRRWA")
                out.append({"R": tf.R, "W": tf.W, "A": tf.A}[kind](word))
            return out
        kernels.append(tf.build_kernel(blocks, warps, 32, ev))
    return tf.make_trace(kernels)


@pytest.mark.parametrize("seed", range(3))
def test_hub_programs_match_oracle(seed):
    tr = hub_trace(seed)
    want = oracle_set(tr)
    assert len(want[0]) > 100
    assert gpu_set(tr) == want
    assert gpu_set(tr, options=NO_STREAMS) == want
    assert gpu_set(tr, compact=True) == want


def test_hub_programs_shards_and_representatives():
    h = hr()
    tr = hub_trace(7)
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    for n in (2, 4, 8):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n))
            ck.replay(h.DeviceTrace.from_trace(tr))
            union += [tuple(x) for x in ck.report()[0]]
            ck.close()
        assert sorted(union) == want
    # representatives: the oracle on the trace restricted to them
    from tests.test_gpu_parity import _only_representatives
    for reps in ((2, 1), (1, 3)):
        assert gpu_set(tr, representatives=reps) == oracle_set(_only_representatives(tr, *reps))


def test_barrier_kernel_falls_back():
    """A long-tailed kernel WITH a __syncwarp row must not take the stream path
    (its count pass cancels the plan): still the oracle's set."""
    rng = random.Random(3)
    blocks, warps = 32, 4
    hub = (3, 1, 7)

    def ev(b, w, l):
        n = 20000 if (b, w, l) == hub else 2
        out = [tf.W(rng.randrange(3000)) for _ in range(n // 2)] + [tf.SYNCWARP] + \
              [tf.R(rng.randrange(3000)) for _ in range(n - n // 2)]
        return out
    tr = tf.make_trace([tf.build_kernel(blocks, warps, 32, ev)])
    assert gpu_set(tr) == oracle_set(tr)


@pytest.mark.parametrize("racy", [True, False])
def test_c4_lv18_streams_vs_oracle(racy):
    g = c4.Graph(18)
    tr = g.trace(racy)
    want = oracle_set(tr)
    assert gpu_set(tr) == want
    assert gpu_set(tr, options=NO_STREAMS) == want
