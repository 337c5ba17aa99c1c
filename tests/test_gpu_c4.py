"""C4 (RMAT BFS levels + degree histogram) parity on the GPU.

2^20 vertices: GPU == oracle on every address, racy and race-free variants.
2^24 vertices (the BASELINE size): GPU == oracle on a seeded sample of words
(the oracle replays the sampled words' full access histories: words are
independent FSMs), plus the race-free variant must report nothing."""
import random

import numpy as np
import pytest

import oracle
from tests.helpers import filter_trace_words
from tracegen import c4

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


@pytest.mark.parametrize("racy", [True, False])
def test_c4_lv20_full_parity(racy):
    g = c4.Graph(20)
    tr = g.trace(racy)
    got, flags = hr().check_trace(tr, ring_capacity=1 << 22)
    want = oracle.check(tr)
    assert flags == want.flags == 0
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races]
    assert (len(got) > 0) == racy


def test_c4_full_size_sampled():
    h = hr()
    g = c4.Graph(24)
    tr = g.trace(True)
    got, flags = h.check_trace(tr, ring_capacity=1 << 24)
    assert flags == 0
    got_set = {(r.word, r.scope) for r in got}
    rng = random.Random(11)
    sample = set(rng.sample(range(g.n), 3000)) | set(range(64)) | set(range(g.n, g.n + 1024))
    ref = oracle.check(filter_trace_words(tr, sample))
    want = {(r.word, r.scope) for r in ref.races}
    assert {x for x in got_set if x[0] in sample} == want
    assert len(want) > 100
    free = g.trace(False)
    got_free, flags = h.check_trace(free, ring_capacity=1 << 20)
    assert got_free == [] and flags == 0
