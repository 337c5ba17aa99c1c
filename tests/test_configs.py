"""CPU-side checks of the BASELINE configs' generators against the oracle:
C2 injected-bug labels, C3 and C5 closed forms, C5 shard partition."""
import numpy as np
import pytest

import oracle
from tracegen import c5, stencil, suite
from paper_2401_04701_b200.multigpu import shard_owner


@pytest.fixture(scope="module")
def c2_cases():
    return suite.suite()


def test_c2_suite_shape(c2_cases):
    # "580 distinct CUDA programs ... 346 contained data races"
    assert 560 <= len(c2_cases) <= 620
    assert len(suite.PATTERNS) == 21
    n_racy = sum(c.racy for c in c2_cases)
    assert 0.4 * len(c2_cases) < n_racy < 0.7 * len(c2_cases)


def test_c2_labels_agree_with_oracle(c2_cases):
    for c in c2_cases:
        res = oracle.check(c.trace)
        assert bool(res.races) == c.racy, c.name
        assert res.flags == 0, c.name


def test_c3_closed_form_small_grid():
    for removed in (None, 0, 20, 40):
        tr = stencil.stencil_trace(removed=removed, n=64)
        res = oracle.check(tr)
        exp = list(stencil.expected_racy_shared_words(removed))
        blocks = {r.block for r in res.races}
        if not exp:
            assert res.races == []
            continue
        assert blocks == set(range(16))
        for b in blocks:
            assert [r.word for r in res.races if r.block == b] == exp
        assert all(r.space == 1 and r.scope == oracle.SCOPE_BLOCK for r in res.races)


def test_c3_access_count():
    tr = stencil.stencil_trace(removed=None, n=64)
    # 648 loads+stores of the halo, 42 x 6 x 256 sweep accesses, 2 x 256 final, per block
    assert tr.n_accesses() == 16 * (648 + 42 * 6 * 256 + 2 * 256)


@pytest.mark.parametrize("lb", [1, 3, 5])
def test_c5_racy_set_is_planted(lb):
    tr = c5.cpu_trace(lb)
    res = oracle.check(tr)
    assert [(r.word, r.scope) for r in res.races] == c5.planted(lb)
    assert res.n_accesses == c5.n_accesses(lb)
    op = tr.rec >> np.uint64(62)
    acc = op != 3
    frac = [float(np.mean(op[acc] == k)) for k in range(3)]
    assert abs(frac[0] - 0.70) < 0.03 and abs(frac[1] - 0.20) < 0.03 and abs(frac[2] - 0.10) < 0.02


@pytest.mark.parametrize("n,g", [(2, 9), (4, 9), (8, 9), (8, 5), (8, 0), (4, 3), (4, 12)])
def test_c5_shards_partition_the_racy_set(n, g):
    lb = 4
    full = [(r.word, r.scope) for r in oracle.check(c5.cpu_trace(lb)).races]
    union = []
    for r in range(n):
        sh = c5.cpu_trace(lb, rank=r, nshard=n, granule_log2=g)
        got = oracle.check(sh).races
        assert all(shard_owner(x.word >> g, n) == r for x in got)
        union += [(x.word, x.scope) for x in got]
    assert sorted(union) == full


@pytest.mark.parametrize("n,g", [(8, 9), (8, 5), (4, 0)])
def test_c5_shard_records_follow_the_owner_function(n, g):
    """The C generator's partition (tracegen/c5gen.h) is hr_shard_owner: every
    access record of shard r has its granule owned by r, the shards together
    hold every access of the full trace, and no rank is starved (the stripe
    rotation spreads a block's warps over the ranks)."""
    lb = 3
    full = c5.cpu_trace(lb)
    fw = full.rec[(full.rec >> np.uint64(62)) != 3] & np.uint64((1 << 61) - 1)
    counts = []
    for r in range(n):
        sh = c5.cpu_trace(lb, rank=r, nshard=n, granule_log2=g)
        acc = sh.rec[(sh.rec >> np.uint64(62)) != 3] & np.uint64((1 << 61) - 1)
        assert np.all(shard_owner(acc >> np.uint64(g), n) == r)
        counts.append(len(acc))
    assert sum(counts) == len(fw)
    assert min(counts) > 0.6 * len(fw) / n
