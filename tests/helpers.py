"""Test-side helpers: per-address access lists, happens-before linear
extensions, and a literal Algorithm-1 simulator over a given FSM table.

The simulator follows PAPER.md:684-718 (Algorithm 1, ``UpdateShadow``)
step by step for ONE word and one commit order: unpack the stored
(state, tid, bc, wc), ``compareTids`` -> relation, ``checkSync`` -> sync
status, ``getTrans`` -> flat index,
lookup, pack.  It is used to verify the product's generated table against
the oracle on the CPU; it is not product code.
"""
from __future__ import annotations

import itertools
from typing import Dict, Iterator, List, Tuple

from oracle.vclock import thread_events

REL_S, REL_W, REL_B, REL_G = 0, 1, 2, 3
US, WS, BS = 0, 1, 2
RACE_BLOCK, RACE_GRID = 30, 31


class Acc(Tuple):
    pass


def accesses_by_address(trace) -> Dict[Tuple, List[Tuple]]:
    """{(kernel, space, ablock, word): [(thread, pidx, bc, wc, kind), ...]}"""
    out: Dict[Tuple, List[Tuple]] = {}
    for k, th in enumerate(thread_events(trace)):
        for t, evs in th.items():
            bc = wc = 0
            for p, e in enumerate(evs):
                if e[0] == "S":
                    bc += 1
                elif e[0] == "WS":
                    wc += 1
                else:
                    _, space, word, kind = e
                    key = (k, space, t[0] if space == 1 else 0xFFFFFFFF, word)
                    out.setdefault(key, []).append((t, p, bc, wc, kind))
    return out


def hb(a, b) -> bool:
    """a happens-before b (program order, block epochs, warp epochs)."""
    (ta, pa, bca, wca, _), (tb, pb, bcb, wcb, _) = a, b
    if ta == tb:
        return pa < pb
    if ta[0] != tb[0]:
        return False
    if bca != bcb:
        return bca < bcb
    if ta[1] != tb[1]:
        return False
    return wca < wcb


def linear_extensions(accs: List[Tuple], cap: int = 5000) -> Iterator[List[Tuple]]:
    n = len(accs)
    preds = [[j for j in range(n) if hb(accs[j], accs[i])] for i in range(n)]
    done = [False] * n
    order: List[int] = []
    count = [0]

    def rec():
        if count[0] >= cap:
            return
        if len(order) == n:
            count[0] += 1
            yield [accs[i] for i in order]
            return
        for i in range(n):
            if not done[i] and all(done[j] for j in preds[i]):
                done[i] = True
                order.append(i)
                yield from rec()
                order.pop()
                done[i] = False

    yield from rec()


def compare_tids(t, o) -> int:
    if t == o:
        return REL_S
    if t[0] == o[0] and t[1] == o[1]:
        return REL_W
    if t[0] == o[0]:
        return REL_B
    return REL_G


def check_sync(rel, bc, obc, wc, owc) -> int:
    if rel != REL_G and bc > obc:
        return BS
    if rel in (REL_S, REL_W) and wc > owc:
        return WS
    return US


def run_word(table: bytes, commits: List[Tuple]) -> Tuple[int, List[int]]:
    """Algorithm 1 over one word; returns (final state, states after each commit)."""
    state, otid, obc, owc = 0, None, 0, 0
    trail = []
    for (t, _p, bc, wc, kind) in commits:
        if state == 0:
            rel, sync = REL_S, US          # INIT ignores the label
        else:
            rel = compare_tids(t, otid)
            sync = check_sync(rel, bc, obc, wc, owc)
        state = table[(state << 6) | (kind << 4) | (sync << 2) | rel]
        otid, obc, owc = t, bc, wc
        trail.append(state)
    return state, trail


def scope_of(state: int) -> int:
    return {RACE_BLOCK: 1, RACE_GRID: 2}.get(state, 0)


def filter_trace_words(trace, words, space: int = 0):
    """Sampled-output check support: a copy of `trace` in which every access
    record not touching one of `words` (in `space`) becomes a NOP; barrier rows
    are kept, so the sampled words keep their exact access history."""
    import numpy as np
    rec = trace.rec.copy()
    op = rec >> np.uint64(62)
    sp = (rec >> np.uint64(61)) & np.uint64(1)
    w = rec & np.uint64((1 << 61) - 1)
    ws = np.asarray(sorted(words), dtype=np.int64)
    table = np.zeros(int(ws.max()) + 2, dtype=bool)        # O(n) lookup, not np.isin's O(n*k)
    table[ws] = True
    idx = np.minimum(w, np.uint64(table.shape[0] - 1)).astype(np.int64)
    keep = (op == 3) | ((sp == space) & table[idx] & (w < np.uint64(table.shape[0] - 1)))
    rec[~keep] = np.uint64(3 << 62)
    return type(trace)(rec, trace.kdesc.copy(), trace.warp_off.copy())
