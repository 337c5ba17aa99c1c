"""Vector-clock race detection along explicit interleavings — TEST INFRASTRUCTURE.

Pure Python, tiny traces only (<= ~8 threads, a handful of events).  Used to
pin hr_oracle.c's static happens-before definition against the classical
dynamic construction (SPEC.md:416-424 ``vclock_check``; FastTrack-style
unbounded history), over every barrier-respecting
interleaving (SPEC.md:159-166 ``enumerate_schedules``).

Semantics of one step of an interleaving (SPEC.md:153 ``run_schedule``):
one event of one runnable thread executes.  A thread reaching
``__syncthreads`` (``__syncwarp``) blocks until every thread of its block
(warp) has reached it; then all are released together and their vector
clocks are joined (the barrier's happens-before edges).
Accesses do not synchronise (atomics included, reading R1).  A ``__syncwarp``
record held by only some lanes of a warp row is ``__syncwarp(mask)`` (PAPER.md:264
"takes a mask argument"): here it synchronises exactly those lanes — the
precise semantics the conservative oracle reading R8 over-approximates.

Decodes the trace records itself (shares no code with the CUDA path).
"""
from __future__ import annotations

import itertools
from typing import Dict, Iterator, List, Optional, Set, Tuple

import numpy as np

Thread = Tuple[int, int, int]          # (block, warp, lane)
Event = Tuple                          # ("acc", space, word, kind) | ("S",) | ("WS",) | ("WS", lanes)


def thread_events(trace) -> List[Dict[Thread, List[Event]]]:
    """Per kernel: each simulated thread's event list, in program order."""
    out = []
    rec = np.asarray(trace.rec, dtype=np.uint64)
    for k in range(trace.kdesc.shape[0]):
        blocks, warps, lanes, _smem, woi = (int(x) for x in trace.kdesc[k, :5])
        tl = int(trace.kdesc[k, 5])              # warp tile (log2 lanes), 0 = whole warps
        th: Dict[Thread, List[Event]] = {}
        for b in range(blocks):
            for w in range(warps):
                gw = b * warps + w
                r0, r1 = int(trace.warp_off[woi + gw]), int(trace.warp_off[woi + gw + 1])
                # per row: the lanes holding a __syncwarp record (the barrier's mask); in a
                # tile kernel each tile's lanes form their own barrier (one __syncwarp(tile
                # mask) per tile)
                ws_mask = {}
                for r in range(r0, r1):
                    m = frozenset(l for l in range(lanes)
                                  if int(rec[r * 32 + l]) & ~(1 << 61) == (3 << 62) | 2)
                    if m and len(m) < lanes:
                        ws_mask[r] = m
                    if m and tl:
                        ws_mask[r] = {l: frozenset(x for x in m if x >> tl == l >> tl) for l in m}
                for l in range(lanes):
                    ev: List[Event] = []
                    for r in range(r0, r1):
                        x = int(rec[r * 32 + l])
                        op, space, word = x >> 62, (x >> 61) & 1, x & ((1 << 61) - 1)
                        if op == 3:
                            if word == 1:
                                ev.append(("S",))
                            elif word == 2:
                                msk = ws_mask.get(r)
                                if isinstance(msk, dict):
                                    msk = msk[l]
                                ev.append(("WS", msk) if msk is not None else ("WS",))
                        else:
                            ev.append(("acc", space, word, op))
                    th[(b, w, l)] = ev
        out.append(th)
    return out


class _Run:
    """Interleaving state machine shared by enumeration and replay."""

    def __init__(self, th: Dict[Thread, List[Event]]):
        self.th = th
        self.ids = sorted(th)
        self.pc = {t: 0 for t in self.ids}
        self.waiting: Dict[Thread, Event] = {}

    def runnable(self) -> List[Thread]:
        return [t for t in self.ids if t not in self.waiting and self.pc[t] < len(self.th[t])]

    def members(self, t: Thread, e: Event) -> List[Thread]:
        b, w, _ = t
        if e[0] == "S":
            return [u for u in self.ids if u[0] == b]
        if len(e) > 1:                                  # __syncwarp(mask): the masked lanes
            return [u for u in self.ids if u[0] == b and u[1] == w and u[2] in e[1]]
        return [u for u in self.ids if u[0] == b and u[1] == w]

    def exec(self, t: Thread):
        """Execute t's next event; returns (event, released_group or None)."""
        e = self.th[t][self.pc[t]]
        if e[0] in ("S", "WS"):
            self.waiting[t] = e
            grp = self.members(t, e)
            if all(self.waiting.get(u) == e for u in grp):
                for u in grp:
                    del self.waiting[u]
                    self.pc[u] += 1
                return e, grp
            return e, None
        self.pc[t] += 1
        return e, None

    def snapshot(self):
        return dict(self.pc), dict(self.waiting)

    def restore(self, snap):
        self.pc, self.waiting = dict(snap[0]), dict(snap[1])


def enumerate_schedules(th: Dict[Thread, List[Event]], cap: Optional[int] = None) -> Iterator[List[Thread]]:
    """Every maximal barrier-respecting interleaving, as a list of thread picks
    (tree enumeration over runnable sets, threads in id order)."""
    run = _Run(th)
    count = [0]

    def rec(prefix):
        if cap is not None and count[0] >= cap:
            return
        rs = run.runnable()
        if not rs:
            count[0] += 1
            yield list(prefix)
            return
        for t in rs:
            snap = run.snapshot()
            run.exec(t)
            prefix.append(t)
            yield from rec(prefix)
            prefix.pop()
            run.restore(snap)

    yield from rec([])


def _leq(a: Dict[Thread, int], b: Dict[Thread, int]) -> bool:
    return all(v <= b.get(k, 0) for k, v in a.items())


def _conflict(k1: int, k2: int) -> bool:
    return not ((k1 == 0 and k2 == 0) or (k1 == 2 and k2 == 2))


def _class(k1: int, k2: int) -> int:
    """bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R (kinds: 0 R, 1 W, 2 A)."""
    s = {k1, k2}
    if s == {1}:
        return 1
    if s == {0, 1}:
        return 2
    if s == {1, 2}:
        return 4
    if s == {0, 2}:
        return 8
    return 0


def vclock_race_classes(th: Dict[Thread, List[Event]], schedule: List[Thread]) -> Dict[Tuple, int]:
    """Like vclock_races, but {address: class mask of all racing pairs seen}."""
    return vclock_races(th, schedule, classes=True)


def vclock_races(th: Dict[Thread, List[Event]], schedule: List[Thread], classes: bool = False) -> Dict[Tuple, int]:
    """Racy addresses along one interleaving: {(space, ablock, word): scope}.

    Each thread keeps a vector clock; an access races with any earlier access
    to the same address by another thread with a conflicting kind whose clock
    is not <= the current thread's clock (unbounded history)."""
    run = _Run(th)
    vc: Dict[Thread, Dict[Thread, int]] = {t: {t: 1} for t in th}
    hist: Dict[Tuple, List[Tuple[Thread, int, Dict[Thread, int]]]] = {}
    races: Dict[Tuple, int] = {}
    for t in schedule:
        e, grp = run.exec(t)
        if e[0] == "acc":
            _, space, word, kind = e
            addr = (space, t[0] if space == 1 else 0xFFFFFFFF, word)
            for (u, k2, c2) in hist.get(addr, []):
                if u != t and _conflict(kind, k2) and not _leq(c2, vc[t]):
                    if classes:
                        races[addr] = races.get(addr, 0) | _class(kind, k2)
                    else:
                        races[addr] = max(races.get(addr, 0), 2 if u[0] != t[0] else 1)
            hist.setdefault(addr, []).append((t, kind, dict(vc[t])))
            vc[t][t] = vc[t].get(t, 0) + 1
        elif grp is not None:
            j: Dict[Thread, int] = {}
            for u in grp:
                for k, v in vc[u].items():
                    j[k] = max(j.get(k, 0), v)
            for u in grp:
                vc[u] = dict(j)
                vc[u][u] = vc[u].get(u, 0) + 1
    return races


def static_races_of(th: Dict[Thread, List[Event]]) -> Dict[Tuple, int]:
    """Convenience: the union over one arbitrary complete interleaving — only
    meaningful together with schedule-independence checks in tests."""
    sched = next(enumerate_schedules(th))
    return vclock_races(th, sched)


def project(th: Dict[Thread, List[Event]], keep: Set[Thread]) -> Dict[Thread, List[Event]]:
    """Two-thread projection: drop every other thread's
    events; barriers then synchronise only the kept threads."""
    return {t: list(ev) for t, ev in th.items() if t in keep}


def thread_pairs(th: Dict[Thread, List[Event]]):
    return itertools.combinations(sorted(th), 2)
