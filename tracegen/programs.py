"""Seeded synthetic trace generators — INPUT ONLY (no method arithmetic).

* The paper's litmus kernels (Listings 1, 2, 4) as traces.
* C1: the single-warp shared-memory tree reduction (BASELINE.json configs[0]).
* Random barrier-uniform programs for the exhaustive / differential families
  (SPEC.md:87-95 ``generate_random_program``).

Expected verdicts are NOT computed here: they live in tests (closed forms,
cited) or come from ``oracle/``.
"""
from __future__ import annotations

import random
from typing import List, Optional, Sequence

from .format import (A, R, W, NOP, SYNCTHREADS, SYNCWARP, SPACE_GLOBAL, SPACE_SHARED,
                     Trace, build_kernel, kernel_from_rows, make_trace, single_kernel)

# ---------------------------------------------------------------------------
# Paper listings
# ---------------------------------------------------------------------------


def listing1(blocks: int, warps: int, lanes: int) -> Trace:
    """``race_noSync``: every thread ``val = data[0]; data[0] = i + val``."""
    return single_kernel(blocks, warps, lanes, lambda b, w, l: [R(0), W(0)])


def listing2(blocks: int, warps: int, lanes: int) -> Trace:
    """``race_blockSync``: ``val = data[0]; __syncthreads();
    if (tid > 0) data[tid-1] = tid;`` with ``tid = threadIdx.x``."""
    def ev(b, w, l):
        tid = w * lanes + l
        e = [R(0), SYNCTHREADS]
        if tid > 0:
            e.append(W(tid - 1))
        return e
    return single_kernel(blocks, warps, lanes, ev)


def listing4(blocks: int, warps: int, lanes: int, length: int) -> Trace:
    """``multiRead_Race``: ``if (tid < len-2) { s = data[tid];
    s += data[tid+1]; data[tid+1] = s; }`` with ``tid = threadIdx.x``."""
    def ev(b, w, l):
        tid = w * lanes + l
        if tid < length - 2:
            return [R(tid), R(tid + 1), W(tid + 1)]
        return []
    return single_kernel(blocks, warps, lanes, ev)


# ---------------------------------------------------------------------------
# C1: shared-memory tree reduction, 1 block x 32 threads (BASELINE configs[0])
# ---------------------------------------------------------------------------

C1_STEPS = (128, 64, 32, 16, 8, 4, 2, 1)
C1_N = 256
C1_ROUNDS = 8


def c1_tree_reduction(removed: Optional[object] = 32, rounds: int = C1_ROUNDS,
                      n: int = C1_N, lanes: int = 32) -> Trace:
    """Tree reduction over ``__shared__ int s[n]`` by one warp.

    Per round: lane loads ``in[r*n + i]`` (global read) into ``s[i]`` (shared
    write) for ``i = lane (mod 32)``; ``__syncthreads``; for ``s`` in
    128..1: for ``i < s`` with ``i = lane (mod 32)``: read ``s[i]``, read
    ``s[i+s]``, write ``s[i]``, then ``__syncthreads``; finally lane 0 reads
    ``s[0]`` and writes ``out[r]`` (global word ``rounds*n + r``);
    ``__syncthreads``.

    ``removed`` selects the barrier to drop: ``None`` (race-free), ``'load'``,
    or one of the step sizes; it is dropped in every round.
    """
    out_base = rounds * n

    def ev(b, w, lane):
        e: List[int] = []
        for r in range(rounds):
            for i in range(lane, n, lanes):
                e += [R(r * n + i), W(i, SPACE_SHARED)]
            if removed != "load":
                e.append(SYNCTHREADS)
            for s in C1_STEPS:
                for i in range(lane, s, lanes):
                    e += [R(i, SPACE_SHARED), R(i + s, SPACE_SHARED), W(i, SPACE_SHARED)]
                if removed != s:
                    e.append(SYNCTHREADS)
            if lane == 0:
                e += [R(0, SPACE_SHARED), W(out_base + r)]
            e.append(SYNCTHREADS)
        return e

    return single_kernel(1, 1, lanes, ev, smem_words=n)


# ---------------------------------------------------------------------------
# Random barrier-uniform programs
# ---------------------------------------------------------------------------


def random_program(rng: random.Random, max_blocks: int = 2, max_warps: int = 2,
                   max_lanes: int = 2, max_slots: int = 4, n_words: int = 2,
                   kinds: Sequence[str] = "RWA", barriers: Sequence[str] = ("S", "WS"),
                   p_barrier: float = 0.3, p_skip: float = 0.25,
                   spaces: Sequence[int] = (SPACE_GLOBAL,), n_kernels: int = 1,
                   grid: Optional[tuple] = None) -> Trace:
    """A random program whose barriers are uniform by construction.

    The body is a list of slots shared by all threads; a slot is a barrier
    (emitted by every thread, "barriers are emitted only at
    top level") or an access slot in which each thread independently skips
    or performs a random (kind, space, word) access.
    """
    kmap = {"R": R, "W": W, "A": A}
    kernels = []
    for _ in range(n_kernels):
        if grid is None:
            nb = rng.randint(1, max_blocks)
            nw = rng.randint(1, max_warps)
            nl = rng.randint(1, max_lanes)
        else:
            nb, nw, nl = grid
        nslots = rng.randint(0, max_slots)
        body = []
        for _s in range(nslots):
            if barriers and rng.random() < p_barrier:
                body.append(("B", rng.choice(list(barriers))))
            else:
                acc = {}
                for b in range(nb):
                    for w in range(nw):
                        for l in range(nl):
                            if rng.random() < p_skip:
                                continue
                            acc[(b, w, l)] = (rng.choice(list(kinds)), rng.choice(list(spaces)),
                                              rng.randrange(n_words))
                body.append(("X", acc))

        def ev(b, w, l, body=body):
            e = []
            for kind, payload in body:
                if kind == "B":
                    e.append(SYNCTHREADS if payload == "S" else SYNCWARP)
                else:
                    a = payload.get((b, w, l))
                    if a is not None:
                        e.append(kmap[a[0]](a[2], a[1]))
            return e

        kernels.append(build_kernel(nb, nw, nl, ev, smem_words=n_words))
    return make_trace(kernels)


def from_thread_events(blocks: int, warps: int, lanes: int, events: dict,
                       smem_words: int = 0) -> Trace:
    """Trace from an explicit ``{(block, warp, lane): [records]}`` map (missing = empty)."""
    return single_kernel(blocks, warps, lanes, lambda b, w, l: events.get((b, w, l), []),
                         smem_words)


def random_tile_program(rng: random.Random, blocks: int = 2, warps: int = 2, lanes: int = 32, tile_log2: int = 2,
                        slots: int = 12, n_words: int = 16, spaces: Sequence[int] = (SPACE_GLOBAL,),
                        p_tile: float = 0.3, p_sync: float = 0.08, p_skip: float = 0.3,
                        kinds: Sequence[str] = "RWA"):
    """A kernel whose warp-level barriers are tiles of 2^tile_log2 lanes
    (cooperative-groups ``tiled_partition<T>().sync()``): each slot is an
    access row (lanes skip at random), a ``__syncthreads`` row (every lane of
    the block), or a tile-barrier row in which every tile of every warp
    independently does or does not hold a ``__syncwarp`` record."""
    import numpy as np
    kmap = {"R": R, "W": W, "A": A}
    T = 1 << tile_log2
    rows = np.full((blocks * warps, slots, 32), NOP, dtype=np.uint64)
    for s in range(slots):
        u = rng.random()
        if u < p_sync:
            rows[:, s, :lanes] = SYNCTHREADS
        elif u < p_sync + p_tile:
            for gw in range(blocks * warps):
                for t0 in range(0, lanes, T):
                    if rng.random() < 0.5:
                        rows[gw, s, t0:min(t0 + T, lanes)] = SYNCWARP
        else:
            for gw in range(blocks * warps):
                for l in range(lanes):
                    if rng.random() >= p_skip:
                        rows[gw, s, l] = kmap[rng.choice(list(kinds))](rng.randrange(n_words), rng.choice(list(spaces)))
    k = kernel_from_rows(blocks, warps, lanes, rows, smem_words=n_words if SPACE_SHARED in spaces else 0)
    k.tile_log2 = tile_log2
    return make_trace([k])
