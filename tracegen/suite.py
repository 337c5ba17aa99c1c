"""C2: race-benchmark-style suite (BASELINE.json configs[1]) — INPUT ONLY.

~580 synthetic kernel traces from 21 pattern generators, each in a bug /
no-bug variant over several grid shapes, memory spaces and (for graph codes)
small inputs of 5..200 nodes — the shape of the paper's Indigo experiment
("21 CUDA kernel generator patterns, which generate up to
580 distinct CUDA programs"; Table II inputs of 5..200 nodes).
Each trace is the recorded access stream of the kernel on its input.

Every case carries the label of its injected bug (racy or not by design);
the ORACLE decides the truth — tests check label == oracle as a sanity check
of the generators and GPU == oracle as the parity gate.
"""
from __future__ import annotations

import random
from dataclasses import dataclass
from typing import Callable, Dict, List, Tuple

from .format import (A, NOP, R, SPACE_GLOBAL, SPACE_SHARED, SYNCTHREADS, SYNCWARP, W, Trace,
                     build_kernel, make_trace)


@dataclass
class Case:
    name: str
    trace: Trace
    racy: bool          # injected-bug label


# ---------------------------------------------------------------------------
# small graphs (CSR), seeded
# ---------------------------------------------------------------------------

def graph(kind: str, n: int, m: int, rng: random.Random):
    edges = set()
    if kind == "dag":
        while len(edges) < m:
            u, v = sorted(rng.sample(range(n), 2))
            edges.add((u, v))
    elif kind == "powerlaw":
        pool = list(range(n))          # preferential attachment: v drawn with weight 1 + indegree
        while len(edges) < m:
            u = rng.randrange(n)
            v = pool[rng.randrange(len(pool))]
            if u != v and (u, v) not in edges:
                edges.add((u, v))
                pool.append(v)
    else:  # ring + chords
        for i in range(n):
            edges.add((i, (i + 1) % n))
        while len(edges) < m:
            u, v = rng.sample(range(n), 2)
            edges.add((u, v))
    adj = [[] for _ in range(n)]
    for u, v in sorted(edges):
        adj[u].append(v)
    return adj


GRAPHS = [("dag", 5, 5), ("dag", 20, 40), ("powerlaw", 50, 150), ("dag", 100, 200),
          ("counter", 200, 1000), ("powerlaw", 200, 1000), ("powerlaw", 2000, 16000)]


def _grid_for(n_threads: int, lanes: int = 32):
    warps = max(1, min(4, (n_threads + lanes - 1) // lanes))
    blocks = max(1, (n_threads + warps * lanes - 1) // (warps * lanes))
    return blocks, warps, lanes


def _gtid(b, w, l, warps, lanes):
    return (b * warps + w) * lanes + l


# ---------------------------------------------------------------------------
# the 21 patterns: f(variant, rng) -> (trace, racy_label)
# ---------------------------------------------------------------------------

def p_nosync(v, rng):
    """Listing 1: all threads read+write data[0]; fix: data[i]."""
    B, Wp, L = v["grid"]
    def ev(b, w, l):
        i = _gtid(b, w, l, Wp, L)
        return [R(0), W(0)] if v["bug"] else [R(i), W(i)]
    return build(B, Wp, L, ev), v["bug"] and B * Wp * L > 1


def p_blocksync(v, rng):
    """Listing 2: racy iff >= 2 blocks."""
    B, Wp, L = v["grid"]
    B = B if v["bug"] else 1
    def ev(b, w, l):
        t = w * L + l
        return [R(0), SYNCTHREADS] + ([W(t - 1)] if t > 0 else [])
    return build(B, Wp, L, ev), B >= 2 and Wp * L >= 2


def p_multiread(v, rng):
    """Listing 4; fix: __syncthreads before the write."""
    B, Wp, L = v["grid"]
    n = Wp * L
    length = n + 2
    def ev(b, w, l):
        t = w * L + l
        e = [R(t), R(t + 1)] if t < length - 2 else []
        e += [] if v["bug"] else [SYNCTHREADS]
        e += [W(t + 1)] if t < length - 2 else []
        return e
    return build(1, Wp, L, ev), v["bug"] and n >= 2


def p_tree_reduce(v, rng):
    """Shared-memory tree reduction with one __syncthreads missing."""
    B, Wp, L = v["grid"]
    n = Wp * L
    sp = v["space"]
    base = lambda b: 0 if sp == SPACE_SHARED else b * n   # noqa: E731
    steps = []
    s = n // 2
    while s >= 1:
        steps.append(s)
        s //= 2
    drop = steps[len(steps) // 2] if v["bug"] and steps else None
    def ev(b, w, l):
        t = w * L + l
        e = [W(base(b) + t, sp), SYNCTHREADS]
        for s in steps:
            if t < s:
                e += [R(base(b) + t, sp), R(base(b) + t + s, sp), W(base(b) + t, sp)]
            if s != drop:
                e.append(SYNCTHREADS)
        return e
    racy = drop is not None and drop < n // 2 and any(True for _ in [0])
    # dropping the barrier after step s races iff the two merged steps use different threads
    racy = drop is not None and (drop // 2) >= 1
    return build(B, Wp, L, ev, smem=n), racy


def p_warp_reduce(v, rng):
    """Warp-level shared reduction; bug: __syncwarp omitted between steps."""
    B, Wp, L = v["grid"]
    sp = v["space"]
    def ev(b, w, l):
        base = w * 32 if sp == SPACE_SHARED else (b * Wp + w) * 32
        e = [W(base + l, sp), SYNCWARP]
        o = 16
        while o >= 1:
            if l < o:
                e += [R(base + l, sp), R(base + l + o, sp), W(base + l, sp)]
            if not v["bug"]:
                e.append(SYNCWARP)
            o //= 2
        return e
    return build(B, Wp, 32, ev, smem=Wp * 32), v["bug"]


def p_scan(v, rng):
    """Hillis-Steele scan with double buffering; bug: single buffer."""
    B, Wp, L = v["grid"]
    n = Wp * L
    sp = v["space"]
    def ev(b, w, l):
        t = w * L + l
        base = 0 if sp == SPACE_SHARED else b * 2 * n
        e = [W(base + t, sp), SYNCTHREADS]
        src, dst = 0, (0 if v["bug"] else n)
        o = 1
        while o < n:
            e.append(R(base + src + t, sp))
            if t >= o:
                e.append(R(base + src + t - o, sp))
            e.append(W(base + dst + t, sp))
            e.append(SYNCTHREADS)
            if not v["bug"]:
                src, dst = dst, src
            o *= 2
        return e
    return build(B, Wp, L, ev, smem=2 * n), v["bug"] and n >= 2


def p_transpose(v, rng):
    """Tile transpose through shared memory; bug: no barrier between write and read."""
    B, Wp, L = v["grid"]
    side = 4 if Wp * L >= 16 else 2
    n = side * side
    def ev(b, w, l):
        t = w * L + l
        if t >= n:
            return [] if v["bug"] else [SYNCTHREADS]
        ty, tx = divmod(t, side)
        e = [R(b * n + t), W(ty * side + tx, SPACE_SHARED)]
        if not v["bug"]:
            e.append(SYNCTHREADS)
        e += [R(tx * side + ty, SPACE_SHARED), W(4096 + b * n + t)]
        return e
    return build(B, Wp, L, ev, smem=n), v["bug"]


def p_stencil1d(v, rng):
    """1D shared stencil with halo; bug: no barrier between load and compute."""
    B, Wp, L = v["grid"]
    n = Wp * L
    def ev(b, w, l):
        t = w * L + l
        e = [R(b * n + t), W(t + 1, SPACE_SHARED)]
        if t == 0:
            e += [R(max(b * n - 1, 0)), W(0, SPACE_SHARED)]
        if t == n - 1:
            e += [R(min((b + 1) * n, B * n - 1)), W(n + 1, SPACE_SHARED)]
        if not v["bug"]:
            e.append(SYNCTHREADS)
        e += [R(t, SPACE_SHARED), R(t + 1, SPACE_SHARED), R(t + 2, SPACE_SHARED), W(8192 + b * n + t)]
        return e
    return build(B, Wp, L, ev, smem=n + 2), v["bug"] and n >= 2


def p_histogram(v, rng):
    """Histogram of input values: atomicAdd (fixed) vs read-modify-write (bug)."""
    B, Wp, L = v["grid"]
    bins = v.get("bins", 4)
    sp = v["space"]
    vals = {}
    def ev(b, w, l):
        t = _gtid(b, w, l, Wp, L)
        bn = (t * 2654435761 + v["seed"]) % bins
        key = bn if sp == SPACE_SHARED else (1 << 20) + bn
        return [R(t), A(key, sp)] if not v["bug"] else [R(t), R(key, sp), W(key, sp)]
    return build(B, Wp, L, ev, smem=bins), v["bug"] and B * Wp * L > 1


def _graph_kernel(v, rng, body):
    adj = graph(*v["graph"], random.Random(v["seed"]))
    n = len(adj)
    B, Wp, L = _grid_for(n)
    def ev(b, w, l):
        u = _gtid(b, w, l, Wp, L)
        if u >= n:
            return []
        return body(u, adj)
    return build(B, Wp, L, ev), adj


def p_bfs(v, rng):
    """BFS level step (thread per vertex): atomicMin (fixed) vs plain R/W (bug).
    Level array at words [0, n); frontier = level L vertices."""
    adj = graph(*v["graph"], random.Random(v["seed"]))
    n = len(adj)
    lvl = [-1] * n
    lvl[0] = 0
    q = [0]
    for u in q:
        for x in adj[u]:
            if lvl[x] < 0:
                lvl[x] = lvl[u] + 1
                q.append(x)
    L0 = v.get("level", 1)
    front = {u for u in range(n) if lvl[u] == L0}
    nxt = {x for u in front for x in adj[u] if lvl[x] < 0 or lvl[x] > L0}
    B, Wp, La = _grid_for(n)
    def ev(b, w, l):
        u = _gtid(b, w, l, Wp, La)
        if u >= n:
            return []
        e = [A(u) if not v["bug"] else R(u)]
        if u in front:
            for x in adj[u]:
                if v["bug"]:
                    e.append(R(x))
                    if x in nxt:
                        e.append(W(x))
                else:
                    e.append(A(x))
        return e
    tr = build(B, Wp, La, ev)
    # racy iff some written vertex is also touched by another thread
    racy = False
    if v["bug"]:
        writers = {}
        for u in front:
            for x in adj[u]:
                if x in nxt:
                    writers.setdefault(x, set()).add(u)
        racy = any(len(s | {x}) >= 2 for x, s in writers.items())
    return tr, racy


def p_sssp(v, rng):
    """SSSP relax: dist[x] = min(dist[x], dist[u] + w): atomicMin vs plain."""
    def body(u, adj):
        e = [R(u)]
        for x in adj[u]:
            e += [A(x)] if not v["bug"] else [R(x), W(x)]
        return e
    tr, adj = _graph_kernel(v, rng, body)
    has_edge = any(adj[u] for u in range(len(adj)))
    return tr, has_edge and (v["bug"] or any(x != u for u in range(len(adj)) for x in adj[u]))


def p_cc(v, rng):
    """Label propagation: in-place (bug: R neighbour labels vs W own label) vs double buffer."""
    n_off = 4096
    def body(u, adj):
        e = [R(u)]
        for x in adj[u]:
            e.append(R(x))
        e.append(W(u) if v["bug"] else W(n_off + u))
        return e
    tr, adj = _graph_kernel(v, rng, body)
    return tr, v["bug"] and any(adj[u] for u in range(len(adj)))


def p_pagerank(v, rng):
    """PageRank push: atomicAdd to neighbour (fixed) vs R+W (bug)."""
    def body(u, adj):
        e = [R(u)]
        for x in adj[u]:
            e += [A(4096 + x)] if not v["bug"] else [R(4096 + x), W(4096 + x)]
        return e
    tr, adj = _graph_kernel(v, rng, body)
    indeg = {}
    for u in range(len(adj)):
        for x in adj[u]:
            indeg[x] = indeg.get(x, 0) + 1
    return tr, v["bug"] and any(c >= 2 for c in indeg.values())


def p_worklist(v, rng):
    """Worklist push: atomic tail (fixed) vs plain read/increment of the tail (bug)."""
    B, Wp, L = v["grid"]
    def ev(b, w, l):
        t = _gtid(b, w, l, Wp, L)
        if t % 3:
            return []
        if v["bug"]:
            return [R(0), W(0), W(16 + t)]
        return [A(0), W(16 + t)]
    tr = build(B, Wp, L, ev)
    pushers = sum(1 for t in range(B * Wp * L) if t % 3 == 0)
    return tr, v["bug"] and pushers >= 2


def p_flag(v, rng):
    """Producer/consumer through a flag: racy under the barrier-only model
    (reading R1: atomics do not synchronise); fixed with __syncthreads."""
    B, Wp, L = v["grid"]
    def ev(b, w, l):
        t = w * L + l
        if v["bug"]:
            if t == 0:
                return [W(b * 2), A(b * 2 + 1)]
            if t == 1:
                return [A(b * 2 + 1), R(b * 2)]
            return []
        e = [W(b * 2)] if t == 0 else []
        e.append(SYNCTHREADS)
        if t == 1:
            e.append(R(b * 2))
        return e
    return build(B, Wp, L, ev), v["bug"] and Wp * L >= 2


def p_pingpong(v, rng):
    """Iterated 1D smoothing across kernels: double buffer (fixed) vs in place (bug)."""
    B, Wp, L = v["grid"]
    n = B * Wp * L
    kernels = []
    for k in range(3):
        src, dst = (k % 2) * n, ((k + 1) % 2) * n
        if v["bug"]:
            src = dst = 0
        def ev(b, w, l, src=src, dst=dst):
            i = _gtid(b, w, l, Wp, L)
            return [R(src + max(i - 1, 0)), R(src + i), R(src + min(i + 1, n - 1)), W(dst + i)]
        kernels.append(build_kernel(B, Wp, L, ev))
    return make_trace(kernels), v["bug"] and n >= 2


def p_gridstride(v, rng):
    """Grid-stride copy; bug: stride one short, so neighbouring threads overlap."""
    B, Wp, L = v["grid"]
    nt = B * Wp * L
    n = 3 * nt
    stride = nt - 1 if v["bug"] else nt
    def ev(b, w, l):
        i = _gtid(b, w, l, Wp, L)
        e = []
        while i < n:
            e += [R(i), W(n + i)]
            i += stride
        return e
    tr = build(B, Wp, L, ev)
    return tr, v["bug"] and nt >= 2


def p_scratch(v, rng):
    """Block-private global scratch; bug: off-by-one overlap with the next block."""
    B, Wp, L = v["grid"]
    S = Wp * L
    def ev(b, w, l):
        t = w * L + l
        span = S + 1 if v["bug"] else S
        e = [W(b * S + t)]
        if v["bug"] and t == S - 1:
            e.append(W(b * S + S))
        e.append(SYNCTHREADS)
        e.append(R(b * S + (t + 1) % span))
        return e
    return build(B, Wp, L, ev), v["bug"] and B >= 2


def p_shared_init(v, rng):
    """Thread 0 initialises shared memory, others read it; bug: no barrier."""
    B, Wp, L = v["grid"]
    n = 8
    def ev(b, w, l):
        t = w * L + l
        e = [W(i, SPACE_SHARED) for i in range(n)] if t == 0 else []
        if not v["bug"]:
            e.append(SYNCTHREADS)
        e.append(R(t % n, SPACE_SHARED))
        return e
    return build(B, Wp, L, ev, smem=n), v["bug"] and Wp * L >= 2


def p_atomic_mix(v, rng):
    """Atomic counters read plainly in the same kernel (bug) or the next one."""
    B, Wp, L = v["grid"]
    def ev(b, w, l):
        t = _gtid(b, w, l, Wp, L)
        e = [A(t % 4)]
        if v["bug"] and t == 0:
            e.append(R(1))
        return e
    k1 = build_kernel(B, Wp, L, ev)
    ks = [k1]
    if not v["bug"]:
        ks.append(build_kernel(1, 1, 1, lambda b, w, l: [R(1)]))
    return make_trace(ks), v["bug"] and B * Wp * L >= 2


def p_warp_sync(v, rng):
    """Lanes exchange through shared memory; bug: legacy warp-synchronous code
    without __syncwarp (lanes are not implicitly synchronised)."""
    B, Wp, L = v["grid"]
    def ev(b, w, l):
        base = w * L
        e = [W(base + l, SPACE_SHARED)]
        if not v["bug"]:
            e.append(SYNCWARP)
        e.append(R(base + (l + 1) % L, SPACE_SHARED))
        return e
    return build(B, Wp, L, ev, smem=Wp * L), v["bug"] and L >= 2


def build(B, Wp, L, ev, smem=0) -> Trace:
    return make_trace([build_kernel(B, Wp, L, ev, smem_words=smem)])


PATTERNS: Dict[str, Callable] = {
    "nosync": p_nosync, "blocksync": p_blocksync, "multiread": p_multiread,
    "tree_reduce": p_tree_reduce, "warp_reduce": p_warp_reduce, "scan": p_scan,
    "transpose": p_transpose, "stencil1d": p_stencil1d, "histogram": p_histogram,
    "bfs": p_bfs, "sssp": p_sssp, "cc": p_cc, "pagerank": p_pagerank, "worklist": p_worklist,
    "flag": p_flag, "pingpong": p_pingpong, "gridstride": p_gridstride, "scratch": p_scratch,
    "shared_init": p_shared_init, "atomic_mix": p_atomic_mix, "warp_sync": p_warp_sync,
}
GRAPH_PATTERNS = {"bfs", "sssp", "cc", "pagerank"}
GRIDS = [(1, 1, 32), (1, 2, 32), (2, 2, 32), (4, 4, 32), (2, 1, 8), (3, 2, 16), (1, 4, 32),
         (8, 4, 32), (16, 8, 32), (5, 3, 20)]


def suite(seed: int = 2401_04701) -> List[Case]:
    """The ~580-trace C2 suite (deterministic for a seed)."""
    rng = random.Random(seed)
    cases: List[Case] = []
    for name, fn in PATTERNS.items():
        variants = []
        if name in GRAPH_PATTERNS:
            for g in GRAPHS:
                for bug in (True, False):
                    for rep in range(3):
                        variants.append({"graph": g, "bug": bug, "seed": rng.randrange(1 << 30),
                                         "level": 1 + rep})
        else:
            spaces = [SPACE_SHARED, SPACE_GLOBAL] if name in ("tree_reduce", "warp_reduce", "scan",
                                                             "histogram") else [None]
            for grid in GRIDS:
                for sp in spaces:
                    for bug in (True, False):
                        variants.append({"grid": grid, "bug": bug, "space": sp,
                                         "seed": rng.randrange(1 << 30)})
        for i, var in enumerate(variants):
            tr, racy = fn(var, rng)
            cases.append(Case(f"{name}/{i}{'-bug' if var['bug'] else ''}", tr, bool(racy)))
    return cases
