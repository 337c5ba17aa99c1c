"""Access-trace container and builders — INPUT ONLY.

This module is the one piece shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2401_04701_b200``): it lays seeded synthetic access
streams out in memory.  It holds none of the method's arithmetic — no
happens-before, no thread relations, no clocks comparisons, no FSM.  Both
sides decode the records independently.

Layout
------------------------------------------------
A trace is a list of *kernels* (kernel boundaries order everything, SURVEY
§8(c) "Kernel boundaries").  Each kernel has a grid of ``blocks`` blocks of
``warps`` warps of ``lanes`` (<= 32) simulated threads (the paper's
T_{bwt} labelling, Fig. ``simple-grid``).

Each record is one uint64::

    bits 63:62  op     0 = read, 1 = write, 2 = atomic, 3 = control
    bit  61     space  0 = global, 1 = shared (__shared__, one instance per block)
    bits 60:0   word   4-byte word index (shadow[k] for data[k])
    control records: word = 0 NOP, 1 __syncthreads, 2 __syncwarp

Records are stored warp-interleaved: row ``r`` holds 32 records, one per
lane; warp ``w`` of kernel ``k`` owns rows ``warp_off[kd.warp_off_index + w]``
up to ``warp_off[kd.warp_off_index + w + 1]`` (so warps may have different
lengths).  Lanes ``>= lanes`` of a row are ignored.  Barrier records are
warp-aligned: when one active lane holds a barrier at some row, every active
lane of that warp holds the same barrier at that row.

``kdesc`` is an (n_kernels, 8) uint64 array:
    [blocks, warps, lanes, smem_words, warp_off_index, tile_log2, 0, 0]
``tile_log2`` (1..4) declares that the kernel's warp-level barriers are tiles of
2^tile_log2 lanes (cooperative-groups ``tiled_partition<T>().sync()``, i.e.
``__syncwarp(tile mask)``): a ``__syncwarp`` record held by whole tiles is one
barrier per tile.  0 = whole-warp ``__syncwarp`` only.
``warp_off`` is a uint64 array of absolute row indices.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Sequence

import numpy as np

OP_READ, OP_WRITE, OP_ATOMIC, OP_CTRL = 0, 1, 2, 3
SPACE_GLOBAL, SPACE_SHARED = 0, 1
CTRL_NOP, CTRL_SYNCTHREADS, CTRL_SYNCWARP = 0, 1, 2
WORD_BITS = 61
WORD_MASK = (1 << WORD_BITS) - 1
LANES_PER_ROW = 32
KDESC_FIELDS = 8


def encode(op: int, space: int, word: int) -> int:
    """Pack one record (layout in the module docstring)."""
    if not 0 <= word <= WORD_MASK:
        raise ValueError(f"word {word} out of range")
    return (op << 62) | (space << 61) | word


NOP = encode(OP_CTRL, 0, CTRL_NOP)
SYNCTHREADS = encode(OP_CTRL, 0, CTRL_SYNCTHREADS)
SYNCWARP = encode(OP_CTRL, 0, CTRL_SYNCWARP)
BARRIERS = (SYNCTHREADS, SYNCWARP)


def R(word: int, space: int = SPACE_GLOBAL) -> int:
    return encode(OP_READ, space, word)


def W(word: int, space: int = SPACE_GLOBAL) -> int:
    return encode(OP_WRITE, space, word)


def A(word: int, space: int = SPACE_GLOBAL) -> int:
    return encode(OP_ATOMIC, space, word)


class BarrierDivergence(ValueError):
    """Threads of one warp (or block) disagree on their barrier sequence."""


@dataclass
class Kernel:
    blocks: int
    warps: int
    lanes: int
    smem_words: int
    rows: List[np.ndarray] = field(default_factory=list)  # per warp: (n_rows, 32) uint64
    tile_log2: int = 0     # warp-level barriers are tiles of 2^tile_log2 lanes (0 = whole warps)

    @property
    def n_warps(self) -> int:
        return self.blocks * self.warps


@dataclass
class Trace:
    rec: np.ndarray        # (n_rows * 32,) uint64
    kdesc: np.ndarray      # (n_kernels, 8) uint64
    warp_off: np.ndarray   # uint64 absolute row offsets

    @property
    def n_kernels(self) -> int:
        return int(self.kdesc.shape[0])

    @property
    def n_rows(self) -> int:
        return int(self.rec.shape[0] // LANES_PER_ROW)

    def n_accesses(self) -> int:
        """Number of memory-access records on active lanes (excludes control and idle lanes)."""
        total = 0
        for k in range(self.n_kernels):
            blocks, warps, lanes, _, woi = (int(x) for x in self.kdesc[k, :5])
            nw = blocks * warps
            offs = self.warp_off[woi: woi + nw + 1].astype(np.int64)
            r0, r1 = int(offs[0]), int(offs[-1])
            rows = self.rec[r0 * 32: r1 * 32].reshape(-1, 32)[:, :lanes]
            total += int(np.count_nonzero((rows >> np.uint64(62)) != OP_CTRL))
        return total

    def save(self, path: str) -> None:
        np.savez_compressed(path, rec=self.rec, kdesc=self.kdesc, warp_off=self.warp_off)

    @staticmethod
    def load(path: str) -> "Trace":
        z = np.load(path)
        return Trace(z["rec"], z["kdesc"], z["warp_off"])


def _split_segments(events: Sequence[int]):
    segs, bars, cur = [], [], []
    for e in events:
        if e in BARRIERS:
            segs.append(cur)
            bars.append(e)
            cur = []
        elif e == NOP:
            cur.append(e)
        else:
            if (e >> 62) == OP_CTRL:
                raise ValueError(f"unknown control record {e:#x}")
            cur.append(e)
    segs.append(cur)
    return segs, bars


def align_warp(lane_events: Sequence[Sequence[int]]) -> np.ndarray:
    """Lay one warp's per-lane event lists out as warp-aligned rows.

    Every lane must execute the same barrier sequence (uniform barriers,
    SURVEY §8(c) "Barrier divergence"); the accesses between two barriers are
    padded with NOPs to the longest lane.
    """
    split = [_split_segments(ev) for ev in lane_events]
    bars0 = split[0][1] if split else []
    for segs, bars in split:
        if bars != bars0:
            raise BarrierDivergence("lanes of a warp disagree on their barrier sequence")
    rows = []
    nseg = len(bars0) + 1
    for i in range(nseg):
        seglen = max((len(s[0][i]) for s in split), default=0)
        for j in range(seglen):
            row = [NOP] * LANES_PER_ROW
            for lane, (segs, _) in enumerate(split):
                if j < len(segs[i]):
                    row[lane] = segs[i][j]
            rows.append(row)
        if i < len(bars0):
            rows.append([bars0[i]] * LANES_PER_ROW)
    if not rows:
        return np.zeros((0, LANES_PER_ROW), dtype=np.uint64)
    return np.array(rows, dtype=np.uint64)


def build_kernel(blocks: int, warps: int, lanes: int,
                 thread_events: Callable[[int, int, int], Sequence[int]],
                 smem_words: int = 0) -> Kernel:
    """Materialise a kernel from a per-thread event function ``f(block, warp, lane)``."""
    if not (blocks >= 1 and warps >= 1 and 1 <= lanes <= LANES_PER_ROW):
        raise ValueError("bad grid")
    k = Kernel(blocks, warps, lanes, smem_words)
    for b in range(blocks):
        nsync = None
        for w in range(warps):
            evs = [list(thread_events(b, w, l)) for l in range(lanes)]
            cnt = sum(1 for e in evs[0] if e == SYNCTHREADS)
            if nsync is None:
                nsync = cnt
            elif cnt != nsync:
                raise BarrierDivergence("warps of a block disagree on their __syncthreads count")
            k.rows.append(align_warp(evs))
    return k


def kernel_from_rows(blocks: int, warps: int, lanes: int, rows: np.ndarray,
                     smem_words: int = 0) -> Kernel:
    """Kernel from a dense (n_warps, n_rows, 32) record array (uniform warp length)."""
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    assert rows.shape[0] == blocks * warps and rows.shape[2] == LANES_PER_ROW
    k = Kernel(blocks, warps, lanes, smem_words)
    k.rows = rows  # type: ignore[assignment]
    return k


def make_trace(kernels: Sequence[Kernel]) -> Trace:
    recs, offs, kd = [], [], []
    row = 0
    for k in kernels:
        woi = sum(len(o) for o in offs)
        if isinstance(k.rows, np.ndarray):
            nw, nr, _ = k.rows.shape
            o = (np.arange(nw + 1, dtype=np.uint64) * np.uint64(nr)) + np.uint64(row)
            recs.append(k.rows.reshape(-1))
            row += nw * nr
        else:
            lens = [r.shape[0] for r in k.rows]
            o = np.zeros(len(lens) + 1, dtype=np.uint64)
            o[0] = row
            o[1:] = row + np.cumsum(np.array(lens, dtype=np.uint64)) if lens else row
            for r in k.rows:
                recs.append(r.reshape(-1))
            row += int(sum(lens))
        offs.append(o)
        kd.append([k.blocks, k.warps, k.lanes, k.smem_words, woi, k.tile_log2, 0, 0])
    rec = np.concatenate(recs) if recs else np.zeros(0, dtype=np.uint64)
    return Trace(np.ascontiguousarray(rec, dtype=np.uint64),
                 np.array(kd, dtype=np.uint64).reshape(-1, KDESC_FIELDS),
                 np.concatenate(offs).astype(np.uint64) if offs else np.zeros(0, np.uint64))


def to_c32(trace: Trace):
    """The HR_TRACE_C32 encoding of a trace (include/hr.h): per record a u32
    word and a byte op | space << 2 (160 B per row).  Requires words < 2^32."""
    word = trace.rec & np.uint64(WORD_MASK)
    if word.size and int(word.max()) >= (1 << 32):
        raise ValueError("C32 encoding needs words < 2^32")
    op = trace.rec >> np.uint64(62)
    sp = (trace.rec >> np.uint64(61)) & np.uint64(1)
    return (np.ascontiguousarray(word.astype(np.uint32)),
            np.ascontiguousarray((op | (sp << np.uint64(2))).astype(np.uint8)))


def single_kernel(blocks, warps, lanes, thread_events, smem_words=0) -> Trace:
    return make_trace([build_kernel(blocks, warps, lanes, thread_events, smem_words)])
