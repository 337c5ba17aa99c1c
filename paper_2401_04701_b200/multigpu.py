"""Address-sharded multi-GPU replay.

Accesses to different words are independent FSMs (the shadow is per word,
PAPER.md:395-396; no transition reads another word), so rank r of N owns the
shadow granules g = (word - base) >> 3 (8 words, 64 B of shadow) with
shard_owner(g) == r (include/hr.h hr_shard_owner: stripes of N granules, one
per rank, rotated per stripe) and the shared instances of simulated blocks
with block % N == r.  Each rank replays every
simulated thread but only its own records, keeping all barrier records so the
per-word commit order stays happens-before consistent; its shadow is 1/N.
The ONE exchange is the race-set allgather (NCCL over NVLink on GPUs, gloo
in the CPU tests): each rank's device report (hr_report_async_to) goes into
a fixed-size device buffer that all_gather_into_tensor moves to every rank
inside the step (DeviceExchange); the concatenate-and-merge in libhirace
(hr_merge_races, host C) runs when the set is collected — shards are
address-disjoint, so the merge only interleaves the per-rank sorted lists.

torch.distributed provides the process group only; the check runs in
libhirace.so.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

RACE_DTYPE = np.dtype([("word", "<u8"), ("block", "<u4"), ("kernel", "<u4"), ("first_tid", "<u4"),
                       ("space", "u1"), ("scope", "u1"), ("first_kind", "u1"), ("prev_state", "u1")])
NOP = np.uint64(3 << 62)


def shard_owner(granule, nshard: int):
    """include/hr.h hr_shard_owner on numpy uint64 granule indices (or an int):
    granule g of stripe s = g >> log2(N) goes to (g + rot(s)) mod N, where
    rot(s) = ((s ^ s >> 32) mod 2^32 * 0x9E3779B1 mod 2^32) >> (32 - log2(N))."""
    l2 = nshard.bit_length() - 1
    assert nshard == 1 << l2, "shard count must be a power of two"
    if l2 == 0:
        return np.zeros_like(np.asarray(granule, dtype=np.uint64)) if not np.isscalar(granule) else 0
    g = np.asarray(granule, dtype=np.uint64)
    s = g >> np.uint64(l2)
    m32 = np.uint64(0xFFFFFFFF)
    rot = ((((s ^ (s >> np.uint64(32))) & m32) * np.uint64(0x9E3779B1)) & m32) >> np.uint64(32 - l2)
    own = ((g & m32) + rot) & np.uint64(nshard - 1)
    return int(own) if np.isscalar(granule) else own


def owner_mask(rows: np.ndarray, block: int, rank: int, nshard: int, base_word: int = 0,
               granule_log2: int = 3) -> np.ndarray:
    """Which records of one warp's rows (n, 32) belong to shard `rank`."""
    op = rows >> np.uint64(62)
    space = (rows >> np.uint64(61)) & np.uint64(1)
    word = rows & np.uint64((1 << 61) - 1)
    gran = (word - np.uint64(base_word)) >> np.uint64(granule_log2)
    glob = (op != 3) & (space == 0) & (shard_owner(gran, nshard) == np.uint64(rank))
    shared = (op != 3) & (space == 1) & ((block % nshard) == rank)
    return glob | shared


def shard_trace(trace, rank: int, nshard: int, base_word: int = 0, granule_log2: int = 3):
    """Host-side shard of a trace: this rank's records compacted per lane inside
    each barrier-delimited segment, padded with NOPs, barrier rows kept."""
    from tracegen.format import Trace   # layout container only
    if nshard == 1:
        return trace
    out_rows, offs, kd = [], [], trace.kdesc.copy()
    row = 0
    for k in range(trace.kdesc.shape[0]):
        blocks, warps = int(trace.kdesc[k, 0]), int(trace.kdesc[k, 1])
        woi = int(trace.kdesc[k, 4])
        kd[k, 4] = len(offs)
        for w in range(blocks * warps):
            r0, r1 = int(trace.warp_off[woi + w]), int(trace.warp_off[woi + w + 1])
            rows = trace.rec[r0 * 32: r1 * 32].reshape(-1, 32)
            keep = owner_mask(rows, w // warps, rank, nshard, base_word, granule_log2)
            op = rows >> np.uint64(62)
            word = rows & np.uint64((1 << 61) - 1)
            is_bar = np.any((op == 3) & (word != 0), axis=1)
            offs.append(row)
            seg_start = 0
            for i in list(np.nonzero(is_bar)[0]) + [rows.shape[0]]:
                seg = rows[seg_start:i]
                km = keep[seg_start:i]
                depth = int(km.sum(axis=0).max()) if seg.shape[0] else 0
                if depth:
                    out = np.full((depth, 32), NOP, dtype=np.uint64)
                    for lane in range(32):
                        v = seg[km[:, lane], lane]
                        out[: v.shape[0], lane] = v
                    out_rows.append(out)
                    row += depth
                if i < rows.shape[0]:
                    out_rows.append(rows[i: i + 1])
                    row += 1
                seg_start = i + 1
        offs.append(row)                 # end of the kernel's last warp (nw + 1 entries)
    rec = np.concatenate([r.reshape(-1) for r in out_rows]) if out_rows else np.zeros(0, np.uint64)
    return Trace(np.ascontiguousarray(rec, dtype=np.uint64), kd, np.array(offs, dtype=np.uint64))


def exchange_races(raw: np.ndarray, flags: int = 0, group=None, device=None) -> Tuple[np.ndarray, int]:
    """Allgather the per-rank race sets and merge: (sorted global set, OR of flags).
    Identical on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    meta = torch.tensor([len(raw), flags], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    allm = torch.stack(metas).cpu()                 # one device->host read
    counts = [int(c) for c in allm[:, 0]]
    all_flags = 0
    for f in allm[:, 1]:
        all_flags |= int(f)
    mx = max(max(counts), 1)
    pad = torch.zeros(mx * 3, dtype=torch.int64, device=dev)
    if len(raw):
        pad[: len(raw) * 3] = torch.from_numpy(np.ascontiguousarray(raw).view(np.int64).copy()).to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    flat = torch.cat([p[: c * 3] for p, c in zip(parts, counts)]).cpu().numpy()
    from .hirace import hr_merge_races          # sort + unique in libhirace (host C), not numpy
    return hr_merge_races(flat.view(RACE_DTYPE)), all_flags


class DeviceExchange:
    """The per-step race-set exchange with no host round trip (SURVEY §8(e)
    step 5): each rank's sorted unique set is written by hr_report_async_to
    into a fixed-size DEVICE buffer (cap records + a 4-word header), and one
    all_gather_into_tensor moves every rank's buffer to every rank (NCCL over
    NVLink: on the launching stream, ordered after the report).  The merge of
    the N address-disjoint sorted lists (hr_merge_races) runs only in
    collect(), off the step's critical path.

    With a gloo group (CPU tests; several ranks sharing one GPU) the buffers
    are staged through host memory for the collective: same result, not the
    device path."""

    def __init__(self, ctx, cap: int = 1 << 17, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.ctx, self.cap, self.group = ctx, int(cap), group
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        dev = device
        self.buf = torch.empty(self.cap * RACE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.hdr = torch.zeros(4, dtype=torch.int32, device=dev)
        gdev = dev if self.nccl else "cpu"
        self.gbuf = torch.empty(self.world * self.buf.numel(), dtype=torch.uint8, device=gdev)
        self.ghdr = torch.empty(self.world * 4, dtype=torch.int32, device=gdev)

    def step(self, stream: Optional[int] = None):
        """Enqueue this rank's report and the allgather (asynchronous on NCCL)."""
        import torch
        import torch.distributed as dist
        from .hirace import hr_report_async_to
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        hr_report_async_to(self.ctx, self.buf.data_ptr(), self.cap, self.hdr.data_ptr(), stream)
        if self.nccl:
            dist.all_gather_into_tensor(self.ghdr, self.hdr, group=self.group)
            dist.all_gather_into_tensor(self.gbuf, self.buf, group=self.group)
        else:
            dist.all_gather_into_tensor(self.ghdr, self.hdr.cpu(), group=self.group)
            dist.all_gather_into_tensor(self.gbuf, self.buf.cpu(), group=self.group)

    def step_from_host(self, raw: np.ndarray, flags: int = 0):
        """Same exchange for a set already on the host (e.g. a CPU-side test of
        the gather / merge logic): the set is written into the device (or, on
        gloo, host) buffer and header, then gathered as in step()."""
        import torch
        import torch.distributed as dist
        raw = np.ascontiguousarray(raw, dtype=RACE_DTYPE)
        n = min(len(raw), self.cap)
        hdr = torch.tensor([len(raw), flags, len(raw), 0], dtype=torch.int32)
        buf = torch.zeros(self.buf.numel(), dtype=torch.uint8)
        if n:
            buf[: n * RACE_DTYPE.itemsize] = torch.from_numpy(raw[:n].view(np.uint8).copy())
        if self.nccl:
            self.hdr.copy_(hdr)
            self.buf.copy_(buf)
            hdr, buf = self.hdr, self.buf
        dist.all_gather_into_tensor(self.ghdr, hdr, group=self.group)
        dist.all_gather_into_tensor(self.gbuf, buf, group=self.group)

    def collect(self, fallback_raw=None) -> Tuple[np.ndarray, int]:
        """(sorted global set, OR of the ranks' flags) of the last step; identical
        on every rank.  A rank whose set overflowed `cap` or whose ring
        overflowed (spill store) is re-read with the full hr_report path
        (`fallback_raw` = that rank's (raw, flags) getter) and re-exchanged."""
        from .hirace import hr_merge_races
        hdr = self.ghdr.cpu().numpy().reshape(self.world, 4).astype(np.int64)
        if np.any(hdr[:, 0] > self.cap) or np.any(hdr[:, 3] != 0):
            if fallback_raw is None:
                raise RuntimeError("race-set exchange overflow: raise DeviceExchange cap or pass fallback_raw")
            raw, flags = fallback_raw()
            return exchange_races(raw, flags, self.group)
        allb = self.gbuf.cpu().numpy().reshape(self.world, -1)
        parts = [allb[r].view(RACE_DTYPE)[: int(hdr[r, 0])] for r in range(self.world)]
        flags = 0
        for f in hdr[:, 1]:
            flags |= int(f)
        flat = np.concatenate(parts) if parts else np.zeros(0, RACE_DTYPE)
        return hr_merge_races(flat), flags


def replay_sharded(trace, group=None, device: Optional[int] = None, base_word: int = 0, cap: int = 1 << 17,
                   **checker_kw):
    """Replay a host trace address-sharded over the ranks of `group` (one GPU per
    rank) and return the global sorted race set (hr_race records) and flags,
    identical on every rank: shard (host), replay (libhirace), device report,
    allgather (DeviceExchange), merge."""
    import torch
    import torch.distributed as dist
    from . import hirace
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    gmax, smem = hirace.trace_extent(trace)
    local = shard_trace(trace, rank, world, base_word)
    ck = hirace.Checker(gmax - base_word, smem, base_word=base_word, device=dev, shard=(rank, world),
                        **checker_kw)
    dt = hirace.DeviceTrace.from_trace(local, device=f"cuda:{dev}")
    dt.flags = hirace.HR_TRACE_F_SHARD_OWNED       # shard_trace kept only this rank's records
    ck.replay(dt)
    ex = DeviceExchange(ck.ctx, cap, group, device=torch.device("cuda", dev))
    ex.step()
    out = ex.collect(fallback_raw=ck.report_raw)
    ck.close()
    return out
