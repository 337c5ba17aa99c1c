"""HR_TRACE_PACKED (include/hr.h): the lossless transfer encoding made by
hr_pack_trace and decoded on the device by hr_unpack_trace and by the packed
replay paths.  Checked two ways: bit-exact round trip of arbitrary 64-bit
records (any op/space/word bits, empty and ragged segments, every delta
width 0..61, the raw escape), and racy sets equal to the oracle's when the
packed trace is replayed from device and from host memory."""
import random

import numpy as np
import pytest

import oracle
from tracegen import c5
from tracegen import format as tf
from tracegen import programs as tp

from tests.test_gpu_parity import _random_batch, oracle_set

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def _dev(rec: np.ndarray, warp_off: np.ndarray):
    import torch
    h = hr()
    return h.DeviceTrace(torch.from_numpy(rec.view(np.int64)).cuda(),
                         torch.from_numpy(warp_off.astype(np.uint64).view(np.int64)).cuda(),
                         np.zeros((0, 8), dtype=np.uint64))


def _roundtrip(rec: np.ndarray, warp_off: np.ndarray):
    import torch
    h = hr()
    ck = h.Checker(1024)
    dt = _dev(rec, warp_off)
    pk = ck.pack(dt)
    out = torch.full((dt.n_rows * 32,), -1, dtype=torch.int64, device="cuda")
    h.hr_unpack_trace(ck.ctx, pk.c(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    po = pk.pack_off.cpu().numpy().view(np.uint64)
    ck.close()
    return out.cpu().numpy().view(np.uint64), po, pk.record_bytes()


def _rows(rng: np.random.Generator, n: int) -> np.ndarray:
    """n rows of 32 records mixing every row shape the encoder distinguishes."""
    M = (1 << 61) - 1
    out = np.zeros((n, 32), dtype=np.uint64)
    lanes = np.arange(32, dtype=np.uint64)
    for i in range(n):
        kind = i % 9
        if kind == 0:                                    # arbitrary 64-bit garbage -> raw escape
            out[i] = rng.integers(0, 2**64, 32, dtype=np.uint64, endpoint=False)
        elif kind == 1:                                  # coalesced row, mixed R/W (affine: bit mask)
            base = int(rng.integers(0, 1 << 40)) if rng.random() < 0.5 else int(rng.integers(0, (1 << 32) - 32))
            ops = rng.integers(0, 2, 32).astype(np.uint64)
            sp = np.uint64(int(rng.integers(0, 2)))
            out[i] = (ops << np.uint64(62)) | (sp << np.uint64(61)) | (np.uint64(base) + lanes)
            if rng.random() < 0.3:                       # one atomic or one NOP lane: nibbles again
                out[i, int(rng.integers(0, 32))] = np.uint64(tf.NOP) if rng.random() < 0.5 else \
                    (np.uint64(2 << 62) | (np.uint64(base) + np.uint64(int(rng.integers(0, 32)))))
        elif kind == 2:                                  # broadcast of one word, uniform op (k == 0)
            out[i] = np.uint64((2 << 62) | (1 << 61) | int(rng.integers(0, M)))
        elif kind == 3:                                  # barrier row / all NOP (no words)
            out[i] = tf.SYNCTHREADS if rng.random() < 0.5 else tf.NOP
        else:                                            # deltas of width k, some NOP / control lanes
            k = int(rng.integers(0, 62))
            base = int(rng.integers(0, M - (1 << k) + 1)) if k < 61 else 0
            if kind in (5, 6) and k < 32:                # bases below 2^32 (the 4-byte base form)
                base = int(rng.integers(0, (1 << 32) - (1 << k) + 1))
            d = rng.integers(0, 1 << k, 32, dtype=np.uint64) if k else np.zeros(32, np.uint64)
            ops = rng.integers(0, 3, 32).astype(np.uint64)
            sp = rng.integers(0, 2, 32).astype(np.uint64)
            row = (ops << np.uint64(62)) | (sp << np.uint64(61)) | (np.uint64(base) + d)
            nop = rng.random(32) < 0.2
            row[nop] = np.uint64(tf.NOP)
            if kind == 8:
                row[rng.integers(0, 32)] = np.uint64(tf.SYNCWARP)
            out[i] = row
    return out.reshape(-1)


def test_roundtrip_arbitrary_records():
    rng = np.random.default_rng(4701)
    n_rows = 3000
    rec = _rows(rng, n_rows)
    # ragged segments, some empty
    cuts = np.sort(rng.integers(0, n_rows + 1, 400))
    warp_off = np.concatenate([[0], cuts, [n_rows]]).astype(np.uint64)
    got, po, nbytes = _roundtrip(rec, warp_off)
    assert np.array_equal(got, rec)
    assert np.all(po % 4 == 0) and np.all(np.diff(po.astype(np.int64)) >= 0)
    assert nbytes == int(po[-1]) + 16


def test_roundtrip_every_delta_width():
    """One row per width k = 1..61: lane l's delta has bit k-1 set, so every
    k-bit field straddles u32 words at all 32 lane positions."""
    rows = []
    for k in range(1, 62):
        top = np.uint64(1) << np.uint64(k - 1)
        low = np.arange(32, dtype=np.uint64) * np.uint64(2654435761) % top if k > 1 else np.zeros(32, np.uint64)
        d = top | low
        d[0] = 0
        rows.append((np.uint64(1) << np.uint64(62)) | d)
    rec = np.concatenate(rows).astype(np.uint64)
    warp_off = np.array([0, 20, 20, 61], dtype=np.uint64)
    got, _, _ = _roundtrip(rec, warp_off)
    assert np.array_equal(got, rec)


def test_row_sizes():
    """Sizes the format in include/hr.h fixes for single-row segments."""
    lanes = np.arange(32, dtype=np.uint64)
    cases = [
        (np.full(32, tf.SYNCTHREADS, np.uint64), 4 + 4),                         # uniform nibble, no words
        (np.uint64(1 << 62) | (np.uint64(4096) + lanes), 4 + 4 + 8),              # uniform W, affine
        ((lanes % np.uint64(2)) << np.uint64(62) | (np.uint64(4096) + lanes), 4 + 4 + 4),    # mixed R/W affine: mask
        ((lanes % np.uint64(2)) << np.uint64(62) | (np.uint64(1 << 40) + lanes), 4 + 4 + 8),  # the same, u64 base
        ((lanes % np.uint64(3) == 0).astype(np.uint64) << np.uint64(62) | np.uint64(1 << 61) | (np.uint64(64) + lanes),
         4 + 4 + 4),                                                             # shared-space R/W affine: mask
        ((lanes % np.uint64(3)) << np.uint64(62) | (np.uint64(4096) + lanes), 4 + 16 + 8),   # R/W/A affine: nibbles
        (np.full(32, 77, np.uint64), 4 + 4 + 8),                                  # broadcast read, k = 0
        (np.uint64(5) * lanes, 4 + 4 + 4 + 4 * 8),                                # reads, max delta 155 -> k = 8, u32 base
        (np.uint64(1 << 40) + np.uint64(5) * lanes, 4 + 4 + 8 + 4 * 8),           # the same above 2^32: u64 base
        (np.uint64(7) + (lanes % np.uint64(2)), 4 + 4 + 8 + 4 * 1),               # k = 1 keeps the u64 base
        (np.full(32, (3 << 62) | 5, np.uint64), 4 + 256),                         # unknown control word -> raw
    ]
    for row, size in cases:
        _, po, _ = _roundtrip(row.astype(np.uint64), np.array([0, 1], np.uint64))
        assert int(po[1]) == size, (row[:2], int(po[1]), size)


@pytest.mark.parametrize("options", [0, 16, 32, 256])
def test_packed_replay_matches_oracle(options):
    tr = _random_batch(91, 40, max_blocks=5, max_warps=8, max_lanes=32, max_slots=12, n_words=700,
                       spaces=(0, 1), p_barrier=0.2, p_skip=0.3)
    o = oracle_set(tr)
    races, fl = hr().check_trace(tr, packed=True, options=options)
    assert ([tuple(r) for r in races], fl) == o
    for t in (tp.c1_tree_reduction(removed=8), tp.listing2(3, 4, 32), tp.listing4(1, 4, 32, 100)):
        races, fl = hr().check_trace(t, packed=True, options=options)
        assert ([tuple(r) for r in races], fl) == oracle_set(t)


@pytest.mark.parametrize("chunk", ["4096", "1000000000"])
def test_packed_host_replay_chunked(chunk, monkeypatch):
    """hr_replay_trace_host on a PACKED host trace: chunks copied, decoded and
    replayed in order; repeated on one context."""
    monkeypatch.setenv("HR_HOST_CHUNK_BYTES", chunk)
    h = hr()
    tr = _random_batch(82, 6, max_blocks=40, max_warps=4, max_lanes=32, max_slots=10, n_words=300,
                       spaces=(0, 1), grid=(37, 3, 32))
    for t in (tr, tp.listing2(33, 2, 32)):
        gmax, smem = h.trace_extent(t)
        ck = h.Checker(gmax, smem)
        host = ck.pack(h.DeviceTrace.from_trace(t)).to_host()
        for _ in range(2):
            ck.reset()
            ck.replay_host(host)
            races, fl, _ = ck.report()
            assert ([tuple(r) for r in races], fl) == oracle_set(t)
        ck.close()


def test_packed_c5_planted_and_size():
    """C5 shape at 2^8 blocks: the packed host replay finds exactly the planted
    set, and the encoding is under half of C32's 160 B/row."""
    import torch
    h = hr()
    lb = 8
    rec, off, kd = c5.gpu_trace(lb, device="cuda")
    ck = h.Checker(c5.total_words(lb))
    dt = h.DeviceTrace(rec, off, kd)
    pk = ck.pack(dt)
    assert pk.record_bytes() < 0.5 * 160 * dt.n_rows
    host = pk.to_host()
    del rec, dt
    torch.cuda.synchronize()
    ck.replay_host(host)
    raw, fl = ck.report_raw()
    assert fl == 0
    assert sorted(zip(raw["word"].tolist(), raw["scope"].tolist())) == c5.planted(lb)
    ck.close()


def test_decreasing_warp_off_rejected():
    h = hr()
    rec = np.zeros(64, np.uint64)
    with pytest.raises(h.HiraceError):
        _roundtrip(rec, np.array([0, 2, 1], np.uint64))


def test_classes_reject_packed():
    h = hr()
    tr = tp.listing2(3, 4, 32)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem)
    pk = ck.pack(h.DeviceTrace.from_trace(tr))
    ck.replay(pk)
    raw, _ = ck.report_raw()
    assert len(raw)
    with pytest.raises(h.HiraceError):
        ck.classes(pk, raw)
    ck.close()
