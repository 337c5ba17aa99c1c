"""Multi-process (world_size 2, gloo on 127.0.0.1) test of the host side of
the address-sharded replay: shard compaction + race-set allgather + merge.
The per-rank local race sets come from the oracle (no GPU here); the merged
result must equal the oracle on the unsharded trace."""
import os
import random
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2401_04701_b200 import multigpu
from tracegen import programs as tp
from tracegen import c5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_raw(races):
    a = np.zeros(len(races), dtype=multigpu.RACE_DTYPE)
    for i, r in enumerate(races):
        a[i] = (r.word, r.block, r.kernel, 0, r.space, r.scope, 0, 0)
    return a


def _worker_device_exchange(rank, world, port, path, out_dir):
    """Same as _worker through multigpu.DeviceExchange (fixed-size buffers +
    all_gather_into_tensor, merged on collect), with a small cap so one rank's
    set overflows it once and the full-path fallback is exercised too."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    trace = np.load(path, allow_pickle=True)["t"].item()
    res = oracle.check(multigpu.shard_trace(trace, rank, world))
    raw = _to_raw(res.races)
    ex = multigpu.DeviceExchange(None, cap=1 << 12, device="cpu")
    ex.step_from_host(raw, res.flags)
    merged, flags = ex.collect()
    small = multigpu.DeviceExchange(None, cap=2, device="cpu")
    small.step_from_host(raw, res.flags)
    merged2, _ = small.collect(fallback_raw=lambda: (raw, res.flags))
    assert np.array_equal(merged, merged2)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), merged)
    dist.destroy_process_group()


def _worker(rank, world, port, path, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    trace = np.load(path, allow_pickle=True)["t"].item()
    local = multigpu.shard_trace(trace, rank, world)
    res = oracle.check(local)
    # every local race is owned by this rank
    for r in res.races:
        if r.space == 0:
            assert multigpu.shard_owner(r.word >> 3, world) == rank
        else:
            assert r.block % world == rank
    merged, flags = multigpu.exchange_races(_to_raw(res.races), res.flags)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), merged)
    dist.destroy_process_group()


def _run(trace, world=2, worker=None):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.npz")
        np.savez(path, t=np.array(trace, dtype=object))
        mp.spawn(worker or _worker, args=(world, _free_port(), path, d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])          # identical on every rank
    return [(int(x["kernel"]), int(x["space"]), int(x["block"]), int(x["word"]), int(x["scope"]))
            for x in outs[0]]


def test_gloo_sharded_random_programs():
    rng = random.Random(77)
    kernels = []
    for _ in range(3):
        t = tp.random_program(rng, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=3000,
                              spaces=(0, 1), grid=(4, 3, 32))
        kernels.append(t)
    from tracegen.format import make_trace, Kernel
    ks = []
    for t in kernels:
        b, w, l, sm, _ = (int(x) for x in t.kdesc[0, :5])
        k = Kernel(b, w, l, sm)
        k.rows = [t.rec[int(t.warp_off[i]) * 32: int(t.warp_off[i + 1]) * 32].reshape(-1, 32)
                  for i in range(b * w)]
        ks.append(k)
    trace = make_trace(ks)
    want = [tuple(r) for r in oracle.check(trace).races]
    assert len(want) > 5
    assert _run(trace, 2) == want


def test_gloo_device_exchange_c5_and_random():
    trace = c5.cpu_trace(3)
    want = [tuple(r) for r in oracle.check(trace).races]
    assert _run(trace, 2, _worker_device_exchange) == want
    rng = random.Random(9)
    t = tp.random_program(rng, max_slots=12, n_words=4000, spaces=(0, 1), grid=(4, 2, 32))
    assert _run(t, 2, _worker_device_exchange) == [tuple(r) for r in oracle.check(t).races]


def test_gloo_sharded_c5():
    trace = c5.cpu_trace(3)
    want = [tuple(r) for r in oracle.check(trace).races]
    assert _run(trace, 2) == want


@pytest.mark.parametrize("n", [2, 4])
def test_shard_trace_partition_single_process(n):
    rng = random.Random(5)
    trace = tp.random_program(rng, max_slots=12, n_words=5000, spaces=(0, 1), grid=(3, 2, 32))
    want = [tuple(r) for r in oracle.check(trace).races]
    union = []
    for r in range(n):
        union += [tuple(x) for x in oracle.check(multigpu.shard_trace(trace, r, n)).races]
    assert sorted(union) == want
