"""C-ABI library: builds for sm_100a, loads, exports every symbol include/hr.h
declares, carries the generated FSM table, and fails loudly without a GPU."""
import ctypes
import re
import os

import numpy as np
import pytest

from paper_2401_04701_b200 import build, hirace
from paper_2401_04701_b200.fsm import generate as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("hr.h", "hr_bench.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        src = re.sub(r"HR_HD[^{;]*\{.*?\n\}", "", src, flags=re.S)     # header-inline helpers, not exports
        names |= set(re.findall(r"\b(hrb?_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


def test_library_builds_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(build.build())
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    from paper_2401_04701_b200 import online
    assert set(names) == set(hirace.EXPORTS) | set(online.EXPORTS)


def test_compiled_table_matches_generator():
    table, flags, _ = G.build_table()
    t, f = hirace.hr_fsm_table()
    assert t == table and f == flags


def test_sass_uses_native_64bit_atomics():
    """ATOMG.E.CAS.64 for global, ATOMS.CAS.64 for shared,
    MATCH.ANY.U64 for coalescing, on sm_100a."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"ATOMG\.E\.CAS\.64", out)
    assert re.search(r"ATOMS\.CAS\.64", out)
    assert "MATCH.ANY.U64" in out


def test_init_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(hirace.HiraceError):
        hirace.hr_init()


def test_config_validation():
    lib = hirace.load()
    ctx = ctypes.c_void_p()
    bad = hirace.HrConfig(5, 27, 20, 20, 16, 0, 0)      # widths must sum to 64
    assert lib.hr_init(ctypes.byref(bad), ctypes.byref(ctx)) == hirace.HR_E_ARG
    bad = hirace.HrConfig(6, 26, 16, 16, 16, 0, 0)
    assert lib.hr_init(ctypes.byref(bad), ctypes.byref(ctx)) == hirace.HR_E_ARG


def test_merge_races_host_only():
    """hr_merge_races (host C, no GPU): the sorted (kernel, space, block, word)
    union of shuffled, duplicated shard reports, one record per address with the
    widest scope."""
    rng = np.random.default_rng(7)
    n = 5000
    a = np.zeros(n, dtype=hirace.RACE_DTYPE)
    a["word"] = rng.integers(0, 1 << 40, n)
    a["kernel"] = rng.integers(0, 3, n)
    a["space"] = rng.integers(0, 2, n)
    a["block"] = np.where(a["space"] == 1, rng.integers(0, 4, n), 0xFFFFFFFF)
    a["scope"] = 1
    dup = a[rng.choice(n, 700, replace=False)].copy()
    dup["scope"] = 2                                   # a later RACE_GRID upgrade of the same address
    parts = np.concatenate([a, dup, a[:300]])
    rng.shuffle(parts)
    got = hirace.hr_merge_races(parts)
    keys = {}
    for r in parts:
        k = (int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]))
        keys[k] = max(keys.get(k, 0), int(r["scope"]))
    want = sorted(keys.items())
    assert [((int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"])), int(r["scope"])) for r in got] == want
    assert len(hirace.hr_merge_races(parts[:0])) == 0


def test_header_shard_owner_matches_python(tmp_path):
    """include/hr.h's inline hr_shard_owner / hr_shard_granule (compiled by
    gcc here) == multigpu.shard_owner, and hr_shard_granule inverts it."""
    import subprocess
    import numpy as np
    from paper_2401_04701_b200.multigpu import shard_owner
    c = tmp_path / "own.c"
    c.write_text("""#include <stdio.h>
#include "hr.h"
int main(void) {
    for (unsigned l = 0; l <= 3; l++)
        for (unsigned long long g = 0; g < 4096; g += 7) {
            unsigned o = hr_shard_owner(g * 977ull + (g << 33), l);
            unsigned long long back = hr_shard_granule((g * 977ull + (g << 33)) >> l, o, l);
            printf("%u %llu %u %d\\n", l, g, o, back == g * 977ull + (g << 33));
        }
    return 0;
}
""")
    exe = tmp_path / "own"
    subprocess.run(["gcc", "-O1", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    n = 0
    for line in out:
        if not line:
            continue
        l, g, o, inv = (int(x) for x in line.split())
        gran = g * 977 + (g << 33)
        assert inv == 1
        assert shard_owner(np.uint64(gran), 1 << l) == o
        n += 1
    assert n == 4 * len(range(0, 4096, 7))
