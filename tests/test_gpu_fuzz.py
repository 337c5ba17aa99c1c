"""Schedule fuzzing (SURVEY §8(c) GPU-path tests): the -DHR_FUZZ build
(libhirace_fuzz.so) sleeps a pseudo-random time before a quarter of the
shadow CASes, folds same-word lane groups in descending lane order, and maps
CUDA blocks to simulated blocks in reverse, so the per-word commit orders
differ from the production build's.  Every order is a linear extension of
happens-before, so the racy set must equal the oracle's in every run.

The fuzz library is loaded in a subprocess (HIRACE_LIB) so this process keeps
the production library."""
import json
import os
import random
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases():
    from tests.test_gpu_parity import _random_batch
    from tracegen import programs as tp, stencil
    out = [("c1_s8", tp.c1_tree_reduction(removed=8)), ("c1_free", tp.c1_tree_reduction(removed=None)),
           ("listing2", tp.listing2(3, 4, 32)), ("listing4", tp.listing4(1, 4, 32, 100)),
           ("stencil64", stencil.stencil_trace(removed=20, n=64))]
    out.append(("wide", _random_batch(100, 40, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                                      spaces=(0, 1), p_barrier=0.25, p_skip=0.5)))
    out.append(("hot", _random_batch(7, 10, max_blocks=16, max_warps=32, max_lanes=32, max_slots=8, n_words=3,
                                     spaces=(0, 1), p_skip=0.2)))
    out.append(("hot_ra", _random_batch(8, 10, max_blocks=16, max_warps=32, max_lanes=32, max_slots=8, n_words=3,
                                        kinds="RA", spaces=(0, 1), p_skip=0.2)))
    out.append(("small", _random_batch(3, 300, max_blocks=2, max_warps=2, max_lanes=2, max_slots=5, n_words=2,
                                       spaces=(0, 1))))
    return out


def worker() -> None:
    """Runs under HIRACE_LIB=libhirace_fuzz.so; prints one JSON line."""
    import oracle
    from paper_2401_04701_b200 import build, hirace
    assert hirace.load()._name == build.LIB_FUZZ
    bad, runs, witnesses = [], 0, []
    for name, tr in _cases():
        exp = ([tuple(r) for r in oracle.check(tr).races], oracle.check(tr).flags)
        for options in (16, 32, 256, 256 | 1024, 512, 1):
            for rep in range(3):
                races, fl = hirace.check_trace(tr, options=options)
                runs += 1
                if ([tuple(r) for r in races], fl) != exp:
                    bad.append((name, options, rep))
                if name == "hot" and options == 16:
                    witnesses.append(_witness(tr))
    print(json.dumps({"runs": runs, "bad": bad, "witnesses": witnesses}))


def _witness(tr):
    """Schedule-dependent diagnostics of the races (hr_race.first_tid,
    first_kind, prev_state): which access moved each word into RACE."""
    from paper_2401_04701_b200 import hirace
    gmax, smem = hirace.trace_extent(tr)
    ck = hirace.Checker(gmax, smem, options=16)
    ck.replay(hirace.DeviceTrace.from_trace(tr))
    raw, _ = ck.report_raw()
    ck.close()
    return sorted((int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["first_tid"]),
                   int(r["first_kind"]), int(r["prev_state"])) for r in raw)


def test_fuzzed_schedules_match_oracle():
    from paper_2401_04701_b200 import build
    lib = build.build_fuzz()
    # additive PYTHONPATH: the driver's load-recording hook (sitecustomize) must stay on the path
    pp = os.environ.get("PYTHONPATH", "")
    env = dict(os.environ, HIRACE_LIB=lib, PYTHONPATH=ROOT + (os.pathsep + pp if pp else ""))
    out = subprocess.run([sys.executable, "-c", "import tests.test_gpu_fuzz as m; m.worker()"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["runs"] == 9 * 6 * 3
    assert res["bad"] == []
    # the fuzzing is effective: the race witnesses (which access entered RACE
    # first) differ between fuzzed runs or from the production build
    prod = [tuple(x) for x in _witness(dict(_cases())["hot"])]
    fuzzed = {tuple(map(tuple, w)) for w in res["witnesses"]}
    assert len(fuzzed) > 1 or fuzzed != {tuple(prod)}


def test_fuzz_build_differs_from_production():
    """The fuzz library really is a different build: jitter sleeps in the check
    path (the production build's only NANOSLEEPs are CUB's scan back-off)."""
    from paper_2401_04701_b200 import build
    lib = build.build_fuzz()
    fuzz = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    prod = subprocess.run(["cuobjdump", "-sass", build.build()], capture_output=True, text=True).stdout
    assert fuzz.count("NANOSLEEP") > prod.count("NANOSLEEP") + 50
