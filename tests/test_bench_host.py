"""Host-side logic of bench.py (no GPU): the clock sampler's window filter and
throttle-reason parsing, and the reference arm's JSON line on a tiny sample."""
import datetime
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _line(ts, sm, reasons=("Not Active",) * 4):
    stamp = datetime.datetime.fromtimestamp(ts).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
    return ", ".join([stamp, "0", str(sm), "1965", "700.0", "0x0"] + list(reasons))


def test_clock_window_and_reasons():
    t0 = 1_800_000_000.0
    text = "\n".join([_line(t0 - 5, 900),                      # before the timed region: ignored
                      _line(t0 + 0.1, 1965), _line(t0 + 0.2, 1965),
                      _line(t0 + 0.3, 1950, ("Not Active", "Not Active", "Not Active", "Active")),
                      _line(t0 + 9, 300, ("Active",) * 4)])    # after it: ignored
    out = bench.Clocks.parse(text, t0, t0 + 1)
    assert out["samples"] == 3 and out["sm_mhz"] == 1965 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]
    assert bench.Clocks.parse(text)["samples"] == 5            # no window: every sample


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-lb", "4"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "accesses/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    cb = d["cpu_baseline"]
    # SURVEY §8(d) "Oracle timing": the host's core count and model, and the labelled extrapolation
    assert cb["host_cpu_count"] == os.cpu_count() and cb["cores"] == 1
    assert "host_cpu_model" in cb and "EXTRAPOLATED" in cb["extrapolation"]
    assert cb["extrapolated_full_step_s"] > 0
