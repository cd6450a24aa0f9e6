"""bench.py contract pieces that run without a GPU: the clock-sample summary
and the reference arm's JSON line (the CPU port of the reference kernels,
timed on a bounded sample of config 2)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_clock_summary_uses_in_region_samples():
    cs = bench.ClockSampler(0)
    cs.lines = ["345, 1965, 0x0, Not Active, Not Active, Not Active, Not Active",   # before the region
                "1965, 1965, 0x0, Not Active, Not Active, Not Active, Active",
                "1950, 1965, 0x0, Not Active, Not Active, Not Active, Not Active"]
    cs.n0 = 1
    s = cs.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1957.5 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]


def test_clock_summary_without_samples():
    cs = bench.ClockSampler(0)
    assert cs.summary()["samples"] == 0


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env={**os.environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
