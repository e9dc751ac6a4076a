"""Host logic of bench.py (CPU): the clock sampler keeps only the samples of the timed region and reports
the throttle reasons the contract asks for."""
import datetime
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _ts(t):
    return datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]


def test_clock_samples_filtered_to_timed_region(tmp_path):
    t0 = 1_800_000_000.0
    rows = [  # timestamp, sm, max, hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        (t0 - 5.0, 1100, 1965, "Not Active", "Not Active", "Not Active", "Not Active"),   # warm-up: dropped
        (t0 + 0.05, 1600, 1965, "Not Active", "Not Active", "Not Active", "Active"),
        (t0 + 0.15, 1700, 1965, "Not Active", "Not Active", "Not Active", "Active"),
        (t0 + 0.25, 1500, 1965, "Not Active", "Not Active", "Not Active", "Not Active"),
        (t0 + 9.0, 900, 1965, "Active", "Not Active", "Not Active", "Not Active"),        # after: dropped
    ]
    p = tmp_path / "clk.csv"
    p.write_text("".join(f"{_ts(r[0])}, {r[1]}, {r[2]}, {r[3]}, {r[4]}, {r[5]}, {r[6]}\n" for r in rows))
    out = bench.ClockSampler.parse(str(p), t0, t0 + 0.3)
    assert out["samples"] == 3
    assert out["sm_mhz"] == 1600 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]
    everything = bench.ClockSampler.parse(str(p), None, None)  # no timed region known: every sample
    assert everything["samples"] == 5 and "hw_slowdown" in everything["reasons"]
