"""CPU: bench.py's clock sampler reports only the samples taken inside the timed region
(between mark() and stop()), falls back to the samples either side of a region shorter
than one polling period, and unions the throttle reasons it saw there."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _sampler(samples, t_mark):
    c = bench.ClockSampler(0)
    c.thread = threading.Thread(target=lambda: None)
    c.thread.start()
    c.done = threading.Event()
    c.max_mhz = 1965.0
    c.samples = samples
    c.t_mark = t_mark
    return c


def test_only_samples_inside_the_timed_region_count():
    now = time.perf_counter()
    samples = [(now - 2.0, 120.0, []),  # idle, before the region
               (now - 0.9, 1965.0, []), (now - 0.5, 1950.0, ["sw_power_cap"]), (now - 0.1, 1965.0, [])]
    clk = _sampler(samples, now - 1.0).stop()
    assert clk["samples"] == 3
    assert clk["sm_mhz"] == 1965.0
    assert clk["sm_max_mhz"] == 1965.0
    assert clk["reasons"] == ["sw_power_cap"]


def test_region_shorter_than_a_period_uses_the_neighbouring_samples():
    now = time.perf_counter()
    samples = [(now - 2.0, 120.0, []), (now - 0.01, 1965.0, []), (now + 5.0, 1965.0, ["hw_slowdown"])]
    c = _sampler(samples, now - 0.005)
    clk = c.stop()
    assert clk["samples"] == 2
    assert clk["reasons"] == ["hw_slowdown"]


def test_no_nvml_and_no_nvidia_smi_reports_none():
    c = bench.ClockSampler(0)
    c.thread = None
    c.proc = None
    assert c.stop() is None
