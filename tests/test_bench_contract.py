"""bench.py host-side pieces that run without a GPU: the clock sampler's
summary (what the JSON line's ``clocks`` key reports) and the config table."""

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_clock_summary_median_and_reasons(bench):
    c = bench.ClockSampler(0)
    c.source = "nvml"
    c.samples = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active"],
                 ["1900", "1965", "Not Active", "Not Active", "Not Active", "Active"],
                 ["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active"]]
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    assert s["samples"] == 3 and s["source"] == "nvml"


def test_clock_summary_flags_throttle(bench):
    c = bench.ClockSampler(0)
    c.samples = [["1200", "1965", "Active", "Not Active", "Active", "Not Active"]]
    assert c.summary()["reasons"] == ["hw_slowdown", "sw_thermal_slowdown"]


def test_clock_summary_unsampled(bench):
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]


def test_sampler_without_gpu_terminates(bench):
    # No GPU here: both NVML and nvidia-smi fail; the thread must still stop.
    with bench.ClockSampler(0) as c:
        pass
    assert not c._t.is_alive()


def test_configs_match_baseline_shapes(bench):
    cfg = bench.CONFIGS
    assert cfg["cfg1"]["N"] == 4096 and cfg["cfg1"]["d"] == 2
    assert cfg["cfg2"]["N"] == 1048576 and cfg["cfg2"]["kernel"] == "log2d"
    assert cfg["cfg3"]["N"] == 1048576 and cfg["cfg3"]["d"] == 3
    for c in cfg.values():
        assert c["n_max"] == 64
