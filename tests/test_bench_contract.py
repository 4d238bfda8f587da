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


def test_default_workload_is_cfg3_and_arms_share_config(bench):
    """The N=1 line is BASELINE configs[2] (the north-star HBM config); both
    arms build their config dict with the same function and keys."""
    import sys
    argv = sys.argv
    cfg = bench.CONFIGS["cfg3"]
    assert (cfg["N"], cfg["d"], cfg["kernel"], cfg["eps"]) == (1048576, 3, "lap3d", 1e-6)
    assert bench.DEFAULT_VARIANTS["cfg3"] == "h2star-bt"
    a = bench.config_dict(cfg, "h2star-bt", 1048576, 5, 11222271705, 1)
    b = bench.config_dict(cfg, "h2star-bt", 1048576, 5, 11222271705, 1)
    assert a == b and a["alg_bytes"] == 8 * 11222271705 + 16 * 1048576
    assert bench.recompute_for(cfg, "auto") == "m2l"
    assert bench.recompute_for(cfg, "none") == ""
    assert bench._is_p2p_phase("down_l5", "m2l") and not bench._is_p2p_phase("leaf", "m2l")
    assert not bench._is_p2p_phase("down_l3_red", "m2l")
    sys.argv = argv


def test_reference_arm_maps_no_repo_library(tmp_path, bench):
    """The reference arm's timing process loads an export written by a
    separate build process and never maps libh2g / libh2b."""
    import json
    import subprocess
    import sys
    code = (
        "import sys, json; sys.path.insert(0, %r); import bench, numpy as np;"
        "info = bench.export_for_reference('cfg1', 'h2star-bt', %r, 2);"
        "from paper_2309_14085_b200.packed import PackedOperator;"
        "op = PackedOperator.load(%r);"
        "from oracle.cpu_reference import time_sampled_matvec;"
        "r = time_sampled_matvec(op, np.random.default_rng(43).standard_normal(op.N), steps=1);"
        "maps = open('/proc/self/maps').read();"
        "print(json.dumps({'v': r['value'], 'so': ('libh2g' in maps) or ('libh2b' in maps)}))"
        % (ROOT, str(tmp_path / "op.npz"), str(tmp_path / "op.npz")))
    out = subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["v"] > 0 and res["so"] is False


def test_shared_build_for_multi_gpu_runs(tmp_path):
    """bench.py N > 1: rank 0 builds once (store=""), every rank loads the
    export and re-evaluates its raw kernel blocks natively -- bitwise the
    operator a stored build holds (reference engine.py:176-179, 309-318)."""
    import numpy as np
    import bench
    from paper_2309_14085_b200.builder import materialize_blocks
    cfg = dict(N=3000, d=3, kernel="lap3d", n_max=32, eps=1e-6, desc="small")
    calls = []
    op, tb = bench.build_op_shared(cfg, "h2star-bt", 0, 1, lambda: calls.append(1),
                                   tmp_root=str(tmp_path))
    assert calls == [1] and tb > 0
    full = materialize_blocks(op)
    ref, _ = bench.build_op(cfg, "h2star-bt")
    assert full.mem_scalars == ref.mem_scalars == op.mem_scalars
    # same blocks; the two blobs order and pad them differently
    from oracle.packed_matvec import packed_matvec
    q = np.random.default_rng(5).standard_normal(cfg["N"])
    assert np.array_equal(packed_matvec(full, q), packed_matvec(ref, q))
    assert bench.recompute_for(cfg, "auto", op) in ("m2l", "near,m2l")
