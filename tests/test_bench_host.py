"""Host-side pieces of bench.py (no GPU): the reference (oracle) arm's JSON line on a small
config, the whole-step roofline arithmetic and the clock-sample reduction."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "freq-bins/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg1")


def test_step_roofline_arithmetic():
    import bench
    st = {"gs_bytes": 6.4708e12, "das_flops": 2 * 36.0e12 * 1e-3}   # 1 s of HBM, 1 ms of fp64 (half)
    r = bench.step_roofline(st, 1000, 6470.8, 2004.0)
    assert abs(r["gs_stream_ms"] - 1000.0) < 1e-6
    assert abs(r["psf_write_ms"] - 1.0) < 1e-9
    assert abs(r["das_fp64_ms"] - 1.0) < 1e-9
    assert abs(r["roofline_ms"] - 1002.0) < 1e-6 and abs(r["frac"] - 0.5) < 1e-9


def test_clock_sampler_reduction():
    import bench
    c = bench.ClockSampler(0)
    c.proc = None
    assert c.stop()["reasons"] == ["nvidia-smi unavailable"]

    class FakeProc:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0
    c.proc = FakeProc()
    c.samples = [["1950", "1965", "900", "Not Active", "Not Active", "Not Active", "Active"],
                 ["1900", "1965", "910", "Not Active", "Not Active", "Not Active", "Not Active"],
                 ["1920", "1965", "905", "Not Active", "Not Active", "Not Active", "Active"]]
    out = c.stop()
    assert out["sm_mhz"] == 1920.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"] and out["samples"] == 3


def test_multi_gpu_value_is_band_over_max_rank_time():
    """N > 1 defaults to strong scaling: value = the band's bins / the max-over-ranks ms (the
    north_star's 256-bin workload sharded); weak (explicit) counts every rank's own band."""
    import bench
    assert abs(bench.bench_value(256, 32, 8, "strong", 20.0) - 256 / 0.020) < 1e-6
    assert abs(bench.bench_value(256, 256, 1, "strong", 50.0) - 256 / 0.050) < 1e-6
    assert abs(bench.bench_value(256, 256, 1, "weak", 50.0) - 256 / 0.050) < 1e-6
    assert abs(bench.bench_value(256, 256, 4, "weak", 50.0) - 4 * 256 / 0.050) < 1e-6
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'args.scaling = "strong" if world > 1' in src


def test_traffic_only_from_a_matching_capture():
    """roofline.traffic is read only under the exact config/variant key it was captured on."""
    import argparse

    import bench
    import synth
    a = argparse.Namespace(order=1, dr=False, alt=False, input="csm", scaling=None)
    b = argparse.Namespace(order=3, dr=False, alt=False, input="csm", scaling=None)
    assert bench.variant_key(synth.CONFIGS["cfg3"], a) != bench.variant_key(synth.CONFIGS["cfg3"], b)
    assert bench.variant_key(synth.CONFIGS["cfg3"], a) != bench.variant_key(synth.CONFIGS["cfg5"], a)
