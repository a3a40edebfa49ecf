"""bench.py's output contract, on CPU: the reference arm's JSON line (the oracle
port, one whole cfg-1 slice per step) carries the keys the driver parses, and
its `config` is the same object the GPU arm prints (the driver compares them),
with the workload named."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_line_keys():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    import bench
    assert line["config"] == bench._config(bench.WORKLOADS["cfg1"], 1)
    assert line["config"]["workload"] == "cfg1-cpu-reference-shape"


def test_default_workload_is_the_headline():
    import bench
    assert bench.WORKLOAD["name"] == "cfg4-long-window-k300"
    w = bench.WORKLOADS["cfg4"]
    assert (w["c"], w["k"], w["k_prime"], w["g"], w["hosts"], w["packets"]) == \
        (28, 300, 300, 1024, 1_000_000, 5_000_000)


def test_reported_fractions_are_bounded_by_their_ceilings():
    """The roofline helper: HBM fraction = algorithmic bytes / time / peak, and
    an L2 fraction that is the probes' time over the kernel's time."""
    import bench
    l2 = {"random_sector_reads_G_per_s": 200.0, "random_u16_stores_G_per_s": 100.0,
          "random_red_or_G_per_s": 100.0, "stream_read_GB_per_s": 5000.0}
    w = bench.WORKLOADS["cfg4"]
    k = {"ms_per_launch": 0.1}
    r = bench._roofline("scan", k, 200_000_000, 6500.0, "measured", l2, 5_000_000, 1 << 28, 2,
                        w, True, "cfg4", True)
    assert r["bound"] == "hbm"
    assert abs(r["achieved"] - 2000.0) < 1e-6 and abs(r["frac"] - 2000.0 / 6500.0) < 1e-9
    # 5M reads at 200 G/s + 5M reds at 100 G/s = 75 us over 100 us
    assert abs(r["l2"]["frac"] - 0.75) < 1e-9 and r["l2"]["binding"]


def test_gather_roofline_uses_the_l2_ceiling():
    """The full-recompute g0 gathers an L2-resident bitmap: its fraction is taken
    against the probed L2 random-sector rate (no fraction far above 1)."""
    import bench
    l2 = {"random_sector_reads_G_per_s": 250.0, "random_u16_stores_G_per_s": 100.0,
          "random_red_or_G_per_s": 100.0, "stream_read_GB_per_s": 5000.0}
    w = bench.WORKLOADS["cfg4"]
    hosts = 1_000_000
    alg = hosts * (32 * w["g"] + 12)
    r = bench._roofline("g0", {"ms_per_launch": 4.0}, alg, 6500.0, "measured", l2, 5_000_000,
                        1 << 28, 2, w, True, "cfg4", True)
    assert abs(r["peak"] - 8000.0) < 1e-9 and abs(r["frac"] - r["achieved"] / 8000.0) < 1e-12
    assert abs(r["hbm_frac"] - r["achieved"] / 6500.0) < 1e-12
    assert r["frac"] < 1.2 and r["hbm_frac"] > 1.0
