"""bench.py's JSON contract: the reference arm on CPU (small sample), and our arm on the GPU
(small env count) -- every key the driver and the judge read, with sane values."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def check_base(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["dtype"] == "f64" and "workload" in d["config"]
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["unit"] == d["unit"]


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3", "--envs", "32")
    check_base(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract(cuda):
    d = run_bench("--steps", "5", "--warmup", "3", "--envs", "256", "--no-cpu", "--secondary", "")
    check_base(d)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] >= d["steps"]  # k_step once per timed step (+ render launches)
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["e2e"]["h2d_bytes_per_step"] == 256 * 3 * 4 and d["e2e"]["d2h_bytes_per_step"] > 0
    # the e2e path's own roofline: host<->device bytes per second over the measured PCIe copy rate
    er = d["e2e"]["roofline"]
    assert er["bound"] == "pcie" and er["peak"] > 1.0 and 0 < er["frac"] <= 1.5
    assert er["pcie_measured_gbs"]["d2h"] > 1.0 and er["pcie_measured_gbs"]["h2d"] > 1.0
    # the issue side of the roofline (ncu counts in profiles/issue.json, scaled to this launch)
    iss = r["issue"]
    assert iss is not None and 0 < iss["frac"] < 1 and 0 < iss["fp64_frac"] < 1
    assert iss["issue_slots_per_launch"] > iss["warp_inst_per_launch"] > 0


@pytest.mark.parametrize("config", ["c4", "c5"])
def test_reference_arm_render_workloads(config):
    """CPU reference arms exist for the rendering configs (BASELINE configs[3], [4]) and carry
    the same config dict as our arm (the driver compares them), the CPU model and the sample."""
    import importlib.util

    d = run_bench("--impl", "reference", "--config", config, "--steps", "1", "--warmup", "3")
    check_base(d)
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert d["config"] == bench.config_for(config, 1)
    cb = d["cpu_baseline"]
    assert "CPU:" in cb["sample"] and "sample of" in cb["sample"] and cb["value"] > 0
