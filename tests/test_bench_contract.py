"""bench.py's JSON line against the driver contract (keys, types, units).

The reference arm (the CPU oracle, tier framing) runs here on the CPU, alone and
under torchrun with two gloo ranks (rank 0 alone prints, the other exits 0);
the GPU arm's line (roofline, clocks, e2e, launch count) is checked on a B200
with a short run.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check_e2e(e, unit):
    assert e["unit"] == unit and e["value"] > 0
    assert isinstance(e["h2d_bytes_per_step"], int) and isinstance(e["d2h_bytes_per_step"], int)


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True and d["value"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    _check_e2e(d["e2e"], d["unit"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_under_torchrun_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29577", "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)   # rank 0 alone prints
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["warmup"] == 3


@pytest.mark.gpu
def test_gpu_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--layers", "4", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["dtype"] == "bf16" and d["scaling"] in ("weak", "strong")
    assert "workload" in d["config"] and "l2" in d["config"]
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and ro["achieved"] > 0 and ro["peak"] > 0
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-6
    assert "traffic" in ro
    clk = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= clk.keys()
    assert isinstance(d["gpu_launches"], int) and d["gpu_launches"] > 0
    _check_e2e(d["e2e"], d["unit"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
