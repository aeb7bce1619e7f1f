"""bench.py's driver contract: one JSON line with the required keys, for our arm and the
reference arm (small settings; the driver's own runs use the defaults)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run(*args: str) -> dict:
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "1", "--warmup", "3", "--replicas", "2", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and "workload" in d["config"]
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    c4 = d["cfg4_circuits"]
    assert c4["circuits"] == 1024 and c4["circuits_per_s"] > 0 and 0 < c4["frac"] < 1
    cf = d["configs"]
    assert {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5"} <= set(cf)
    assert all(0 < cf[k]["frac"] < 1 for k in ("cfg3", "cfg4", "cfg5"))
    assert cf["cfg1"]["s"] > 0 and cf["cfg2"]["energies_per_s"] > 0 and cf["cfg2"]["vectors"] == 64


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert {"kind", "cores", "sample", "value"} <= set(d["cpu_baseline"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
