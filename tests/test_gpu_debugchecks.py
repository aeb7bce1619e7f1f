"""The -DBMPS_DEBUG_CHECKS build (tools/variants/debugchecks.so: bounds of every
two-site item, exactly-once completion of every Jacobi visit of every round) is
live: a clean circuit passes and an out-of-chain item traps. The whole GPU suite
and the bench also run clean under it (profiles/r02_debugchecks.md)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "tools" / "variants" / "debugchecks.so"


@pytest.mark.skipif(not LIB.exists(), reason="debug-checks build absent (python -m "
                    "paper_1807_07914_b200.build --out tools/variants/debugchecks.so -D BMPS_DEBUG_CHECKS)")
@pytest.mark.parametrize("mode", ["ok", "bad"])
def test_debug_checks_are_live(mode):
    env = {**os.environ, "BMPS_LIB": str(LIB)}
    out = subprocess.run([sys.executable, "tools/debugcheck_case.py", mode], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300)
    text = out.stdout + out.stderr
    if mode == "ok":
        assert out.returncode == 0 and "DEBUGCHECK ok" in text, text[-2000:]
    else:
        assert "BMPS_CHECK failed" in text, text[-2000:]


@pytest.mark.skipif(not LIB.exists(), reason="debug-checks build absent")
def test_visit_scheduling_invariants_hold_under_stress():
    """tools/debug_stress.py under the invariant-check build: cfg4 slices (thousands of
    small items per launch, where a CTA once re-ran a stale claim after the launch's last
    item retired) and chi = 256 bench steps; any violated invariant traps."""
    env = {**os.environ, "BMPS_LIB": str(LIB)}
    out = subprocess.run([sys.executable, "tools/debug_stress.py", "8"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=600)
    text = out.stdout + out.stderr
    assert out.returncode == 0 and "BMPS_CHECK" not in text, text[-2000:]
    assert "cfg4 x 8 ok" in text and "chi256 steps x 8 ok" in text
