"""Shared fixtures. ``-m gpu`` tests need a B200; everything else runs on CPU."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and libbmps.so")


def load_golden(name: str):
    d = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return d, json.loads(str(d["meta"]))


def assert_scaled_close(got, ref, rtol=1e-10, what=""):
    """|got - ref| <= rtol * max|ref| over the output set (SURVEY §8(c) check)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if ref.size == 0:
        return
    scale = float(np.max(np.abs(ref)))
    err = np.abs(got - ref)
    worst = float(err.max())
    assert worst <= rtol * max(scale, 1e-300), (
        f"{what}: max |delta| {worst:.3e} > {rtol:g} * {scale:.3e}")


def split_lams(flat, dims):
    out, o = [], 0
    for d in dims:
        out.append(flat[o:o + d])
        o += d
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(2024)
