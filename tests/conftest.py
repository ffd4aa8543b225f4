"""Shared test plumbing: the gpu marker, golden fixtures, case builders."""

from __future__ import annotations

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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "cases.json").read_text())


@pytest.fixture(scope="session")
def golden_renders():
    return dict(np.load(GOLDEN / "renders.npz"))


@pytest.fixture(scope="session")
def golden_prep():
    return dict(np.load(GOLDEN / "prep.npz"))


@pytest.fixture(scope="session")
def golden_sampling():
    return dict(np.load(GOLDEN / "sampling.npz"))


from oracle.oracle import PRESET_POINTS  # noqa: E402  (transfer.py:207-228)


def tf_arrays(spec):
    """(values, rgba, domain) of a golden TF spec, independent of the product."""
    if "preset" in spec:
        pts = PRESET_POINTS[spec["preset"]]
        dom = (-1000.0, 2000.0)
    else:
        pts = [tuple(p) for p in spec["points"]]
        dom = tuple(spec["domain"]) if spec["domain"] else (pts[0][0], pts[-1][0])
    v = np.array([p[0] for p in pts], dtype=np.float64)
    c = np.array([p[1:] for p in pts], dtype=np.float64)
    return v, c, (float(dom[0]), float(dom[1]))


DEFAULT_SETTINGS = dict(step=None, interpolation="trilinear", classification="post", mode="dvr",
                        isovalue=None, lighting=True, early_termination_alpha=0.99,
                        use_blocks=False, block_size=64, overlap=3, background=(0.0, 0.0, 0.0, 1.0),
                        ambient=0.1, diffuse=0.7, specular=0.2, shininess=32.0)


def settings_dict(case):
    s = dict(DEFAULT_SETTINGS)
    s.update(case["settings"])
    s["background"] = tuple(s["background"])
    return s


def compare_render(name, golden, out, pixels, stats, taken=None, blocks_hit=None):
    """Assert bit-exact parity with a golden render; returns (max|d out|, max|d px|)."""
    g_out = golden[name + "__out"]
    d_out = float(np.abs(out.reshape(-1, 4) - g_out).max())
    d_px = int(np.abs(pixels.astype(int) - golden[name + "__pixels"].astype(int)).max())
    assert list(stats) == golden[name + "__stats"].tolist(), (name, list(stats), golden[name + "__stats"].tolist())
    if taken is not None:
        assert np.array_equal(taken, golden[name + "__taken"]), name
    if blocks_hit is not None:
        assert np.array_equal(blocks_hit, golden[name + "__blocks_hit"]), name
    return d_out, d_px
