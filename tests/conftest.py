"""Shared pytest configuration.

``-m gpu`` tests need a B200 and call the CUDA library through its C ABI;
everything else runs on the CPU (oracle vs golden vectors, host logic,
library symbol exports, gloo multi-process view sharding).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name: str) -> dict:
    """{case: {key: array}} from tests/golden/<name>.npz."""
    out: dict = {}
    with np.load(GOLDEN / f"{name}.npz") as z:
        for key in z.files:
            case, field = key.split("/", 1)
            out.setdefault(case, {})[field] = z[key]
    return out


def cam_from_row(row, view_id=0):
    """CameraView from the golden camera row [W, H, fx, fy, cx, cy, near, w2c(16)]."""
    from paper_2409_08270_b200.scene import CameraView
    return CameraView(view_id=view_id, width=int(row[0]), height=int(row[1]), fx=float(row[2]),
                      fy=float(row[3]), cx=float(row[4]), cy=float(row[5]),
                      world_to_camera=np.asarray(row[7:23]).reshape(4, 4), near_clip=float(row[6]))


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(20240811)
