"""Closed-form label assignment on the GPU (reference ``solver.py:33-172``).

``assign_binary`` / ``assign_scene`` keep the reference signatures, checks,
messages and ``Assignment`` result; the one-vs-rest argmax runs in the CUDA
kernel ``fs_assign`` (``csrc/fs_assign.cu``), which reproduces the
reference's float32 operation sequence bit for bit.  The exhaustive
objective / brute-force certification oracles (``solver.py:175-239``) stay
on the CPU in the reference and are not part of this path.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .contributions import ContributionMatrix

UNOBSERVED_EPS = 1e-12  # reference solver.py:29


@dataclass
class Assignment:
    """Per-Gaussian membership (reference ``solver.py:33-108``).

    Binary mode: ``labels`` (N uint8, 1 = foreground).  Scene mode:
    ``membership`` (E x N uint8), row 0 = complement of the object rows.
    """

    mode: str
    gamma: float
    labels: Optional[np.ndarray] = None
    membership: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        if self.mode not in ("binary", "scene"):
            raise ValueError(f"unknown assignment mode {self.mode!r}")
        if self.labels is not None:
            self.labels = np.asarray(self.labels, dtype=np.uint8)
        if self.membership is not None:
            self.membership = np.asarray(self.membership, dtype=np.uint8)

    @property
    def num_gaussians(self) -> int:
        return int(self.labels.shape[0] if self.mode == "binary" else self.membership.shape[1])

    @property
    def num_objects(self) -> int:
        return 2 if self.mode == "binary" else int(self.membership.shape[0])

    def members(self, object_id: int) -> np.ndarray:
        if not 0 <= object_id < self.num_objects:
            raise ValueError(f"unknown object id {object_id}")
        if self.mode == "binary":
            fg = self.labels.astype(bool)
            return fg if object_id == 1 else ~fg
        return self.membership[object_id].astype(bool)

    def member_counts(self) -> list:
        cached = getattr(self, "_device_counts", None)  # counted on the GPU by LabelSolver.assign
        if cached is not None:
            return list(cached)
        if self.mode == "binary":
            fg = int(np.count_nonzero(self.labels))
            return [self.num_gaussians - fg, fg]
        return self.membership.sum(axis=1, dtype=np.int64).tolist()

    def save(self, path) -> None:
        head = json.dumps({"mode": self.mode, "gamma": self.gamma, "E": self.num_objects,
                           "N": self.num_gaussians}).encode("ascii")
        payload = self.labels if self.mode == "binary" else self.membership
        with open(path, "wb") as fh:
            fh.write(struct.pack("<I", len(head)) + head)
            fh.write(np.ascontiguousarray(payload).tobytes())

    @classmethod
    def load(cls, path) -> "Assignment":
        with open(path, "rb") as fh:
            (hlen,) = struct.unpack("<I", fh.read(4))
            header = json.loads(fh.read(hlen).decode("ascii"))
            payload = np.frombuffer(fh.read(), dtype=np.uint8)
        mode, e, n = header["mode"], header["E"], header["N"]
        if mode == "binary":
            if payload.size != n:
                raise ValueError(f"{path}: expected {n} labels, got {payload.size}")
            return cls(mode=mode, gamma=header["gamma"], labels=payload.copy())
        if payload.size != e * n:
            raise ValueError(f"{path}: expected {e}x{n} membership payload")
        return cls(mode=mode, gamma=header["gamma"], membership=payload.reshape(e, n).copy())


def _check_gamma(gamma: float) -> float:
    gamma = float(gamma)
    if not -1.0 <= gamma <= 1.0:
        raise ValueError(f"gamma must lie in [-1, 1], got {gamma}")
    return gamma


def assign_binary(matrix: ContributionMatrix, gamma: float) -> Assignment:
    """Foreground / background argmax with background bias (``solver.py:140-153``)."""
    from . import _native

    gamma = _check_gamma(gamma)
    if matrix.num_objects != 2:
        raise ValueError(f"binary assignment requires E=2, got E={matrix.num_objects}")
    labels = _native.assign(matrix.values, gamma, _native.MODE_BINARY)
    return Assignment(mode="binary", gamma=gamma, labels=labels)


def assign_scene(matrix: ContributionMatrix, gamma: float) -> Assignment:
    """One-vs-rest argmax for every object in one pass (``solver.py:156-172``)."""
    from . import _native

    gamma = _check_gamma(gamma)
    e, n = matrix.values.shape
    if e < 2:
        raise ValueError(f"scene assignment requires E>=2, got E={e}")
    membership = _native.assign(matrix.values, gamma, _native.MODE_SCENE)
    return Assignment(mode="scene", gamma=gamma, membership=membership)
