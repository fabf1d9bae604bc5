"""Fused label solve with a device-resident contribution matrix.

The reference runs two calls, ``accumulate_contributions`` then
``assign_binary`` / ``assign_scene`` (``contributions.py:90``,
``solver.py:140/156``), and its service re-runs only the argmax when the
bias changes (``service.py:56-66,101-127``).  ``LabelSolver`` keeps the
float32 matrix on the GPU after one accumulation so every further gamma
costs one K4 launch plus the D2H of the labels.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .contributions import ContributionMatrix, validate_views
from .rasterizer import DEFAULT_BLEND, BlendConfig
from .solver import Assignment, _check_gamma


class LabelSolver:
    def __init__(self, scene, device: Optional[int] = None):
        from . import _native

        self._native = _native
        self.scene = scene
        self.ctx = _native.context(device)
        self.num_objects = 0
        self._A = None  # device float32 E x N
        self._out = None
        self.stats: dict = {}

    def accumulate(self, views: Sequence, num_objects: int,
                   blend: BlendConfig = DEFAULT_BLEND, download: bool = True):
        views = list(views)
        validate_views(views, int(num_objects))
        n = len(self.scene)
        e = int(num_objects)
        ctx = self.ctx
        with ctx.lock:
            ctx.set_scene(self.scene)
            acc = ctx.alloc(8 * e * max(n, 1)).zero()
            self.stats = ctx.accumulate([v for v, _ in views], [m.labels for _, m in views], e,
                                        blend.alpha_floor, blend.transmittance_floor, acc.ptr)
            if self._A is None or self._A.nbytes < 4 * e * max(n, 1):
                self._A = ctx.alloc(4 * e * max(n, 1))
                self._out = ctx.alloc(e * max(n, 1))
            if n:
                ctx.finalize(acc.ptr, e * n, out_ptr=self._A.ptr)
            acc.release()
        self.num_objects = e
        if not download:
            return None
        values = np.empty((e, n), dtype=np.float32)
        if values.size:
            self._A.to_host(values)
        return ContributionMatrix(values=values)

    def assign(self, gamma: float, mode: str = "binary") -> Assignment:
        if self._A is None:
            raise ValueError("accumulate() must run before assign()")
        gamma = _check_gamma(gamma)
        e, n = self.num_objects, len(self.scene)
        nat = self._native
        if mode == "binary":
            if e != 2:
                raise ValueError(f"binary assignment requires E=2, got E={e}")
            nat.assign(None, gamma, nat.MODE_BINARY, ctx=self.ctx, on_device_ptr=self._A.ptr,
                       n=n, e=e, out_ptr=self._out.ptr)
            labels = np.empty(n, np.uint8)
            self._out.to_host(labels)
            return Assignment(mode="binary", gamma=gamma, labels=labels)
        if mode == "scene":
            if e < 2:
                raise ValueError(f"scene assignment requires E>=2, got E={e}")
            nat.assign(None, gamma, nat.MODE_SCENE, ctx=self.ctx, on_device_ptr=self._A.ptr,
                       n=n, e=e, out_ptr=self._out.ptr)
            member = np.empty((e, n), np.uint8)
            self._out.to_host(member)
            return Assignment(mode="scene", gamma=gamma, membership=member)
        raise ValueError(f"unknown assignment mode {mode!r}")


def solve(scene, views: Sequence, num_objects: int, gamma: float = 0.0, mode: str = "binary",
          blend: BlendConfig = DEFAULT_BLEND, device: Optional[int] = None):
    """(ContributionMatrix, Assignment) for one scene: the north-star entry point."""
    s = LabelSolver(scene, device)
    matrix = s.accumulate(views, num_objects, blend)
    return matrix, s.assign(gamma, mode)
