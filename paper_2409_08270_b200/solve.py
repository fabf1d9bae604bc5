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
                   blend: BlendConfig = DEFAULT_BLEND, download: bool = True,
                   process_group=None):
        """Accumulate A on the device (and keep it there); optionally view-sharded.

        With ``process_group`` every rank validates all views (same errors on
        every rank), accumulates its shard and one all-reduce joins them.
        """
        views = list(views)
        e = int(num_objects)
        validate_views(views, e)
        n = len(self.scene)
        ctx = self.ctx
        acc_t = None
        sel = views
        if process_group is not None:
            import torch
            import torch.distributed as dist

            from .distributed import shard_views
            rank = dist.get_rank(process_group)
            world = dist.get_world_size(process_group)
            sel = [views[i] for i in shard_views(len(views), rank, world)]
            acc_t = torch.zeros(e * max(n, 1), dtype=torch.float64, device=f"cuda:{ctx.device}")
            acc_ptr = acc_t.data_ptr()
        with ctx.lock:
            ctx.set_scene(self.scene)
            if acc_t is None:
                acc = ctx.alloc(8 * e * max(n, 1)).zero()
                acc_ptr = acc.ptr
            self.stats = ctx.accumulate([v for v, _ in sel], [m.labels for _, m in sel], e,
                                        blend.alpha_floor, blend.transmittance_floor, acc_ptr)
        if acc_t is not None:
            import torch.distributed as dist
            dist.all_reduce(acc_t, group=process_group)
        with ctx.lock:
            if self._A is None or self._A.nbytes < 4 * e * max(n, 1):
                self._A = ctx.alloc(4 * e * max(n, 1))
                self._out = ctx.alloc(e * max(n, 1))
            if n:
                ctx.finalize(acc_ptr, e * n, out_ptr=self._A.ptr)
            if acc_t is None:
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
          blend: BlendConfig = DEFAULT_BLEND, device: Optional[int] = None, process_group=None):
    """(ContributionMatrix, Assignment) for one scene: the north-star entry point.

    Host numpy inputs in, host results out; with ``process_group`` the views
    are sharded over the group's GPUs and every rank returns the full result.
    """
    s = LabelSolver(scene, device)
    matrix = s.accumulate(views, num_objects, blend, process_group=process_group)
    return matrix, s.assign(gamma, mode)
