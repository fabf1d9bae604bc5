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

from .contributions import (ContributionMatrix, acc_kind_of, check_shapes, run_device_accumulate,
                            validate_views)
from .rasterizer import DEFAULT_BLEND, BlendConfig
from .solver import Assignment, _check_gamma


class LabelSolver:
    """Accumulate once, then re-run the argmax for any gamma on the device.

    ``own_buffers=False`` borrows the context's scratch buffers (one-shot
    solves); the default keeps a private device copy of the matrix alive for
    the solver's lifetime (the interactive-gamma service case).
    """

    def __init__(self, scene, device: Optional[int] = None, own_buffers: bool = True,
                 deterministic: bool = True):
        from . import _native

        self._native = _native
        self.scene = scene
        self.ctx = _native.context(device)
        self.own = own_buffers
        self.deterministic = deterministic
        self._torch_A = None  # keeps a torch-owned matrix (sharded solves) alive
        self.num_objects = 0
        self._A = None  # device float32 E x N
        self._out = None
        self.stats: dict = {}

    def _buffers(self, e: int, n: int):
        need_a, need_o = 4 * e * max(n, 1), e * max(n, 1)
        if not self.own:
            return self.ctx.buffer("A32", need_a), self.ctx.buffer("labels", need_o)
        if self._A is None or self._A.nbytes < need_a:
            self._A = self.ctx.alloc(need_a)
            self._out = self.ctx.alloc(need_o)
        return self._A, self._out

    def accumulate(self, views: Sequence, num_objects: int,
                   blend: BlendConfig = DEFAULT_BLEND, download: bool = True,
                   process_group=None, devices: Optional[Sequence[int]] = None):
        """Accumulate A on the device (and keep it there); optionally view-sharded.

        With ``process_group`` every rank validates all views (same errors on
        every rank), accumulates its shard, and a reduce-scatter + all-gather
        leave the full matrix on every rank's device.  With ``devices`` the
        views are split over those GPUs from this process (multidevice.py) and
        the matrix is then kept on this solver's device for the re-assignments.
        """
        views = list(views)
        e = int(num_objects)
        n = len(self.scene)
        if n == 0:
            validate_views(views, e)
        else:
            check_shapes(views, e)
        ctx = self.ctx
        kind = acc_kind_of(self.deterministic, blend)
        if devices is not None and n:
            from .multidevice import solve_multi
            values, _ = solve_multi(self.scene, views, e, blend, devices, kind)
            with ctx.lock:
                A, out = self._buffers(e, n)
                A.from_host(values)
                self._A_cur, self._out_cur = A, out
            self.num_objects = e
            return ContributionMatrix(values=values) if download else None
        if process_group is not None and n:
            # reduce-scatter + sliced cast + all-gather (distributed.py); the
            # gathered E x N matrix stays on this rank's device
            from .distributed import sharded_matrix_device
            A_t, self.stats = sharded_matrix_device(self.scene, views, e, blend, process_group,
                                                    ctx.device, kind)
            with ctx.lock:
                A, out = self._buffers(e, n)
                self._torch_A = A_t
                self._A_cur, self._out_cur = _TorchView(A_t, ctx), out
        else:
            with ctx.lock:
                ctx.set_scene(self.scene)
                acc_ptr = ctx.acc_buffer(e, n, kind).zero().ptr
                self.stats = run_device_accumulate(ctx, views, e, blend, acc_ptr, kind) if n else {}
                A, out = self._buffers(e, n)
                self._A_cur, self._out_cur = A, out
                if n:
                    ctx.finalize(acc_ptr, n, e, out_ptr=A.ptr, acc_kind=kind)
        A = self._A_cur
        self.num_objects = e
        if not download:
            return None
        values = ctx.pinned_empty((e, n), np.float32)  # full-speed D2H
        if values.size:
            A.to_host(values)
        return ContributionMatrix(values=values)

    def assign(self, gamma: float, mode: str = "binary") -> Assignment:
        if getattr(self, "_A_cur", None) is None:
            raise ValueError("accumulate() must run before assign()")
        gamma = _check_gamma(gamma)
        e, n = self.num_objects, len(self.scene)
        nat = self._native
        if mode == "binary":
            if e != 2:
                raise ValueError(f"binary assignment requires E=2, got E={e}")
            nat.assign(None, gamma, nat.MODE_BINARY, ctx=self.ctx, on_device_ptr=self._A_cur.ptr,
                       n=n, e=e, out_ptr=self._out_cur.ptr)
            labels = self.ctx.pinned_empty((n,), np.uint8)
            self._out_cur.to_host(labels)
            asn = Assignment(mode="binary", gamma=gamma, labels=labels)
            fg = self.ctx.member_counts(self._out_cur.ptr, n, 1)[0]
            asn._device_counts = [n - fg, fg]  # member_counts() without a host pass
            return asn
        if mode == "scene":
            if e < 2:
                raise ValueError(f"scene assignment requires E>=2, got E={e}")
            nat.assign(None, gamma, nat.MODE_SCENE, ctx=self.ctx, on_device_ptr=self._A_cur.ptr,
                       n=n, e=e, out_ptr=self._out_cur.ptr)
            member = self.ctx.pinned_empty((e, n), np.uint8)
            self._out_cur.to_host(member)
            asn = Assignment(mode="scene", gamma=gamma, membership=member)
            asn._device_counts = self.ctx.member_counts(self._out_cur.ptr, n, e)
            return asn
        raise ValueError(f"unknown assignment mode {mode!r}")


class _TorchView:
    """A torch CUDA tensor seen through the DeviceBuffer interface (ptr, to_host)."""

    def __init__(self, t, ctx):
        self.t, self.ctx = t, ctx
        self.ptr = t.data_ptr()
        self.nbytes = t.numel() * t.element_size()

    def to_host(self, out: np.ndarray) -> np.ndarray:
        import torch
        torch.from_numpy(out.reshape(-1)).copy_(self.t.reshape(-1)[:out.size])
        return out


def pin_inputs(scene, views: Sequence, device: Optional[int] = None):
    """(scene, views) backed by page-locked host memory, for repeated solves.

    The returned scene is a shallow copy whose float64 arrays live in pinned
    blocks and every mask is a view into one pinned uint16 block, so each
    later ``solve`` / ``accumulate_contributions`` DMA-copies them to the GPU
    directly instead of through the library's staging buffers (the serving
    setup: inputs stay pinned, every solve still transfers them).  Values
    are identical; the originals are not modified.
    """
    import copy

    from . import _native
    from .contributions import LabelMask

    ctx = _native.context(device)

    def pin(a):
        b = ctx.pinned_empty(a.shape, a.dtype)
        b[...] = a
        return b

    sc = copy.copy(scene)
    for name in ("means", "rotations", "scales", "opacities"):
        setattr(sc, name, pin(np.ascontiguousarray(getattr(scene, name), dtype=np.float64)))
    views = list(views)
    total = sum(int(m.labels.size) for _, m in views)
    block = ctx.pinned_empty((max(total, 1),), np.uint16)
    out, at = [], 0
    for cam, m in views:
        k = int(m.labels.size)
        dst = block[at:at + k].reshape(m.labels.shape)
        dst[...] = m.labels
        out.append((cam, LabelMask(m.view_id, dst)))
        at += k
    return sc, out


def solve(scene, views: Sequence, num_objects: int, gamma: float = 0.0, mode: str = "binary",
          blend: BlendConfig = DEFAULT_BLEND, device: Optional[int] = None, process_group=None,
          devices: Optional[Sequence[int]] = None, deterministic: bool = True,
          stats: Optional[dict] = None):
    """(ContributionMatrix, Assignment) for one scene: the north-star entry point.

    Host numpy inputs in, host results out.  ``devices``: split the views over
    these GPUs from this process (multidevice.py); ``process_group``: shard them
    over a torch.distributed group (every rank returns the full result).
    """
    if devices is not None:
        from .multidevice import solve_multi
        gamma = _check_gamma(gamma)
        views = list(views)
        e = int(num_objects)
        if mode not in ("binary", "scene"):
            raise ValueError(f"unknown assignment mode {mode!r}")
        if mode == "binary" and e != 2:
            raise ValueError(f"binary assignment requires E=2, got E={e}")
        if mode == "scene" and e < 2:
            raise ValueError(f"scene assignment requires E>=2, got E={e}")
        check_shapes(views, e)
        if len(scene) == 0:
            validate_views(views, e)
        values, labels = solve_multi(scene, views, e, blend, devices,
                                     acc_kind_of(deterministic, blend),
                                     gamma=gamma, mode=mode, stats=stats)
        if mode == "binary":
            return ContributionMatrix(values=values), Assignment(mode, gamma, labels=labels)
        return ContributionMatrix(values=values), Assignment(mode, gamma, membership=labels)
    s = LabelSolver(scene, device, own_buffers=False, deterministic=deterministic)
    matrix = s.accumulate(views, num_objects, blend, process_group=process_group)
    if stats is not None:
        stats.update(s.stats)
    return matrix, s.assign(gamma, mode)
