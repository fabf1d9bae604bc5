"""Contribution accumulation: the E x N alpha*T mass matrix on the GPU.

``accumulate_contributions`` keeps the reference signature
(``contributions.py:90-95``), validation order and messages
(``contributions.py:104-114``) and result type; the work runs in the CUDA
library (``fs_accumulate``: projection, tile binning and the raster kernel --
in-kernel per-tile depth sort, exact float64 walk, atomics -- per view,
float64 accumulation on the device, one float32 cast at the end --
``contributions.py:116``).

Views are independent and A is additive over views
(``contributions.py:103-116``), so the views can be split over GPUs:
``devices=[...]`` runs one host thread per GPU in this process with a shared
dynamic view queue and reduces the per-GPU accumulators over NVLink peer
memory inside the finalize (``multidevice.py``); ``process_group`` (a
``torch.distributed`` group, one process per GPU) shards the views over the
ranks and joins them with a reduce-scatter + all-gather (``distributed.py``).

The accumulator is deterministic by default: fixed-point integer sums
(``FS_ACC_FIXED``), so the matrix is bit-identical for any schedule and any
number of GPUs (test_contributions.py:160-168).
``deterministic=False`` -- and blends without floors (``EXACT_BLEND``), whose
weights can underflow below any fixed-point resolution -- use float64 atomics.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .rasterizer import DEFAULT_BLEND, BlendConfig
from .scene import GaussianScene

MATRIX_MAGIC = b"FSA1"  # reference contributions.py:26


@dataclass
class LabelMask:
    """H x W uint16 object-id grid for one view; 0 is background (``contributions.py:29-43``)."""

    view_id: int
    labels: np.ndarray

    def __post_init__(self) -> None:
        self.labels = np.asarray(self.labels, dtype=np.uint16)
        if self.labels.ndim != 2:
            raise ValueError("mask labels must be a 2D grid")

    @property
    def num_objects(self) -> int:
        return int(self.labels.max()) + 1 if self.labels.size else 1


@dataclass
class ContributionMatrix:
    """Dense E x N float32 alpha*T mass per label (``contributions.py:46-87``)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        self.values = np.ascontiguousarray(self.values, dtype=np.float32)
        if self.values.ndim != 2:
            raise ValueError("contribution matrix must be 2D (E x N)")

    @property
    def num_objects(self) -> int:
        return int(self.values.shape[0])

    @property
    def num_gaussians(self) -> int:
        return int(self.values.shape[1])

    @property
    def observed(self) -> np.ndarray:
        """Columns that received any mass (float64 column sum > 0)."""
        return self.values.sum(axis=0, dtype=np.float64) > 0.0

    def save(self, path) -> None:
        e, n = self.values.shape
        with open(path, "wb") as fh:
            fh.write(MATRIX_MAGIC + struct.pack("<II", e, n))
            self.values.tofile(fh)

    @classmethod
    def load(cls, path) -> "ContributionMatrix":
        with open(path, "rb") as fh:
            magic = fh.read(4)
            if magic != MATRIX_MAGIC:
                raise ValueError(f"{path}: bad magic {magic!r}")
            e, n = struct.unpack("<II", fh.read(8))
            data = np.fromfile(fh, dtype=np.float32, count=e * n)
        if data.size != e * n:
            raise ValueError(f"{path}: truncated contribution matrix")
        return cls(values=data.reshape(e, n))


def validate_views(views: Sequence, num_objects: int) -> None:
    """Reference checks in view order (``contributions.py:104-114``), on the host."""
    for view, mask in views:
        labels = mask.labels
        if labels.shape != (view.height, view.width):
            raise ValueError(
                f"view {view.view_id}: mask shape {labels.shape} does not "
                f"match view dimensions {(view.height, view.width)}")
        top = int(labels.max()) if labels.size else 0
        if top >= num_objects:
            j, k = np.unravel_index(int(np.argmax(labels)), labels.shape)
            raise ValueError(
                f"view {view.view_id}: label {top} at pixel ({j}, {k}) "
                f"exceeds object count {num_objects}")


def check_shapes(views: Sequence, num_objects: int) -> None:
    """Shape checks on the host; label ranges are checked on the device.

    If a view has the wrong shape, the reference would still have raised for
    an out-of-range label in an earlier view first, so those views get the
    full host check (``contributions.py:103-114`` order).
    """
    for i, (view, mask) in enumerate(views):
        if mask.labels.shape != (view.height, view.width):
            validate_views(views[: i + 1], num_objects)


# The fixed-point accumulator resolves 2^-60 per add; every add carries at least
# one weight w = alpha*T >= alpha_floor * T_floor (T is checked against its
# floor before the update, contributions.py:148-157), so its relative error is
# at most 2^-60 / (alpha_floor * T_floor) -- 2e-12 for the default blend, far
# inside the float32 result.  Without floors (EXACT_BLEND) weights can underflow
# towards 1e-300 and only float64 covers that range.
FIXED_MIN_WEIGHT = 2.0 ** -26


def acc_kind_of(deterministic: bool, blend=None) -> int:
    """Accumulator kind: fixed-point when deterministic and the blend's floors
    bound the weights from below, float64 atomics otherwise."""
    from . import _native
    if not deterministic:
        return _native.ACC_F64
    if blend is not None and blend.alpha_floor * blend.transmittance_floor < FIXED_MIN_WEIGHT:
        return _native.ACC_F64
    return _native.ACC_FIXED


def run_device_accumulate(ctx, views: Sequence, num_objects: int, blend, acc_ptr,
                          acc_kind: Optional[int] = None) -> dict:
    """ctx.accumulate with the reference's label error reproduced on failure."""
    from . import _native

    if acc_kind is None:
        acc_kind = _native.ACC_DEFAULT
    try:
        return ctx.accumulate([v for v, _ in views], [m.labels for _, m in views], num_objects,
                              blend.alpha_floor, blend.transmittance_floor, acc_ptr,
                              acc_kind=acc_kind)
    except _native.LabelRangeError as err:
        validate_views([views[err.view]], num_objects)  # raises the reference message
        raise


def accumulate_contributions(
    scene: GaussianScene,
    views: Sequence[tuple],
    num_objects: int,
    blend: BlendConfig = DEFAULT_BLEND,
    *,
    device: Optional[int] = None,
    devices: Optional[Sequence[int]] = None,
    process_group=None,
    stats: Optional[dict] = None,
    deterministic: bool = True,
) -> ContributionMatrix:
    """Scatter every pixel's surviving alpha*T samples into label rows, on the GPU.

    ``device``: CUDA ordinal (default: ``LOCAL_RANK`` or 0).  ``devices``: split
    the views over these GPUs from this process (dynamic queue, peer-memory
    reduction).  ``process_group``: shard the views over a ``torch.distributed``
    group (every rank returns the full matrix).  ``stats``: filled with the
    library's counters (instances, tile steps, exact evaluations, ...).
    ``deterministic``: fixed-point accumulator (default), bit-identical for any
    schedule and GPU count; False: float64 atomics.
    """
    views = list(views)
    num_objects = int(num_objects)
    check_shapes(views, num_objects)
    if len(scene) == 0:
        validate_views(views, num_objects)
        return ContributionMatrix(values=np.zeros((num_objects, 0), dtype=np.float32))
    kind = acc_kind_of(deterministic, blend)
    if process_group is not None:
        # shapes were checked above on every rank; label ranges are checked per
        # shard and agreed on (distributed.accumulate_shard_checked)
        from .distributed import accumulate_sharded
        values = accumulate_sharded(scene, views, num_objects, blend, process_group,
                                    device=device, stats=stats, acc_kind=kind)
        return ContributionMatrix(values=values)
    if devices is not None:
        from .multidevice import solve_multi
        values, _ = solve_multi(scene, views, num_objects, blend, devices, kind, stats=stats)
        return ContributionMatrix(values=values)
    from . import _native

    ctx = _native.context(device)
    n = len(scene)
    with ctx.lock:
        ctx.set_scene(scene)
        acc = ctx.acc_buffer(num_objects, n, kind).zero()
        st = run_device_accumulate(ctx, views, num_objects, blend, acc.ptr, kind)
        out = ctx.pinned_empty((num_objects, n), np.float32)  # full-speed D2H (768 MB at C4)
        ctx.finalize(acc.ptr, n, num_objects, out=out, acc_kind=kind)
    if stats is not None:
        stats.update(st)
    return ContributionMatrix(values=out)
