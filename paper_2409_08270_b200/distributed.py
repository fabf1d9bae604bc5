"""View sharding across GPUs: one process per GPU, one all-reduce.

A is additive over views (reference ``contributions.py:103-116``; pinned by
the reference's additivity / permutation tests ``test_contributions.py:79-95``),
so the views are split into disjoint contiguous shards, each rank
accumulates its shard on its own GPU into a float64 E x N buffer, and a
single ``all_reduce(SUM)`` joins the partials.  Mask shapes are checked on
the host for every view; label ranges on the device for the rank's own
shard, with one tiny MIN all-reduce so that every rank raises the
reference's error for the same view.  With NCCL the buffer never
leaves the device; the float32 cast (``contributions.py:116``) runs after the
reduction on every rank.  Summation order differs between GPU counts only at
the float64 rounding level (~1e-16 relative), far below the float32 result.

``partial_fn`` lets host-only backends (gloo, used by the CPU test-suite)
plug a host implementation of the per-shard partial; the product path on
NCCL always runs the CUDA library.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np


def shard_views(n_views: int, rank: int, world: int) -> list:
    """Contiguous balanced shard of view indices for ``rank`` of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return list(range(start, stop))


_NO_ERROR = 1 << 62


def accumulate_shard_checked(ctx, views: Sequence, mine: Sequence, num_objects: int, blend,
                             acc_ptr: int, group, device) -> dict:
    """Accumulate this rank's views ``mine`` (indices into ``views``) on the device.

    Label ranges (contributions.py:108-114) are checked on the device for the
    shard only; one MIN all-reduce of the first offending view index makes
    every rank raise the reference's error for the same (globally first)
    view.  Shapes were checked on the host for every view beforehand.
    """
    import torch
    import torch.distributed as dist

    from . import _native
    from .contributions import validate_views

    sel = [views[i] for i in mine]
    bad = _NO_ERROR
    st: dict = {}
    try:
        st = ctx.accumulate([v for v, _ in sel], [m.labels for _, m in sel], num_objects,
                            blend.alpha_floor, blend.transmittance_floor, acc_ptr)
    except _native.LabelRangeError as err:
        bad = int(mine[err.view])
    on = "cpu" if dist.get_backend(group) == "gloo" else f"cuda:{device}"
    t = torch.tensor([bad], dtype=torch.int64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    first = int(t.item())
    if first != _NO_ERROR:
        validate_views([views[first]], num_objects)  # raises the reference message
        raise ValueError(f"view {views[first][0].view_id}: label out of range")
    return st


def _device_partial_path(scene, views, mine, num_objects, blend, group, device, stats):
    import torch
    import torch.distributed as dist

    from . import _native

    if device is None:
        device = torch.cuda.current_device()
    ctx = _native.context(device)
    n = len(scene)
    acc = torch.zeros(num_objects * max(n, 1), dtype=torch.float64, device=f"cuda:{device}")
    with ctx.lock:
        ctx.set_scene(scene)
        torch.cuda.synchronize(device)
        st = accumulate_shard_checked(ctx, views, mine, num_objects, blend, acc.data_ptr(), group,
                                      device)
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    torch.cuda.synchronize(device)
    host = ctx.pinned_empty((num_objects, n), np.float32)  # finalize D2H straight into it
    if host.size:
        with ctx.lock:
            ctx.finalize(acc.data_ptr(), n, num_objects, out=host)
    if stats is not None:
        stats.update(st)
    return host


def _gpu_partial_host(scene, views, num_objects, blend) -> np.ndarray:
    from . import _native

    ctx = _native.context()
    n = len(scene)
    with ctx.lock:
        ctx.set_scene(scene)
        acc = ctx.buffer("acc64", 8 * num_objects * max(n, 1)).zero()
        ctx.accumulate([v for v, _ in views], [m.labels for _, m in views], num_objects,
                       blend.alpha_floor, blend.transmittance_floor, acc.ptr)
        out = np.zeros((num_objects, n), dtype=np.float64)
        if out.size:
            acc.to_host(out)
    return out


def accumulate_sharded(scene, views: Sequence, num_objects: int, blend, group,
                       device: Optional[int] = None, stats: Optional[dict] = None,
                       partial_fn: Optional[Callable] = None) -> np.ndarray:
    """E x N float32 contribution matrix from a view-sharded accumulation."""
    import torch
    import torch.distributed as dist

    from .contributions import validate_views

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    idx = shard_views(len(views), rank, world)
    if partial_fn is None and dist.get_backend(group) == "nccl":
        return _device_partial_path(scene, views, idx, num_objects, blend, group, device, stats)
    # host-only backends: every rank checks every view on the host
    validate_views(views, num_objects)
    fn = partial_fn or _gpu_partial_host
    part = np.ascontiguousarray(fn(scene, [views[i] for i in idx], num_objects, blend),
                                dtype=np.float64)
    t = torch.from_numpy(part.reshape(-1).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy().reshape(num_objects, len(scene)).astype(np.float32)
