"""View sharding across GPUs: one process per GPU (torchrun), NCCL collectives.

A is additive over views (reference ``contributions.py:103-116``; pinned by
the reference's additivity / permutation tests ``test_contributions.py:79-95``),
so the views are split into disjoint contiguous shards and every rank
accumulates its shard on its own GPU into an N x E accumulator.  The ranks
then join the partials without ever materialising the full sum on every GPU:

* ``reduce_scatter`` of the accumulator by Gaussian slices (the layout is
  Gaussian-major, so rank r's slice is one contiguous block);
* rank r casts its reduced slice to float32 (``contributions.py:116``);
* ``all_gather`` of the float32 slices.

Bytes on NVLink per GPU: (g-1)/g * N*E*(entry + 4) instead of an all-reduce's
2 (g-1)/g * N*E*entry -- 25% less for float64 entries.  With the default
fixed-point accumulator the integer sum is exact, so the matrix is
bit-identical to a single-GPU solve for any world size.

Mask shapes are checked on the host for every view; label ranges on the
device for the rank's own shard, with one tiny MIN all-reduce so that every
rank raises the reference's error for the same view.

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
                             acc_ptr: int, group, device, acc_kind: Optional[int] = None) -> dict:
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
    if acc_kind is None:
        acc_kind = _native.ACC_DEFAULT
    try:
        st = ctx.accumulate([v for v, _ in sel], [m.labels for _, m in sel], num_objects,
                            blend.alpha_floor, blend.transmittance_floor, acc_ptr,
                            acc_kind=acc_kind)
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


def padded_rows(n: int, world: int) -> int:
    """Gaussian rows of the accumulator: a multiple of the world size (equal slices)."""
    return -(-max(n, 1) // world) * world


def alloc_accumulator(n: int, num_objects: int, world: int, acc_kind: int, device):
    """Zeroed torch accumulator of padded_rows(n, world) x E entries of acc_kind."""
    import torch

    from . import _native
    words = _native.acc_entry_bytes(acc_kind) // 8
    dtype = torch.int64 if acc_kind == _native.ACC_FIXED else torch.float64
    return torch.zeros(padded_rows(n, world) * num_objects * words, dtype=dtype, device=device)


def reduce_scatter_finalize(ctx, acc, n: int, num_objects: int, acc_kind: int, group, device):
    """E x N float32 device tensor on every rank from the ranks' accumulators.

    reduce_scatter by Gaussian slices -> float32 cast of this rank's slice
    (fs_reduce_finalize) -> all_gather of the slices -> the API's E x N layout.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    e = int(num_objects)
    chunk = padded_rows(n, world) // world
    part = torch.empty(acc.numel() // world, dtype=acc.dtype, device=acc.device)
    dist.reduce_scatter_tensor(part, acc, group=group)
    sl = torch.zeros((e, chunk), dtype=torch.float32, device=acc.device)
    g0, g1 = rank * chunk, min(n, rank * chunk + chunk)
    if g1 > g0:
        with ctx.lock:
            if acc.is_cuda:
                ctx.set_stream(torch.cuda.current_stream(acc.device).cuda_stream)
            ctx.reduce_finalize([part.data_ptr()], g0, n, e, g0, g1, sl.data_ptr(), chunk,
                                out_on_device=True, acc_kind=acc_kind)
    gathered = torch.empty(world * e * chunk, dtype=torch.float32, device=acc.device)
    dist.all_gather_into_tensor(gathered, sl.reshape(-1), group=group)
    return (gathered.view(world, e, chunk).permute(1, 0, 2).reshape(e, world * chunk)[:, :n]
            .contiguous())


def sharded_matrix_device(scene, views, num_objects: int, blend, group, device, acc_kind: int):
    """(E x N float32 device tensor, this rank's counters) for a view-sharded solve (NCCL)."""
    import torch
    import torch.distributed as dist

    from . import _native

    if device is None:
        device = torch.cuda.current_device()
    ctx = _native.context(device)
    n = len(scene)
    world = dist.get_world_size(group)
    mine = shard_views(len(views), dist.get_rank(group), world)
    acc = alloc_accumulator(n, num_objects, world, acc_kind, f"cuda:{device}")
    with ctx.lock:
        ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
        ctx.set_scene(scene)
        st = accumulate_shard_checked(ctx, views, mine, num_objects, blend, acc.data_ptr(), group,
                                      device, acc_kind)
    return reduce_scatter_finalize(ctx, acc, n, num_objects, acc_kind, group, device), st


def _device_partial_path(scene, views, num_objects, blend, group, device, stats, acc_kind):
    from . import _native

    A, st = sharded_matrix_device(scene, views, num_objects, blend, group, device, acc_kind)
    ctx = _native.context(A.device.index)
    host = ctx.pinned_empty((num_objects, len(scene)), np.float32)
    if host.size:
        import torch
        torch.from_numpy(host).copy_(A)
    if stats is not None:
        stats.update(st)
    return host


def _gpu_partial_host(scene, views, num_objects, blend) -> np.ndarray:
    from . import _native

    ctx = _native.context()
    n = len(scene)
    with ctx.lock:
        ctx.set_scene(scene)
        acc = ctx.acc_buffer(num_objects, n, _native.ACC_F64).zero()
        ctx.accumulate([v for v, _ in views], [m.labels for _, m in views], num_objects,
                       blend.alpha_floor, blend.transmittance_floor, acc.ptr,
                       acc_kind=_native.ACC_F64)
        out = np.zeros((n, num_objects), dtype=np.float64)  # N x E (Gaussian-major)
        if out.size:
            acc.to_host(out)
    return np.ascontiguousarray(out.T)


def accumulate_sharded(scene, views: Sequence, num_objects: int, blend, group,
                       device: Optional[int] = None, stats: Optional[dict] = None,
                       partial_fn: Optional[Callable] = None,
                       acc_kind: Optional[int] = None) -> np.ndarray:
    """E x N float32 contribution matrix from a view-sharded accumulation."""
    import torch
    import torch.distributed as dist

    from .contributions import validate_views

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    idx = shard_views(len(views), rank, world)
    if partial_fn is None and dist.get_backend(group) == "nccl":
        if acc_kind is None:
            from . import _native
            acc_kind = _native.ACC_DEFAULT
        return _device_partial_path(scene, views, num_objects, blend, group, device, stats,
                                    acc_kind)
    # host-only backends: every rank checks every view on the host
    validate_views(views, num_objects)
    fn = partial_fn or _gpu_partial_host
    part = np.ascontiguousarray(fn(scene, [views[i] for i in idx], num_objects, blend),
                                dtype=np.float64)
    t = torch.from_numpy(part.reshape(-1).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy().reshape(num_objects, len(scene)).astype(np.float32)
