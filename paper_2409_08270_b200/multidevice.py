"""Single-process multi-GPU solve: ``devices=[...]`` on the public entry points.

The reference's own callers -- ``splatlift accumulate`` (cli.py:96-107, the
accumulate call at :104) and the service (service.py:56-66) -- run in one
process, so a torchrun-only multi-GPU path never reaches them.  This path
does, from one process:

* one library context (streams + workspaces) per GPU; the host scene is
  uploaded to the first and copied device to device to the others
  (``fs_copy_scene``, NVLink peer copies), so it crosses PCIe once;
* ``fs_accumulate_multi``: one native host thread per GPU pops views from a
  shared queue whenever one of its streams frees up, so faster GPUs take
  more views (A is additive over views, contributions.py:103-116);
* ``fs_finalize_multi``: GPU i reduces column slice i of A by reading every
  GPU's accumulator over NVLink peer memory (the reduce half of a
  reduce-scatter fused into the float32 cast), runs the biased argmax on
  the slice (solver.py:118-172) and copies both straight into the host
  outputs -- no all-gather, the host is the destination.

With the default deterministic accumulator (``FS_ACC_FIXED``) the result is
bit-identical to a single-GPU solve whatever the queue hands to which GPU.
A device may be listed more than once (independent contexts on one GPU);
``devices=[0, 0]`` exercises the whole path on a single GPU.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence

import numpy as np


def device_contexts(devices: Sequence[int]) -> list:
    """One library context per entry of ``devices`` (repeats get their own slot)."""
    from . import _native

    seen: dict = {}
    out = []
    for d in devices:
        d = int(d)
        slot = seen.get(d, 0)
        seen[d] = slot + 1
        out.append(_native.context(d, slot))
    return out


def solve_multi(scene, views: Sequence, num_objects: int, blend, devices: Sequence[int],
                acc_kind: int, gamma: float = 0.0, mode: Optional[str] = None,
                stats: Optional[dict] = None):
    """(E x N float32 matrix, labels or membership or None) over ``devices``.

    Views are [(CameraView, LabelMask)] already shape-checked by the caller;
    label ranges are checked on the devices and the reference's error is
    raised for the first offending view (contributions.py:104-114).
    """
    from . import _native
    from .contributions import validate_views

    devices = list(devices)
    if not devices:
        raise ValueError("devices must name at least one GPU")
    if len(devices) > 16:
        raise ValueError(f"at most 16 devices are supported, got {len(devices)}")
    ctxs = device_contexts(devices)
    e, n = int(num_objects), len(scene)
    locks = sorted({id(c): c for c in ctxs}.values(), key=id)
    for c in locks:
        c.lock.acquire()
    try:
        # the host scene crosses PCIe once: the first GPU uploads it, the others copy
        # the resident arrays device to device (NVLink peer copies between GPUs)
        ctxs[0].set_scene(scene)
        with ThreadPoolExecutor(len(ctxs)) as pool:
            list(pool.map(lambda c: c.copy_scene_from(ctxs[0])
                          if c._scene_key != ctxs[0]._scene_key or c._scene_key is None else None,
                          ctxs[1:]))
            accs = list(pool.map(lambda c: c.acc_buffer(e, n, acc_kind, role="acc_multi").zero(),
                                 ctxs))
        try:
            st, owner = _native.accumulate_multi(
                ctxs, [v for v, _ in views], [m.labels for _, m in views], e, blend.alpha_floor,
                blend.transmittance_floor, [a.ptr for a in accs], acc_kind)
        except _native.LabelRangeError as err:
            validate_views([views[err.view]], e)  # raises the reference message
            raise
        out = ctxs[0].pinned_empty((e, n), np.float32)
        labels, code = None, -1
        if mode == "binary":
            labels, code = ctxs[0].pinned_empty((n,), np.uint8), _native.MODE_BINARY
        elif mode == "scene":
            labels, code = ctxs[0].pinned_empty((e, n), np.uint8), _native.MODE_SCENE
        elif mode is not None:
            raise ValueError(f"unknown assignment mode {mode!r}")
        _native.finalize_multi(ctxs, [a.ptr for a in accs], n, e, out, gamma, code, labels,
                               acc_kind)
    finally:
        for c in locks:
            c.lock.release()
    if stats is not None:
        stats.update(st)
        stats["view_device"] = [devices[int(i)] for i in owner]
        stats["views_per_device"] = [int(np.count_nonzero(owner == i)) for i in range(len(ctxs))]
    return out, labels
