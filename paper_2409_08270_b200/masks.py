"""Mask ingestion: 16-bit label PNGs -> the device.

``save_mask_png`` / ``load_mask_png`` mirror the reference's wire format and
checks (``masks.py:25-40``: pixel value = object id, modes I;16 / I / L / P,
uint16 range); grayscale PNGs are decoded by ``fs_decode_mask_png`` (C++,
zlib), the rest by Pillow.  ``read_masks`` mirrors the CLI's pairing of views with
``{view_id}.png`` files (``cli.py:74-83``) but decodes on a thread pool.

``accumulate_mask_files`` is the pipelined form of "read every mask, then
accumulate_contributions": masks are decoded (one pool task per view, up to
``lookahead`` chunks ahead) while the GPU accumulates the previous chunk into
one float64 device buffer, so decode and the H2D copies overlap the kernels.  Errors are
the reference's, in view order (shape checks on the host per chunk, label
ranges on the device).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from .rasterizer import DEFAULT_BLEND, BlendConfig


def save_mask_png(path, labels: np.ndarray) -> None:
    """uint16 label grid -> 16-bit grayscale PNG (reference ``masks.py:25-27``)."""
    from PIL import Image

    labels = np.ascontiguousarray(labels, dtype=np.uint16)
    Image.fromarray(labels).save(path, format="PNG")


def load_mask_png(path) -> np.ndarray:
    """16-bit (or 8-bit / palette) PNG -> uint16 labels (reference ``masks.py:30-40``).

    Grayscale 8/16-bit PNGs -- the wire format -- are decoded natively
    (``fs_decode_mask_png``: zlib inflate + row unfiltering in C++, no GIL);
    every other flavour (palette, interlaced, ...) goes through Pillow exactly as
    the reference does.  No silent fallback: without the library this raises
    ``NativeUnavailable`` like every other entry point.
    """
    from PIL import Image

    from . import _native

    data = Path(path).read_bytes()
    arr = _native.decode_mask_png(data)  # raises NativeUnavailable without the library
    if arr is not None:
        return arr
    with Image.open(path) as im:
        if im.mode not in ("I;16", "I", "L", "P"):
            raise ValueError(f"{path}: unsupported mask mode {im.mode}")
        if im.mode == "I;16":
            arr = np.asarray(im, dtype=np.uint16)  # already the wire format
            return np.ascontiguousarray(arr)
        arr = np.asarray(im.convert("I"), dtype=np.int32)
    if arr.min() < 0 or arr.max() > np.iinfo(np.uint16).max:
        raise ValueError(f"{path}: mask values outside uint16 range")
    return arr.astype(np.uint16)


def _workers(workers: Optional[int]) -> int:
    return max(1, workers if workers else min(16, os.cpu_count() or 1))


def mask_paths(masks_dir, views: Sequence) -> list:
    """(view, path) for every view with a ``{view_id}.png`` mask (``cli.py:74-83``)."""
    out = []
    for view in views:
        path = Path(masks_dir) / f"{view.view_id}.png"
        if path.exists():
            out.append((view, path))
    return out


def read_masks(masks_dir, views: Sequence, workers: Optional[int] = None) -> list:
    """The CLI's ``_read_masks`` on a thread pool: [(view, LabelMask)] in view order."""
    from .contributions import LabelMask

    pairs = mask_paths(masks_dir, views)
    with ThreadPoolExecutor(_workers(workers)) as pool:
        labels = list(pool.map(lambda vp: load_mask_png(vp[1]), pairs))
    return [(v, LabelMask(view_id=v.view_id, labels=lab)) for (v, _), lab in zip(pairs, labels)]


def accumulate_mask_files(scene, view_paths: Sequence, num_objects: int,
                          blend: BlendConfig = DEFAULT_BLEND, *, chunk: int = 16,
                          lookahead: int = 2, workers: Optional[int] = None,
                          device: Optional[int] = None, stats: Optional[dict] = None,
                          deterministic: bool = True):
    """accumulate_contributions over ``[(view, png_path)]`` with decode overlapped.

    Equivalent to ``accumulate_contributions(scene, [(v, LabelMask(v.view_id,
    load_mask_png(p))) ...], num_objects, blend)``; the matrix differs only in
    float64 summation order (atomics), i.e. not at all after the float32 cast
    in practice (and not at all with the default deterministic accumulator).
    """
    from . import _native
    from .contributions import (ContributionMatrix, LabelMask, acc_kind_of, check_shapes,
                                run_device_accumulate, validate_views)

    view_paths = list(view_paths)
    num_objects = int(num_objects)
    n = len(scene)
    chunk = max(1, int(chunk))
    starts = list(range(0, len(view_paths), chunk))
    window = chunk * max(1, int(lookahead))  # views decoded ahead of the GPU

    ctx = _native.context(device)
    kind = acc_kind_of(deterministic, blend)
    totals: dict = {}
    with ThreadPoolExecutor(_workers(workers)) as pool:
        # one decode task per view, at most `window` views ahead of the device
        futs = {}
        nxt = [0]

        def submit_until(k):
            while nxt[0] < min(k, len(view_paths)):
                futs[nxt[0]] = pool.submit(load_mask_png, view_paths[nxt[0]][1])
                nxt[0] += 1

        submit_until(window)
        with ctx.lock:
            ctx.set_scene(scene)
            acc = ctx.acc_buffer(num_objects, n, kind).zero()
            for s in starts:
                e = min(s + chunk, len(view_paths))
                pairs = [(view_paths[j][0], LabelMask(view_id=view_paths[j][0].view_id,
                                                      labels=futs.pop(j).result()))
                         for j in range(s, e)]
                submit_until(e + window)
                check_shapes(pairs, num_objects)
                if n == 0:
                    validate_views(pairs, num_objects)
                    continue
                st = run_device_accumulate(ctx, pairs, num_objects, blend, acc.ptr, kind)
                for k, v in st.items():
                    if isinstance(v, (int, float)):
                        totals[k] = totals.get(k, 0) + v
            out = ctx.pinned_empty((num_objects, n), np.float32)
            if out.size:
                ctx.finalize(acc.ptr, n, num_objects, out=out, acc_kind=kind)
    if stats is not None:
        stats.update(totals)
    return ContributionMatrix(values=out)
