"""Blend configuration, tile binning and novel-view compositing
(reference ``rasterizer.py:31-252``).

``TileBinning`` keeps the reference's attributes (``tiles_x``, ``tiles_y``,
packed ``indices`` / ``means2d`` / ``inv_cov`` / ``depths`` / ``radii`` and
per-tile ``tile_lists`` ordered by (depth, gaussian_index)); the lists are
built on the GPU by the same binning + per-tile ordering that feeds the
raster kernel (``fs_bin_splats``).

``render_property`` / ``render_view`` / ``render_subset_alpha_depth``
 run the raster kernel in its compositing form: per
pixel, float64 sums of w = alpha*T, depth*w and channel*w in list order, the
same expressions as rasterizer.py:176-203 (``fs_render`` /
``fs_render_splats``).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .scene import CameraView, GaussianScene

TILE_SIZE = 16  # reference rasterizer.py:31


@dataclass(frozen=True)
class BlendConfig:
    """Throughput floors of the blending walk (reference ``rasterizer.py:34-49``).

    ``alpha_floor``: samples below it are dropped (no weight, no
    transmittance update).  ``transmittance_floor``: a pixel stops once its
    transmittance falls below it, after the sample that crossed it was added.
    Zero disables either rule.
    """

    alpha_floor: float = 1.0 / 255.0
    transmittance_floor: float = 1e-4

    @classmethod
    def exact(cls) -> "BlendConfig":
        return cls(alpha_floor=0.0, transmittance_floor=0.0)


DEFAULT_BLEND = BlendConfig()
EXACT_BLEND = BlendConfig.exact()


def tile_range(mx: float, my: float, radius: int, tiles_x: int, tiles_y: int):
    """Inclusive tile box of a splat's radius box (reference ``rasterizer.py:106-113``)."""
    tx0 = max(0, int(math.floor((mx - radius) / TILE_SIZE)))
    tx1 = min(tiles_x - 1, int(math.floor((mx + radius) / TILE_SIZE)))
    ty0 = max(0, int(math.floor((my - radius) / TILE_SIZE)))
    ty1 = min(tiles_y - 1, int(math.floor((my + radius) / TILE_SIZE)))
    return tx0, tx1, ty0, ty1


class TileBinning:
    """Per-tile depth-ordered splat lists, built on the device."""

    def __init__(self, view: CameraView, projected: Sequence, device: int = None):
        from . import _native

        self.tiles_x = (view.width + TILE_SIZE - 1) // TILE_SIZE
        self.tiles_y = (view.height + TILE_SIZE - 1) // TILE_SIZE
        k = len(projected)
        self.indices = np.fromiter((p.gaussian_index for p in projected), dtype=np.int64, count=k)
        self.means2d = np.array([p.mean2d for p in projected], dtype=np.float64).reshape(k, 2)
        self.inv_cov = np.array([(p.inv_cov2d[0, 0], p.inv_cov2d[0, 1], p.inv_cov2d[1, 1])
                                 for p in projected], dtype=np.float64).reshape(k, 3)
        self.depths = np.fromiter((p.depth for p in projected), dtype=np.float64, count=k)
        self.radii = np.fromiter((p.radius for p in projected), dtype=np.int64, count=k)
        offsets, items = _native.bin_splats(self.means2d, self.depths, self.radii, self.indices,
                                            view.width, view.height, device=device)
        self.tile_offsets = offsets
        self.tile_items = items
        self.tile_lists = [items[offsets[t]:offsets[t + 1]] for t in range(len(offsets) - 1)]

    def tile_count(self, tx: int, ty: int) -> int:
        return len(self.tile_lists[ty * self.tiles_x + tx])


def bin_gaussians_to_tiles(projected: Sequence, view: CameraView) -> TileBinning:
    """Reference ``bin_gaussians_to_tiles`` (``rasterizer.py:116-120``)."""
    return TileBinning(view, projected)


def _tile_pixel_grid(view: CameraView, tx: int, ty: int):
    """Tile pixel bounds and sample centres (reference ``rasterizer.py:123-130``)."""
    x0, y0 = tx * TILE_SIZE, ty * TILE_SIZE
    x1, y1 = min(x0 + TILE_SIZE, view.width), min(y0 + TILE_SIZE, view.height)
    us = np.arange(x0, x1, dtype=np.float64) + 0.5
    vs = np.arange(y0, y1, dtype=np.float64) + 0.5
    return x0, y0, x1, y1, us[None, :], vs[:, None]


@dataclass
class RenderOutput:
    """Per-pixel blend results (reference ``rasterizer.py:56-66``): property
    value, accumulated alpha, and depth -- the alpha-blended expected depth
    normalised by the accumulated alpha, zero wherever ``alpha`` is zero."""

    value: Optional[np.ndarray]
    alpha: np.ndarray
    depth: np.ndarray


def _check_channel(scene: GaussianScene, channel):
    if channel is None:
        return None
    channel = np.asarray(channel, dtype=np.float64)
    if channel.shape[0] != len(scene):  # rasterizer.py:146-148
        raise ValueError(f"channel length {channel.shape[0]} != scene size {len(scene)}")
    if channel.ndim == 2 and channel.shape[1] != 3:
        raise ValueError(f"vector channels must have 3 components, got {channel.shape[1]}")
    if channel.ndim > 2:
        raise ValueError(f"channel must be N or N x 3, got shape {channel.shape}")
    return np.ascontiguousarray(channel)


def render_property(scene: GaussianScene, binning: TileBinning, view: CameraView,
                    channel: Optional[np.ndarray], blend: BlendConfig = DEFAULT_BLEND,
                    *, device: Optional[int] = None) -> RenderOutput:
    """Alpha-composite a per-Gaussian channel (scalar or 3-vector) per pixel over
    the given binning (reference ``rasterizer.py:133-203``).  ``channel=None``
    skips value accumulation and returns alpha/depth only."""
    from . import _native

    channel = _check_channel(scene, channel)
    lists = binning.tile_lists
    offsets = np.zeros(len(lists) + 1, np.int64)
    offsets[1:] = np.cumsum([len(x) for x in lists])
    items = (np.concatenate([np.asarray(x, np.int64) for x in lists]) if offsets[-1]
             else np.zeros(0, np.int64))
    idx = np.asarray(binning.indices, np.int64)
    opac = np.asarray(scene.opacities, np.float64)[idx]
    ch = None if channel is None else channel[idx]
    value, alpha, depth = _native.render_splats(
        view.width, view.height, binning.means2d, binning.inv_cov, binning.depths, opac, offsets,
        items, blend.alpha_floor, blend.transmittance_floor, ch, device=device)
    return RenderOutput(value=value, alpha=alpha, depth=depth)


def _render_scene(scene, view, member, channel, blend, device):
    from . import _native

    ctx = _native.context(device)
    with ctx.lock:
        ctx.set_scene(scene)
        value, alpha, depth = ctx.render(view, member, blend.alpha_floor,
                                         blend.transmittance_floor, channel)
    return RenderOutput(value=value, alpha=alpha, depth=depth)


def render_view(scene: GaussianScene, view: CameraView, channel: Optional[np.ndarray] = None,
                blend: BlendConfig = DEFAULT_BLEND, *,
                device: Optional[int] = None) -> RenderOutput:
    """Project, bin and composite a view in one call (reference
    ``rasterizer.py:206-215``) -- fused on the device (``fs_render``)."""
    return _render_scene(scene, view, None, _check_channel(scene, channel), blend, device)


def render_subset_alpha_depth(scene: GaussianScene, view: CameraView, member_mask: np.ndarray,
                              blend: BlendConfig = DEFAULT_BLEND, *,
                              device: Optional[int] = None) -> RenderOutput:
    """Accumulated alpha and blended depth of a member subset (reference
    ``rasterizer.py:218-234``): projection, binning and walk run over the
    subset only, so transmittance reflects subset-internal occlusion."""
    member = np.asarray(member_mask, dtype=bool).reshape(len(scene))
    return _render_scene(scene, view, member, None, blend, device)


def save_render_grid(path, grid: np.ndarray) -> None:
    """Write a float32 grid with an 8-byte (width, height) LE header
    (reference ``rasterizer.py:237-243``)."""
    grid = np.asarray(grid, dtype=np.float32)
    h, w = grid.shape
    with open(path, "wb") as fh:
        fh.write(struct.pack("<II", w, h))
        grid.tofile(fh)


def load_render_grid(path) -> np.ndarray:
    """Reference ``rasterizer.py:246-252``."""
    with open(path, "rb") as fh:
        w, h = struct.unpack("<II", fh.read(8))
        data = np.fromfile(fh, dtype=np.float32, count=w * h)
    if data.size != w * h:
        raise ValueError(f"{path}: truncated render grid")
    return data.reshape(h, w)
