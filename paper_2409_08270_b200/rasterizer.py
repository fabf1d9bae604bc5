"""Blend configuration and tile binning (reference ``rasterizer.py:31-130``).

``TileBinning`` keeps the reference's attributes (``tiles_x``, ``tiles_y``,
packed ``indices`` / ``means2d`` / ``inv_cov`` / ``depths`` / ``radii`` and
per-tile ``tile_lists`` ordered by (depth, gaussian_index)), but the lists are
built on the GPU by the same depth radix sort + instance emission + tile
radix sort that feeds the raster kernel (``fs_bin_splats``).  Novel-view
rendering (``render_property`` / ``render_view``) is out of scope for this
tier.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .scene import CameraView

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
