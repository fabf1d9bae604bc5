"""Seeded synthetic label-solver workloads at benchmark scale (configs C1-C5).

The reference's own fixture generators (``synth.make_two_cluster`` /
``synth.make_random``, reference ``synth.py:124-223``) render ground-truth
masks with the CPU rasteriser and are only practical up to ~10 k Gaussians.
The north-star configurations (1 M-3 M Gaussians, 200-300 views of
1008x756 / 1920x1080) need masks that cost O(pixels) to make, so this module
builds them analytically:

* geometry follows ``make_random`` (means U(-1.2, 1.2)^3, random unit
  quaternions, opacity U(0.1, 0.95), ring cameras of radius 5 with focal = W
  and elevation U(-1, 1); reference ``synth.py:180-206``) with scales
  U(0.002, 0.01) (make_random's U(0.08, 0.4) / 40) so a 1008x756 view sees
  ~5 px splats;
* objects are ``E - 1`` uniform-density balls of Gaussians on a 3-D grid
  (the sampling of reference ``synth.py:104-121``); everything else is
  background (label 0);
* each view's mask paints every ball's silhouette disk (radius f*R/z around
  its projected centre), nearest ball last, so overlaps go to the nearer ball;
* ``label_noise`` replaces that fraction of pixels with U{0..E-1} (config C5).

Everything is numpy with ``default_rng(seed)``; identical seeds give
identical inputs on every machine with the same numpy.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from .scene import CameraView, GaussianScene


def look_at(position, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """4x4 world->camera with camera axes x right, y down, z forward."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    w2c = np.eye(4)
    w2c[:3, :3] = np.stack([right, down, fwd])
    w2c[:3, 3] = -w2c[:3, :3] @ pos
    return w2c


def ring_camera(view_id: int, azimuth: float, radius: float, width: int, height: int,
                focal: float, elevation: float = 0.0) -> CameraView:
    pos = (radius * math.cos(azimuth), elevation, radius * math.sin(azimuth))
    return CameraView(view_id=view_id, width=width, height=height, fx=focal, fy=focal,
                      cx=width / 2.0, cy=height / 2.0, world_to_camera=look_at(pos))


def _ball(rng, count, center, radius, scale_range, opacity_range):
    d = rng.normal(size=(count, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = radius * rng.random(count) ** (1.0 / 3.0)
    means = center + d * r[:, None]
    q = rng.normal(size=(count, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = rng.uniform(*scale_range, size=(count, 3))
    o = rng.uniform(*opacity_range, size=count)
    return means, q, s, o


@dataclass
class Workload:
    scene: GaussianScene
    views: list
    masks: np.ndarray  # V x H x W uint16
    num_objects: int
    membership: np.ndarray  # N uint16 ground-truth label
    ball_centers: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    ball_radius: float = 0.0
    name: str = ""

    def pairs(self):
        from .contributions import LabelMask
        return [(v, LabelMask(view_id=v.view_id, labels=self.masks[i]))
                for i, v in enumerate(self.views)]

    def view_pixels(self) -> int:
        return int(sum(v.width * v.height for v in self.views))

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.scene.means, self.scene.rotations, self.scene.scales,
                  self.scene.opacities, self.masks):
            h.update(np.ascontiguousarray(a).tobytes())
        for v in self.views:
            h.update(np.ascontiguousarray(v.world_to_camera).tobytes())
        return h.hexdigest()


def _ball_grid(n_balls: int, extent: float = 0.8):
    if n_balls <= 0:
        return np.zeros((0, 3)), 0.0
    if n_balls == 1:
        return np.zeros((1, 3)), 0.5
    side = int(math.ceil(n_balls ** (1.0 / 3.0)))
    lin = np.linspace(-extent, extent, side) if side > 1 else np.zeros(1)
    grid = np.stack(np.meshgrid(lin, lin, lin, indexing="ij"), axis=-1).reshape(-1, 3)
    spacing = (2 * extent / (side - 1)) if side > 1 else 1.0
    return grid[:n_balls], 0.35 * spacing


def analytic_masks(views, centers, radius, num_objects, rng=None, label_noise=0.0):
    """Silhouette-disk masks (nearest ball wins), optional iid label noise."""
    nv = len(views)
    h, w = views[0].height, views[0].width
    masks = np.zeros((nv, h, w), dtype=np.uint16)
    for i, v in enumerate(views):
        m = masks[i]
        rot, t = v.world_to_camera[:3, :3], v.world_to_camera[:3, 3]
        cam = centers @ rot.T + t
        order = np.argsort(-cam[:, 2])  # far first, near painted last
        for b in order:
            z = cam[b, 2]
            if z <= v.near_clip + radius:
                continue
            u = v.fx * cam[b, 0] / z + v.cx
            vv = v.fy * cam[b, 1] / z + v.cy
            rp = v.fx * radius / z
            x0, x1 = max(0, int(u - rp)), min(w, int(u + rp) + 2)
            y0, y1 = max(0, int(vv - rp)), min(h, int(vv + rp) + 2)
            if x0 >= x1 or y0 >= y1:
                continue
            xs = np.arange(x0, x1) + 0.5
            ys = np.arange(y0, y1) + 0.5
            inside = (xs[None, :] - u) ** 2 + (ys[:, None] - vv) ** 2 <= rp * rp
            m[y0:y1, x0:x1][inside] = b + 1
        if label_noise > 0.0:
            flip = rng.random((h, w)) < label_noise
            m[flip] = rng.integers(0, num_objects, size=int(flip.sum()), dtype=np.uint16)
    return masks


def make_workload(seed: int, n_gaussians: int, n_views: int, width: int, height: int,
                  num_objects: int, label_noise: float = 0.0,
                  scale_range=(0.002, 0.01), object_fraction=None,
                  iid_masks: bool = False, name: str = "") -> Workload:
    """Box-geometry scene with E-1 ball objects and analytic (or iid) masks.

    ``object_fraction`` (default: the balls' share of the box volume, i.e. a
    uniform Gaussian density everywhere) of the Gaussians sit in the balls.
    """
    rng = np.random.default_rng(seed)
    centers, radius = _ball_grid(num_objects - 1)
    if object_fraction is None:
        object_fraction = min(0.9, (num_objects - 1) * (4.0 / 3.0) * math.pi * radius ** 3 / 2.4 ** 3)
    n_obj_total = int(n_gaussians * object_fraction) if num_objects > 1 else 0
    per = n_obj_total // max(num_objects - 1, 1) if num_objects > 1 else 0
    parts, member = [], []
    for b in range(num_objects - 1):
        parts.append(_ball(rng, per, centers[b], radius, scale_range, (0.1, 0.95)))
        member.append(np.full(per, b + 1, dtype=np.uint16))
    n_bg = n_gaussians - per * (num_objects - 1)
    bg_means = rng.uniform(-1.2, 1.2, size=(n_bg, 3))
    q = rng.normal(size=(n_bg, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    parts.append((bg_means, q, rng.uniform(*scale_range, size=(n_bg, 3)),
                  rng.uniform(0.1, 0.95, size=n_bg)))
    member.append(np.zeros(n_bg, dtype=np.uint16))
    # interleave objects and background so Gaussian ids carry no spatial order
    perm = rng.permutation(n_gaussians)
    cat = [np.concatenate([p[k] for p in parts])[perm] for k in range(4)]
    membership = np.concatenate(member)[perm]
    scene = GaussianScene(means=cat[0], rotations=cat[1], scales=cat[2], opacities=cat[3])
    views = [ring_camera(i, 2.0 * math.pi * i / max(n_views, 1), 5.0, width, height,
                         float(width), elevation=float(rng.uniform(-1.0, 1.0)))
             for i in range(n_views)]
    if iid_masks:
        masks = rng.integers(0, num_objects, size=(n_views, height, width), dtype=np.uint16)
    else:
        masks = analytic_masks(views, centers, radius, num_objects, rng, label_noise)
    return Workload(scene=scene, views=views, masks=masks, num_objects=num_objects,
                    membership=membership, ball_centers=centers, ball_radius=radius,
                    name=name)


# The BASELINE.json configurations.  C1 is the reference's own
# two-cluster generator and is loaded from tests/golden instead.
CONFIGS = {
    "C2": dict(seed=2, n_gaussians=1_000_000, n_views=200, width=1008, height=756, num_objects=2),
    "C3": dict(seed=3, n_gaussians=1_000_000, n_views=200, width=1008, height=756, num_objects=32),
    "C4": dict(seed=4, n_gaussians=3_000_000, n_views=300, width=1920, height=1080, num_objects=64),
    "C5": dict(seed=5, n_gaussians=1_000_000, n_views=100, width=1008, height=756, num_objects=2,
               label_noise=0.2),
}


def config_workload(name: str, **overrides) -> Workload:
    kw = dict(CONFIGS[name])
    kw.update(overrides)
    return make_workload(name=name, **kw)
