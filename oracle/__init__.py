"""CPU oracle for the FlashSplat label-solver hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product package ``paper_2409_08270_b200`` never imports it and has no CPU
fallback.

Parity status: PINNED against golden vectors produced by the reference
package (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; checked by
``tests/test_oracle_golden.py``).

Two halves:

* ``fs_oracle.c`` (built by ``oracle/Makefile`` into ``oracle/build/liborc.so``):
  float64 restatement of projection (scene.py:228-312), binning
  (rasterizer.py:72-130), the blending walk / accumulation
  (contributions.py:90-160, view-parallel with an ordered f64 merge) and
  novel-view compositing (rasterizer.py:133-203; ``render_view`` /
  ``render_mask`` below follow rasterizer.py:206-234 and maskrender.py:45-95).
* ``one_vs_rest_wins`` / ``assign_binary`` / ``assign_scene`` below: numpy
  restatement of the float32 op sequence of solver.py:111-172.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liborc.so"
_lib = None

UNOBSERVED_EPS = np.float32(1e-12)  # solver.py:29 compared against a float32 total


class OrcCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("w2c", ctypes.c_double * 16),
        ("near_clip", ctypes.c_double),
    ]


def build() -> Path:
    """Compile the C restatement (idempotent)."""
    src = _HERE / "fs_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        L.orc_project.argtypes = [ctypes.c_int64, P, P, P, P, P, P, P, P, P, P]
        L.orc_project.restype = None
        L.orc_bin.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, ctypes.c_int, P, P]
        L.orc_bin.restype = ctypes.c_int64
        L.orc_accumulate_view.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, P, P]
        L.orc_accumulate_view.restype = ctypes.c_int
        L.orc_accumulate.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, P, P, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_int, P]
        L.orc_accumulate.restype = ctypes.c_int
        L.orc_render.argtypes = [ctypes.c_int64, P, P, P, P, P, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, P, P, ctypes.c_double, ctypes.c_double, P, P, P]
        L.orc_render.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def camera(width, height, fx, fy, cx, cy, world_to_camera, near_clip=0.01) -> OrcCamera:
    c = OrcCamera()
    c.width, c.height = int(width), int(height)
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    w = np.ascontiguousarray(world_to_camera, dtype=np.float64).reshape(16)
    for i in range(16):
        c.w2c[i] = float(w[i])
    c.near_clip = float(near_clip)
    return c


def camera_of(view) -> OrcCamera:
    """Accepts any object with the reference CameraView attributes."""
    return camera(view.width, view.height, view.fx, view.fy, view.cx, view.cy,
                  view.world_to_camera, view.near_clip)


def _scene_arrays(means, quats, scales, opac=None):
    means = np.ascontiguousarray(means, dtype=np.float64).reshape(-1, 3)
    n = means.shape[0]
    quats = np.ascontiguousarray(quats, dtype=np.float64).reshape(n, 4)
    scales = np.ascontiguousarray(scales, dtype=np.float64).reshape(n, 3)
    out = [means, quats, scales]
    if opac is not None:
        out.append(np.ascontiguousarray(opac, dtype=np.float64).reshape(n))
    return out


def project(means, quats, scales, cam: OrcCamera):
    """_project_arrays (scene.py:252-312): (alive, mean2d, conic, depth, radius, stats)."""
    means, quats, scales = _scene_arrays(means, quats, scales)
    n = means.shape[0]
    alive = np.zeros(n, np.uint8)
    mean2d = np.zeros((n, 2))
    conic = np.zeros((n, 3))
    depth = np.zeros(n)
    radius = np.zeros(n, np.int64)
    stats = np.zeros(5, np.int64)
    lib().orc_project(n, _ptr(means), _ptr(quats), _ptr(scales), ctypes.addressof(cam),
                      _ptr(alive), _ptr(mean2d), _ptr(conic), _ptr(depth), _ptr(radius),
                      _ptr(stats))
    return alive.astype(bool), mean2d, conic, depth, radius, stats


def bin_tiles(alive, mean2d, depth, radius, width, height):
    """TileBinning (rasterizer.py:72-100) as CSR: (offsets[ntiles+1], gaussian indices)."""
    alive = np.ascontiguousarray(alive, dtype=np.uint8)
    mean2d = np.ascontiguousarray(mean2d, dtype=np.float64)
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    radius = np.ascontiguousarray(radius, dtype=np.int64)
    n = alive.shape[0]
    ntiles = ((width + 15) // 16) * ((height + 15) // 16)
    offs = np.zeros(ntiles + 1, np.int64)
    total = lib().orc_bin(n, _ptr(alive), _ptr(mean2d), _ptr(depth), _ptr(radius),
                          int(width), int(height), _ptr(offs), None)
    items = np.zeros(max(total, 1), np.int64)
    lib().orc_bin(n, _ptr(alive), _ptr(mean2d), _ptr(depth), _ptr(radius),
                  int(width), int(height), _ptr(offs), _ptr(items))
    return offs, items[:total]


def accumulate_view(means, quats, scales, opac, cam: OrcCamera, mask, num_objects,
                    alpha_floor=1.0 / 255.0, t_floor=1e-4):
    """_accumulate_view (contributions.py:119-160): E x N float64 partial + walk counters."""
    means, quats, scales, opac = _scene_arrays(means, quats, scales, opac)
    n = means.shape[0]
    mask = np.ascontiguousarray(mask, dtype=np.uint16)
    part = np.zeros((num_objects, n))
    ws = np.zeros(5, np.int64)
    lib().orc_accumulate_view(n, _ptr(means), _ptr(quats), _ptr(scales), _ptr(opac),
                              ctypes.addressof(cam), _ptr(mask), int(num_objects),
                              float(alpha_floor), float(t_floor), _ptr(part), _ptr(ws))
    stats = dict(zip(("tile_steps", "lockstep_evals", "active_evals", "contrib_pairs",
                      "instances"), ws.tolist()))
    return part, stats


def accumulate(means, quats, scales, opac, cams, masks, num_objects,
               alpha_floor=1.0 / 255.0, t_floor=1e-4, threads=None, as_float32=True):
    """accumulate_contributions (contributions.py:90-116) without the input validation.

    Views run on ``threads`` host threads; per-view f64 partials are merged in
    view order, so the result does not depend on the thread count.
    """
    means, quats, scales, opac = _scene_arrays(means, quats, scales, opac)
    n = means.shape[0]
    nv = len(cams)
    cam_arr = (OrcCamera * max(nv, 1))(*cams)
    masks = [np.ascontiguousarray(m, dtype=np.uint16) for m in masks]
    mptrs = (ctypes.c_void_p * max(nv, 1))(*[m.ctypes.data for m in masks])
    total = np.zeros((num_objects, n))
    if threads is None:
        threads = os.cpu_count() or 1
    lib().orc_accumulate(n, _ptr(means), _ptr(quats), _ptr(scales), _ptr(opac), nv,
                         ctypes.addressof(cam_arr), ctypes.addressof(mptrs), int(num_objects),
                         float(alpha_floor), float(t_floor), int(threads), _ptr(total))
    return total.astype(np.float32) if as_float32 else total


def render_splats(mean2d, conic, depth, opac, channel, width, height, offsets, items,
                  alpha_floor=1.0 / 255.0, t_floor=1e-4):
    """render_property (rasterizer.py:133-203) over a binning given as CSR.

    Splat arrays (and ``opac`` / ``channel``, already gathered per splat) are
    indexed by ``items``.  Returns (value | None, alpha, depth).
    """
    mean2d = np.ascontiguousarray(mean2d, dtype=np.float64).reshape(-1, 2)
    k = mean2d.shape[0]
    conic = np.ascontiguousarray(conic, dtype=np.float64).reshape(k, 3)
    depth = np.ascontiguousarray(depth, dtype=np.float64).reshape(k)
    opac = np.ascontiguousarray(opac, dtype=np.float64).reshape(k)
    channels = 0
    ch = np.zeros(1)
    if channel is not None:
        ch = np.ascontiguousarray(channel, dtype=np.float64)
        channels = 1 if ch.ndim == 1 else ch.shape[1]
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    items = np.ascontiguousarray(items, dtype=np.int64)
    if items.size == 0:
        items = np.zeros(1, np.int64)
    rho = np.zeros((height, width))
    dep = np.zeros((height, width))
    value = np.zeros((height, width, channels) if channels > 1 else (height, width)) \
        if channels else np.zeros(1)
    lib().orc_render(k, _ptr(mean2d), _ptr(conic), _ptr(depth), _ptr(opac), _ptr(ch), channels,
                     int(width), int(height), _ptr(offsets), _ptr(items), float(alpha_floor),
                     float(t_floor), _ptr(value), _ptr(rho), _ptr(dep))
    return (value if channels else None), rho, dep


def render_view(means, quats, scales, opac, cam: OrcCamera, channel=None, member=None,
                alpha_floor=1.0 / 255.0, t_floor=1e-4):
    """render_view / render_subset_alpha_depth (rasterizer.py:206-234):
    project (scene.py:252-312), bin (rasterizer.py:72-100) and composite."""
    means, quats, scales, opac = _scene_arrays(means, quats, scales, opac)
    alive, mean2d, conic, depth, radius, _ = project(means, quats, scales, cam)
    if member is not None:
        alive = alive & np.asarray(member, dtype=bool)
    offs, items = bin_tiles(alive, mean2d, depth, radius, cam.width, cam.height)
    return render_splats(mean2d, conic, depth, opac, channel, cam.width, cam.height, offs, items,
                         alpha_floor, t_floor)


def render_mask(means, quats, scales, opac, cam: OrcCamera, membership, tau,
                alpha_floor=1.0 / 255.0, t_floor=1e-4):
    """render_scene_mask (maskrender.py:69-95); render_binary_mask is the E = 2 case
    with membership [~fg, fg] (maskrender.py:45-66).  uint16 H x W labels."""
    membership = np.asarray(membership).astype(bool)
    labels = np.zeros((cam.height, cam.width), np.uint16)
    best = np.full((cam.height, cam.width), np.inf)
    for obj in range(1, membership.shape[0]):
        if not membership[obj].any():
            continue
        _, rho, dep = render_view(means, quats, scales, opac, cam, None, membership[obj],
                                  alpha_floor, t_floor)
        wins = (rho > tau) & (dep < best)
        labels[wins] = obj
        best[wins] = dep[wins]
    return labels


# ---------------------------------------------------------------------------
# solver.py:111-172 restated in numpy (float32 op sequence, no fusion).
# ---------------------------------------------------------------------------

def check_gamma(gamma: float) -> float:
    gamma = float(gamma)
    if not -1.0 <= gamma <= 1.0:
        raise ValueError(f"gamma must lie in [-1, 1], got {gamma}")
    return gamma


def one_vs_rest_wins(values: np.ndarray, gamma: float) -> np.ndarray:
    """solver.py:118-137: E x N bool wins; every step separately rounded in f32."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    e = values.shape[0]
    total = values[0].copy()
    for row in range(1, e):  # sequential row order, as numpy's axis-0 reduce
        total += values[row]
    observed = total > UNOBSERVED_EPS
    inv = np.zeros_like(total)
    np.divide(np.float32(1.0), total, out=inv, where=observed)
    fg = values * inv
    rest = total - values
    rest *= inv
    rest += np.float32(gamma)
    return (fg > rest) & observed


def assign_binary(values: np.ndarray, gamma: float) -> np.ndarray:
    """solver.py:140-153: N uint8 labels."""
    gamma = check_gamma(gamma)
    return one_vs_rest_wins(values, gamma)[1].astype(np.uint8)


def assign_scene(values: np.ndarray, gamma: float) -> np.ndarray:
    """solver.py:156-172: E x N uint8 membership, row 0 = complement of the union."""
    gamma = check_gamma(gamma)
    wins = one_vs_rest_wins(values, gamma)
    member = np.zeros(values.shape, dtype=np.uint8)
    member[1:] = wins[1:]
    member[0] = ~member[1:].any(axis=0)
    return member


def decision_margin(values: np.ndarray, gamma: float) -> np.ndarray:
    """fg - rest per (row, column) from the reference's own f32 sequence."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    total = values.sum(axis=0, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = np.where(total > 0, 1.0 / total, 0.0)
    fg = values * inv
    rest = (total - values) * inv + gamma
    return fg - rest
