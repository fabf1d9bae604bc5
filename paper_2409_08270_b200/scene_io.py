"""Scene ingestion: splat checkpoints in binary PLY.

Semantics follow the reference loader / writer (``ply.py:63-141``): vertex
properties are little-endian float32 pre-activation parameters; loading
applies exp to the log-scales, the logistic to the opacity logit and (in
``GaussianScene``) normalises the quaternions; writing applies the inverses
(opacity clamped to [1e-7, 1 - 1e-7] before the logit).  Errors are the
reference's ``SceneFormatError`` / ``SceneDataError`` with the same texts.

The vertex block is memory-mapped and converted column by column, so a
multi-million-splat checkpoint is read without an intermediate copy of the
whole record array; the activations are the same float64 numpy expressions
as the reference's.

``load_scene_ply(path, device=d)`` is the device path:
the float32 records go to the GPU as the file stores them (one upload of
4 * properties bytes per splat -- 68 B for a 17-property checkpoint instead
of the 88 B float64 scene) and one kernel applies the activations and the
scene's validation (``fs_set_scene_ply``).  The returned ``PlyScene`` is a
GaussianScene whose float64 host arrays are only computed -- with the
reference's numpy expressions -- if something reads them; solving never does.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .scene import GaussianScene, SceneDataError, SceneFormatError

# vertex properties a checkpoint must carry (reference ply.py:17-23)
SPLAT_PROPERTIES = ("x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity",
                    "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3")
REQUIRED_PROPERTIES = SPLAT_PROPERTIES


def _read_header(raw: bytes):
    """(vertex count, property names, byte offset of the payload)."""
    if not raw.startswith(b"ply\n") and not raw.startswith(b"ply\r\n"):
        raise SceneFormatError("not a PLY file (missing 'ply' magic)")
    end = raw.find(b"end_header")
    if end < 0:
        raise SceneFormatError("unterminated PLY header")
    nl = raw.find(b"\n", end)
    payload = len(raw) if nl < 0 else nl + 1
    count, names, element = None, [], None
    for text in raw[:end].decode("ascii", errors="replace").splitlines()[1:]:
        words = text.split()
        if not words:
            continue
        key = words[0]
        if key == "format" and "binary_little_endian" not in text:
            raise SceneFormatError(
                f"unsupported PLY format: {text.strip()!r} (need binary_little_endian)")
        if key == "element":
            element = words[1]
            if element == "vertex":
                count = int(words[2])
        elif key == "property" and element == "vertex":
            if words[1] not in ("float", "float32"):
                raise SceneFormatError(f"unsupported property type {words[1]!r} for {words[2]!r}")
            names.append(words[2])
    if count is None:
        raise SceneFormatError("PLY header has no vertex element")
    return count, names, payload


class PlyScene(GaussianScene):
    """A checkpoint resident on the GPU from its raw float32 records.

    Behaves as the reference's GaussianScene: ``means`` / ``rotations`` /
    ``scales`` / ``opacities`` / ``colors_dc`` are the loader's float64 arrays
    (ply.py:94-98, normalised quaternions scene.py:96-100), computed on the
    host on first access.  The solver uploads ``_ply_block`` to every GPU it
    uses instead (``Context.set_scene``).
    """

    def __init__(self, path, count: int, names: list, block: np.ndarray, verts: np.ndarray):
        self.source_path = str(path)
        self._ply_count = int(count)
        self._ply_block = block          # count x len(names) float32 records (memmap)
        self._ply_stride = len(names)
        self._ply_offsets = np.array([names.index(p) for p in SPLAT_PROPERTIES], np.int32)
        self._ply_verts = verts          # the same bytes as a structured array
        self._host = None

    def __len__(self) -> int:
        return self._ply_count

    def _arrays(self) -> dict:
        if self._host is None:
            cols = {p: np.asarray(self._ply_verts[p]) for p in SPLAT_PROPERTIES}
            s = _activated_scene(cols, self.source_path)
            self._host = {k: getattr(s, k) for k in
                          ("means", "rotations", "scales", "opacities", "colors_dc")}
        return self._host

    means = property(lambda self: self._arrays()["means"])
    rotations = property(lambda self: self._arrays()["rotations"])
    scales = property(lambda self: self._arrays()["scales"])
    opacities = property(lambda self: self._arrays()["opacities"])
    colors_dc = property(lambda self: self._arrays()["colors_dc"])


def _activated_scene(cols: dict, source_path: str) -> GaussianScene:
    def f64(*keys):
        return np.stack([cols[k].astype(np.float64) for k in keys], axis=1)

    return GaussianScene(
        means=f64("x", "y", "z"),
        rotations=f64("rot_0", "rot_1", "rot_2", "rot_3"),
        scales=np.exp(f64("scale_0", "scale_1", "scale_2")),
        opacities=1.0 / (1.0 + np.exp(-cols["opacity"].astype(np.float64))),
        colors_dc=f64("f_dc_0", "f_dc_1", "f_dc_2"),
        source_path=source_path)


def load_scene_ply(path, device=None) -> GaussianScene:
    """Splat checkpoint -> GaussianScene with activations applied (reference ``ply.py:63-106``).

    ``device``: CUDA ordinal -- upload the raw records and activate / validate
    them on that GPU (returns a ``PlyScene``, already resident there); the
    errors are the reference's, for the same vertex.
    """
    path = Path(path)
    with open(path, "rb") as fh:
        head = fh.read(1 << 16)
    count, names, offset = _read_header(head)
    for required in SPLAT_PROPERTIES:
        if required not in names:
            raise SceneFormatError(f"{path}: missing required vertex property '{required}'")
    if count < 1:
        raise SceneDataError(f"{path}: scene has no vertices")
    rec = np.dtype([(p, "<f4") for p in names])
    avail = (path.stat().st_size - offset) // rec.itemsize
    if avail < count:
        raise SceneFormatError(f"{path}: truncated payload ({avail}/{count} vertices)")
    verts = np.memmap(path, dtype=rec, mode="r", offset=offset, shape=(count,))
    if device is not None:
        block = np.memmap(path, dtype=np.float32, mode="r", offset=offset,
                          shape=(count, len(names)))
        return _load_on_device(path, PlyScene(path, count, names, block, verts), device)
    cols = {p: np.asarray(verts[p]) for p in SPLAT_PROPERTIES}
    ok = np.ones(count, bool)
    for p in SPLAT_PROPERTIES:
        ok &= np.isfinite(cols[p])
    if not ok.all():
        raise SceneDataError(f"{path}: non-finite values at vertex {int(np.argmin(ok))}")

    scene = _activated_scene(cols, str(path))
    del verts
    return scene


def _load_on_device(path, scene: PlyScene, device: int) -> PlyScene:
    """Upload + activate + validate on the GPU; the reference's first error."""
    from . import _native

    ctx = _native.context(device)
    with ctx.lock:
        bad = ctx.set_scene_ply(scene)
        ok = not (bad >= 0).any()
        if ok:
            ctx._scene_key = ("ply", id(scene), len(scene))
            ctx._scene_ref = scene
    if bad[0] >= 0:  # ply.py:84-88, before the scene is built
        raise SceneDataError(f"{path}: non-finite values at vertex {int(bad[0])}")
    if bad[1] >= 0:  # scene.py:96-99
        raise SceneDataError(f"quaternion {int(bad[1])} has zero or non-finite norm")
    if bad[2] >= 0:
        raise SceneDataError(f"gaussian {int(bad[2])} has non-positive scale")
    if bad[3] >= 0:
        raise SceneDataError(f"gaussian {int(bad[3])} has opacity outside [0, 1]")
    return scene


def export_ply(scene: GaussianScene, path) -> None:
    """GaussianScene -> checkpoint with inverse activations (reference ``ply.py:109-141``)."""
    path = Path(path)
    n = len(scene)
    rec = np.zeros(n, dtype=np.dtype([(p, "<f4") for p in SPLAT_PROPERTIES]))
    for k, axis in zip(("x", "y", "z"), scene.means.T):
        rec[k] = axis
    if scene.colors_dc is not None:
        for k, axis in zip(("f_dc_0", "f_dc_1", "f_dc_2"), scene.colors_dc.T):
            rec[k] = axis
    clipped = np.clip(scene.opacities, 1e-7, 1.0 - 1e-7)
    rec["opacity"] = np.log(clipped / (1.0 - clipped))
    for k, axis in zip(("scale_0", "scale_1", "scale_2"), np.log(scene.scales).T):
        rec[k] = axis
    for k, axis in zip(("rot_0", "rot_1", "rot_2", "rot_3"), scene.rotations.T):
        rec[k] = axis
    lines = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    lines += [f"property float {p}" for p in SPLAT_PROPERTIES] + ["end_header"]
    try:
        with open(path, "wb") as fh:
            fh.write(("\n".join(lines) + "\n").encode("ascii"))
            rec.tofile(fh)
    except OSError as exc:
        raise OSError(f"cannot write scene to {path}: {exc}") from exc
