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


def load_scene_ply(path) -> GaussianScene:
    """Splat checkpoint -> GaussianScene with activations applied (reference ``ply.py:63-106``)."""
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
    cols = {p: np.asarray(verts[p]) for p in SPLAT_PROPERTIES}
    ok = np.ones(count, bool)
    for p in SPLAT_PROPERTIES:
        ok &= np.isfinite(cols[p])
    if not ok.all():
        raise SceneDataError(f"{path}: non-finite values at vertex {int(np.argmin(ok))}")

    def f64(*keys):
        return np.stack([cols[k].astype(np.float64) for k in keys], axis=1)

    scene = GaussianScene(
        means=f64("x", "y", "z"),
        rotations=f64("rot_0", "rot_1", "rot_2", "rot_3"),
        scales=np.exp(f64("scale_0", "scale_1", "scale_2")),
        opacities=1.0 / (1.0 + np.exp(-cols["opacity"].astype(np.float64))),
        colors_dc=f64("f_dc_0", "f_dc_1", "f_dc_2"),
        source_path=str(path))
    del verts
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
