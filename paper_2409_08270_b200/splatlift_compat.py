"""Drop-in switch for code written against the reference package ``splatlift``.

``install()`` rebinds the hot-path entry points everywhere the reference
imports them, so its CLI (``splatlift accumulate`` / ``splatlift assign``),
its FastAPI service and user code run on the B200 kernels unchanged:

    splatlift.accumulate_contributions / splatlift.contributions.accumulate_contributions
    splatlift.cli.accumulate_contributions                (reference cli.py:17)
    splatlift.assign_binary / assign_scene, splatlift.solver.*,
    splatlift.cli.*  (cli.py:25), splatlift.service.*     (service.py:28)
    splatlift.render_view / render_property / render_subset_alpha_depth,
    splatlift.rasterizer.*, splatlift.maskrender.*        (maskrender.py:15-21)
    splatlift.render_binary_mask / render_scene_mask,
    splatlift.maskrender.*, splatlift.cli.* (cli.py:19), splatlift.service.* (service.py:24-26)
    splatlift.load_mask_png, splatlift.masks/cli/metrics   (cli.py:20, metrics.py:10)

The replacement functions accept the reference's own ``GaussianScene``,
``CameraView``, ``LabelMask`` and ``ContributionMatrix`` objects (they only
read the documented attributes) and return objects with the reference's
attributes and file formats (``values`` / ``save`` / ``load``;
``labels`` / ``membership`` / ``save``).  ``uninstall()`` restores the
originals.

Multi-GPU: ``install(devices=...)`` makes the rebound
``accumulate_contributions`` -- the CLI's ``splatlift accumulate``
(cli.py:96-107) and any user code -- split the views over those GPUs from
the calling process (``multidevice.py``: one native thread per GPU, dynamic
view queue, peer-memory reduction).  The default ``"auto"`` uses every
visible GPU when there is more than one (``FLASHSPLAT_DEVICES=0,1,...`` or
``all`` overrides); ``None`` keeps one GPU.
"""

from __future__ import annotations

import importlib

from . import contributions as _contrib
from . import maskrender as _maskrender
from . import rasterizer as _rasterizer
from . import solver as _solver

_TARGETS = {
    "accumulate_contributions": ["splatlift", "splatlift.contributions", "splatlift.cli"],
    "assign_binary": ["splatlift", "splatlift.solver", "splatlift.cli", "splatlift.service"],
    "assign_scene": ["splatlift", "splatlift.solver", "splatlift.cli", "splatlift.service"],
    "render_view": ["splatlift", "splatlift.rasterizer", "splatlift.service"],
    "render_property": ["splatlift", "splatlift.rasterizer", "splatlift.maskrender"],
    "render_subset_alpha_depth": ["splatlift", "splatlift.rasterizer", "splatlift.maskrender"],
    "render_binary_mask": ["splatlift", "splatlift.maskrender", "splatlift.cli",
                           "splatlift.service"],
    "render_scene_mask": ["splatlift", "splatlift.maskrender", "splatlift.cli",
                          "splatlift.service"],
    "load_mask_png": ["splatlift", "splatlift.masks", "splatlift.cli", "splatlift.metrics"],
    "load_scene_ply": ["splatlift", "splatlift.ply", "splatlift.cli"],
}
_saved: dict = {}
_devices = None  # GPU list the rebound accumulate_contributions spreads views over
_device_ply = False  # load_scene_ply uploads + activates on the GPU (scene_io.PlyScene)


def resolve_devices(devices="auto"):
    """None, or the list of CUDA ordinals to use (``"auto"``: all GPUs if > 1)."""
    import os
    env = os.environ.get("FLASHSPLAT_DEVICES")
    if devices == "auto" and env:
        devices = "all" if env.strip() == "all" else [int(x) for x in env.split(",") if x.strip()]
    if devices in ("auto", "all"):
        from . import _native
        try:
            count = _native.device_count()
        except _native.NativeUnavailable:
            count = 0
        if devices == "auto" and count < 2:
            return None
        return list(range(count)) if count else None
    if devices is None:
        return None
    devices = [int(d) for d in devices]
    return devices if len(devices) > 1 else None


def _replacement(name):
    if name == "load_mask_png":
        from .masks import load_mask_png  # same array, native decode of the wire format
        return load_mask_png
    if name == "load_scene_ply":
        ref_scene = importlib.import_module("splatlift.scene").GaussianScene
        from .scene_io import load_scene_ply as impl

        def load_scene_ply(path):
            if _device_ply:
                # raw records activated on the GPU; a GaussianScene whose float64 host
                # arrays are built only if read (scene_io.PlyScene)
                return impl(path, device=_devices[0] if _devices else 0)
            s = impl(path)  # memory-mapped columns; the caller's own scene type
            return ref_scene(means=s.means, rotations=s.rotations, scales=s.scales,
                             opacities=s.opacities, colors_dc=s.colors_dc,
                             source_path=s.source_path)

        return load_scene_ply
    if name.startswith("render_") and name.endswith("_mask"):
        ref_mask = importlib.import_module("splatlift.maskrender").RenderedMask
        impl = getattr(_maskrender, name)

        def render_mask(*args, **kw):
            m = impl(*args, **kw)
            return ref_mask(view_id=m.view_id, labels=m.labels, gamma=m.gamma, tau=m.tau)

        render_mask.__name__ = name
        return render_mask
    if name.startswith("render_"):
        ref_out = importlib.import_module("splatlift.rasterizer").RenderOutput
        impl = getattr(_rasterizer, name)

        def render(*args, **kw):
            o = impl(*args, **kw)
            return ref_out(value=o.value, alpha=o.alpha, depth=o.depth)

        render.__name__ = name
        return render
    if name == "accumulate_contributions":
        ref_matrix = importlib.import_module("splatlift.contributions").ContributionMatrix

        def accumulate_contributions(scene, views, num_objects, blend=None, **kw):
            from .rasterizer import DEFAULT_BLEND
            if _devices is not None and "device" not in kw and "process_group" not in kw:
                kw.setdefault("devices", list(_devices))
            m = _contrib.accumulate_contributions(scene, views, num_objects,
                                                  blend if blend is not None else DEFAULT_BLEND,
                                                  **kw)
            return ref_matrix(values=m.values)  # the caller's own type

        return accumulate_contributions
    ref_assignment = importlib.import_module("splatlift.solver").Assignment
    impl = getattr(_solver, name)

    def assign(matrix, gamma):
        a = impl(matrix, gamma)
        return ref_assignment(mode=a.mode, gamma=a.gamma, labels=a.labels,
                              membership=a.membership)

    assign.__name__ = name
    return assign


def install(devices="auto", device_ply: bool = False) -> None:
    """Rebind the reference's entry points.  ``devices``: see resolve_devices.
    ``device_ply``: the rebound ``load_scene_ply`` (the CLI's, cli.py:97) uploads the
    checkpoint's raw records and activates them on the GPU (scene_io.PlyScene) instead
    of returning the reference's host-activated scene type."""
    global _devices, _device_ply
    _devices = resolve_devices(devices)
    _device_ply = bool(device_ply)
    for name, modules in _TARGETS.items():
        fn = _replacement(name)
        for modname in modules:
            try:
                mod = importlib.import_module(modname)
            except ImportError:
                continue
            if hasattr(mod, name):
                _saved.setdefault((modname, name), getattr(mod, name))
                setattr(mod, name, fn)


def uninstall() -> None:
    global _devices, _device_ply
    _devices = None
    _device_ply = False
    for (modname, name), fn in _saved.items():
        setattr(importlib.import_module(modname), name, fn)
    _saved.clear()
