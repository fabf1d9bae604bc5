"""Time fs_set_scene / the PLY device loader with and without the spatial order."""
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_08270_b200 import _native, export_ply, load_scene_ply, synth  # noqa: E402

wl = synth.config_workload("C2", n_views=2)
ctx = _native.context(0)
with tempfile.TemporaryDirectory() as d:
    path = Path(d) / "s.ply"
    export_ply(wl.scene, path)
    for rep in range(4):
        with ctx.lock:
            t0 = time.perf_counter()
            ctx.set_scene(wl.scene)
            t1 = time.perf_counter()
            ctx._scene_key = None
        t2 = time.perf_counter()
        sc = load_scene_ply(path, device=0)
        t3 = time.perf_counter()
        ctx._scene_key = None
        print(os.environ.get("FS_SCENE_ORDER", "1"), "set_scene %.1f ms" % ((t1 - t0) * 1e3),
              "ply device load %.1f ms" % ((t3 - t2) * 1e3))
