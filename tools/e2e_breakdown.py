"""Time the phases of the public solve() path on the workload of bench.py (diagnostic)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2409_08270_b200 import _native, synth  # noqa: E402
from paper_2409_08270_b200.contributions import validate_views  # noqa: E402
from paper_2409_08270_b200.solve import LabelSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = synth.config_workload(name)
pairs = wl.pairs()
E, N = wl.num_objects, len(wl.scene)
ctx = _native.context(0)
for rep in range(3):
    t = {}
    t0 = time.perf_counter()
    validate_views(pairs, E)
    t["validate"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ctx._scene_key = None
    ctx.set_scene(wl.scene)
    t["scene_upload"] = time.perf_counter() - t0
    acc = ctx.acc_buffer(E, N).zero()
    t0 = time.perf_counter()
    st = ctx.accumulate([v for v, _ in pairs], [m.labels for _, m in pairs], E, 1 / 255, 1e-4, acc.ptr)
    t["accumulate_host_masks"] = time.perf_counter() - t0
    t["accumulate_gpu_ms"] = st["gpu_ms"] / 1e3
    out = np.empty((E, N), np.float32)
    t0 = time.perf_counter()
    ctx.finalize(acc.ptr, N, E, out=out)
    t["finalize_d2h"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _native.assign(out, 0.0, _native.MODE_BINARY if E == 2 else _native.MODE_SCENE)
    t["assign_host"] = time.perf_counter() - t0
    s = LabelSolver(wl.scene)
    ctx._scene_key = None
    t0 = time.perf_counter()
    s.accumulate(pairs, E)
    s.assign(0.0, "binary" if E == 2 else "scene")
    t["solve_total"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 1) for k, v in t.items()}, flush=True)
