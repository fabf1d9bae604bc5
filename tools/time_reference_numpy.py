"""Times the REFERENCE implementation itself (splatlift, numpy) on this host -- the
build container, where /root/reference exists (it does not exist on the GPU box,
so bench.py's CPU arm is the pinned C port instead).

One process per core runs the reference's own per-view kernel
``contributions._accumulate_view`` (contributions.py:119-160) on one view of the
C2 workload each (SURVEY 8(d) view-parallel harness); the parent sums the float64
partials in view order and casts once, exactly as accumulate_contributions does
(contributions.py:103-116).  Reports view-px/s for 1 process and for P processes.

usage: python tools/time_reference_numpy.py [--views 16] [--gaussians 1000000] [--out JSON]
"""

import argparse
import json
import os
import platform
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

_WL = None


def _init(n, views):
    global _WL
    from paper_2409_08270_b200 import synth
    _WL = synth.config_workload("C2", n_gaussians=n, n_views=views)


def _one(i):
    import splatlift as ref
    from splatlift import contributions as rc
    wl = _WL
    sc = ref.GaussianScene(means=wl.scene.means, rotations=wl.scene.rotations,
                           scales=wl.scene.scales, opacities=wl.scene.opacities)
    v = wl.views[i]
    rv = ref.CameraView(view_id=v.view_id, width=v.width, height=v.height, fx=v.fx, fy=v.fy,
                        cx=v.cx, cy=v.cy, world_to_camera=v.world_to_camera,
                        near_clip=v.near_clip)
    t0 = time.perf_counter()
    part = rc._accumulate_view(sc, rv, ref.LabelMask(v.view_id, wl.masks[i]), 2,
                               ref.DEFAULT_BLEND)
    return i, part, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    procs = min(a.views, os.cpu_count() or 1)
    px = 1008 * 756
    t0 = time.perf_counter()
    with ProcessPoolExecutor(procs, initializer=_init, initargs=(a.gaussians, a.views)) as ex:
        res = sorted(ex.map(_one, range(a.views)))
    wall = time.perf_counter() - t0
    total = np.zeros_like(res[0][1])
    for _, part, _ in res:
        total += part
    per_view = [t for _, _, t in res]
    out = {"implementation": "reference splatlift (numpy), contributions._accumulate_view",
           "host": platform.processor() or platform.machine(), "cpus": os.cpu_count(),
           "workload": f"C2 scene ({a.gaussians} Gaussians), {a.views} views 1008x756, E=2",
           "single_process_view_px_per_s": px / float(np.median(per_view)),
           "median_s_per_view_one_core": float(np.median(per_view)),
           "processes": procs, "wall_s": wall,
           "parallel_view_px_per_s": a.views * px / wall,
           "note": "measured in the build container (the reference does not exist on the GPU "
                   "box); wall includes the workers' workload generation"}
    print(json.dumps(out))
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
