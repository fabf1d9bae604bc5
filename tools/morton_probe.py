"""Upper bound of a spatially coherent Gaussian order: the same workload solved
with its Gaussians in generator order and re-ordered along a 3-D Morton curve
(host-side permutation, no kernel change).  Prints per-solve device ms.

    python tools/morton_probe.py C2 [C4]
"""
import sys
import time

import numpy as np

from paper_2409_08270_b200 import GaussianScene, solve, synth


def morton_order(means, bits=10):
    lo, hi = means.min(0), means.max(0)
    q = ((means - lo) / np.maximum(hi - lo, 1e-30) * ((1 << bits) - 1)).astype(np.uint64)
    code = np.zeros(len(means), np.uint64)
    for b in range(bits):
        for a in range(3):
            code |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(code, kind="stable")


def timed(scene, pairs, e, reps=3):
    best = 1e9
    for _ in range(reps):
        st = {}
        solve(scene, pairs, e, 0.0, "binary" if e == 2 else "scene", stats=st)
        best = min(best, st.get("gpu_ms", 1e9))
    return best


for name in sys.argv[1:] or ["C2"]:
    wl = synth.config_workload(name)
    s = wl.scene
    e = wl.num_objects
    pairs = wl.pairs()
    perm = morton_order(s.means)
    s2 = GaussianScene(s.means[perm], s.rotations[perm], s.scales[perm], s.opacities[perm])
    solve(s, pairs[:4], e, 0.0, "binary" if e == 2 else "scene")  # warm-up
    t0 = timed(s, pairs, e)
    t1 = timed(s2, pairs, e)
    st0, st1 = {}, {}
    solve(s, pairs, e, 0.0, "binary" if e == 2 else "scene", stats=st0)
    solve(s2, pairs, e, 0.0, "binary" if e == 2 else "scene", stats=st1)
    print(name, "generator order %.2f ms, Morton order %.2f ms" % (t0, t1),
          {k: (round(st0[k], 2), round(st1[k], 2)) for k in ("prep_ms", "bin_ms", "raster_ms") if k in st0})
