import sys, time, numpy as np
sys.path.insert(0, ".")
from paper_2409_08270_b200 import synth, render_scene_mask, Assignment, _native
wl = synth.make_workload(seed=2, n_gaussians=1000000, n_views=2, width=1008, height=756, num_objects=32)
rng = np.random.default_rng(1)
memb = np.zeros((32, len(wl.scene)), np.uint8)
memb[rng.integers(0, 32, size=len(wl.scene)), np.arange(len(wl.scene))] = 1
asn = Assignment(mode="scene", gamma=0.0, membership=memb)
render_scene_mask(wl.scene, asn, wl.views[1])
ctx = _native.context(0)
ctx.set_scene(wl.scene)
for _ in range(3):
    t0 = time.perf_counter(); ctx.render_mask(wl.views[1], memb, 0.5, 1/255, 1e-4); t1 = time.perf_counter()
    print("native render_mask", (t1 - t0) * 1e3, "ms")
