"""Dump one fuzz render case's GPU outputs (scene mask + per-object alpha/depth)
to gpurun_out/ for comparison with the oracle / reference here."""
import sys

import numpy as np

sys.path.insert(0, "tests")
from conftest import cam_from_row  # noqa: E402
from fuzz_cases import case_arrays, render_extras  # noqa: E402
from paper_2409_08270_b200 import (Assignment, BlendConfig, GaussianScene, render_scene_mask,  # noqa: E402
                                   render_subset_alpha_depth)

seed = int(sys.argv[1])
c = case_arrays(seed)
scene = GaussianScene(c["means"], c["quats"], c["scales"], c["opac"])
pairs = [(cam_from_row(r, i), None) for i, r in enumerate(c["cams"])]
E, blend = c["E"], BlendConfig(*c["floors"])
_, memb, tau = render_extras(seed, len(scene), E)
out = {}
for vi, (cam, _) in enumerate(pairs):
    out[f"mask{vi}"] = render_scene_mask(scene, Assignment(mode="scene", gamma=0.0, membership=memb),
                                         cam, tau, blend).labels
    for obj in range(1, E):
        r = render_subset_alpha_depth(scene, cam, memb[obj].astype(bool), blend)
        out[f"alpha{vi}_{obj}"] = r.alpha
        out[f"depth{vi}_{obj}"] = r.depth
np.savez(f"gpurun_out/fuzz_case_{seed}.npz", **out)
print("saved", len(out))
