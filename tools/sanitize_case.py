"""Small GPU workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library at least once, without torch.

  C1        the two-cluster golden (8 views 128x128, 10k Gaussians), both
            accumulator kinds, finalize, assign (binary + scene), render, bin
  C2 view   one 1008x756 view of the C2 scene, fixed-point accumulator
  long      buckets past the in-smem sort (the chunk-sort + global-merge path)
  multi     devices=[0, 0]: the dynamic view queue and the two-part finalize

usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py [c1|c2|long|multi|all]
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import cam_from_row, load_golden  # noqa: E402
from paper_2409_08270_b200 import (  # noqa: E402
    EXACT_BLEND, CameraView, GaussianScene, LabelMask, accumulate_contributions, assign_binary,
    assign_scene, render_view, solve, synth)
from paper_2409_08270_b200 import _native  # noqa: E402


def c1():
    c = load_golden("accumulate")["C1_default"]
    scene = GaussianScene(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"])
    pairs = [(cam_from_row(r, i), LabelMask(i, m)) for i, (r, m) in enumerate(zip(c["cams"],
                                                                                c["masks"]))]
    A = accumulate_contributions(scene, pairs, 2).values
    A64 = accumulate_contributions(scene, pairs, 2, deterministic=False).values
    assign_binary(fs_matrix(A), 0.0)
    assign_scene(fs_matrix(np.vstack([A, A64[1:]])), 0.1)
    accumulate_contributions(scene, pairs[:2], 2, EXACT_BLEND)
    render_view(scene, pairs[0][0], np.linspace(0, 1, len(scene)))
    ctx = _native.context(0)
    with ctx.lock:
        ctx.set_scene(scene)
        ctx.bin(pairs[0][0])
    print("c1 ok", float(A.sum()))


def fs_matrix(v):
    from paper_2409_08270_b200 import ContributionMatrix
    return ContributionMatrix(values=v)


def c2():
    wl = synth.config_workload("C2", n_views=1)
    M, asn = solve(wl.scene, wl.pairs(), 2, 0.0, "binary")
    print("c2 view ok", float(M.values.sum()), int(asn.labels.sum()))


def long():
    rng = np.random.default_rng(17)
    n = 10000
    means = np.stack([rng.uniform(-0.3, 0.3, n), rng.uniform(-0.2, 0.2, n),
                      rng.choice(np.linspace(3.0, 4.0, 50), size=n)], axis=1)
    scene = GaussianScene(means, rng.normal(size=(n, 4)), rng.uniform(0.05, 0.4, (n, 3)),
                          rng.uniform(0.01, 0.05, n))
    view = CameraView(0, 64, 48, 60.0, 60.0, 32.0, 24.0, np.eye(4))
    m = LabelMask(0, rng.integers(0, 3, (48, 64), dtype=np.uint16))
    A = accumulate_contributions(scene, [(view, m)], 3).values
    print("long buckets ok", float(A.sum()))


def multi():
    wl = synth.make_workload(seed=25, n_gaussians=50000, n_views=6, width=256, height=192,
                             num_objects=4)
    M, asn = solve(wl.scene, wl.pairs(), 4, 0.1, "scene", devices=[0, 0])
    print("multi ok", float(M.values.sum()))


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("c1", c1), ("c2", c2), ("long", long), ("multi", multi)):
        if which in (name, "all"):
            fn()
