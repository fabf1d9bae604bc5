"""C2 scene seen through a 3x narrower field of view (about 1/9 of the Gaussians
in frame): device time of the solve -- the case where culled splats dominate."""
import dataclasses
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_08270_b200 import LabelMask, solve, synth  # noqa: E402

wl = synth.config_workload("C2")
pairs = [(dataclasses.replace(v, fx=v.fx * 3, fy=v.fy * 3), LabelMask(v.view_id, m.labels))
         for v, m in wl.pairs()]
solve(wl.scene, pairs[:4], 2, 0.0, "binary")
best = 1e9
for _ in range(4):
    st = {}
    solve(wl.scene, pairs, 2, 0.0, "binary", stats=st)
    best = min(best, st["gpu_ms"])
print("narrow FOV C2: %.2f ms, emitted per view %.0f" % (best, st["emitted"] / len(pairs)))
