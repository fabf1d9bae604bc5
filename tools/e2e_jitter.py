"""Distribution of end-to-end solve times (pinned inputs, scene re-uploaded every
solve) -- the bench's e2e loop, many reps.  usage: python tools/e2e_jitter.py [reps]"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_08270_b200 import _native, pin_inputs, solve, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wl = synth.config_workload("C2")
scene_h, pairs = pin_inputs(wl.scene, wl.pairs(), device=0)
solve(scene_h, pairs, 2, 0.0, "binary")
ts = []
for _ in range(reps):
    ctx = _native.context(0)
    ctx._scene_key = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solve(scene_h, pairs, 2, 0.0, "binary")
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
ts = np.array(ts)
print(os.environ.get("FS_SCENE_ORDER", "1"), "median %.1f  p90 %.1f  max %.1f  >100ms: %d" % (
    np.median(ts), np.percentile(ts, 90), ts.max(), int((ts > 100).sum())), np.round(ts[:12], 1))
