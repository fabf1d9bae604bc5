"""Full-size parity check: one config end to end on the GPU against the C oracle
(all host threads), reported the way the north star states the bar.

  * A: max |dA| / (atol + rtol |A_ref|) with rtol 1e-4, atol 1e-6 (north star),
    and the fraction of float32 entries bit-identical;
  * labels: bit-exact count; flips inside the reference's decision band
    (|margin| <= 4 (rtol + atol / total)) are reported apart.

usage: python tools/parity_full.py [--config C2] [--views V] [--out JSON]
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (checker only)
from paper_2409_08270_b200 import solve, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--views", type=int, default=None)
    ap.add_argument("--gamma", type=float, default=0.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wl = (synth.config_workload(a.config, n_views=a.views) if a.views
          else synth.config_workload(a.config))
    E = wl.num_objects
    mode = "binary" if E == 2 else "scene"
    t0 = time.perf_counter()
    A, asn = solve(wl.scene, wl.pairs(), E, a.gamma, mode)
    t_gpu = time.perf_counter() - t0
    cams = [oracle.camera_of(v) for v in wl.views]
    t0 = time.perf_counter()
    ref64 = oracle.accumulate(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                              wl.scene.opacities, cams, list(wl.masks), E, 1 / 255, 1e-4,
                              threads=os.cpu_count(), as_float32=False)
    t_cpu = time.perf_counter() - t0
    ref = ref64.astype(np.float32)
    got = A.values
    rtol, atol = 1e-4, 1e-6
    ratio = np.abs(got.astype(np.float64) - ref64) / (atol + rtol * np.abs(ref64))
    if mode == "binary":
        ref_lab = oracle.assign_binary(ref, a.gamma)
        lab = asn.labels
    else:
        ref_lab = oracle.assign_scene(ref, a.gamma)
        lab = asn.membership
    margin = oracle.decision_margin(ref, a.gamma)
    total = ref.astype(np.float64).sum(axis=0)
    band = np.abs(margin) <= 4 * (rtol + atol / np.maximum(total, 1e-30))
    flips = (lab != ref_lab)
    if flips.ndim == 2:
        flips = flips.any(axis=0)
    band = band[1] if mode == "binary" else band.any(axis=0)  # binary decides on row 1
    out = {
        "config": a.config, "views": len(wl.views), "gaussians": len(wl.scene), "E": E,
        "matrix": {"max_err_over_tolerance": float(ratio.max()),
                   "entries_bit_identical": float(np.mean(got == ref)),
                   "max_abs_diff": float(np.abs(got - ref).max())},
        "labels": {"mode": mode, "gamma": a.gamma, "flips": int(flips.sum()),
                   "flips_outside_band": int((flips & ~band).sum()),
                   "band_size": int(band.sum()), "gaussians": int(flips.size)},
        "seconds": {"gpu_solve_e2e": t_gpu, "cpu_oracle": t_cpu, "cpu_threads": os.cpu_count()},
    }
    print(json.dumps(out))
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
