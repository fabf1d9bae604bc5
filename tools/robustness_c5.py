"""Noisy-mask robustness sweep (BASELINE config C5): one accumulation over
100 views whose masks carry 20% iid label noise, then the biased argmax for
gamma in {0, 0.2, 0.5} on the device-resident matrix; labels scored against the
ground-truth membership of the synthetic scene (and, for reference, the same
scene with clean masks).

usage: python tools/robustness_c5.py [--out JSON]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import synth  # noqa: E402
from paper_2409_08270_b200.solve import LabelSolver  # noqa: E402


def scores(pred_fg: np.ndarray, gt_fg: np.ndarray, observed: np.ndarray) -> dict:
    tp = int(np.count_nonzero(pred_fg & gt_fg))
    fp = int(np.count_nonzero(pred_fg & ~gt_fg))
    fn = int(np.count_nonzero(~pred_fg & gt_fg))
    obs = observed
    return {"accuracy": float(np.mean(pred_fg == gt_fg)),
            "accuracy_observed": float(np.mean(pred_fg[obs] == gt_fg[obs])),
            "iou_fg": tp / max(tp + fp + fn, 1), "precision": tp / max(tp + fp, 1),
            "recall": tp / max(tp + fn, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {}
    for name, noise in (("C5_noisy", 0.2), ("C5_clean", 0.0)):
        wl = synth.config_workload("C5", label_noise=noise)
        gt_fg = wl.membership != 0
        s = LabelSolver(wl.scene)
        t0 = time.perf_counter()
        M = s.accumulate(wl.pairs(), wl.num_objects)
        t_acc = time.perf_counter() - t0
        observed = M.observed
        res = {"label_noise": noise, "gaussians": len(wl.scene), "views": len(wl.views),
               "observed": int(observed.sum()), "accumulate_s": t_acc, "gamma": {}}
        for g in (0.0, 0.2, 0.5):
            t0 = time.perf_counter()
            asn = s.assign(g, "binary")
            dt = time.perf_counter() - t0
            r = scores(asn.labels.astype(bool), gt_fg, observed)
            r["assign_ms"] = dt * 1e3
            res["gamma"][str(g)] = r
        out[name] = res
        print(name, json.dumps(res["gamma"]), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
