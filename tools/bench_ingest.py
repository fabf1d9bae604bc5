"""Mask ingestion on the C2 workload: 200 16-bit PNG masks.

  serial    -- the reference CLI's flow: load_mask_png per view in order, then
               accumulate_contributions (cli.py:74-104), on this package's GPU path
  pipelined -- accumulate_mask_files: thread-pool decode overlapped with the
               device accumulation
Wall clock, PNGs written once to a scratch directory first.

usage: python tools/bench_ingest.py [--views V] [--dir DIR]
"""

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import (LabelMask, accumulate_contributions,  # noqa: E402
                                   accumulate_mask_files, load_mask_png, save_mask_png, synth)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--dir", default=None)
    a = ap.parse_args()
    wl = synth.config_workload("C2", n_views=a.views)
    d = Path(a.dir or tempfile.mkdtemp(prefix="fs_masks_"))
    d.mkdir(parents=True, exist_ok=True)
    paths = []
    for v, m in zip(wl.views, wl.masks):
        p = d / f"{v.view_id}.png"
        save_mask_png(p, m)
        paths.append((v, p))
    E = wl.num_objects
    accumulate_mask_files(wl.scene, paths[:8], E)  # warm: context, scene
    t0 = time.perf_counter()
    pairs = [(v, LabelMask(v.view_id, load_mask_png(p))) for v, p in paths]
    t1 = time.perf_counter()
    accumulate_contributions(wl.scene, pairs, E)
    t2 = time.perf_counter()
    accumulate_mask_files(wl.scene, paths, E)
    t3 = time.perf_counter()
    png_mb = sum(p.stat().st_size for _, p in paths) / 1e6
    print(json.dumps({
        "views": len(paths), "png_MB": round(png_mb, 1), "raw_MB": round(wl.masks.nbytes / 1e6, 1),
        "serial_s": {"decode": t1 - t0, "accumulate": t2 - t1, "total": t2 - t0},
        "pipelined_s": t3 - t2}))


if __name__ == "__main__":
    main()
