"""bench.py host logic on CPU: clock-sample windowing, the atomic roofline
lookup and the --impl reference JSON line (C1, oracle on the host)."""

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import bench

ROOT = Path(__file__).resolve().parents[1]


def test_clock_window_keeps_timed_region_samples():
    c = bench.ClockSampler(0)
    busy = "1965, 1965, 900, 0x0, Not Active, Not Active, Not Active, Not Active"
    slow = "1200, 1965, 900, 0x0, Active, Not Active, Not Active, Not Active"
    c.lines = [(0.0, slow)] + [(1.0 + 0.1 * i, busy) for i in range(5)] + [(9.0, slow)]
    c.t_begin, c.t_end = 1.0, 1.5
    s = c.summary()
    assert s["window"] == "timed region" and s["samples"] == 5
    assert s["sm_mhz"] == 1965.0 and s["reasons"] == []
    # too few samples inside: warm-up + timed region, throttle reasons surface
    c.t_begin, c.t_end = 5.0, 5.0
    s = c.summary()
    assert s["window"] == "warm-up + timed region" and s["samples"] == 7
    assert s["reasons"] == ["hw_slowdown"]


def test_atomic_roofline_uses_the_l2_ceiling():
    peak, key, sized = bench.atomic_peak(16 << 20)
    assert key == "16MB_C2" and peak > 0 and sized == peak
    peak2, key2, sized2 = bench.atomic_peak(1536 << 20)
    assert key2 == "1536MB_C4" and peak2 == peak and sized2 < peak
    # the fixed-point accumulator: its own (pair-of-REDs) ceiling, classes of twice the bytes
    pf, kf, sf = bench.atomic_peak(32 << 20, fixed=True)
    assert kf == "16MB_C2" and 0 < pf < peak and sf == pf
    pf2, kf2, sf2 = bench.atomic_peak(3072 << 20, fixed=True)
    assert kf2 == "1536MB_C4" and sf2 < pf


def test_reference_arm_line(capsys):
    args = argparse.Namespace(config="C1", views=None, gaussians=None, iid=False, steps=1,
                              warmup=0, cpu_views=2, impl="reference")
    bench.run_reference(args, rank=0, world=1)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "view-px/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "view-px/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # other ranks print nothing
    bench.run_reference(args, rank=1, world=2)
    assert capsys.readouterr().out == ""


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (here on
    gloo, --launch-check: rank layout only) and reports n_gpus = 2."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-check",
                        "--views", "7"], capture_output=True, text=True, timeout=300, env=env,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["requested"] == 2
    # contiguous balanced view shards: rank 0 views 0..3, rank 1 views 4..6
    assert rec["ranks"] == [[0, 4, 0], [1, 3, 4]]
