#!/usr/bin/env python
"""bench.py -- FlashSplat label-solver throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one full label solve of the configuration's scene: for every view
project -> depth sort -> bin -> raster-accumulate into the N x E accumulator
(deterministic fixed-point by default, ``--acc f64`` for float64 atomics);
N>1: reduce-scatter of the accumulator, float32 cast + biased argmax of the
rank's Gaussian slice, all-gather of the matrix and labels; N=1: cast +
argmax.  Views are sharded over ranks (strong scaling: the scene is fixed,
more GPUs split its views).  ``--gpus N`` without torchrun re-launches itself
under ``torch.distributed.run`` with N ranks (one per GPU).  After the timed
region rank 0 re-solves the whole scene on its own GPU and compares: with the
fixed-point accumulator the sharded matrix must be bit-identical
(``shard_check``; at N=1 a 1-stream re-run checks schedule independence).  ``value`` = view-pixels of the scene / device time per
step with inputs resident in HBM (CUDA events on the launching side, barrier
+ synchronize around the K steps, max over ranks).  ``e2e`` = the same
metric through the public API ``solve()`` from host numpy inputs (scene +
masks H2D, matrix + labels D2H every step).

``--impl reference`` times the reference algorithm on the host CPU cores:
the pinned CPU restatement in oracle/ (float64, view-parallel over all
threads), on a bounded sample of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# algorithmic bytes of one raster-accumulate launch
BYTES_PER_PIXEL = 2          # uint16 label
BYTES_PER_TILE_STEP = 36     # 4 B instance index + 32 B projected record
BYTES_PER_ATOMIC = {0: 8, 1: 16}  # accumulator add: float64 / fixed-point (hi, lo) words


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--views", type=int, default=None, help="override the view count")
    ap.add_argument("--gaussians", type=int, default=None, help="override the Gaussian count")
    ap.add_argument("--streams", type=int, default=6)
    ap.add_argument("--iid", action="store_true",
                    help="worst case: iid uniform labels per pixel instead of object silhouettes")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-views", type=int, default=None)
    ap.add_argument("--acc", default="fixed", choices=["fixed", "f64"],
                    help="accumulator: deterministic fixed-point (default) or float64 atomics")
    ap.add_argument("--no-check", action="store_true", help="skip the shard / rerun identity check")
    ap.add_argument("--launch-check", action="store_true",
                    help="(tests) only report the rank layout; runs without a GPU (gloo)")
    return ap.parse_args()


def self_launch(args) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run, N ranks."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator / NVLS setup in the log ...
    env.setdefault("NCCL_DEBUG_FILE", "/tmp/flashsplat_nccl.%h.%p.log")  # ... not on stdout
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def launch_check(args, rank, world):
    """Rank layout only (CPU test of the --gpus N launch path, gloo backend)."""
    import torch
    import torch.distributed as dist

    from paper_2409_08270_b200.distributed import shard_views
    dist.init_process_group("gloo")
    n_views = args.views or 200
    mine = shard_views(n_views, rank, world)
    t = torch.tensor([rank, len(mine), mine[0] if mine else -1], dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "requested": args.gpus,
                          "ranks": [[int(x) for x in o] for o in out]}), flush=True)
    dist.destroy_process_group()


def load_workload(name, views=None, gaussians=None, iid=False):
    from paper_2409_08270_b200 import synth
    from paper_2409_08270_b200.scene import CameraView, GaussianScene
    if name == "C1":
        with np.load(ROOT / "tests" / "golden" / "accumulate.npz") as z:
            c = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith("C1_default/")}
        scene = GaussianScene(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"])
        cams = [CameraView(i, int(r[0]), int(r[1]), r[2], r[3], r[4], r[5],
                           np.asarray(r[7:23]).reshape(4, 4), r[6]) for i, r in enumerate(c["cams"])]
        return synth.Workload(scene=scene, views=cams, masks=np.ascontiguousarray(c["masks"]),
                              num_objects=2, membership=np.zeros(len(scene), np.uint16), name="C1")
    over = {}
    if views:
        over["n_views"] = views
    if gaussians:
        over["n_gaussians"] = gaussians
    if iid:
        over["iid_masks"] = True
    return synth.config_workload(name, **over)


CONFIG_TEXT = {
    "C1": "make_two_cluster(seed=0) 10k Gaussians, 8 views 128x128, binary",
    "C2": "synthetic 1M Gaussians, 200 views 1008x756, binary (E=2)",
    "C3": "synthetic 1M Gaussians, 200 views 1008x756, scene L=32",
    "C4": "synthetic 3M Gaussians, 300 views 1920x1080, L=64",
    "C5": "synthetic 1M Gaussians, 100 views 1008x756, E=2, 20% label noise",
}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []  # (arrival time, csv line)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, begin: bool):
        """Bracket the timed region (samples outside it are dropped when enough lie inside)."""
        if begin:
            self.t_begin = time.perf_counter()
        else:
            self.t_end = time.perf_counter()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = getattr(self, "t_begin", None), getattr(self, "t_end", None)
        lines = [ln for t, ln in self.lines]
        if lo is not None and hi is not None:
            inside = [ln for t, ln in self.lines if lo <= t <= hi + 0.25]
            window = "timed region"
            if len(inside) < 3:  # short region: include the warm-up steps (also under load)
                inside, window = lines, "warm-up + timed region"
            lines = inside
        else:
            window = "run"
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": window}


def workload_config(args, wl):
    """The workload's `config` object -- identical in both arms (--impl ours / reference)."""
    return {"workload": CONFIG_TEXT[args.config] + (" (iid labels)" if args.iid else ""),
            "name": args.config + ("-iid" if args.iid else ""),
            "gaussians": len(wl.scene), "views": len(wl.views),
            "image": f"{wl.views[0].width}x{wl.views[0].height}", "num_objects": wl.num_objects,
            # timing rule: inputs larger than L2 (126 MB) between timed steps
            "l2": "inputs larger than L2 (masks %.0f MB + scene %.0f MB)" % (
                wl.masks.nbytes / 1e6, len(wl.scene) * 88 / 1e6)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def atomic_peak(acc_bytes, fixed=False):
    """R_atom (tools/atomic_peak.cu): the L2 ceiling of the accumulator adds -- 16 random
    lanes per warp instruction into an L2-resident buffer (float64 RED, or the fixed-point
    accumulator's pair of uint64 REDs) -- plus, for context, the uniform-random rate into a
    buffer of the accumulator's size (a floor: real scatters have far more locality)."""
    p = ROOT / "profiles" / "r2_atomic_peak.json"
    if not p.exists():
        p = ROOT / "profiles" / "r1_atomic_peak.json"
    if not p.exists():
        return None, None, None
    res = json.loads(p.read_text())["results"]
    key = "fixed_pair_rand16" if fixed and "fixed_pair_rand16" in res["16MB_C2"] else "f64_rand16"
    scale = 2 if key == "fixed_pair_rand16" else 1  # the fixed classes hold twice the bytes
    cls = ("16MB_C2" if acc_bytes <= scale * (64 << 20) else
           ("256MB_C3" if acc_bytes <= scale * (768 << 20) else "1536MB_C4"))
    return res["16MB_C2"][key] * 1e9, cls, res[cls][key] * 1e9


def pipe_peaks():
    """Measured pipe rates of this B200 (tools/pipe_peak.cu -> profiles/r2_pipe_peak.json):
    DFMA / FFMA / MUFU.EX2 thread-ops per SM per clock."""
    p = ROOT / "profiles" / "r2_pipe_peak.json"
    if not p.exists():
        return None
    return json.loads(p.read_text())


def cpu_baseline(wl, views_override=None):
    """Oracle (float64 restatement, pinned to the reference) on all host threads."""
    import oracle
    cores = os.cpu_count() or 1
    k = views_override or min(len(wl.views), max(cores, 2))
    k = min(k, len(wl.views))
    sel = list(range(k))
    cams = [oracle.camera_of(wl.views[i]) for i in sel]
    masks = [wl.masks[i] for i in sel]
    threads = min(cores, k)
    t0 = time.perf_counter()
    A = oracle.accumulate(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                          wl.scene.opacities, cams, masks, wl.num_objects, threads=threads)
    # the whole solve path: the biased argmax over all N columns (solver.py:118-172)
    (oracle.assign_binary if wl.num_objects == 2 else oracle.assign_scene)(A, 0.0)
    dt = time.perf_counter() - t0
    px = sum(wl.views[i].width * wl.views[i].height for i in sel)
    return {"value": px / dt, "unit": "view-px/s", "cores": threads, "kind": "port",
            "sample": f"{k} of {len(wl.views)} views ({px} view-px), all {len(wl.scene)} Gaussians, "
                      f"accumulate + argmax, {dt:.2f} s wall", "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    wl = load_workload(args.config, args.views, args.gaussians, args.iid)
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    k = args.cpu_views or min(len(wl.views), max(cores, 2))
    times = []
    for step in range(args.warmup + args.steps):
        r = cpu_baseline(wl, k)
        if step >= args.warmup:
            times.append(r["seconds"])
    px = sum(wl.views[i].width * wl.views[i].height for i in range(min(k, len(wl.views))))
    mean_s = float(np.mean(times))
    value = px / mean_s
    line = {
        "impl": "reference", "metric": "view-pixels/sec of contribution accumulation",
        "value": value, "unit": "view-px/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, wl),
        "cpu_baseline": {"value": value, "unit": "view-px/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": "view-px/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:
        return launch_check(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2409_08270_b200 import _native, solve
    from paper_2409_08270_b200.distributed import alloc_accumulator, padded_rows, shard_views

    if local >= torch.cuda.device_count():
        sys.exit(f"bench.py: rank {rank} needs cuda:{local} but only "
                 f"{torch.cuda.device_count()} GPU(s) are visible (--gpus {args.gpus})")
    torch.cuda.set_device(local)
    group = None
    if world > 1 or "RANK" in os.environ:  # torchrun: NCCL path even for one rank
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD

    wl = load_workload(args.config, args.views, args.gaussians, args.iid)
    E, N = wl.num_objects, len(wl.scene)
    mine = shard_views(len(wl.views), rank, world)
    views = [wl.views[i] for i in mine]
    total_px = wl.view_pixels()

    ctx = _native.Context(local, streams=args.streams)
    ctx.set_scene(wl.scene)
    # inputs resident in HBM before the timed region: this rank's masks
    masks_dev = torch.from_numpy(np.ascontiguousarray(wl.masks[mine]).view(np.int16)).cuda()
    mask_ptrs = [masks_dev[i].data_ptr() for i in range(len(mine))]
    kind = _native.ACC_FIXED if args.acc == "fixed" else _native.ACC_F64
    acc = alloc_accumulator(N, E, world, kind, "cuda")
    A32 = torch.empty(E * N, dtype=torch.float32, device="cuda")
    mode = _native.MODE_BINARY if E == 2 else _native.MODE_SCENE
    rows = 1 if mode == _native.MODE_BINARY else E
    out = torch.empty(rows * N, dtype=torch.uint8, device="cuda")
    floors = (1.0 / 255.0, 1e-4)
    chunk = padded_rows(N, world) // world
    g0, g1 = rank * chunk, min(N, rank * chunk + chunk)
    part = torch.empty(acc.numel() // world, dtype=acc.dtype, device="cuda")
    A_sl = torch.zeros((E, chunk), dtype=torch.float32, device="cuda")
    L_sl = torch.zeros((rows, chunk), dtype=torch.uint8, device="cuda")
    A_all = torch.empty(world * E * chunk, dtype=torch.float32, device="cuda")
    L_all = torch.empty(world * rows * chunk, dtype=torch.uint8, device="cuda")
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def step(timing=False):
        acc.zero_()
        st = ctx.accumulate(views, mask_ptrs, E, floors[0], floors[1], acc.data_ptr(),
                            masks_on_device=True, acc_kind=kind)
        if group is None:
            ctx.finalize(acc.data_ptr(), N, E, out_ptr=A32.data_ptr(), acc_kind=kind)
            _native.assign(None, 0.0, mode, ctx=ctx, on_device_ptr=A32.data_ptr(), n=N, e=E,
                           out_ptr=out.data_ptr())
            return st
        # reduce-scatter by Gaussian slices -> cast + argmax of this rank's
        # slice -> all-gather of matrix and labels -> the API's E x N layout
        dist.reduce_scatter_tensor(part, acc, group=group)
        if g1 > g0:
            ctx.reduce_finalize([part.data_ptr()], g0, N, E, g0, g1, A_sl.data_ptr(), chunk,
                                out_on_device=True, acc_kind=kind)
        _native.assign(None, 0.0, mode, ctx=ctx, on_device_ptr=A_sl.data_ptr(), n=chunk, e=E,
                       out_ptr=L_sl.data_ptr())
        dist.all_gather_into_tensor(A_all, A_sl.reshape(-1), group=group)
        dist.all_gather_into_tensor(L_all, L_sl.reshape(-1), group=group)
        A32.view(E, N).copy_(A_all.view(world, E, chunk).permute(1, 0, 2)
                             .reshape(E, world * chunk)[:, :N])
        out.view(rows, N).copy_(L_all.view(world, rows, chunk).permute(1, 0, 2)
                                .reshape(rows, world * chunk)[:, :N])
        return st

    stats = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.warmup):
            step()
        ctx.set_timing(True)
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        clk.mark(True)
        t0.record()
        for _ in range(args.steps):
            stats.append(step())
        t1.record()
        torch.cuda.synchronize()
        clk.mark(False)
    ctx.set_timing(False)
    elapsed = t0.elapsed_time(t1) / 1e3
    if group is not None:
        e = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
        dist.all_reduce(e, op=dist.ReduceOp.MAX, group=group)
        elapsed = float(e.item())
        dist.barrier()
    s_per_step = elapsed / args.steps
    value = total_px / s_per_step

    # ---- end to end through the public API (host inputs, host outputs) ----
    e2e = None
    det = kind == _native.ACC_FIXED
    if not args.no_e2e:
        from paper_2409_08270_b200 import pin_inputs
        # inputs staged once in page-locked host memory (the serving setup);
        # every timed solve still copies them host -> device
        scene_h, pairs = pin_inputs(wl.scene, wl.pairs(), device=local)
        h2d = int(wl.masks[mine].nbytes + wl.scene.means.nbytes + wl.scene.rotations.nbytes
                  + wl.scene.scales.nbytes + wl.scene.opacities.nbytes)
        d2h = int(E * N * 4 + (N if E == 2 else E * N))
        reps = max(1, min(args.steps, 5))
        solve(scene_h, pairs, E, 0.0, "binary" if E == 2 else "scene",
              process_group=group, deterministic=det)  # warm
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        # each solve timed on its own (events around it); the line reports the
        # median solve next to the mean and every rep
        rep_s = []
        for _ in range(reps):
            ctx_cached = _native.context(local)
            ctx_cached._scene_key = None  # re-upload the scene every step
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            solve(scene_h, pairs, E, 0.0, "binary" if E == 2 else "scene", process_group=group,
                  deterministic=det)
            b.record()
            torch.cuda.synchronize()
            rep_s.append(a.elapsed_time(b) / 1e3)
        e_s = float(np.median(rep_s)) * reps
        # one more (warm) solve from the plain pageable numpy inputs, for reference
        pairs_pg = wl.pairs()
        solve(wl.scene, pairs_pg, E, 0.0, "binary" if E == 2 else "scene", process_group=group,
              deterministic=det)
        ctx_cached._scene_key = None
        torch.cuda.synchronize()
        c = torch.cuda.Event(enable_timing=True)
        c.record()
        solve(wl.scene, pairs_pg, E, 0.0, "binary" if E == 2 else "scene", process_group=group,
              deterministic=det)
        d = torch.cuda.Event(enable_timing=True)
        d.record()
        torch.cuda.synchronize()
        pageable_s = c.elapsed_time(d) / 1e3
        if group is not None:
            t = torch.tensor([e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            e_s = float(t.item())
        e2e = {"value": total_px / (e_s / reps), "unit": "view-px/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "s_per_scene": e_s / reps, "estimator": f"median of {reps} timed solves",
               "s_per_scene_mean": float(np.mean(rep_s)),
               "s_per_solve": [round(x, 6) for x in rep_s],
               "inputs": "page-locked host arrays (pin_inputs)",
               "s_per_scene_pageable_inputs": pageable_s}

    if rank != 0:
        if group is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (raster-accumulate) ----
    # The timed steps overlap views on several streams, so per-kernel event times
    # there include other streams' work.  The kernel's own duration is taken
    # from one more (untimed for `value`) pass on a 1-stream context with CUDA
    # events around every raster launch on its stream.
    ctx1 = _native.Context(local, streams=1)
    ctx1.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx1.set_scene(wl.scene)
    ctx1.set_timing(True)
    iso = None
    A_ts = A32.clone()  # the timed run's matrix and labels (all-gathered when sharded)
    L_ts = out.clone()
    for _ in range(2):
        acc.zero_()
        iso = ctx1.accumulate(views, mask_ptrs, E, floors[0], floors[1], acc.data_ptr(),
                              masks_on_device=True, acc_kind=kind)
    # ---- identity check: the whole scene re-solved on this GPU alone, on one
    # stream (a different schedule), against the timed run's matrix / labels ----
    check = None
    if not args.no_check:
        ctx1.set_timing(False)
        if world > 1:
            acc_c = alloc_accumulator(N, E, 1, kind, "cuda")
            ctx1.accumulate(wl.views, list(wl.masks), E, floors[0], floors[1], acc_c.data_ptr(),
                            acc_kind=kind)
        else:
            acc_c = acc  # the 1-stream pass above covered every view
        A_c = torch.empty(E * N, dtype=torch.float32, device="cuda")
        ctx1.finalize(acc_c.data_ptr(), N, E, out_ptr=A_c.data_ptr(), acc_kind=kind)
        L_c = torch.empty_like(out)
        _native.assign(None, 0.0, mode, ctx=ctx1, on_device_ptr=A_c.data_ptr(), n=N, e=E,
                       out_ptr=L_c.data_ptr())
        torch.cuda.synchronize()
        diff = (A_c - A_ts).abs()
        check = {"reference": "single-GPU 1-stream re-solve of all %d views" % len(wl.views),
                 "timed_run": f"{world} GPU(s), {args.streams} streams",
                 "accumulator": args.acc,
                 "matrix_bit_identical": bool(torch.equal(A_c.view(torch.int32),
                                                          A_ts.view(torch.int32))),
                 "entries_differing": int((A_c != A_ts).sum().item()),
                 "max_abs_diff": float(diff.max().item()) if diff.numel() else 0.0,
                 "label_flips": int((L_c != L_ts).sum().item())}
    ctx1.close()
    st = stats[-1]
    views_n = max(iso["views"], 1)
    raster_avg_s = iso["raster_ms"] / views_n / 1e3
    alg_bytes = (BYTES_PER_PIXEL * iso["view_pixels"] + BYTES_PER_TILE_STEP * iso["tile_steps"]
                 + BYTES_PER_ATOMIC[kind] * iso["atomics"]) / views_n
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / raster_avg_s / 1e9 if raster_avg_s > 0 else None
    traffic = None
    instr = None
    rec = {}
    tp = ROOT / "profiles" / "raster_traffic.json"
    if tp.exists():
        try:
            rec = json.loads(tp.read_text()).get(args.config, {})
            traffic = rec.get("dram_bytes_per_launch")
            instr = rec.get("warp_instructions_per_launch")
        except Exception:
            traffic = None
    atom_rate = iso["atomics"] / views_n / raster_avg_s if raster_avg_s > 0 else None
    atom_peak, atom_key, atom_sized = atomic_peak(E * N * BYTES_PER_ATOMIC[kind],
                                                  fixed=kind == _native.ACC_FIXED)
    clk_summary = clk.summary()
    sm_hz = (clk_summary.get("sm_mhz") or 1965.0) * 1e6
    issue_peak = 148 * 4 * sm_hz  # warp-instructions / s (one issue slot per scheduler per clock)
    # work-normalised compute roofline, measured this run: exact alpha evaluations
    # per second of raster time; the FP64 work per evaluation and the warp
    # instructions per evaluation are properties of this build (ncu, raster_traffic.json)
    evals_per_launch = iso["exact_evals"] / views_n
    eval_rate = evals_per_launch / raster_avg_s if raster_avg_s > 0 else None
    pk = pipe_peaks()
    compute = None
    if eval_rate and rec.get("fp64_thread_ops_per_exact_eval"):
        f64_peak = pk["dfma_per_sm_clk"] * 148 * sm_hz if pk else 64 * 148 * sm_hz
        f64_ach = eval_rate * rec["fp64_thread_ops_per_exact_eval"]
        inst_ach = eval_rate * rec["warp_instructions_per_exact_eval"]
        compute = {
            "exact_alpha_evals_per_launch": evals_per_launch,
            "exact_alpha_evals_per_s": eval_rate,
            "fp64": {"ops_per_exact_eval": rec["fp64_thread_ops_per_exact_eval"],
                     "achieved_ops_per_s": f64_ach, "peak_ops_per_s": f64_peak,
                     "frac": f64_ach / f64_peak,
                     "peak_source": "profiles/r2_pipe_peak.json (tools/pipe_peak.cu, DFMA "
                                    "thread-ops/SM/clk) x 148 SMs x this run's SM clock"},
            "issue": {"warp_instructions_per_exact_eval": rec["warp_instructions_per_exact_eval"],
                      "achieved_per_s": inst_ach, "peak_per_s": issue_peak,
                      "frac": inst_ach / issue_peak},
            "per_eval_constants_source": rec.get("source")}
    stage_sum = st["prep_ms"] + st["bin_ms"] + st["raster_ms"]
    line = {
        "metric": "view-pixels/sec of contribution accumulation",
        "value": value, "unit": "view-px/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": s_per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, wl),
        "run": {"parallelism": f"views sharded over {world} GPU(s)" + (
                    ", reduce-scatter + sliced cast/argmax + all-gather (NCCL)" if world > 1 else ""),
                "accumulator": "fixed-point (deterministic)" if kind == _native.ACC_FIXED
                else "float64 atomics",
                "streams": args.streams},
        "solve_s_per_scene": s_per_step,
        "e2e": e2e,
        "gpu_launches": int(sum(s["launches"] for s in stats) + 2 * args.steps),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": peak_kind, "kernel": "raster_kernel (K3)",
                     "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": raster_avg_s * 1e3,
                     "share_of_serial_step": iso["raster_ms"] / iso["gpu_ms"] if iso["gpu_ms"] else None,
                     "timing": "CUDA events around each raster launch on its stream, 1-stream pass",
                     "compute": compute,
                     "binding": {
                         "resource": "SM warp-instruction issue (not HBM: see DESIGN.md)",
                         "warp_instructions_per_launch": instr,
                         "achieved_winst_per_s": (instr / raster_avg_s) if instr else None,
                         "peak_winst_per_s": issue_peak,
                         "frac": (instr / raster_avg_s / issue_peak) if instr else None,
                         "instructions_source": "profiles/raster_traffic.json (ncu --set full)"},
                     "atomics": {
                         "per_launch": iso["atomics"] / views_n,
                         "achieved_per_s": atom_rate,
                         "peak_per_s": atom_peak,
                         "frac": (atom_rate / atom_peak) if (atom_rate and atom_peak) else None,
                         "peak_source": "profiles/r2_atomic_peak.json 16MB_C2 "
                                        + ("fixed_pair_rand16 (two uint64 REDs per add" if kind
                                           == _native.ACC_FIXED else "f64_rand16 (float64 RED")
                                        + ", 16 random lanes per warp instruction, L2-resident "
                                        "buffer; tools/atomic_peak.cu)",
                         "uniform_random_per_s_at_accumulator_size": atom_sized,
                         "accumulator_size_class": atom_key,
                         "l2_red_pct_of_peak_ncu": rec.get("l2_red_pct_of_peak")},
                     "warp_efficiency": {
                         "threads_per_inst": rec.get("warp_efficiency_threads_per_inst"),
                         "pred_on_threads_per_inst":
                             rec.get("warp_efficiency_pred_on_threads_per_inst"),
                         "source": "ncu smsp__thread_inst_executed[_pred_on]_per_inst_executed"}},
        "stages_ms_per_step": {"prep": st["prep_ms"], "bin": st["bin_ms"],
                               "raster": st["raster_ms"], "sum": stage_sum},
        "counters_per_step": {k: st[k] for k in ("emitted", "instances", "tile_steps",
                                                 "exact_evals", "atomics", "retried_views")},
        "clocks": clk_summary,
        "shard_check": check,
    }
    if world == 1 and not args.no_cpu:
        # ~10 s of wall time on the host: three views per core (one per core per step in
        # the --impl reference arm, which repeats it warmup + steps times)
        k = args.cpu_views or 3 * (os.cpu_count() or 1)
        line["cpu_baseline"] = {k2: v for k2, v in cpu_baseline(wl, k).items() if k2 != "seconds"}
        ref_np = ROOT / "profiles" / "r2_reference_numpy_c2.json"
        if args.config == "C2" and ref_np.exists():
            # the reference itself (numpy) cannot run on the GPU box (/root/reference is not
            # there): its C2 per-view rate, measured in the build container, for context
            r = json.loads(ref_np.read_text())
            line["cpu_baseline"]["reference_numpy_build_host"] = {
                "view_px_per_s_one_core": r["single_process_view_px_per_s"],
                "view_px_per_s_parallel": r["parallel_view_px_per_s"],
                "processes": r["processes"], "source": "profiles/r2_reference_numpy_c2.json",
                "note": "tools/time_reference_numpy.py, build container, not the GPU box"}
    print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
