"""World-size-2 view sharding over gloo on the CPU: the sharded matrix equals
the unsharded one (A is additive over views).  The per-shard partial is the
CPU oracle here (test-only); on NCCL the product path runs the CUDA library."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2409_08270_b200 import DEFAULT_BLEND
from paper_2409_08270_b200.distributed import accumulate_sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_partial(scene, views, num_objects, blend):
    cams = [oracle.camera_of(v) for v, _ in views]
    masks = [m.labels for _, m in views]
    return oracle.accumulate(scene.means, scene.rotations, scene.scales, scene.opacities, cams,
                             masks, num_objects, blend.alpha_floor, blend.transmittance_floor,
                             threads=2, as_float32=False)


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2409_08270_b200 import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = synth.make_workload(seed=13, n_gaussians=3000, n_views=5, width=64, height=48,
                             num_objects=3)
    A = accumulate_sharded(wl.scene, wl.pairs(), 3, DEFAULT_BLEND, dist.group.WORLD,
                           partial_fn=_oracle_partial)
    np.save(f"{out_path}.{rank}.npy", A)
    dist.destroy_process_group()


def test_two_rank_sharding_equals_single(tmp_path):
    from paper_2409_08270_b200 import synth
    port = _free_port()
    out = str(tmp_path / "A")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    a0, a1 = np.load(out + ".0.npy"), np.load(out + ".1.npy")
    assert np.array_equal(a0, a1)
    wl = synth.make_workload(seed=13, n_gaussians=3000, n_views=5, width=64, height=48,
                             num_objects=3)
    full = _oracle_partial(wl.scene, wl.pairs(), 3, DEFAULT_BLEND).astype(np.float32)
    np.testing.assert_allclose(a0, full, rtol=1e-6, atol=1e-9)


class _FakeCtx:
    """Stands in for the CUDA context: reports the device label check's outcome
    (first offending view of the shard) the way Context.accumulate does."""

    def __init__(self, bad_local):
        self.bad_local = bad_local

    def accumulate(self, views, masks, *args, **kw):
        from paper_2409_08270_b200._native import LabelRangeError
        if self.bad_local is not None:
            raise LabelRangeError("label out of range", self.bad_local)
        return {"views": len(views)}


def _agree_worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2409_08270_b200 import LabelMask, synth
    from paper_2409_08270_b200.distributed import accumulate_shard_checked, shard_views
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = synth.make_workload(seed=14, n_gaussians=100, n_views=6, width=32, height=24,
                             num_objects=2)
    pairs = wl.pairs()
    # bad labels in views 4 (rank 1's shard) and 1 (rank 0's shard): every rank must
    # raise the reference's error for view 1, the first in view order
    for v, lab in ((4, 7), (1, 5)):
        m = pairs[v][1].labels.copy()
        m[2, 3] = lab
        pairs[v] = (pairs[v][0], LabelMask(pairs[v][0].view_id, m))
    mine = shard_views(len(pairs), rank, world)
    local_bad = next((i for i, g in enumerate(mine) if g in (1, 4)), None)
    try:
        accumulate_shard_checked(_FakeCtx(local_bad), pairs, mine, 2, DEFAULT_BLEND, 0,
                                 dist.group.WORLD, 0)
        msg = "no error"
    except ValueError as exc:
        msg = str(exc)
    with open(f"{out_path}.{rank}.txt", "w") as fh:
        fh.write(msg)
    dist.destroy_process_group()


def test_two_rank_label_error_agreement(tmp_path):
    port = _free_port()
    out = str(tmp_path / "err")
    mp.spawn(_agree_worker, args=(2, port, out), nprocs=2, join=True)
    msgs = [open(f"{out}.{r}.txt").read() for r in (0, 1)]
    assert msgs[0] == msgs[1]
    assert "view 1: label 5 at pixel (2, 3) exceeds object count 2" in msgs[0]


class _HostFinalizeCtx:
    """CPU stand-in for the library's fs_reduce_finalize (fixed-point parts ->
    float32 slice), so the reduce-scatter / all-gather reassembly of
    distributed.reduce_scatter_finalize runs on gloo."""

    def __init__(self):
        import threading
        self.lock = threading.Lock()

    def set_stream(self, handle):
        pass

    def reduce_finalize(self, parts, part_g0, n, e, g0, g1, out_ptr, ld, out_on_device=True,
                        acc_kind=1):
        import ctypes
        rows = g1 - part_g0
        words = np.ctypeslib.as_array((ctypes.c_uint64 * (rows * e * 2)).from_address(parts[0]))
        w = words.reshape(rows, e, 2)[g0 - part_g0:]
        val = ((w[..., 0].astype(object) << 32) + w[..., 1].astype(object))
        f = np.array([[float(x) * 2.0 ** -59 for x in r] for r in val], np.float64)
        out = np.ctypeslib.as_array((ctypes.c_float * (e * ld)).from_address(out_ptr)).reshape(e, ld)
        out[:, :g1 - g0] = f.T.astype(np.float32)


def _rs_worker(rank, world, port, out_path, n, e):
    import torch
    import torch.distributed as dist

    from paper_2409_08270_b200 import _native
    from paper_2409_08270_b200.distributed import alloc_accumulator, reduce_scatter_finalize
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    acc = alloc_accumulator(n, e, world, _native.ACC_FIXED, "cpu")
    rng = np.random.default_rng(100 + rank)
    words = acc.view(-1, e, 2)
    words[:n] = torch.from_numpy(rng.integers(0, 2 ** 40, (n, e, 2), dtype=np.int64))
    A = reduce_scatter_finalize(_HostFinalizeCtx(), acc, n, e, _native.ACC_FIXED,
                                dist.group.WORLD, None)
    np.save(f"{out_path}.{rank}.npy", A.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 7), (3, 10), (2, 1)])
def test_reduce_scatter_finalize_reassembles_the_matrix(tmp_path, world, n):
    """Padding to equal Gaussian slices, reduce-scatter of the fixed-point words,
    per-slice cast and all-gather give every rank the E x N matrix of the summed
    accumulators (distributed.py; the NCCL path runs the same code on GPUs)."""
    e = 3
    port = _free_port()
    out = str(tmp_path / "A")
    mp.spawn(_rs_worker, args=(world, port, out, n, e), nprocs=world, join=True)
    total = np.zeros((n, e, 2), dtype=object)
    for r in range(world):
        total += np.random.default_rng(100 + r).integers(0, 2 ** 40, (n, e, 2),
                                                         dtype=np.int64).astype(object)
    val = (total[..., 0] << 32) + total[..., 1]
    expect = np.array([[float(x) * 2.0 ** -59 for x in row] for row in val]).T.astype(np.float32)
    for r in range(world):
        got = np.load(f"{out}.{r}.npy")
        assert got.shape == (e, n)
        assert np.array_equal(got, expect)
