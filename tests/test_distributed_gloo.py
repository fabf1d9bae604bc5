"""World-size-2 view sharding over gloo on the CPU: the sharded matrix equals
the unsharded one (A is additive over views).  The per-shard partial is the
CPU oracle here (test-only); on NCCL the product path runs the CUDA library."""

import os
import socket

import numpy as np
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
