"""The NCCL product path of view sharding on the one GPU of the test box: a
single-rank process group exercises accumulate_shard_checked (device label
check + MIN agreement), the SUM all-reduce and solve(process_group=...)
exactly as every rank runs them under torchrun.  Multi-rank host logic is
covered by tests/test_distributed_gloo.py."""

import socket

import numpy as np
import pytest

from conftest import cam_from_row, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

from paper_2409_08270_b200 import (  # noqa: E402
    GaussianScene,
    LabelMask,
    accumulate_contributions,
    solve,
)

ACC = load_golden("accumulate")


@pytest.fixture(scope="module")
def group():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def case_inputs(name):
    c = ACC[name]
    scene = GaussianScene(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"])
    views = [(cam_from_row(r, i), LabelMask(i, m)) for i, (r, m) in
             enumerate(zip(c["cams"], c["masks"]))]
    return c, scene, views


def test_sharded_accumulate_matches_reference(group):
    c, scene, views = case_inputs("C1_default")
    m = accumulate_contributions(scene, views, int(c["E"]), process_group=group)
    np.testing.assert_allclose(m.values, c["A"], rtol=1e-6, atol=1e-9)
    A, asn = solve(scene, views, int(c["E"]), 0.0, "binary", process_group=group)
    assert np.array_equal(A.values, m.values)
    assert asn.labels.shape == (len(scene),)


def test_sharded_label_error_is_the_reference_error(group):
    c, scene, views = case_inputs("C1_default")
    bad = [(v, LabelMask(m.view_id, m.labels.copy())) for v, m in views]
    bad[3][1].labels[5, 7] = 9
    bad[5][1].labels[0, 0] = 4
    with pytest.raises(ValueError, match=r"view 3: label 9 at pixel \(5, 7\) exceeds object count 2"):
        accumulate_contributions(scene, bad, 2, process_group=group)
    with pytest.raises(ValueError, match=r"view 3: label 9 at pixel \(5, 7\)"):
        solve(scene, bad, 2, 0.0, "binary", process_group=group)
    # a shape error after a label error: the label error (earlier view) wins
    shp = list(bad)
    shp[4] = (shp[4][0], LabelMask(4, np.zeros((3, 3), np.uint16)))
    with pytest.raises(ValueError, match="view 3: label 9"):
        accumulate_contributions(scene, shp, 2, process_group=group)


def test_sharded_scene_solve_and_resident_matrix(group):
    """The reduce-scatter + sliced cast + all-gather path with E > 2: the matrix,
    scene membership and re-assignment on the gathered device matrix (LabelSolver)
    equal the single-GPU results bit for bit (fixed-point accumulator)."""
    from paper_2409_08270_b200 import LabelSolver, synth
    wl = synth.make_workload(seed=41, n_gaussians=30001, n_views=5, width=200, height=150,
                             num_objects=5)
    M1, a1 = solve(wl.scene, wl.pairs(), 5, 0.2, "scene")
    M2, a2 = solve(wl.scene, wl.pairs(), 5, 0.2, "scene", process_group=group)
    assert np.array_equal(M1.values, M2.values)
    assert np.array_equal(a1.membership, a2.membership)
    s = LabelSolver(wl.scene)
    s.accumulate(wl.pairs(), 5, process_group=group)
    for g in (-0.3, 0.0, 0.6):
        ref = solve(wl.scene, wl.pairs(), 5, g, "scene")[1].membership
        got = s.assign(g, "scene")
        assert np.array_equal(got.membership, ref)
        assert got.member_counts() == ref.sum(axis=1, dtype=np.int64).tolist()
