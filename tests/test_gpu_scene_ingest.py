"""Device-side scene ingestion: ``load_scene_ply(path, device=0)``
uploads the checkpoint's float32 records and activates / validates them in the
scene-setup kernel (fs_set_scene_ply).

Pinned against ``tests/golden/scene_ply.npz``: two checkpoints (one with extra,
interleaved properties) and the arrays the REFERENCE loader produced from them
(ply.py:63-106, scene.py:96-100; tests/golden/make_golden.py ``ply``).  Means
and normalised quaternions must be bit-identical.  The activations use
float64 exp, which is not bit-reproducible across implementations: numpy's
own (its AVX-512 SIMD exp on these hosts) misses the correctly rounded value
in ~4% of inputs by 1 ulp, libm in ~0.1%.  So exp(scale) must agree within
1 ulp, and the logistic 1 / (1 + exp(-x)) -- whose add and divide can turn a
1-ulp exp difference into 2 -- within 2 ulps; downstream the matrix and
labels are compared against a solve on the reference arrays.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2409_08270_b200")
from paper_2409_08270_b200 import CameraView, GaussianScene, load_scene_ply, solve  # noqa: E402
from paper_2409_08270_b200 import _native  # noqa: E402
from paper_2409_08270_b200.scene import SceneDataError  # noqa: E402

PLY = load_golden("scene_ply")


def _ulps(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    assert np.array_equal(np.signbit(a), np.signbit(b))
    return np.abs(a.view(np.int64) - b.view(np.int64))


def _write(tmp_path, name, data):
    p = tmp_path / f"{name}.ply"
    p.write_bytes(bytes(data))
    return p


@pytest.mark.parametrize("case", sorted(PLY))
def test_device_activations_match_reference_loader(tmp_path, case):
    c = PLY[case]
    path = _write(tmp_path, case, c["ply"])
    sc = load_scene_ply(path, device=0)
    assert isinstance(sc, fs.scene_io.PlyScene) and len(sc) == len(c["means"])
    params = np.zeros((len(sc), 8))
    ctx = _native.context(0)
    with ctx.lock:
        bad = ctx.set_scene_ply(sc, params)
        ctx._scene_key = None
    assert (bad < 0).all()
    # normalised quaternions: same sequential norm and division as numpy -> bit-exact
    assert _ulps(params[:, 4:8], c["rotations"]).max() == 0
    # exp / logistic: the device's float64 exp against numpy's
    su = _ulps(params[:, 0:3], c["scales"])
    ou = _ulps(params[:, 3], c["opacities"])
    assert su.max() <= 1 and ou.max() <= 2, (su.max(), ou.max())
    assert np.mean(su == 0) > 0.9 and np.mean(ou == 0) > 0.9
    # the lazily built host arrays are the reference loader's, bit for bit
    for k, ref in (("means", "means"), ("rotations", "rotations"), ("scales", "scales"),
                   ("opacities", "opacities"), ("colors_dc", "colors")):
        assert np.array_equal(getattr(sc, k), c[ref]), k


def test_solve_from_device_loaded_scene_matches_host_loaded(tmp_path):
    c = PLY["interleaved"]
    path = _write(tmp_path, "s", c["ply"])
    host = GaussianScene(c["means"], c["rotations"], c["scales"], c["opacities"])
    dev = load_scene_ply(path, device=0)
    cams = [CameraView(view_id=i, width=160, height=120, fx=90.0, fy=90.0, cx=80.5 + 3 * i,
                       cy=60.5, world_to_camera=np.eye(4), near_clip=0.01) for i in range(3)]
    rng = np.random.default_rng(4)
    masks = [rng.integers(0, 3, (120, 160)).astype(np.uint16) for _ in cams]
    pairs = [(v, fs.LabelMask(v.view_id, m)) for v, m in zip(cams, masks)]
    A_dev, a_dev = solve(dev, pairs, 3, 0.0, "scene")
    A_host, a_host = solve(host, pairs, 3, 0.0, "scene")
    np.testing.assert_allclose(A_dev.values, A_host.values, rtol=1e-6, atol=1e-9)
    assert np.mean(A_dev.values == A_host.values) >= 0.999
    assert np.mean(a_dev.membership == a_host.membership) >= 0.999
    assert A_host.values.sum() > 0


def _patched(c, props, edits):
    """Checkpoint bytes with values overwritten: edits = [(vertex, property, value)]."""
    raw = bytes(c["ply"])
    head_end = raw.index(b"end_header\n") + len(b"end_header\n")
    names = [ln.split()[2] for ln in raw[:head_end].decode().splitlines()
             if ln.startswith("property")]
    rec = np.frombuffer(raw[head_end:], dtype=np.dtype([(p, "<f4") for p in names])).copy()
    for v, p, val in edits:
        rec[p][v] = val
    return raw[:head_end] + rec.tobytes()


@pytest.mark.parametrize("edits,message", [
    ([(40, "f_dc_1", np.nan), (7, "rot_0", 0.0), (7, "rot_1", 0.0), (7, "rot_2", 0.0),
      (7, "rot_3", 0.0)], "non-finite values at vertex 40"),
    ([(9, "nx", np.inf)], "non-finite values at vertex 9"),
    ([(30, "rot_0", 0.0), (30, "rot_1", 0.0), (30, "rot_2", 0.0), (30, "rot_3", 0.0),
      (12, "rot_0", 0.0), (12, "rot_1", 0.0), (12, "rot_2", 0.0), (12, "rot_3", 0.0)],
     "quaternion 12 has zero or non-finite norm"),
    ([(25, "scale_1", -800.0), (3, "scale_2", -900.0)], "gaussian 3 has non-positive scale"),
])
def test_device_load_errors_match_host_loader(tmp_path, edits, message):
    c = PLY["plain"]
    path = tmp_path / "bad.ply"
    path.write_bytes(_patched(c, None, edits))
    with pytest.raises(SceneDataError) as host_err:
        load_scene_ply(path)  # the reference-semantics host loader
    with pytest.raises(SceneDataError) as dev_err:
        load_scene_ply(path, device=0)
    assert message in str(host_err.value)
    assert str(dev_err.value) == str(host_err.value)
    # the failed upload leaves no scene resident: a good checkpoint loads afterwards
    good = _write(tmp_path, "good", c["ply"])
    assert len(load_scene_ply(good, device=0)) == len(c["means"])


def test_device_loaded_scene_on_several_contexts(tmp_path):
    """A PlyScene resident on one context reaches the others by fs_copy_scene
    (devices=[0, 0]): same matrix and labels as the single-context solve."""
    c = PLY["plain"]
    dev = load_scene_ply(_write(tmp_path, "m", c["ply"]), device=0)
    cams = [CameraView(view_id=i, width=128, height=96, fx=80.0, fy=80.0, cx=64.5, cy=48.5 - 2 * i,
                       world_to_camera=np.eye(4), near_clip=0.01) for i in range(4)]
    rng = np.random.default_rng(6)
    pairs = [(v, fs.LabelMask(v.view_id, rng.integers(0, 2, (96, 128)).astype(np.uint16)))
             for v in cams]
    M1, a1 = solve(dev, pairs, 2, 0.0, "binary")
    M2, a2 = solve(dev, pairs, 2, 0.0, "binary", devices=[0, 0])
    assert np.array_equal(M1.values, M2.values) and np.array_equal(a1.labels, a2.labels)
    assert M1.values.sum() > 0


@pytest.mark.parametrize("seed", range(80))
def test_device_loader_fuzz_matches_host_loader(tmp_path, seed):
    """The special-value checkpoints of tests/test_scene_io.py's fuzz (host loader
    == reference loader there): the device path raises the same error, or
    produces the same arrays (quaternions and means bit-exact, exp activations
    within the ulp bounds above; +-inf / 0 where exp overflows / underflows)."""
    from fuzz_cases import patch_ply, ply_edits

    c = PLY["plain" if seed % 2 else "interleaved"]
    _, names = patch_ply(c["ply"], [])
    data, _ = patch_ply(c["ply"], ply_edits(seed, len(c["means"]), names))
    path = _write(tmp_path, "f", data)
    try:
        host = load_scene_ply(path)
        host_err = None
    except SceneDataError as e:
        host, host_err = None, e
    if host_err is not None:
        with pytest.raises(SceneDataError) as dev_err:
            load_scene_ply(path, device=0)
        assert str(dev_err.value) == str(host_err)
        return
    sc = load_scene_ply(path, device=0)
    params = np.zeros((len(sc), 8))
    ctx = _native.context(0)
    with ctx.lock:
        bad = ctx.set_scene_ply(sc, params)
        ctx._scene_key = None
    assert (bad < 0).all()
    assert np.array_equal(params[:, 4:8], host.rotations)
    fin = np.isfinite(host.scales) & (host.scales > 0)
    assert np.array_equal(params[:, 0:3][~fin], host.scales[~fin])  # inf / 0 exactly
    assert _ulps(params[:, 0:3][fin], host.scales[fin]).max() <= 1
    assert _ulps(params[:, 3], host.opacities).max() <= 2
    assert np.array_equal(sc.means, host.means)
