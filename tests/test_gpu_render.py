"""GPU parity of novel-view rendering: render_property /
render_view / render_subset_alpha_depth (reference rasterizer.py:133-234) and
render_binary_mask / render_scene_mask (maskrender.py:45-95) through the C
ABI (fs_render, fs_render_splats, fs_render_mask) against the reference's
golden vectors (tests/golden/render.npz) and the pinned oracle."""

import numpy as np
import pytest

import oracle
from conftest import cam_from_row, load_golden

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2409_08270_b200")
from paper_2409_08270_b200 import (  # noqa: E402
    DEFAULT_BLEND,
    EXACT_BLEND,
    Assignment,
    BlendConfig,
    GaussianScene,
    bin_gaussians_to_tiles,
    project_scene,
    render_binary_mask,
    render_property,
    render_scene_mask,
    render_subset_alpha_depth,
    render_view,
)
from paper_2409_08270_b200 import synth  # noqa: E402

REN = load_golden("render")
RENDER_CASES = sorted(k for k in REN if "labels" not in REN[k])
MASK_CASES = sorted(k for k in REN if "labels" in REN[k])
# per-pixel float64 sums in the reference's order; CUDA exp vs numpy exp differ
# by an ulp at most, so the outputs agree to ~1e-15 relative
RTOL, ATOL = 1e-11, 1e-15


def scene_of(c):
    return GaussianScene(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"])


def blend_of(c):
    return BlendConfig(float(c["floors"][0]), float(c["floors"][1]))


@pytest.mark.parametrize("case", RENDER_CASES)
def test_render_matches_reference(case):
    c = REN[case]
    scene, view, blend = scene_of(c), cam_from_row(c["cam"]), blend_of(c)
    if "member" in c:
        out = render_subset_alpha_depth(scene, view, c["member"].astype(bool), blend)
        assert out.value is None
    else:
        out = render_view(scene, view, c.get("channel"), blend)
    np.testing.assert_allclose(out.alpha, c["alpha"], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(out.depth, c["depth"], rtol=RTOL, atol=ATOL)
    if "value" in c:
        assert out.value.shape == c["value"].shape
        np.testing.assert_allclose(out.value, c["value"], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_render_property_over_a_binning_equals_render_view(case):
    """render_property over bin_gaussians_to_tiles(project_scene(...)) -- the
    caller's binning through fs_render_splats -- is bit-identical to the fused
    render_view / subset path (same walk, same order)."""
    c = REN[case]
    scene, view, blend = scene_of(c), cam_from_row(c["cam"]), blend_of(c)
    member = c["member"].astype(bool) if "member" in c else None
    splats, _ = project_scene(scene, view, member_mask=member)
    binning = bin_gaussians_to_tiles(splats, view)
    ch = None if member is not None else c.get("channel")
    a = render_property(scene, binning, view, ch, blend)
    if member is not None:
        b = render_subset_alpha_depth(scene, view, member, blend)
    else:
        b = render_view(scene, view, ch, blend)
    assert np.array_equal(a.alpha, b.alpha)
    assert np.array_equal(a.depth, b.depth)
    if ch is not None:
        assert np.array_equal(a.value, b.value)


@pytest.mark.parametrize("case", MASK_CASES)
def test_masks_match_reference(case):
    c = REN[case]
    scene, view = scene_of(c), cam_from_row(c["cam"])
    if bytes(c["mode"]).decode() == "binary":
        asn = Assignment(mode="binary", gamma=0.0, labels=c["assignment"])
        out = render_binary_mask(scene, asn, view, float(c["tau"]))
    else:
        asn = Assignment(mode="scene", gamma=0.0, membership=c["assignment"])
        out = render_scene_mask(scene, asn, view, float(c["tau"]))
    assert out.labels.dtype == np.uint16
    assert np.array_equal(out.labels, c["labels"])


@pytest.mark.parametrize("blend", [DEFAULT_BLEND, EXACT_BLEND], ids=["default", "exact"])
def test_render_medium_scene_matches_oracle(blend):
    """A denser synthetic view (C2 geometry at 20 k Gaussians, ragged edge
    tiles) against the C oracle, scalar and vector channels."""
    wl = synth.make_workload(seed=21, n_gaussians=20_000, n_views=1, width=250, height=190,
                             num_objects=2)
    view = wl.views[0]
    rng = np.random.default_rng(5)
    ch = rng.random((len(wl.scene), 3))
    out = render_view(wl.scene, view, ch, blend)
    cam = oracle.camera_of(view)
    value, alpha, depth = oracle.render_view(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                                             wl.scene.opacities, cam, ch, None,
                                             blend.alpha_floor, blend.transmittance_floor)
    assert alpha.max() > 0.5
    np.testing.assert_allclose(out.alpha, alpha, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out.depth, depth, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out.value, value, rtol=1e-10, atol=1e-14)
    # scene-mask path against the oracle on the same view
    memb = np.zeros((3, len(wl.scene)), np.uint8)
    obj = rng.integers(0, 3, size=len(wl.scene))
    memb[obj, np.arange(len(wl.scene))] = 1
    asn = Assignment(mode="scene", gamma=0.0, membership=memb)
    got = render_scene_mask(wl.scene, asn, view, 0.3, blend).labels
    ref = oracle.render_mask(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                             wl.scene.opacities, cam, memb, 0.3, blend.alpha_floor,
                             blend.transmittance_floor)
    assert np.array_equal(got, ref)


def test_render_properties():
    """Reference test_rasterizer.py:127-165 properties on the device."""
    c = REN["rand_exact"]
    scene, view = scene_of(c), cam_from_row(c["cam"])
    rng = np.random.default_rng(1)
    ch = rng.random((len(scene), 3))
    out = render_view(scene, view, ch, EXACT_BLEND)
    assert out.value.shape == (view.height, view.width, 3)
    for axis in range(3):
        single = render_view(scene, view, ch[:, axis], EXACT_BLEND)
        assert np.array_equal(out.value[:, :, axis], single.value)
    x, y = rng.random(len(scene)), rng.random(len(scene))
    comb = render_view(scene, view, 2.75 * x + y)
    px, py = render_view(scene, view, x), render_view(scene, view, y)
    assert np.abs(comb.value - (2.75 * px.value + py.value)).max() < 1e-12
    assert out.alpha.min() >= 0.0 and out.alpha.max() <= 1.0 + 1e-12
    again = render_view(scene, view, ch, EXACT_BLEND)
    assert np.array_equal(again.value, out.value) and np.array_equal(again.alpha, out.alpha)
    empty = render_subset_alpha_depth(scene, view, np.zeros(len(scene), bool))
    assert not empty.alpha.any() and not empty.depth.any()
    full = render_subset_alpha_depth(scene, view, np.ones(len(scene), bool))
    ref = render_view(scene, view, None)
    assert np.array_equal(full.alpha, ref.alpha) and np.array_equal(full.depth, ref.depth)


def test_render_validation_messages():
    c = REN["rand_default"]
    scene, view = scene_of(c), cam_from_row(c["cam"])
    with pytest.raises(ValueError, match="channel length"):
        render_view(scene, view, np.ones(len(scene) + 1))
    asn_b = Assignment(mode="binary", gamma=0.0, labels=np.ones(len(scene), np.uint8))
    for bad in (0.0, 1.0, -0.2, 7.0):
        with pytest.raises(ValueError, match="tau"):
            render_binary_mask(scene, asn_b, view, tau=bad)
    asn_s = Assignment(mode="scene", gamma=0.0, membership=np.zeros((2, len(scene)), np.uint8))
    with pytest.raises(ValueError, match="binary"):
        render_binary_mask(scene, asn_s, view)
    with pytest.raises(ValueError, match="scene"):
        render_scene_mask(scene, asn_b, view)
    assert not render_scene_mask(scene, asn_s, view).labels.any()


def test_tau_monotone_and_single_object_equals_binary():
    c = REN["rand_default"]
    scene, view = scene_of(c), cam_from_row(c["cam"])
    member = np.random.default_rng(2).random(len(scene)) < 0.5
    asn = Assignment(mode="binary", gamma=0.0, labels=member.astype(np.uint8))
    prev = None
    for tau in (0.05, 0.1, 0.3, 0.6, 0.9):
        lab = render_binary_mask(scene, asn, view, tau).labels > 0
        if prev is not None:
            assert not np.any(lab & ~prev)
        prev = lab
    sc = Assignment(mode="scene", gamma=0.0,
                    membership=np.stack([~member, member]).astype(np.uint8))
    assert np.array_equal(render_scene_mask(scene, sc, view).labels,
                          render_binary_mask(scene, asn, view).labels)


def test_render_at_benchmark_resolution_matches_reference():
    """GPU render_view / render_scene_mask against the reference at 1008 x 756 (100 k
    Gaussians of the C2 recipe; golden accumulate_fullres)."""
    G = load_golden("accumulate_fullres")
    c = G["c2res_coherent"]
    wl = synth.make_workload(**dict(eval(bytes(c["gen_args"]).decode())))
    assert wl.digest() == bytes(c["digest"]).decode()
    r = G["c2res_coherent_render"]
    ch = np.random.default_rng(5).random(len(wl.scene))
    out = render_view(wl.scene, wl.views[0], ch)
    for got, key in ((out.alpha, "alpha"), (out.depth, "depth"), (out.value, "value")):
        np.testing.assert_allclose(np.asarray(got).ravel()[r["idx"]], r[key], rtol=1e-11,
                                   atol=1e-14)
    np.testing.assert_allclose([out.alpha.sum(), out.depth.sum(), out.value.sum()], r["sums"],
                               rtol=1e-11)
    m = G["c2res_coherent_mask"]
    asn = Assignment(mode="scene", gamma=0.0, membership=c["labels_g0"])
    got = render_scene_mask(wl.scene, asn, wl.views[1], float(m["tau"]))
    assert np.array_equal(got.labels, m["labels"])
