"""Pin the oracle's novel-view rendering to the reference (rasterizer.py:133-234,
maskrender.py:45-95) through tests/golden/render.npz (make_golden.py render)."""

import numpy as np
import pytest

import oracle
from conftest import cam_from_row, load_golden

REN = load_golden("render")
RENDER_CASES = sorted(k for k in REN if "labels" not in REN[k])
MASK_CASES = sorted(k for k in REN if "labels" in REN[k])


def scene_of(c):
    return c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"]


@pytest.mark.parametrize("case", RENDER_CASES)
def test_oracle_render_matches_reference(case):
    c = REN[case]
    af, tf = c["floors"]
    cam = oracle.camera_of(cam_from_row(c["cam"]))
    value, alpha, depth = oracle.render_view(*scene_of(c), cam, c.get("channel"),
                                             c.get("member"), af, tf)
    # per-pixel sums run in the reference's order; only libm exp vs numpy exp differ
    np.testing.assert_allclose(alpha, c["alpha"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(depth, c["depth"], rtol=1e-12, atol=1e-15)
    if "value" in c:
        np.testing.assert_allclose(value, c["value"], rtol=1e-12, atol=1e-15)
    else:
        assert value is None


@pytest.mark.parametrize("case", MASK_CASES)
def test_oracle_masks_match_reference(case):
    c = REN[case]
    cam = oracle.camera_of(cam_from_row(c["cam"]))
    asn = c["assignment"]
    if bytes(c["mode"]).decode() == "binary":
        fg = asn.astype(bool)
        asn = np.stack([~fg, fg])
    labels = oracle.render_mask(*scene_of(c), cam, asn, float(c["tau"]))
    assert np.array_equal(labels, c["labels"])


def test_render_known_answers():
    c = REN["single"]
    assert c["alpha"][8, 8] == pytest.approx(0.6, abs=1e-12)
    assert c["value"][8, 8] == pytest.approx(0.6, abs=1e-12)
    assert c["depth"][8, 8] == pytest.approx(2.0, abs=1e-12)
    c = REN["two"]
    assert c["alpha"][8, 8] == pytest.approx(0.75, abs=1e-12)
    assert c["value"][8, 8] == pytest.approx(0.5, abs=1e-12)
    assert REN["subset_local"]["alpha"][8, 8] == pytest.approx(0.7, abs=1e-12)
    assert not REN["subset_empty"]["alpha"].any()
    assert REN["scene_tie"]["labels"][8, 8] == 1


def test_oracle_render_at_benchmark_resolution():
    """render_view (sampled pixels + whole-image sums) and render_scene_mask (all pixels)
    of the reference at 1008 x 756, 100 k Gaussians (golden accumulate_fullres)."""
    from paper_2409_08270_b200 import synth
    G = load_golden("accumulate_fullres")
    c = G["c2res_coherent"]
    wl = synth.make_workload(**dict(eval(bytes(c["gen_args"]).decode())))
    assert wl.digest() == bytes(c["digest"]).decode()
    sc = (wl.scene.means, wl.scene.rotations, wl.scene.scales, wl.scene.opacities)
    r = G["c2res_coherent_render"]
    ch = np.random.default_rng(5).random(len(wl.scene))
    value, alpha, depth = oracle.render_view(*sc, oracle.camera_of(wl.views[0]), ch)
    for got, key in ((alpha, "alpha"), (depth, "depth"), (value, "value")):
        np.testing.assert_allclose(got.ravel()[r["idx"]], r[key], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose([alpha.sum(), depth.sum(), value.sum()], r["sums"], rtol=1e-12)
    m = G["c2res_coherent_mask"]
    labels = oracle.render_mask(*sc, oracle.camera_of(wl.views[1]), c["labels_g0"],
                                float(m["tau"]))
    assert np.array_equal(labels, m["labels"])
