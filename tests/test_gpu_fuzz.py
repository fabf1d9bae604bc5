"""Randomised adversarial parity (tests/fuzz_cases.py builds the cases: near-plane
and behind-camera Gaussians, exact duplicates, sub-pixel to whole-image
footprints, opacities at 0 / 1 / the alpha floor, 1-400 px rotated cameras,
E 2-40, seven blend-floor settings, random gamma), each checked against the
pinned oracle through the public API and the C ABI: projection (bit-identical,
same op order), tile lists (identical), the accumulated matrix with both
accumulators (within rtol 1e-6 of the oracle's float64 walk, almost every
float32 entry bit-identical), both assignments (bit-exact against the oracle's
argmax of the same matrix); every other case also renders alpha, depth, a
3-channel property and the scene mask.  tests/golden/fuzz.npz holds the
REFERENCE's own outputs for a subset of the same cases (make_golden.py fuzz).
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2409_08270_b200")
from paper_2409_08270_b200 import (  # noqa: E402
    Assignment,
    BlendConfig,
    ContributionMatrix,
    GaussianScene,
    LabelMask,
    accumulate_contributions,
    assign_binary,
    assign_scene,
    render_scene_mask,
    render_view,
)
from paper_2409_08270_b200 import _native  # noqa: E402

from conftest import cam_from_row, load_golden  # noqa: E402
from fuzz_cases import (  # noqa: E402
    N_CASES, ambiguous_mask_pixels, case_arrays, digest, label_band, render_extras)

REF = load_golden("fuzz")  # the reference's outputs for the cases small enough for it
REF_SEEDS = sorted(int(k[1:]) for k in REF)


def _case(seed):
    c = case_arrays(seed)
    scene = GaussianScene(c["means"], c["quats"], c["scales"], c["opac"])
    pairs = [(cam_from_row(r, i), LabelMask(i, m)) for i, (r, m) in enumerate(zip(c["cams"], c["masks"]))]
    return scene, pairs, c["E"], BlendConfig(*c["floors"]), c["gamma"]


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_case_matches_oracle(seed):
    scene, pairs, E, blend, gamma = _case(seed)
    ctx = _native.context(0)
    for cam, _ in pairs:
        with ctx.lock:
            ctx.set_scene(scene)
            g = ctx.project(cam)
            offs, items = ctx.bin(cam)
        o = oracle.project(scene.means, scene.rotations, scene.scales, oracle.camera_of(cam))
        assert np.array_equal(g[0], o[0])
        for k in (1, 2, 3, 4):
            assert np.array_equal(g[k][g[0]], o[k][o[0]]), k
        assert list(g[5]) == list(o[5])
        o_offs, o_items = oracle.bin_tiles(o[0], o[1], o[3], o[4], cam.width, cam.height)
        assert np.array_equal(offs, o_offs) and np.array_equal(items, o_items)

    ref = oracle.accumulate(scene.means, scene.rotations, scene.scales, scene.opacities,
                            [oracle.camera_of(c) for c, _ in pairs], [m.labels for _, m in pairs],
                            E, blend.alpha_floor, blend.transmittance_floor, threads=4,
                            as_float32=False)
    for det in (True, False):
        A = accumulate_contributions(scene, pairs, E, blend, deterministic=det).values
        assert A.dtype == np.float32 and A.shape == (E, len(scene))
        np.testing.assert_allclose(A, ref, rtol=1e-6, atol=1e-9)
        differ = int(np.count_nonzero(A != ref.astype(np.float32)))
        assert differ <= max(2, A.size // 1000), f"{differ} of {A.size} entries differ"
    M = ContributionMatrix(A)
    assert np.array_equal(assign_scene(M, gamma).membership, oracle.assign_scene(A, gamma))
    if E == 2:
        assert np.array_equal(assign_binary(M, gamma).labels, oracle.assign_binary(A, gamma))


@pytest.mark.parametrize("seed", range(0, N_CASES, 2))
def test_fuzz_render_matches_oracle(seed):
    """render_view (alpha, depth, a 3-channel property) and render_scene_mask on
    the same adversarial cases, against the oracle's compositing."""
    scene, pairs, E, blend, gamma = _case(seed)
    ch, memb, tau = render_extras(seed, len(scene), E)
    for cam, _ in pairs:
        out = render_view(scene, cam, ch, blend)
        o = oracle.camera_of(cam)
        value, alpha, depth = oracle.render_view(scene.means, scene.rotations, scene.scales,
                                                 scene.opacities, o, ch, None, blend.alpha_floor,
                                                 blend.transmittance_floor)
        np.testing.assert_allclose(out.alpha, alpha, rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(out.depth, depth, rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(out.value, value, rtol=1e-10, atol=1e-14)
        got = render_scene_mask(scene, Assignment(mode="scene", gamma=0.0, membership=memb), cam,
                                tau, blend).labels
        ref = oracle.render_mask(scene.means, scene.rotations, scene.scales, scene.opacities, o,
                                 memb, tau, blend.alpha_floor, blend.transmittance_floor)
        differ = got != ref
        if differ.any():
            # only where the reference's own decision is ill-conditioned: float64
            # exp / BLAS rounding (~1e-16) decides an alpha-vs-tau test or an exact
            # depth tie (duplicated Gaussians in different objects)
            amb = ambiguous_mask_pixels(oracle, scene.means, scene.rotations, scene.scales,
                                        scene.opacities, o, memb, tau,
                                        (blend.alpha_floor, blend.transmittance_floor))
            assert not (differ & ~amb).any(), f"{int((differ & ~amb).sum())} clear pixels differ"
            assert differ.sum() <= max(4, differ.size // 500)


@pytest.mark.parametrize("seed", REF_SEEDS)
def test_fuzz_case_matches_reference_golden(seed):
    """The device path against the REFERENCE's own outputs (tests/golden/fuzz.npz)
    on the same case: the float32 matrix, the labels (flips only inside the
    north-star decision band), and the first view's render + scene mask."""
    ref = REF[f"s{seed}"]
    c = case_arrays(seed)
    assert digest(c) == bytes(ref["digest"]).decode(), "fuzz generator drifted"
    scene, pairs, E, blend, gamma = _case(seed)
    A = accumulate_contributions(scene, pairs, E, blend).values
    np.testing.assert_allclose(A, ref["A"], rtol=1e-6, atol=1e-9)
    differ = int(np.count_nonzero(A != ref["A"]))
    assert differ <= max(2, A.size // 1000), f"{differ} of {A.size} entries differ"
    M = ContributionMatrix(A)
    memb = assign_scene(M, gamma).membership
    flips = (memb != ref["membership"]).any(axis=0)
    assert not (flips & ~label_band(oracle, ref["A"], gamma, True)).any()
    if "labels" in ref:
        lab = assign_binary(M, gamma).labels
        assert not ((lab != ref["labels"]) & ~label_band(oracle, ref["A"], gamma, False)).any()
    if "r_alpha" in ref:
        ch, rmemb, tau = render_extras(seed, len(scene), E)
        cam = pairs[0][0]
        out = render_view(scene, cam, ch, blend)
        # float64 exp (CUDA vs numpy's SIMD exp) and BLAS rounding: ~1e-15 relative
        np.testing.assert_allclose(out.alpha, ref["r_alpha"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(out.depth, ref["r_depth"], rtol=1e-10, atol=1e-14)
        got = render_scene_mask(scene, Assignment(mode="scene", gamma=0.0, membership=rmemb), cam,
                                tau, blend).labels
        differ = got != ref["r_mask"]
        if differ.any():
            amb = ambiguous_mask_pixels(oracle, scene.means, scene.rotations, scene.scales,
                                        scene.opacities, oracle.camera_of(cam), rmemb, tau,
                                        (blend.alpha_floor, blend.transmittance_floor))
            assert not (differ & ~amb).any()


@pytest.mark.parametrize("seed", range(0, N_CASES, 4))
def test_fuzz_multi_context_matches_single(seed):
    """The single-process multi-GPU path (three contexts on one GPU: dynamic view
    queue, peer-memory reduce fused into the cast and argmax) on the adversarial
    cases: with the fixed-point accumulator, bit-identical to the one-context
    solve; with float64 atomics, within the summation-order tolerance."""
    from paper_2409_08270_b200 import solve

    scene, pairs, E, blend, gamma = _case(seed)
    A1, m1 = solve(scene, pairs, E, gamma, "scene", blend)
    A3, m3 = solve(scene, pairs, E, gamma, "scene", blend, devices=[0, 0, 0])
    if blend.alpha_floor * blend.transmittance_floor >= 2.0 ** -26:  # fixed-point accumulator
        assert A3.values.tobytes() == A1.values.tobytes()
        assert np.array_equal(m3.membership, m1.membership)
    else:
        np.testing.assert_allclose(A3.values, A1.values, rtol=1e-6, atol=1e-9)
        assert np.array_equal(m3.membership, oracle.assign_scene(A3.values, gamma))
