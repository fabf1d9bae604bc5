"""Pin the CPU oracle to golden vectors produced by the reference itself.

tests/golden/*.npz were written by tests/golden/make_golden.py, which runs the
reference package (splatlift) on seeded inputs.  If these pass, the oracle
(oracle/fs_oracle.c + oracle/__init__.py) restates the reference's algorithm
and can stand in for it at sizes the reference cannot reach.
"""

import numpy as np
import pytest

import oracle
from conftest import cam_from_row, load_golden

PROJ = load_golden("projection")
BIN = load_golden("binning")
ACC = load_golden("accumulate")
ASG = load_golden("assign")


def orc_cam(row):
    return oracle.camera_of(cam_from_row(row))


@pytest.mark.parametrize("case", sorted(PROJ))
def test_projection_matches_reference(case):
    c = PROJ[case]
    alive, mean2d, conic, depth, radius, stats = oracle.project(
        c["in_means"], c["in_quats"], c["in_scales"], orc_cam(c["cam"]))
    assert np.array_equal(alive, c["alive"])
    assert np.array_equal(stats, c["stats"])
    a = c["alive"]
    assert np.array_equal(radius[a], c["radius"][a])
    np.testing.assert_allclose(mean2d[a], c["mean2d"][a], rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(conic[a], c["conic"][a], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(depth, c["depth"], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("case", sorted(k for k in BIN if k != "tile_range"))
def test_binning_matches_reference(case):
    c = BIN[case]
    cam = orc_cam(c["cam"])
    alive, mean2d, _, depth, radius, _ = oracle.project(
        c["in_means"], c["in_quats"], c["in_scales"], cam)
    offs, items = oracle.bin_tiles(alive, mean2d, depth, radius, cam.width, cam.height)
    assert np.array_equal(offs, c["offsets"])
    assert np.array_equal(items, c["items"])


def _inputs(c, case):
    if "in_means" in c:
        return c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"]
    src = ACC["C1_default"]
    return src["in_means"], src["in_quats"], src["in_scales"], src["in_opac"]


@pytest.mark.parametrize("case", sorted(k for k in ACC if not k.startswith("synth")))
def test_accumulate_matches_reference(case):
    c = ACC[case]
    means, quats, scales, opac = _inputs(c, case)
    cams_rows = c["cams"] if "cams" in c else ACC["C1_default"]["cams"]
    masks = c["masks"] if "masks" in c else ACC["C1_default"]["masks"]
    if case == "C1_exact_2views":
        cams_rows, masks = cams_rows[:2], masks[:2]
    cams = [orc_cam(r) for r in cams_rows]
    af, tf = c["floors"]
    total = oracle.accumulate(means, quats, scales, opac, cams, list(masks), int(c["E"]),
                              af, tf, threads=4, as_float32=False)
    ref64 = c["A64"]
    # float64 restatement: agreement to a few ulps of the largest entry
    np.testing.assert_allclose(total, ref64, rtol=1e-10, atol=1e-12)
    f32 = total.astype(np.float32)
    mism = int(np.count_nonzero(f32 != c["A"]))
    assert mism <= max(2, f32.size // 10000), mism


def test_accumulate_synthetic_workloads_match_reference():
    from paper_2409_08270_b200 import synth
    for name in ("synth_coherent", "synth_iid", "synth_dense"):
        c = ACC[name]
        kw = dict(eval(bytes(c["gen_args"]).decode()))
        wl = synth.make_workload(**kw)
        assert wl.digest() == bytes(c["digest"]).decode(), f"{name}: generator drifted"
        cams = [oracle.camera_of(v) for v in wl.views]
        A = oracle.accumulate(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                              wl.scene.opacities, cams, list(wl.masks), wl.num_objects,
                              threads=4)
        np.testing.assert_allclose(A, c["A"], rtol=1e-6, atol=1e-9)


def test_kat_single_gaussian():
    # test_contributions.py:26-36 known answer, reproduced by the oracle
    c = ACC["kat_single_default"]
    assert abs(float(c["A"][1, 0]) - 17.71578278407129) < 1e-4
    assert c["A"][0, 0] == 0.0


def test_tile_range_corner_cases():
    c = BIN["tile_range"]
    # restated via the binning routine on single splats
    for args, expect in zip(c["args"], c["out"]):
        mx, my, r, tx_n, ty_n = args
        W, H = int(tx_n) * 16, int(ty_n) * 16
        offs, items = oracle.bin_tiles(np.array([1], np.uint8), np.array([[mx, my]]),
                                       np.array([1.0]), np.array([int(r)]), W, H)
        tx0, tx1, ty0, ty1 = expect
        counts = np.diff(offs).reshape(int(ty_n), int(tx_n))
        want = np.zeros_like(counts)
        if tx0 <= tx1 and ty0 <= ty1:
            want[ty0:ty1 + 1, tx0:tx1 + 1] = 1
        assert np.array_equal(counts, want), (args, expect)


@pytest.mark.parametrize("case", sorted(ASG))
def test_assignment_matches_reference(case):
    c = ASG[case]
    for i, g in enumerate(c["gammas"]):
        assert np.array_equal(oracle.assign_scene(c["A"], g), c["scene"][i]), (case, g)
        if "binary" in c:
            assert np.array_equal(oracle.assign_binary(c["A"], g), c["binary"][i]), (case, g)


def test_gamma_range_error_message():
    with pytest.raises(ValueError, match=r"gamma must lie in \[-1, 1\], got 1.5"):
        oracle.assign_binary(np.ones((2, 3), np.float32), 1.5)


def test_oracle_matches_reference_at_benchmark_resolution():
    """1008 x 756 (C2 camera geometry), 100 k Gaussians, 2 views, E = 4, straight from the
    reference (tests/golden/make_golden.py fullres)."""
    from conftest import load_golden
    from paper_2409_08270_b200 import synth
    c = load_golden("accumulate_fullres")["c2res_coherent"]
    kw = dict(eval(bytes(c["gen_args"]).decode()))
    wl = synth.make_workload(**kw)
    assert wl.digest() == bytes(c["digest"]).decode(), "generator drifted"
    cams = [oracle.camera_of(v) for v in wl.views]
    A = oracle.accumulate(wl.scene.means, wl.scene.rotations, wl.scene.scales,
                          wl.scene.opacities, cams, list(wl.masks), wl.num_objects, threads=4)
    assert np.count_nonzero(A != c["A"]) <= A.size // 10000
    np.testing.assert_allclose(A, c["A"], rtol=1e-6, atol=1e-9)
    assert np.array_equal(oracle.assign_scene(c["A"], 0.0), c["labels_g0"])


def test_oracle_on_acceptance_instances():
    """The oracle reproduces the reference's matrices and labels on the 200
    optimality instances and the two-cluster fixture (tests/golden/acceptance.npz)."""
    from conftest import cam_from_row
    acc = load_golden("acceptance")
    for k, c in acc.items():
        if not (k.startswith("opt") or k == "cluster"):
            continue
        cams = [oracle.camera_of(cam_from_row(r, i)) for i, r in enumerate(c["cams"])]
        floors = (0.0, 0.0) if k.startswith("opt") else (1 / 255, 1e-4)
        A = oracle.accumulate(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"], cams,
                              list(c["masks"]), 2, *floors, threads=4)
        np.testing.assert_allclose(A, c["A"], rtol=1e-6, atol=1e-12)
        if k.startswith("opt"):
            assert np.array_equal(oracle.assign_binary(A, 0.0), c["labels"]), k


FUZZ = load_golden("fuzz")


@pytest.mark.parametrize("case", sorted(FUZZ, key=lambda k: int(k[1:])))
def test_oracle_on_adversarial_fuzz_cases(case):
    """The oracle against the reference's own outputs on the adversarial cases of
    tests/fuzz_cases.py (near plane, duplicates, floors, 1-400 px cameras, E up
    to 40, seven blend settings; tests/golden/fuzz.npz)."""
    from fuzz_cases import ambiguous_mask_pixels, case_arrays, digest, render_extras
    from paper_2409_08270_b200 import GaussianScene

    ref = FUZZ[case]
    seed = int(case[1:])
    c = case_arrays(seed)
    assert digest(c) == bytes(ref["digest"]).decode(), "fuzz generator drifted"
    s = GaussianScene(c["means"], c["quats"], c["scales"], c["opac"])  # reference normalisation
    cams = [orc_cam(r) for r in c["cams"]]
    A = oracle.accumulate(s.means, s.rotations, s.scales, s.opacities, cams, c["masks"], c["E"],
                          *c["floors"], threads=4)
    np.testing.assert_allclose(A, ref["A"], rtol=1e-6, atol=1e-9)
    differ = int(np.count_nonzero(A != ref["A"]))
    assert differ <= max(2, A.size // 1000), f"{differ} of {A.size} entries differ"
    assert np.array_equal(oracle.assign_scene(ref["A"], c["gamma"]), ref["membership"])
    if "labels" in ref:
        assert np.array_equal(oracle.assign_binary(ref["A"], c["gamma"]), ref["labels"])
    if "r_alpha" in ref:
        ch, memb, tau = render_extras(seed, len(s), c["E"])
        _, alpha, depth = oracle.render_view(s.means, s.rotations, s.scales, s.opacities, cams[0],
                                             ch, None, *c["floors"])
        np.testing.assert_allclose(alpha, ref["r_alpha"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(depth, ref["r_depth"], rtol=1e-10, atol=1e-14)
        mask = oracle.render_mask(s.means, s.rotations, s.scales, s.opacities, cams[0], memb, tau,
                                  *c["floors"])
        differ = mask != ref["r_mask"]
        if differ.any():
            amb = ambiguous_mask_pixels(oracle, s.means, s.rotations, s.scales, s.opacities,
                                        cams[0], memb, tau, c["floors"])
            assert not (differ & ~amb).any(), f"{int((differ & ~amb).sum())} clear pixels differ"
