"""Scene ingestion: binary PLY checkpoints (reference ply.py)."""

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2409_08270_b200 import GaussianScene, export_ply, load_scene_ply
from paper_2409_08270_b200.scene import SceneDataError, SceneFormatError

REF = Path("/root/reference/pkg/src")


def scene(n=50, seed=0):
    rng = np.random.default_rng(seed)
    return GaussianScene(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)),
                         rng.uniform(0.01, 0.3, (n, 3)), rng.uniform(0.05, 0.95, n),
                         colors_dc=rng.normal(size=(n, 3)))


def test_round_trip(tmp_path):
    s = scene()
    export_ply(s, tmp_path / "s.ply")
    t = load_scene_ply(tmp_path / "s.ply")
    assert len(t) == len(s) and t.source_path == str(tmp_path / "s.ply")
    np.testing.assert_allclose(t.means, s.means.astype(np.float32), rtol=0, atol=0)
    np.testing.assert_allclose(t.scales, s.scales, rtol=1e-6)
    np.testing.assert_allclose(t.opacities, s.opacities, rtol=1e-6)
    np.testing.assert_allclose(np.abs(np.sum(t.rotations * s.rotations, axis=1)), 1.0, rtol=1e-6)


def test_errors(tmp_path):
    p = tmp_path / "bad.ply"
    p.write_bytes(b"plx\n")
    with pytest.raises(SceneFormatError, match="missing 'ply' magic"):
        load_scene_ply(p)
    p.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 1\nend_header\n")
    with pytest.raises(SceneFormatError, match="binary_little_endian"):
        load_scene_ply(p)
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                  b"property float x\nend_header\n")
    with pytest.raises(SceneFormatError, match="missing required vertex property 'y'"):
        load_scene_ply(p)
    s = scene(4)
    export_ply(s, p)
    data = p.read_bytes()
    p.write_bytes(data[:-10])
    with pytest.raises(SceneFormatError, match=r"truncated payload \(3/4 vertices\)"):
        load_scene_ply(p)
    raw = bytearray(data)
    head = raw.index(b"end_header\n") + len(b"end_header\n")
    raw[head + 2 * 68 + 4:head + 2 * 68 + 8] = np.array([np.nan], "<f4").tobytes()  # vertex 2, y
    p.write_bytes(bytes(raw))
    with pytest.raises(SceneDataError, match="non-finite values at vertex 2"):
        load_scene_ply(p)


def test_matches_reference_loader(tmp_path):
    if not REF.exists():
        pytest.skip("reference package not available here")
    sys.path.insert(0, str(REF))
    try:
        import splatlift.ply as ref_ply
        from splatlift import GaussianScene as RefScene
    except ImportError as exc:
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(str(REF))
    s = scene(200, seed=3)
    rs = RefScene(means=s.means, rotations=s.rotations, scales=s.scales, opacities=s.opacities,
                  colors_dc=s.colors_dc)
    ref_ply.export_ply(rs, tmp_path / "r.ply")
    export_ply(s, tmp_path / "m.ply")
    assert (tmp_path / "r.ply").read_bytes() == (tmp_path / "m.ply").read_bytes()
    a, b = ref_ply.load_scene_ply(tmp_path / "r.ply"), load_scene_ply(tmp_path / "r.ply")
    for k in ("means", "rotations", "scales", "opacities", "colors_dc"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_host_loader_matches_reference_golden(tmp_path):
    """The host loader against the arrays the reference's load_scene_ply produced
    (tests/golden/scene_ply.npz, make_golden.py ``ply``), bit for bit; the lazy
    PlyScene (device path) builds the same host arrays."""
    from conftest import load_golden
    from paper_2409_08270_b200.scene_io import PlyScene, _read_header

    for case, c in load_golden("scene_ply").items():
        p = tmp_path / f"{case}.ply"
        p.write_bytes(bytes(c["ply"]))
        s = load_scene_ply(p)
        count, names, offset = _read_header(p.read_bytes()[:1 << 16])
        verts = np.memmap(p, dtype=np.dtype([(q, "<f4") for q in names]), mode="r",
                          offset=offset, shape=(count,))
        block = np.memmap(p, dtype=np.float32, mode="r", offset=offset, shape=(count, len(names)))
        lazy = PlyScene(p, count, names, block, verts)
        for k, ref in (("means", "means"), ("rotations", "rotations"), ("scales", "scales"),
                       ("opacities", "opacities"), ("colors_dc", "colors")):
            assert np.array_equal(getattr(s, k), c[ref]), (case, k)
            assert np.array_equal(getattr(lazy, k), c[ref]), (case, k)
        assert len(lazy) == count
        # offsets of the required properties in the record, reference order
        assert [names[i] for i in lazy._ply_offsets] == list(
            ("x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity",
             "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"))


@pytest.mark.parametrize("seed", range(80))
def test_host_loader_fuzz_matches_reference_loader(tmp_path, seed):
    """Checkpoints with special values (NaN, inf, +-0, denormals, exp overflow /
    underflow arguments, zero quaternions) in random properties: the host loader
    raises the reference loader's error, or returns its arrays bit for bit."""
    if not REF.exists():
        pytest.skip("reference package not available here")
    sys.path.insert(0, str(REF))
    try:
        import splatlift.ply as ref_ply
    finally:
        sys.path.remove(str(REF))
    from conftest import load_golden
    from fuzz_cases import patch_ply, ply_edits

    c = load_golden("scene_ply")["plain" if seed % 2 else "interleaved"]
    _, names = patch_ply(c["ply"], [])
    data, _ = patch_ply(c["ply"], ply_edits(seed, len(c["means"]), names))
    p = tmp_path / "f.ply"
    p.write_bytes(data)
    try:
        want = ref_ply.load_scene_ply(p)
        want_err = None
    except Exception as e:  # noqa: BLE001 -- the reference's own error is the expectation
        want, want_err = None, e
    if want_err is not None:  # same exception class (by name: two packages) and message
        with pytest.raises(Exception) as got:
            load_scene_ply(p)
        assert type(got.value).__name__ == type(want_err).__name__
        assert str(got.value) == str(want_err)
    else:
        got = load_scene_ply(p)
        for k in ("means", "rotations", "scales", "opacities", "colors_dc"):
            assert np.array_equal(getattr(got, k), getattr(want, k), equal_nan=True), k
