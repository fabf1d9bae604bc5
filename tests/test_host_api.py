"""Host-side logic of the package: types, validation order and messages,
serialisation formats, tile_range, view sharding.  No GPU needed."""

import numpy as np
import pytest

from paper_2409_08270_b200 import (
    Assignment,
    BlendConfig,
    CameraView,
    ContributionMatrix,
    DEFAULT_BLEND,
    EXACT_BLEND,
    GaussianScene,
    LabelMask,
    SceneDataError,
    tile_range,
)
from paper_2409_08270_b200.contributions import validate_views
from paper_2409_08270_b200.distributed import shard_views
from paper_2409_08270_b200.solver import _check_gamma


def frontal(w=16, h=16, f=24.0):
    return CameraView(0, w, h, f, f, w / 2 + 0.5, h / 2 + 0.5, np.eye(4))


def test_blend_constants():
    assert DEFAULT_BLEND.alpha_floor == 1.0 / 255.0
    assert DEFAULT_BLEND.transmittance_floor == 1e-4
    assert EXACT_BLEND == BlendConfig(0.0, 0.0)


def test_scene_validation_messages():
    with pytest.raises(SceneDataError, match="quaternion 1"):
        GaussianScene([[0, 0, 1]] * 2, [[1, 0, 0, 0], [0, 0, 0, 0]], [[1] * 3] * 2, [0.5] * 2)
    with pytest.raises(SceneDataError, match="gaussian 0 has non-positive scale"):
        GaussianScene([[0, 0, 1]], [[1, 0, 0, 0]], [[0, 1, 1]], [0.5])
    with pytest.raises(SceneDataError, match="gaussian 0 has opacity outside"):
        GaussianScene([[0, 0, 1]], [[1, 0, 0, 0]], [[1, 1, 1]], [1.5])
    s = GaussianScene([[0, 0, 1]], [[2, 0, 0, 0]], [[1, 1, 1]], [0.5])
    assert np.allclose(s.rotations, [[1, 0, 0, 0]])


def test_camera_validation():
    with pytest.raises(ValueError, match="orthonormal"):
        CameraView(3, 4, 4, 1.0, 1.0, 2, 2, np.diag([2.0, 1, 1, 1]))
    with pytest.raises(ValueError, match="focal"):
        CameraView(0, 4, 4, 0.0, 1.0, 2, 2, np.eye(4))


def test_validate_views_order_and_messages():
    v = frontal()
    good = LabelMask(0, np.zeros((16, 16), np.uint16))
    bad_shape = LabelMask(0, np.zeros((8, 16), np.uint16))
    lab = np.zeros((16, 16), np.uint16)
    lab[3, 7] = 5
    with pytest.raises(ValueError, match=r"view 0: mask shape \(8, 16\) does not match"):
        validate_views([(v, good), (v, bad_shape)], 2)
    with pytest.raises(ValueError, match=r"view 0: label 5 at pixel \(3, 7\) exceeds object count 2"):
        validate_views([(v, LabelMask(0, lab))], 2)
    validate_views([(v, good)], 1)


def test_contribution_matrix_file_roundtrip(tmp_path, rng):
    m = ContributionMatrix(rng.random((3, 7)).astype(np.float32))
    p = tmp_path / "A.bin"
    m.save(p)
    assert p.read_bytes()[:4] == b"FSA1"
    assert np.array_equal(ContributionMatrix.load(p).values, m.values)
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(ValueError, match="truncated"):
        ContributionMatrix.load(p)
    p.write_bytes(b"NOPE" + bytes(16))
    with pytest.raises(ValueError, match="magic"):
        ContributionMatrix.load(p)
    z = ContributionMatrix(np.array([[0, 1.0], [0, 0]], np.float32))
    assert z.observed.tolist() == [False, True]


def test_assignment_roundtrip(tmp_path, rng):
    a = Assignment("binary", 0.25, labels=rng.integers(0, 2, 17))
    a.save(tmp_path / "a.bin")
    b = Assignment.load(tmp_path / "a.bin")
    assert b.mode == "binary" and b.gamma == 0.25 and np.array_equal(a.labels, b.labels)
    mem = rng.integers(0, 2, (4, 9)).astype(np.uint8)
    s = Assignment("scene", -0.4, membership=mem)
    s.save(tmp_path / "s.bin")
    t = Assignment.load(tmp_path / "s.bin")
    assert np.array_equal(t.membership, mem) and t.member_counts() == mem.sum(1).tolist()
    with pytest.raises(ValueError):
        Assignment("weird", 0.0)


def test_gamma_check():
    assert _check_gamma(-1) == -1.0
    with pytest.raises(ValueError, match=r"gamma must lie in \[-1, 1\], got 1.5"):
        _check_gamma(1.5)


def test_tile_range_matches_golden():
    from conftest import load_golden
    c = load_golden("binning")["tile_range"]
    for args, expect in zip(c["args"], c["out"]):
        mx, my, r, tx, ty = args
        assert tile_range(mx, my, int(r), int(tx), int(ty)) == tuple(expect)


def test_shard_views_partition():
    for n in (0, 1, 7, 200):
        for world in (1, 2, 3, 8):
            shards = [shard_views(n, r, world) for r in range(world)]
            flat = [i for s in shards for i in s]
            assert flat == list(range(n))
            assert max(map(len, shards)) - min(map(len, shards)) <= 1


def test_render_grid_round_trip(tmp_path):
    """save_render_grid / load_render_grid (reference rasterizer.py:237-252)."""
    from paper_2409_08270_b200 import load_render_grid, save_render_grid
    grid = np.random.default_rng(0).random((12, 9)).astype(np.float32)
    path = tmp_path / "rho.f32"
    save_render_grid(path, grid)
    assert path.stat().st_size == 8 + 12 * 9 * 4
    assert np.array_equal(load_render_grid(path), grid)
    path.write_bytes(path.read_bytes()[:-4])
    with pytest.raises(ValueError, match="truncated"):
        load_render_grid(path)


def test_mask_png_round_trip_and_errors(tmp_path):
    """load_mask_png / save_mask_png keep the reference wire format (masks.py:25-40)."""
    from PIL import Image

    from paper_2409_08270_b200 import CameraView, load_mask_png, read_masks, save_mask_png
    lab = np.random.default_rng(0).integers(0, 65536, size=(13, 17)).astype(np.uint16)
    lab[0, 0] = 65535
    save_mask_png(tmp_path / "0.png", lab)
    assert np.array_equal(load_mask_png(tmp_path / "0.png"), lab)
    Image.fromarray(np.full((4, 5), 7, np.uint8)).save(tmp_path / "1.png")  # 8-bit L
    assert np.array_equal(load_mask_png(tmp_path / "1.png"), np.full((4, 5), 7, np.uint16))
    Image.fromarray(np.zeros((4, 5, 3), np.uint8)).save(tmp_path / "2.png")  # RGB
    with pytest.raises(ValueError, match="unsupported mask mode"):
        load_mask_png(tmp_path / "2.png")
    views = [CameraView(view_id=i, width=17, height=13, fx=10, fy=10, cx=8, cy=6,
                        world_to_camera=np.eye(4)) for i in (0, 3, 1)]
    pairs = read_masks(tmp_path, views, workers=2)  # view 3 has no file: skipped
    assert [v.view_id for v, _ in pairs] == [0, 1]
    assert np.array_equal(pairs[0][1].labels, lab)


def test_native_png_decoder_matches_pillow():
    """fs_decode_mask_png (C++, zlib) == Pillow on 8/16-bit grayscale PNGs with every
    filter mix Pillow produces; palette PNGs are declined (Pillow path)."""
    import io

    from PIL import Image

    from paper_2409_08270_b200 import _native
    rng = np.random.default_rng(0)
    for trial in range(40):
        h, w = (int(x) for x in rng.integers(1, 200, 2))
        kind = trial % 4
        if kind == 0:
            a = rng.integers(0, 65536, (h, w)).astype(np.uint16)
        elif kind == 1:
            a = (rng.integers(0, 4, (h, w)) * 1000).astype(np.uint16)
        elif kind == 2:
            a = np.cumsum(rng.integers(0, 3, (h, w)), axis=1).astype(np.uint16)
        else:
            a = rng.integers(0, 256, (h, w)).astype(np.uint8)
        buf = io.BytesIO()
        Image.fromarray(a).save(buf, format="PNG", optimize=trial % 2 == 0)
        data = buf.getvalue()
        ref = np.asarray(Image.open(io.BytesIO(data)).convert("I"), np.int32).astype(np.uint16)
        got = _native.decode_mask_png(data)
        assert got is not None and np.array_equal(got, ref)
    pal = Image.fromarray(rng.integers(0, 5, (9, 9)).astype(np.uint8)).convert("P")
    buf = io.BytesIO()
    pal.save(buf, format="PNG")
    assert _native.decode_mask_png(buf.getvalue()) is None
    assert _native.decode_mask_png(b"not a png") is None


def test_native_png_decoder_on_corrupted_files_defers_to_pillow():
    """Corrupted / truncated mask files: the native decoder either declines
    (None -> the Pillow path, which raises or decodes exactly as the reference
    does) or returns exactly what Pillow decodes -- never data from a file the
    reference would reject (e.g. a damaged IHDR: Pillow checks chunk CRCs)."""
    import io

    from PIL import Image, PngImagePlugin

    from paper_2409_08270_b200 import _native

    def pillow(data):
        try:
            with Image.open(io.BytesIO(data)) as im:
                return np.asarray(im.convert("I"), np.int32).astype(np.uint16)
        except Exception:
            return None

    rng = np.random.default_rng(3)
    for trial in range(1500):
        h, w = (int(x) for x in rng.integers(1, 40, 2))
        a = (rng.integers(0, 65536, (h, w)).astype(np.uint16) if trial % 2
             else rng.integers(0, 256, (h, w)).astype(np.uint8))
        info = None
        if trial % 5 == 0:
            info = PngImagePlugin.PngInfo()
            info.add_text("k", "v" * int(rng.integers(1, 30)))
        buf = io.BytesIO()
        Image.fromarray(a).save(buf, format="PNG", pnginfo=info)
        d = bytearray(buf.getvalue())
        mode = trial % 3
        if mode == 0:
            for _ in range(int(rng.integers(1, 4))):
                d[int(rng.integers(8, len(d)))] = int(rng.integers(0, 256))
        elif mode == 1:
            d = d[:int(rng.integers(8, len(d)))]
        else:
            d[int(rng.integers(8, len(d)))] ^= 1 << int(rng.integers(0, 8))
        got = _native.decode_mask_png(bytes(d))
        if got is not None:
            ref = pillow(bytes(d))
            assert ref is not None, f"trial {trial}: native decoded a file Pillow rejects"
            assert np.array_equal(got, ref), f"trial {trial}"
