"""splatlift_compat rebinds the reference package's import sites (CPU check; the
reference package is importable only in the build container)."""

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture
def splatlift():
    if not REF.exists():
        pytest.skip("reference package not available here")
    sys.path.insert(0, str(REF))
    try:
        import splatlift  # noqa: F401
        import splatlift.cli  # noqa: F401
        import splatlift.service  # noqa: F401
    except ImportError as exc:
        pytest.skip(f"reference not importable: {exc}")
    yield sys.modules["splatlift"]
    sys.path.remove(str(REF))


def test_install_rebinds_every_import_site(splatlift):
    from paper_2409_08270_b200 import splatlift_compat
    import splatlift.cli as cli
    import splatlift.contributions as contrib
    import splatlift.service as service
    import splatlift.solver as solver
    before = (cli.accumulate_contributions, solver.assign_binary, service.assign_scene)
    splatlift_compat.install()
    try:
        for mod in (splatlift, contrib, cli):
            assert mod.accumulate_contributions.__module__ == "paper_2409_08270_b200.splatlift_compat"
        for mod in (splatlift, solver, cli, service):
            assert mod.assign_binary.__module__ == "paper_2409_08270_b200.splatlift_compat"
            assert mod.assign_scene.__module__ == "paper_2409_08270_b200.splatlift_compat"
    finally:
        splatlift_compat.uninstall()
    assert (cli.accumulate_contributions, solver.assign_binary, service.assign_scene) == before


def test_install_rebinds_render_import_sites(splatlift):
    from paper_2409_08270_b200 import splatlift_compat
    import splatlift.cli as cli
    import splatlift.maskrender as maskrender
    import splatlift.rasterizer as rasterizer
    before = (rasterizer.render_view, maskrender.render_subset_alpha_depth, cli.render_scene_mask)
    splatlift_compat.install()
    try:
        mod_name = "paper_2409_08270_b200.splatlift_compat"
        for mod in (splatlift, rasterizer):
            assert mod.render_view.__module__ == mod_name
        for mod in (splatlift, rasterizer, maskrender):
            assert mod.render_property.__module__ == mod_name
            assert mod.render_subset_alpha_depth.__module__ == mod_name
        for mod in (splatlift, maskrender, cli):
            assert mod.render_binary_mask.__module__ == mod_name
            assert mod.render_scene_mask.__module__ == mod_name
    finally:
        splatlift_compat.uninstall()
    assert (rasterizer.render_view, maskrender.render_subset_alpha_depth,
            cli.render_scene_mask) == before


def test_install_rebinds_mask_loading(splatlift):
    from paper_2409_08270_b200 import splatlift_compat
    import splatlift.cli as cli
    import splatlift.masks as masks
    before = masks.load_mask_png
    splatlift_compat.install()
    try:
        for mod in (splatlift, masks, cli):
            assert mod.load_mask_png.__module__ == "paper_2409_08270_b200.masks"
    finally:
        splatlift_compat.uninstall()
    assert masks.load_mask_png is before


def test_file_formats_byte_identical_to_reference(splatlift, tmp_path):
    """FSA1 matrices and assignment files written by either package are byte-identical
    and load in the other (contributions.py:70-87, solver.py:79-108)."""
    import numpy as np
    from paper_2409_08270_b200 import Assignment, ContributionMatrix
    rng = np.random.default_rng(4)
    A = rng.random((3, 11)).astype(np.float32)
    ContributionMatrix(A).save(tmp_path / "ours.fsa")
    splatlift.ContributionMatrix(A).save(tmp_path / "ref.fsa")
    assert (tmp_path / "ours.fsa").read_bytes() == (tmp_path / "ref.fsa").read_bytes()
    assert np.array_equal(splatlift.ContributionMatrix.load(tmp_path / "ours.fsa").values, A)
    assert np.array_equal(ContributionMatrix.load(tmp_path / "ref.fsa").values, A)
    for mode, kw in (("binary", dict(labels=rng.integers(0, 2, 13).astype(np.uint8))),
                     ("scene", dict(membership=rng.integers(0, 2, (4, 13)).astype(np.uint8)))):
        Assignment(mode, 0.25, **kw).save(tmp_path / f"ours_{mode}.bin")
        splatlift.Assignment(mode=mode, gamma=0.25, **kw).save(tmp_path / f"ref_{mode}.bin")
        assert ((tmp_path / f"ours_{mode}.bin").read_bytes()
                == (tmp_path / f"ref_{mode}.bin").read_bytes())
        back = splatlift.Assignment.load(tmp_path / f"ours_{mode}.bin")
        assert back.mode == mode and back.member_counts() == Assignment(mode, 0.25, **kw).member_counts()


def test_install_devices_reach_the_multi_gpu_path(splatlift, monkeypatch):
    """install(devices=[...]) makes the rebound accumulate (the CLI's, cli.py:104)
    split views over those GPUs; one device / None keeps the single-GPU path."""
    from paper_2409_08270_b200 import splatlift_compat
    from paper_2409_08270_b200 import contributions as contrib
    import splatlift.cli as cli
    import numpy as np
    seen = {}

    def fake(scene, views, num_objects, blend, **kw):
        seen.update(kw)
        return contrib.ContributionMatrix(values=np.zeros((num_objects, 1), np.float32))

    monkeypatch.setattr(contrib, "accumulate_contributions", fake)
    for devices, expect in (([0, 1, 2], [0, 1, 2]), ([3], None), (None, None)):
        seen.clear()
        splatlift_compat.install(devices=devices)
        try:
            cli.accumulate_contributions(object(), [], 2)
        finally:
            splatlift_compat.uninstall()
        assert seen.get("devices") == expect
    monkeypatch.setenv("FLASHSPLAT_DEVICES", "1,0")
    assert splatlift_compat.resolve_devices("auto") == [1, 0]


def test_install_device_ply_routes_the_cli_loader(splatlift, monkeypatch):
    """install(device_ply=True): the CLI's load_scene_ply (cli.py:97) goes through the
    device ingestion path (scene_io.load_scene_ply(path, device=...))."""
    from paper_2409_08270_b200 import scene_io, splatlift_compat
    import splatlift.cli as cli
    seen = {}

    def fake(path, device=None):
        seen["device"] = device
        return "scene"

    monkeypatch.setattr(scene_io, "load_scene_ply", fake)
    splatlift_compat.install(devices=[2, 3], device_ply=True)
    try:
        assert cli.load_scene_ply("x.ply") == "scene" and seen["device"] == 2
    finally:
        splatlift_compat.uninstall()
