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
