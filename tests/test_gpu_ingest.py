"""Pipelined mask ingestion: accumulate_mask_files equals
accumulate_contributions over the same PNG masks, with the reference's errors."""

import numpy as np
import pytest

from conftest import cam_from_row, load_golden

pytestmark = pytest.mark.gpu

from paper_2409_08270_b200 import (  # noqa: E402
    GaussianScene,
    LabelMask,
    accumulate_contributions,
    accumulate_mask_files,
    load_mask_png,
    save_mask_png,
)

ACC = load_golden("accumulate")


def c1(tmp_path):
    c = ACC["C1_default"]
    scene = GaussianScene(c["in_means"], c["in_quats"], c["in_scales"], c["in_opac"])
    views = [cam_from_row(r, i) for i, r in enumerate(c["cams"])]
    paths = []
    for v, m in zip(views, c["masks"]):
        p = tmp_path / f"{v.view_id}.png"
        save_mask_png(p, m)
        paths.append((v, p))
    return c, scene, views, paths


@pytest.mark.parametrize("chunk", [1, 3, 16])
def test_pipelined_ingest_matches_accumulate(tmp_path, chunk):
    c, scene, views, paths = c1(tmp_path)
    m = accumulate_mask_files(scene, paths, 2, chunk=chunk, workers=3)
    np.testing.assert_allclose(m.values, c["A"], rtol=1e-6, atol=1e-9)
    ref = accumulate_contributions(
        scene, [(v, LabelMask(v.view_id, load_mask_png(p))) for v, p in paths], 2)
    assert np.array_equal(np.argmax(m.values, axis=0), np.argmax(ref.values, axis=0))


def test_pipelined_ingest_errors_in_view_order(tmp_path):
    c, scene, views, paths = c1(tmp_path)
    lab = c["masks"][5].copy()
    lab[2, 3] = 7
    save_mask_png(paths[5][1], lab)
    save_mask_png(paths[6][1], np.zeros((5, 5), np.uint16))  # shape error later
    with pytest.raises(ValueError, match=r"view 5: label 7 at pixel \(2, 3\) exceeds object count 2"):
        accumulate_mask_files(scene, paths, 2, chunk=3)
    save_mask_png(paths[5][1], c["masks"][5])
    with pytest.raises(ValueError, match="view 6: mask shape"):
        accumulate_mask_files(scene, paths, 2, chunk=3)
